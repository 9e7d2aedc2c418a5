"""CPU: the float64 decoder restatement (oracle/beam.py) reproduces the
reference's staged greedy program (traced and executed by the
reference: tests/golden/greedy_*.json) token for token at beam 1."""
import numpy as np
import pytest

from oracle import beam, fixtures


@pytest.mark.parametrize("name", [c["name"] for c in fixtures.GREEDY_CASES])
def test_beam1_oracle_is_the_reference_greedy_program(name):
    doc = fixtures.load_golden(name)
    case = doc["case"]
    f = fixtures.make_greedy_feeds(case)
    exp_toks = doc["expected"]["outputs"][0]["tensor"]["data"]
    exp_t = doc["expected"]["outputs"][1]["tensor"]["data"][0]
    r = beam.decode("rnn", f["h0"], f["emb"][:, 0, :], (f["w_in"], f["u"], f["w_out"]), 1, case["eos"],
                    case["max_len"], exact=True)
    assert r["steps"] == exp_t
    assert list(r["tokens"][0, 0, :exp_t + 1]) == exp_toks


def test_beam_search_properties():
    rng = np.random.default_rng(0)
    S, V, E, H, K = 3, 40, 6, 8, 4
    W = rng.uniform(-1, 1, (E + H, 4 * H))
    r = beam.decode("lstm", rng.uniform(-1, 1, (S, H)), rng.uniform(-1, 1, (V, E)),
                    (W, rng.uniform(-0.1, 0.1, 4 * H), rng.uniform(-2, 2, (H, V)), rng.uniform(-1, 1, V)),
                    K, 3, 12)
    s = r["scores"]
    assert np.all(np.diff(s, axis=1) <= 0)          # beams sorted best first
    assert np.all(s <= 0)                             # log-probabilities
    assert r["steps"] <= 12
