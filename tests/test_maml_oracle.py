"""CPU: the closed-form float64 MAML meta-gradient (oracle/maml.py) against
the reference's gradient() of the staged one-task program
(tests/golden/maml_*.json)."""
import numpy as np
import pytest

from oracle import fixtures
from oracle import maml as omaml
from oracle.gen_stream_golden import MAML_CASES


@pytest.mark.parametrize("case", MAML_CASES, ids=lambda c: c["name"])
def test_meta_grad_matches_reference_gradient(case):
    doc = fixtures.load_golden(case["name"])
    th = omaml.init_theta(case["H"], case["seed"])
    xs, ys, xq, yq = omaml.sinusoid_tasks(case["tasks"], case["K"], case["seed"] + 1)
    loss, g = omaml.meta_grad(th, xs, ys, xq, yq, case["alpha"])
    for t, outs in enumerate(doc["outputs"]):
        assert abs(loss[t] - outs[0][0]) < 1e-10 * max(1, abs(outs[0][0]))
        for k, name in enumerate(omaml.NAMES):
            ref = np.asarray(outs[1 + k])
            assert np.allclose(g[name][t].reshape(-1), ref, rtol=1e-9, atol=1e-11), name
