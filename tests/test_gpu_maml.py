"""C5 MAML on the GPU (csrc/maml.cu via paper_1810_08061_b200.maml) against
the reference's gradient() goldens (tests/golden/maml_*.json) and the
closed-form float64 oracle at 4096 tasks.  fp32: rtol 1e-4 (stated bound)."""
import numpy as np
import pytest
import torch

from oracle import fixtures
from oracle import maml as omaml
from oracle.gen_stream_golden import MAML_CASES
from paper_1810_08061_b200.maml import MamlTrainer, flatten_theta, unflatten

pytestmark = pytest.mark.gpu


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a[..., 0], dtype=np.float32)).cuda()


@pytest.mark.parametrize("case", MAML_CASES, ids=lambda c: c["name"])
def test_meta_grad_matches_reference(case):
    doc = fixtures.load_golden(case["name"])
    H, K, n = case["H"], case["K"], case["tasks"]
    th = omaml.init_theta(H, case["seed"])
    xs, ys, xq, yq = omaml.sinusoid_tasks(n, K, case["seed"] + 1)
    tr = MamlTrainer(H, K, n, alpha=case["alpha"], theta=th)
    g, loss = tr.meta_grad(_t(xs), _t(ys), _t(xq), _t(yq))
    ref = np.mean([np.concatenate([np.asarray(o[1 + k]) for k in range(6)]) for o in doc["outputs"]], axis=0)
    ref_loss = np.mean([o[0][0] for o in doc["outputs"]])
    got = g.cpu().numpy().astype(np.float64)
    assert np.allclose(got, ref, rtol=1e-4, atol=1e-4 * np.max(np.abs(ref)))
    assert abs(float(loss.item()) - ref_loss) <= 1e-4 * max(1, abs(ref_loss))


def test_meta_grad_4096_tasks_and_step():
    H, K, n = 40, 10, 4096
    th = omaml.init_theta(H, 3)
    xs, ys, xq, yq = omaml.sinusoid_tasks(n, K, 4)
    loss_ref, g_ref = omaml.meta_grad(th, xs, ys, xq, yq, 0.01)
    ref = np.concatenate([g_ref[k].mean(axis=0).reshape(-1) for k in omaml.NAMES])
    tr = MamlTrainer(H, K, n, alpha=0.01, beta=0.5, theta=th)
    args = (_t(xs), _t(ys), _t(xq), _t(yq))
    g, loss = tr.meta_grad(*args)
    got = g.cpu().numpy().astype(np.float64)
    assert np.allclose(got, ref, rtol=1e-4, atol=1e-4 * np.max(np.abs(ref)))
    assert abs(float(loss.item()) - loss_ref.mean()) <= 1e-4 * loss_ref.mean()
    tr.step(*args)   # meta-SGD: theta - beta * meta_grad
    new = tr.theta.cpu().numpy().astype(np.float64)
    assert np.allclose(new, flatten_theta(th) - 0.5 * got, rtol=1e-5, atol=1e-6)
