"""f3: autograd through the C ABI — forward wn_eval (A), backward wn_eval_adjoint (Aᵀ)."""
import numpy as np
import pytest

import oracle
from paper_2405_16634_b200 import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ag():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2405_16634_b200.autograd as ag

    return ag


def test_backward_is_the_transpose(ag):
    import paper_2405_16634_b200.wn as wn

    p, nr = synth.sphere(3000, seed=31)
    rng = np.random.default_rng(32)
    mu0 = (nr * 0.004 * (1 + 0.2 * rng.standard_normal((3000, 1)))).astype(np.float32)
    g = rng.standard_normal(3000).astype(np.float32)
    w = float(np.float32(0.005))
    t = wn.wn_build_tree(torch.from_numpy(p).cuda())
    mu = torch.from_numpy(mu0).cuda().requires_grad_(True)
    F = ag.winding_number(t, mu, w, adjoint="transpose")
    (F * torch.from_numpy(g).cuda()).sum().backward()
    cl = oracle.Cloud(p)
    ref = cl.AT_transpose(g, mu0, w)           # exact transpose of the treecode at g(μ)
    got = mu.grad.cpu().numpy()
    err = np.linalg.norm(got - ref, axis=1)
    assert np.all(err <= 1e-4 * np.linalg.norm(ref, axis=1) + 1e-5 * np.abs(ref).max())
    # ⟨A μ, g⟩ is linear in μ at fixed geometry: its gradient contracted with μ reproduces it
    lhs = float((F.detach() * torch.from_numpy(g).cuda()).sum())
    rhs = float((mu.grad * mu.detach()).sum())
    assert abs(lhs - rhs) <= 1e-4 * abs(lhs)


def test_gather_backward(ag):
    import paper_2405_16634_b200.wn as wn

    p, nr = synth.sphere(2000, seed=33)
    g = np.random.default_rng(34).standard_normal(2000).astype(np.float32)
    w = float(np.float32(0.01))
    t = wn.wn_build_tree(torch.from_numpy(p).cuda())
    mu = torch.from_numpy((nr * 0.006).astype(np.float32)).cuda().requires_grad_(True)
    ag.winding_number(t, mu, w, adjoint="gather").backward(torch.from_numpy(g).cuda())
    ref = oracle.Cloud(p).AT(g, w)
    err = np.linalg.norm(mu.grad.cpu().numpy() - ref, axis=1)
    assert np.all(err <= 1e-4 * np.linalg.norm(ref, axis=1) + 1e-5 * np.abs(ref).max())
