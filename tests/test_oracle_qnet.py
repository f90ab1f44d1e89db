"""Pins for oracle/qnet.py -- torch float64 autograd (independent library) and finite
differences."""
import numpy as np
import pytest
import torch

from oracle import qnet as QN
from oracle import space as SP
from oracle import actions as A


def _torch_forward(theta, dims, x):
    o = 0
    h = x
    for i in range(len(dims) - 1):
        fi, fo = dims[i], dims[i + 1]
        Wm = theta[o:o + fi * fo].view(fo, fi)
        o += fi * fo
        b = theta[o:o + fo]
        o += fo
        h = torch.nn.functional.linear(h, Wm, b)
        if i < len(dims) - 2:
            h = torch.relu(h)
    return h


@pytest.mark.parametrize("dims", [[17, 9], [34, 16, 12], [68, 64, 64, 54]])
def test_forward_backward_vs_torch(dims):
    rng = np.random.default_rng(0)
    n = QN.n_params(dims)
    theta = rng.normal(0, 0.3, n)
    x = rng.normal(0, 1, (5, dims[0]))
    dz = rng.normal(0, 1, (5, dims[-1]))
    z, acts = QN.forward(theta, dims, x)
    g = QN.backward(theta, dims, acts, dz)
    th = torch.tensor(theta, dtype=torch.float64, requires_grad=True)
    zt = _torch_forward(th, dims, torch.tensor(x))
    (zt * torch.tensor(dz)).sum().backward()
    np.testing.assert_allclose(z, zt.detach().numpy(), rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(g, th.grad.numpy(), rtol=1e-10, atol=1e-12)


def test_backward_finite_differences():
    rng = np.random.default_rng(1)
    dims = [6, 5, 4]
    theta = rng.normal(0, 0.5, QN.n_params(dims))
    x = rng.normal(0, 1, (3, 6))
    dz = rng.normal(0, 1, (3, 4))
    z, acts = QN.forward(theta, dims, x)
    g = QN.backward(theta, dims, acts, dz)
    eps = 1e-6
    for k in range(len(theta)):
        tp, tm = theta.copy(), theta.copy()
        tp[k] += eps
        tm[k] -= eps
        fd = ((QN.forward(tp, dims, x)[0] - QN.forward(tm, dims, x)[0]) * dz).sum() / (2 * eps)
        assert abs(fd - g[k]) < 1e-6 * max(1, abs(fd))


def test_structured_head_gradient_vs_autograd():
    sp = SP.build_space(5, 3, (25, 50, 75))
    rng = np.random.default_rng(2)
    off = A.offsets(sp)
    for _ in range(30):
        idx = int(rng.integers(A.n_actions(sp)))
        l, g, s = A.decode(sp, idx, off)
        z = rng.normal(0, 1, sp.H)
        zt = torch.tensor(z, requires_grad=True)
        v = zt[0]
        aL = zt[1:1 + sp.L]
        aJ = zt[1 + sp.L:].view(sp.W, sp.T)
        cL = aL - aL.mean()
        cJ = aJ - aJ.mean(0, keepdim=True)
        q = v + cL[l] + sum(cJ[g[i], sp.slot_type[l][s[i]]] for i in range(len(g)))
        q.backward()
        np.testing.assert_allclose(QN.dq_dz(sp, l, g, s), zt.grad.numpy(), atol=1e-14)
        vv, aLn, aJn = QN.split_head(z, sp)
        cLn, cJn = QN.center(aLn, aJn)
        assert QN.q_value(vv, cLn, cJn, sp, l, g, s) == pytest.approx(q.item(), abs=1e-12)


def test_fixed_point_half_even():
    assert QN.fixed(0.5 / 4294967296.0) == 0
    assert QN.fixed(1.5 / 4294967296.0) == 2
    assert QN.fixed(-2.5 / 4294967296.0) == -2
    assert QN.fixed(1.0) == 4294967296
