"""a3/a4/a10/a11 -- the duelling Q-network (ORACLE, test infrastructure only), float64.

Paper: fully connected layers with ReLU (Table VI); duelling architecture
Q = V + (A - mean A) (Wang et al.); double DQN with separate online and
target networks (van Hasselt); Q-learning update
Q <- Q + alpha (r + gamma max_a Q(s', a) - Q), i.e. SGD on (1/2) delta^2.

Factorised duelling head (reading R1/A1): z = [v | aL (L) | aJ (W x T)];
  cL = aL - mean(aL);  cJ[j][tau] = aJ[j][tau] - mean_j aJ[.][tau]   (means over all
  layouts / all window positions, reading R20);
  Q(s, a=(l, g, sigma)) = v + cL[l] + sum_i cJ[g_i][tau(l, sigma(i))]   (summed in that order).
Argmax key: Q^ = F(v) + F(cL[l]) + sum_i F(cJ[g_i][tau]) with F(x) = rint_half_even(x 2^32)
as an exact integer (reading R15).

Parameter layout (shared with synth.init_weights): per Linear layer W [out][in] row-major,
then b [out].

Pins: tests/test_oracle_qnet.py -- forward/backward against torch float64 autograd on CPU
(an independent library implementation) and central finite differences; the structured
head gradient against autograd of the Q formula; the tabular special case of P:178
(tests/test_oracle_dqn.py).
"""
from __future__ import annotations

import numpy as np


def net_dims(space, net) -> list:
    fin = space.W * (12 + 5)
    return [fin] + [net.hidden_width] * net.hidden_layers + [space.H]


def n_params(dims) -> int:
    return sum(dims[i] * dims[i + 1] + dims[i + 1] for i in range(len(dims) - 1))


def unflatten(theta, dims):
    out = []
    o = 0
    for i in range(len(dims) - 1):
        fi, fo = dims[i], dims[i + 1]
        Wm = theta[o:o + fi * fo].reshape(fo, fi)
        o += fi * fo
        b = theta[o:o + fo]
        o += fo
        out.append((Wm, b))
    return out


def forward(theta, dims, x, pre=None):
    """x [M][in] -> (z [M][H], acts) where acts[l] is the input of layer l.  If `pre` is a
    list, the hidden layers' pre-activations are appended to it."""
    layers = unflatten(np.asarray(theta, np.float64), dims)
    h = np.asarray(x, np.float64)
    acts = []
    for i, (Wm, b) in enumerate(layers):
        acts.append(h)
        y = h @ Wm.T + b
        if i < len(layers) - 1 and pre is not None:
            pre.append(y)
        h = np.maximum(y, 0.0) if i < len(layers) - 1 else y
    return h, acts


def backward(theta, dims, acts, dz, masks=None):
    """Gradient of sum(dz * z) w.r.t. the flat parameters.  ReLU'(h) = [h > 0] for the input of
    layer i > 0, or masks[i - 1] when given (the near-zero lockstep of reading R25)."""
    layers = unflatten(np.asarray(theta, np.float64), dims)
    grads = [None] * len(layers)
    d = np.asarray(dz, np.float64)
    for i in range(len(layers) - 1, -1, -1):
        Wm, _ = layers[i]
        h = acts[i]
        grads[i] = (d.T @ h, d.sum(0))
        if i > 0:
            d = (d @ Wm) * (h > 0 if masks is None else masks[i - 1])
    return np.concatenate([np.concatenate([gw.ravel(), gb]) for gw, gb in grads])


def split_head(z, space):
    """z [H] -> v, aL [L], aJ [W][T] (all zero for the sequential agent's flat head, R28)."""
    L, W, T = space.L, space.W, space.T
    if getattr(space, "seq", False):
        return z[0], z[1:1 + L], np.zeros((W, T))
    return z[0], z[1:1 + L], z[1 + L:1 + L + W * T].reshape(W, T)


def center(aL, aJ):
    return aL - aL.mean(), aJ - aJ.mean(axis=0, keepdims=True)


def fixed(x) -> int:
    """F(x) = round-half-even(x * 2^32) as an exact integer."""
    return int(np.rint(float(x) * 4294967296.0))


def q_value(v, cL, cJ, space, l, g, sigma) -> float:
    st = space.slot_type[l]
    q = float(v) + float(cL[l])
    for i, gi in enumerate(g):
        q += float(cJ[gi, st[sigma[i]]])
    return q


def q_fixed(Fv, FcL, FcJ, space, l, g, sigma) -> int:
    st = space.slot_type[l]
    q = Fv + FcL[l]
    for i, gi in enumerate(g):
        q += FcJ[gi][st[sigma[i]]]
    return q


def dq_dz(space, l, g, sigma) -> np.ndarray:
    """Structured gradient of Q(s, a) w.r.t. the head output z:
    dQ/dv = 1; dQ/daL[l'] = [l' = l] - 1/L; dQ/daJ[j][tau] = #{i: g_i = j, tau_i = tau}
    - #{i: tau_i = tau} / W."""
    L, W, T = space.L, space.W, space.T
    d = np.zeros(space.H)
    d[0] = 1.0
    d[1:1 + L] = -1.0 / L
    d[1 + l] += 1.0
    if getattr(space, "seq", False):
        return d                                  # flat head: no job-advantage block
    dJ = np.zeros((W, T))
    st = space.slot_type[l]
    for i, gi in enumerate(g):
        tau = st[sigma[i]]
        dJ[gi, tau] += 1.0
        dJ[:, tau] -= 1.0 / W
    d[1 + L:] = dJ.ravel()
    return d
