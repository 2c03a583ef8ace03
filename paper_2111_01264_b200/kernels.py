"""The reference's kernel plugin module on the B200 (fp64, bit-exact with numba).

Same contract as pkg/src/paraq/_kernels_numba.py:14-121 / _kernels_numpy.py: C-contiguous
float64 numpy arrays in, fresh arrays out, inputs never mutated, no validation (the
callers in nn.py validate).  Each call moves its operands to HBM, runs one sm_100a fp64
kernel that keeps the reference's per-element accumulation order with explicitly
rounded multiply / add (no FMA, like numba), and copies the result back -- so the
values are bit-identical to the numba backend (tests/test_gpu_plugin.py), which lets
the reference's own nn.py / agent.py run unchanged on the GPU:

    import paraq.backend, paraq.nn
    import paper_2111_01264_b200.kernels as b200
    paraq.nn.K = b200          # the reference's nn module now computes on the B200

``spin`` is the env busy-wait model (envs.py:108-117, :166): host CPU work by
definition, implemented on the host exactly like the numba kernel's FMA-free chain.
"""

from __future__ import annotations

import numpy as np

from . import _native as N

BACKEND_NAME = "b200"


def _dev(a, dtype=np.float64):
    torch = N.require_cuda()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=dtype)).cuda()


def _out(shape):
    torch = N.require_cuda()
    return torch.empty(shape, dtype=torch.float64, device="cuda")


def _host(t):
    return t.cpu().numpy()


def affine_rows(w, b, x):
    n, d = np.shape(x)
    o = np.shape(w)[0]
    W, B, X, out = _dev(w), _dev(b), _dev(x), _out((n, o))
    N.check(N.load().pq64_affine_rows(W.data_ptr(), B.data_ptr(), X.data_ptr(), n, o, d,
                                      out.data_ptr(), N.stream_ptr()), "affine_rows")
    return _host(out)


def relu(x):
    X = _dev(x)
    out = _out(X.shape)
    N.check(N.load().pq64_relu(X.data_ptr(), X.numel(), out.data_ptr(), N.stream_ptr()), "relu")
    return _host(out)


def output_delta(q, actions, targets):
    n, o = np.shape(q)
    Q, A, T, out = _dev(q), _dev(actions, np.int64), _dev(targets), _out((n, o))
    N.check(N.load().pq64_output_delta(Q.data_ptr(), A.data_ptr(), T.data_ptr(), n, o,
                                       out.data_ptr(), N.stream_ptr()), "output_delta")
    return _host(out)


def weight_grad(delta, acts):
    n, o = np.shape(delta)
    d = np.shape(acts)[1]
    D, X, out = _dev(delta), _dev(acts), _out((o, d))
    N.check(N.load().pq64_weight_grad(D.data_ptr(), X.data_ptr(), n, o, d, out.data_ptr(),
                                      N.stream_ptr()), "weight_grad")
    return _host(out)


def bias_grad(delta):
    n, o = np.shape(delta)
    D, out = _dev(delta), _out((o,))
    N.check(N.load().pq64_bias_grad(D.data_ptr(), n, o, out.data_ptr(), N.stream_ptr()),
            "bias_grad")
    return _host(out)


def hidden_delta(delta, w, pre):
    n, o = np.shape(delta)
    d = np.shape(w)[1]
    D, W, P, out = _dev(delta), _dev(w), _dev(pre), _out((n, d))
    N.check(N.load().pq64_hidden_delta(D.data_ptr(), W.data_ptr(), P.data_ptr(), n, o, d,
                                       out.data_ptr(), N.stream_ptr()), "hidden_delta")
    return _host(out)


def rmsprop_flat(p, g, m, v, lr, rho, kappa):
    P, G, M, V = _dev(p), _dev(g), _dev(m), _dev(v)
    p2, m2, v2 = _out(P.shape), _out(P.shape), _out(P.shape)
    N.check(N.load().pq64_rmsprop_flat(P.data_ptr(), G.data_ptr(), M.data_ptr(), V.data_ptr(),
                                       P.numel(), lr, rho, kappa, p2.data_ptr(), m2.data_ptr(),
                                       v2.data_ptr(), N.stream_ptr()), "rmsprop_flat")
    return _host(p2), _host(m2), _host(v2)


def spin(units: int) -> float:
    acc = 1.0
    for _ in range(units):
        acc = acc * 1.0000000001 + 1e-12
    return acc
