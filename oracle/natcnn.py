"""Nature-CNN DQN learner in fp64 -- TEST INFRASTRUCTURE ONLY (the parity oracle).

Composition of the reference kernel module (restated bit-exactly in
oracle/kernels.c) through im2col, following the reference line by line:

* forward          -- nn.forward (nn.py:123-131): affine_rows then relu per layer,
                      last layer linear.  A conv layer is affine_rows over its
                      im2col patch rows.
* gradient         -- nn.gradient (nn.py:134-170): forward keeping pre-activations,
                      output_delta, then for k = last..0: weight_grad, bias_grad,
                      hidden_delta.  For a conv layer the hidden delta is taken in
                      patch space (hidden_delta with an all-pass mask), scattered
                      back by col2im (kh, kw ascending) and then masked by the
                      previous layer's pre-activation > 0 -- the restatement of
                      hidden_delta's [pre > 0] factor for overlapping patches.
* rmsprop_step     -- nn.rmsprop_step (nn.py:173-203) incl. the non-finite check.
* td_targets       -- agent.td_targets (agent.py:69-81).
* train_minibatch  -- agent.train_minibatch (agent.py:84-105): gradient of the mean
                      loss, x n, centered RMSProp.

Restatement choices (the reference has no conv net):
* inputs are uint8 frame stacks [n, 4, 84, 84]; x = u8 / 255.0 in fp64;
* conv1 weights flatten (out, c, kh, kw) over the planar input; conv2 and conv3
  weights flatten (out, kh, kw, c) over NHWC activations; fc1 reads conv3's
  output flattened (h, w, c);
* init: the reference init_network bound sqrt(6/(fan_in+fan_out)) over each
  flattened (out, in*kh*kw) matrix, drawn layer by layer from one
  default_rng(seed) (nn.py:93-109).

Two optional knobs, both off by default (the fp64 reference arithmetic):
* ``K`` -- the kernel module: ``oracle._lib`` (kernels.c, bit-exact with numba, the
  default) or ``oracle.blas`` (the reference numpy backend with batched rows, for
  batch 1024 / W 512 in seconds);
* ``store`` -- a storage model (``Bf16Storage``): the points where the device path
  keeps a value in bf16 (the tensor-core operands W1..W4, the conv activations, the
  data gradients).  The oracle still computes in fp64 but rounds exactly there, so a
  comparison with the bf16 tensor-core path is well posed: what remains is fp32
  accumulation order, which is what the stated tolerance (rel 1e-3) bounds.
* ``huber`` -- the opt-in Huber TD loss (north star); None = the reference's
  half-squared loss (Huber with delta = infinity).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib as _K_EXACT


@dataclass(frozen=True)
class Layer:
    kind: str              # "conv" or "fc"
    out: int
    k: int = 0             # conv kernel size
    s: int = 0             # conv stride
    planar: bool = False   # conv input is (c, h, w) instead of NHWC


@dataclass(frozen=True)
class NetSpec:
    in_shape: tuple        # (c, h, w) for conv nets, (d,) for MLPs
    layers: tuple

    def shapes(self):
        """Per layer: (in_shape, out_shape, weight_shape)."""
        res = []
        cur = self.in_shape
        for L in self.layers:
            if L.kind == "conv":
                if L.planar:
                    c, h, w = cur
                else:
                    h, w, c = cur
                oh = (h - L.k) // L.s + 1
                ow = (w - L.k) // L.s + 1
                res.append((cur, (oh, ow, L.out), (L.out, c * L.k * L.k)))
                cur = (oh, ow, L.out)
            else:
                d = int(np.prod(cur))
                res.append((cur, (L.out,), (L.out, d)))
                cur = (L.out,)
        return res

    @property
    def n_params(self) -> int:
        return sum(o * i + o for _, _, (o, i) in self.shapes())


def nature_cnn(actions: int = 18, frame: int = 84, stack: int = 4) -> NetSpec:
    return NetSpec(
        (stack, frame, frame),
        (
            Layer("conv", 32, 8, 4, planar=True),
            Layer("conv", 64, 4, 2),
            Layer("conv", 64, 3, 1),
            Layer("fc", 512),
            Layer("fc", actions),
        ),
    )


def mlp(sizes) -> NetSpec:
    return NetSpec((sizes[0],), tuple(Layer("fc", s) for s in sizes[1:]))


@dataclass
class Params:
    weights: list
    biases: list


@dataclass
class Opt:
    m_weights: list
    m_biases: list
    v_weights: list
    v_biases: list
    step: int = 0

    @classmethod
    def zeros(cls, p: Params) -> "Opt":
        z = lambda xs: [np.zeros_like(x) for x in xs]  # noqa: E731
        return cls(z(p.weights), z(p.biases), z(p.weights), z(p.biases))


def bf16_round(x) -> np.ndarray:
    """fp64 -> fp32 (round to nearest even) -> bf16 (round to nearest even), as fp64:
    the device's fp32 value stored with __float2bfloat16_rn."""
    f = np.ascontiguousarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def fp32_round(x) -> np.ndarray:
    return np.asarray(x, dtype=np.float32).astype(np.float64)


class Bf16Storage:
    """Where the B200 learner / acting path stores bf16:

    * weights of layers 0..3 (conv1..fc1): the bf16 shadow of the fp32 master;
      fc2 and all biases stay fp32;
    * forward activations of the conv layers (act1..act3, NHWC bf16); fc1's output
      h1 and the Q-values stay fp32;
    * data gradients: fc1's output delta dh1 feeds the fc1 weight gradient and data
      gradient as bf16 (its bias gradient sums the fp32 values), dY3 / dY2 / dY1
      (post-mask) are stored bf16 and every consumer reads those.

    By default the oracle rounds its own fp64 value at each of those points.  Two
    device inputs can be substituted (teacher forcing; every value is still computed
    by the oracle in fp64 from them):

    * ``masks[k]``: the ReLU mask of layer k (the device's stored activation > 0).  A
      mask bit is a discrete decision on a value that is ~0: where fp32 and fp64 land
      on opposite sides of 0 the whole data gradient of that unit flips, which no
      tolerance on the rest can absorb (a few per 10^4 fc1 units at batch 32);
    * ``acts[k]`` / ``deltas[k]``: the device's stored bf16 tensor at that point.
      Chained bf16 roundings are not well conditioned either: a value within the
      accumulation error of a rounding boundary lands one ulp (2^-8) apart, and each
      rounding stage turns an upstream error e into ~sqrt(e * 2^-8).  With the
      device's stored tensors as the next stage's inputs, each stage is compared on
      identical inputs, and ``seen`` keeps the oracle's own (unrounded) value at every
      point for the stage check.
    """

    def __init__(self, bf16_layers=(0, 1, 2, 3), masks=None, acts=None, deltas=None):
        self.bf16_layers = set(bf16_layers)
        self.masks = masks
        self.acts = acts or {}
        self.deltas = deltas or {}
        self.seen = {}

    @property
    def forced(self) -> bool:
        return self.masks is not None or bool(self.acts)

    def weight(self, k, w):
        return bf16_round(w) if k in self.bf16_layers else w

    def act(self, k, spec, x):
        if spec.layers[k].kind != "conv":
            return x
        self.seen[("act", k)] = x
        if k in self.acts:
            return np.asarray(self.acts[k], dtype=np.float64).reshape(x.shape)
        return bf16_round(x)

    def delta(self, k, x):
        self.seen[("delta", k)] = x
        if k in self.deltas:
            return np.asarray(self.deltas[k], dtype=np.float64).reshape(x.shape)
        return bf16_round(x)

    def relu_mask(self, k, pre):
        if self.masks is not None and k < len(self.masks) and self.masks[k] is not None:
            return np.asarray(self.masks[k], dtype=bool).reshape(pre.shape)
        if k in self.acts:
            return (np.asarray(self.acts[k]) > 0).reshape(pre.shape)
        return pre > 0.0


def init_params(spec: NetSpec, seed: int) -> Params:
    """nn.init_network (nn.py:93-109) over the flattened weight matrices."""
    rng = np.random.default_rng(seed)
    ws, bs = [], []
    for _, _, (o, i) in spec.shapes():
        bound = np.sqrt(6.0 / (i + o))
        ws.append(rng.uniform(-bound, bound, size=(o, i)))
        bs.append(np.zeros(o, dtype=np.float64))
    return Params(ws, bs)


# --- im2col / col2im -------------------------------------------------------------

def _patch_index(L: Layer, in_shape):
    """Flat input index of every (patch row, patch column)."""
    if L.planar:
        c, h, w = in_shape
    else:
        h, w, c = in_shape
    oh = (h - L.k) // L.s + 1
    ow = (w - L.k) // L.s + 1
    oy, ox = np.meshgrid(np.arange(oh), np.arange(ow), indexing="ij")
    oy, ox = oy.reshape(-1, 1), ox.reshape(-1, 1)
    if L.planar:   # columns (c, kh, kw)
        cc, ky, kx = np.meshgrid(np.arange(c), np.arange(L.k), np.arange(L.k), indexing="ij")
        cc, ky, kx = cc.reshape(1, -1), ky.reshape(1, -1), kx.reshape(1, -1)
        return (cc * h + (oy * L.s + ky)) * w + (ox * L.s + kx)
    # columns (kh, kw, c)
    ky, kx, cc = np.meshgrid(np.arange(L.k), np.arange(L.k), np.arange(c), indexing="ij")
    ky, kx, cc = ky.reshape(1, -1), kx.reshape(1, -1), cc.reshape(1, -1)
    return ((oy * L.s + ky) * w + (ox * L.s + kx)) * c + cc


def im2col(x, L: Layer, in_shape):
    """x: [n, prod(in_shape)] -> patches [n*OH*OW, C*k*k] (rows (b, oy, ox))."""
    idx = _patch_index(L, in_shape)
    n = x.shape[0]
    return x.reshape(n, -1)[:, idx].reshape(n * idx.shape[0], idx.shape[1])


def col2im(dpatch, L: Layer, in_shape, n):
    """Scatter-add patch-space gradients back to the input layout.  For every input
    element the contributions are summed in (patch row, patch column) ascending
    order (np.add.at applies the flattened index list sequentially)."""
    idx = _patch_index(L, in_shape)
    out = np.zeros((n, int(np.prod(in_shape))), dtype=np.float64)
    dp = dpatch.reshape(n, idx.size)
    flat = idx.reshape(-1)
    for b in range(n):
        np.add.at(out[b], flat, dp[b])
    return out


def col2im_fast(dpatch, L: Layer, in_shape, n):
    """col2im for NHWC layers as k*k strided slice-adds (fp64 order differs from col2im's
    np.add.at only by rounding; used with the batched kernel module)."""
    h, w, c = in_shape
    oh = (h - L.k) // L.s + 1
    ow = (w - L.k) // L.s + 1
    dp = dpatch.reshape(n, oh, ow, L.k, L.k, c)
    out = np.zeros((n, h, w, c), dtype=np.float64)
    for ky in range(L.k):
        for kx in range(L.k):
            out[:, ky:ky + L.s * (oh - 1) + 1:L.s, kx:kx + L.s * (ow - 1) + 1:L.s, :] += \
                dp[:, :, :, ky, kx, :]
    return out.reshape(n, -1)


# --- forward / gradient ----------------------------------------------------------

def _inputs(spec: NetSpec, states):
    states = np.asarray(states)
    feat = int(np.prod(spec.in_shape))
    if states.ndim == len(spec.in_shape) + 1 or (states.ndim == 2 and states.shape[1] == feat):
        n = states.shape[0]
    else:
        n = 1
    x = states.reshape(n, -1)
    if states.dtype == np.uint8:
        x = x.astype(np.float64) / 255.0
    else:
        x = np.ascontiguousarray(x, dtype=np.float64)
    if x.shape[1] != int(np.prod(spec.in_shape)):
        raise ValueError(f"state batch has {x.shape[1]} features, expected {spec.in_shape}")
    return x


def _layer_rows(spec, k, act, n):
    """GEMM-row view of layer k's input activation."""
    in_shape, _, _ = spec.shapes()[k]
    L = spec.layers[k]
    if L.kind == "conv":
        return im2col(act, L, in_shape)
    return act.reshape(n, -1)


def _weights(p: Params, store):
    if store is None:
        return p.weights
    return [store.weight(k, w) for k, w in enumerate(p.weights)]


def _relu(K, store, k, pre):
    if store is None or not store.forced:
        return K.relu(pre)
    return np.where(store.relu_mask(k, pre), pre, 0.0)


def forward(spec: NetSpec, p: Params, states, K=None, store=None) -> np.ndarray:
    """nn.forward (nn.py:123-131)."""
    K = K or _K_EXACT
    x = _inputs(spec, states)
    n = x.shape[0]
    last = len(spec.layers) - 1
    act = x
    for k, (w, b) in enumerate(zip(_weights(p, store), p.biases)):
        pre = K.affine_rows(w, b, _layer_rows(spec, k, act, n))
        act = _relu(K, store, k, pre) if k < last else pre
        act = act.reshape(n, -1)
        if store is not None and k < last:
            act = store.act(k, spec, act)
    return act


def forward_trace(spec: NetSpec, p: Params, states, K=None, store=None):
    """Forward keeping every layer input (GEMM rows), pre-activation and output."""
    K = K or _K_EXACT
    x = _inputs(spec, states)
    n = x.shape[0]
    last = len(spec.layers) - 1
    rows, pres, acts = [], [], [x]
    for k, (w, b) in enumerate(zip(_weights(p, store), p.biases)):
        r = _layer_rows(spec, k, acts[-1], n)
        pre = K.affine_rows(w, b, r)
        rows.append(r)
        pres.append(pre)
        a = (_relu(K, store, k, pre) if k < last else pre).reshape(n, -1)
        if store is not None and k < last:
            a = store.act(k, spec, a)
        acts.append(a)
    return rows, pres, acts


def huber_delta(q, actions, targets, huber):
    """Output delta of the mean Huber TD loss: clip(q[a] - target, -huber, huber) / n at
    the taken action (the north star's "Huber TD loss"; the reference's half-squared
    loss, _kernels_numpy.py:30-35, is huber = infinity)."""
    n = q.shape[0]
    delta = np.zeros_like(q)
    rows = np.arange(n)
    delta[rows, actions] = np.clip(q[rows, actions] - targets, -huber, huber) / n
    return delta


def gradient(spec: NetSpec, p: Params, states, actions, targets, K=None, store=None,
             huber=None):
    """nn.gradient (nn.py:134-170): exact gradient of the mean half-squared TD error
    (or of the mean Huber loss when ``huber`` is set)."""
    K = K or _K_EXACT
    x = _inputs(spec, states)
    n = x.shape[0]
    actions = np.ascontiguousarray(actions, dtype=np.int64)
    targets = np.ascontiguousarray(targets, dtype=np.float64)
    if actions.shape != (n,) or targets.shape != (n,):
        raise ValueError("states, actions and targets must have matching batch sizes")
    n_out = spec.layers[-1].out
    if actions.size and (actions.min() < 0 or actions.max() >= n_out):
        raise ValueError("action index out of range")
    rows, pres, acts = forward_trace(spec, p, x, K, store)
    weights = _weights(p, store)
    last = len(spec.layers) - 1
    shapes = spec.shapes()
    if huber is None:
        delta = K.output_delta(acts[-1], actions, targets)
    else:
        delta = huber_delta(acts[-1], actions, targets, huber)
    gw = [None] * len(spec.layers)
    gb = [None] * len(spec.layers)
    for k in range(last, -1, -1):
        gb_src = delta
        if store is not None and k < last:
            # the stored (bf16) data gradient feeds this layer's weight gradient and the
            # next data gradient; fc1's bias gradient sums the fp32 values
            delta = store.delta(k, delta)
            if k < last - 1:
                gb_src = delta
        gw[k] = K.weight_grad(delta, rows[k])
        gb[k] = K.bias_grad(gb_src)
        if k == 0:
            break
        L = spec.layers[k]
        in_shape = shapes[k][0]
        prev_pre = pres[k - 1].reshape(n, -1)
        if store is not None:
            prev_pre = store.relu_mask(k - 1, pres[k - 1]).reshape(n, -1).astype(np.float64)
        if L.kind == "fc":
            delta = K.hidden_delta(delta, weights[k], prev_pre)
        else:
            dpatch = K.hidden_delta(delta, weights[k], np.ones_like(rows[k]))
            dx = (col2im_fast if K is not _K_EXACT and not L.planar else col2im)(
                dpatch, L, in_shape, n)
            dx = dx * (prev_pre > 0.0)
            delta = dx
        # delta rows for layer k-1: pixels x channels for a conv, samples x units for fc
        if spec.layers[k - 1].kind == "conv":
            delta = delta.reshape(-1, spec.layers[k - 1].out)
    return Params(gw, gb)


def rmsprop_step(opt: Opt, p: Params, g: Params, lr=2.5e-4, rho=0.95, kappa=0.01, K=None):
    """nn.rmsprop_step (nn.py:173-203)."""
    K = K or _K_EXACT
    for a in g.weights + g.biases:
        if not np.all(np.isfinite(a)):
            raise ValueError("gradient contains non-finite entries")
    nw, nmw, nvw = [], [], []
    for w, gw, m, v in zip(p.weights, g.weights, opt.m_weights, opt.v_weights):
        p2, m2, v2 = K.rmsprop_flat(w.reshape(-1), gw.reshape(-1), m.reshape(-1),
                                    v.reshape(-1), lr, rho, kappa)
        nw.append(p2.reshape(w.shape))
        nmw.append(m2.reshape(w.shape))
        nvw.append(v2.reshape(w.shape))
    nb, nmb, nvb = [], [], []
    for b, gb, m, v in zip(p.biases, g.biases, opt.m_biases, opt.v_biases):
        p2, m2, v2 = K.rmsprop_flat(b, gb, m, v, lr, rho, kappa)
        nb.append(p2)
        nmb.append(m2)
        nvb.append(v2)
    return Params(nw, nb), Opt(nmw, nmb, nvw, nvb, opt.step + 1)


def td_targets(spec, target: Params, rewards, next_states, terminals, gamma, K=None,
               store=None):
    """agent.td_targets (agent.py:69-81)."""
    q_next = forward(spec, target, next_states, K, store)
    out = np.empty(len(rewards), dtype=np.float64)
    for i in range(len(rewards)):
        r = float(rewards[i])
        out[i] = r if terminals[i] else r + gamma * q_next[i].max()
    return out


def train_minibatch(spec, theta: Params, opt: Opt, batch, target: Params, gamma,
                    lr=2.5e-4, rho=0.95, kappa=0.01, *, return_grad=False, K=None, store=None,
                    huber=None, target_store=None):
    """agent.train_minibatch (agent.py:84-105).  batch = (states, actions, rewards,
    next_states, terminals) as arrays."""
    states, actions, rewards, next_states, terminals = batch
    targets = td_targets(spec, target, rewards, next_states, terminals, gamma, K,
                         target_store if target_store is not None else store)
    g = gradient(spec, theta, states, actions, targets, K, store, huber)
    n = float(len(actions))
    summed = Params([w * n for w in g.weights], [b * n for b in g.biases])
    p2, o2 = rmsprop_step(opt, theta, summed, lr, rho, kappa, K)
    if return_grad:
        return p2, o2, summed, targets
    return p2, o2


def loss_value(spec, p, states, actions, targets, K=None):
    q = forward(spec, p, states, K)
    err = targets - q[np.arange(len(actions)), actions]
    return float(np.mean(0.5 * err ** 2))


def copy_params(p: Params) -> Params:
    return Params([w.copy() for w in p.weights], [b.copy() for b in p.biases])


FNV_OFFSET = 0xCBF29CE484222325
FNV_PRIME = 0x100000001B3


def parameter_bytes(p: Params) -> bytes:
    """nn.parameter_bytes (nn.py:214-220): LE f64, per layer weights then bias."""
    out = []
    for w, b in zip(p.weights, p.biases):
        out.append(np.ascontiguousarray(w, dtype="<f8").tobytes())
        out.append(np.ascontiguousarray(b, dtype="<f8").tobytes())
    return b"".join(out)


def theta_hash(p: Params) -> str:
    """nn.theta_hash (nn.py:223-229): 64-bit FNV-1a, 16 hex digits."""
    h = FNV_OFFSET
    for byte in parameter_bytes(p):
        h ^= byte
        h = (h * FNV_PRIME) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"
