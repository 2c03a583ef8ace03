"""Device-resident Nature-CNN Q-network with the reference's numeric-core API.

Mirrors pkg/src/paraq/nn.py (names, argument meaning, error behaviour):

* ``init_network``  -- nn.py:93-109: U(+-sqrt(6/(fan_in+fan_out))) per flattened
  (out, in*kh*kw) weight matrix drawn from default_rng(seed), zero biases.
* ``forward``       -- nn.py:123-131 (tcgen05 implicit-GEMM conv/FC on the B200).
* ``gradient``      -- nn.py:134-170: mean half-squared TD-error gradient.
* ``rmsprop_step``  -- nn.py:173-203: centered RMSProp, raises ValueError on a
  non-finite gradient, returns fresh Parameters / OptState.
* ``copy_parameters``, ``parameter_bytes``, ``theta_hash`` -- nn.py:206-229.

Parameters live on the GPU as an fp32 master vector in nn.parameter_bytes order
plus bf16 shadow copies of the conv1..fc1 weights that the tensor-core GEMMs read.
Arithmetic is bf16 x bf16 -> fp32 on the tensor cores, fp32 elsewhere; parity with
the fp64 reference is a stated tolerance (tests/test_gpu_parity.py).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _native as N

FRAME = 84
STACK = 4
FRAME_BYTES = FRAME * FRAME
HIDDEN = 512
STATE_DIM = STACK * FRAME_BYTES


def layer_shapes(actions: int = 18):
    """Flattened (out, in) weight shapes: conv1, conv2, conv3, fc1, fc2."""
    return [(32, 4 * 8 * 8), (64, 4 * 4 * 32), (64, 3 * 3 * 64), (512, 3136), (actions, 512)]


def num_params(actions: int = 18) -> int:
    return sum(o * i + o for o, i in layer_shapes(actions))


@dataclass
class Parameters:
    """Host view: layered weights (out, in) and biases, float64 (nn.py:24-45)."""

    weights: list
    biases: list

    @property
    def n_layers(self) -> int:
        return len(self.weights)

    @property
    def output_dim(self) -> int:
        return self.weights[-1].shape[0]

    def flat(self) -> np.ndarray:
        parts = []
        for w, b in zip(self.weights, self.biases):
            parts.append(np.asarray(w, dtype=np.float64).reshape(-1))
            parts.append(np.asarray(b, dtype=np.float64).reshape(-1))
        return np.concatenate(parts)

    @classmethod
    def from_flat(cls, flat: np.ndarray, actions: int) -> "Parameters":
        ws, bs, off = [], [], 0
        for o, i in layer_shapes(actions):
            ws.append(np.asarray(flat[off:off + o * i], dtype=np.float64).reshape(o, i).copy())
            off += o * i
            bs.append(np.asarray(flat[off:off + o], dtype=np.float64).copy())
            off += o
        return cls(ws, bs)


Gradients = Parameters


@dataclass
class OptConfig:
    """Centered-RMSProp constants (nn.py:56-70)."""

    learning_rate: float = 2.5e-4
    rho: float = 0.95
    kappa: float = 0.01

    def validate(self) -> None:
        if not self.learning_rate > 0:
            raise ValueError("learning rate must be positive")
        if not 0.0 <= self.rho < 1.0:
            raise ValueError("rho must lie in [0, 1)")
        if not self.kappa > 0:
            raise ValueError("kappa must be positive")


def _torch():
    return N.require_cuda()


class QNet:
    """One device-resident parameter set (theta or theta-minus)."""

    def __init__(self, master, shadow, actions: int):
        self.master = master          # torch.float32 [P]
        self.shadow = shadow          # torch.int16 (bf16 bits) [S]
        self.actions = actions

    # -- construction --------------------------------------------------------------
    @classmethod
    def empty(cls, actions: int = 18) -> "QNet":
        torch = _torch()
        lib = N.load()
        master = torch.zeros(lib.pq_num_params(actions), dtype=torch.float32, device="cuda")
        shadow = torch.zeros(lib.pq_num_shadow(), dtype=torch.int16, device="cuda")
        return cls(master, shadow, actions)

    @classmethod
    def from_flat(cls, flat, actions: int = 18) -> "QNet":
        torch = _torch()
        net = cls.empty(actions)
        src = torch.as_tensor(np.asarray(flat, dtype=np.float32))
        if src.numel() != net.master.numel():
            raise ValueError(f"expected {net.master.numel()} parameters, got {src.numel()}")
        net.master.copy_(src)
        net.sync_shadow()
        return net

    @classmethod
    def from_params(cls, params: Parameters) -> "QNet":
        return cls.from_flat(params.flat(), params.output_dim)

    def sync_shadow(self, stream=None) -> None:
        N.check(N.load().pq_net_sync_shadow(self.struct(), N.stream_ptr(stream)), "sync_shadow")

    def struct(self) -> N.PqNet:
        return N.PqNet(self.master.data_ptr(), self.shadow.data_ptr())

    # -- host views ----------------------------------------------------------------
    def flat(self) -> np.ndarray:
        return self.master.detach().cpu().numpy().astype(np.float64)

    def to_params(self) -> Parameters:
        return Parameters.from_flat(self.flat(), self.actions)

    @property
    def weights(self):
        return self.to_params().weights

    @property
    def biases(self):
        return self.to_params().biases

    @property
    def n_layers(self) -> int:
        return 5

    @property
    def output_dim(self) -> int:
        return self.actions

    def copy(self) -> "QNet":
        dst = QNet(self.master.clone(), self.shadow.clone(), self.actions)
        return dst


@dataclass
class OptState:
    """Per-parameter first (m) and second (v) moments, device fp32 (nn.py:73-90)."""

    m: object
    v: object
    step: int = 0

    @classmethod
    def zeros(cls, params: QNet) -> "OptState":
        torch = _torch()
        return cls(torch.zeros_like(params.master), torch.zeros_like(params.master))

    def struct(self) -> N.PqOpt:
        return N.PqOpt(self.m.data_ptr(), self.v.data_ptr())


def network_sizes(actions: int = 18) -> list:
    """The reference's layer-size list for this network: [state_dim, hidden, actions]
    (executor.py:352-354 builds it from the env and hp.hidden)."""
    return [STATE_DIM, HIDDEN, int(actions)]


def init_network(layer_sizes, seed: int) -> QNet:
    """nn.init_network(layer_sizes, seed) (nn.py:93-109) over the flattened Nature-CNN
    weight matrices.  layer_sizes is the reference's [state_dim, hidden, actions] list:
    state_dim must be 4*84*84 (uint8 frame stacks) and hidden 512 (fc1); the conv stack
    between them is the Nature-CNN's."""
    sizes = [int(s) for s in layer_sizes]
    if len(sizes) != 3 or sizes[0] != STATE_DIM or sizes[1] != HIDDEN:
        raise ValueError(f"layer sizes must be [{STATE_DIM}, {HIDDEN}, actions] "
                         f"(Nature-CNN over 4x84x84 frames); got {list(layer_sizes)}")
    actions = sizes[2]
    if not 1 <= actions <= 32:
        raise ValueError("actions must lie in [1, 32]")
    rng = np.random.default_rng(seed)
    parts = []
    for o, i in layer_shapes(actions):
        bound = np.sqrt(6.0 / (i + o))
        parts.append(rng.uniform(-bound, bound, size=(o, i)).reshape(-1))
        parts.append(np.zeros(o, dtype=np.float64))
    return QNet.from_flat(np.concatenate(parts), actions)


# ------------------------------------------------------------------- workspaces
_WS: dict = {}


def workspace(max_batch: int, actions: int):
    """Cached device workspace for batches up to max_batch (rounded up to 64)."""
    torch = _torch()
    cap = max(64, 1 << (int(max_batch) - 1).bit_length())
    key = (cap, actions, torch.cuda.current_device())
    if key not in _WS:
        nbytes = N.load().pq_workspace_bytes(cap, actions)
        _WS[key] = (torch.zeros(nbytes, dtype=torch.uint8, device="cuda"), cap)
    return _WS[key]


def _stage_states(states):
    """Host or device uint8 states [n, 4, 84, 84] -> (ring [4n, 7056], refs [n, 4])."""
    torch = _torch()
    if isinstance(states, np.ndarray) or not hasattr(states, "is_cuda"):
        arr = np.asarray(states)
        if arr.dtype != np.uint8:
            raise ValueError("states must be uint8 frame stacks")
        if arr.ndim == 3:
            arr = arr[None]
        if arr.ndim != 4 or arr.shape[1:] != (STACK, FRAME, FRAME):
            raise ValueError(f"state batch has shape {arr.shape}, expected (n, 4, 84, 84)")
        t = torch.from_numpy(np.ascontiguousarray(arr)).cuda(non_blocking=False)
    else:
        t = states
        if t.dim() == 3:
            t = t.unsqueeze(0)
        if t.dtype != torch.uint8 or tuple(t.shape[1:]) != (STACK, FRAME, FRAME):
            raise ValueError(f"state batch has shape {tuple(t.shape)}, expected (n, 4, 84, 84)")
        t = t.contiguous()
    n = t.shape[0]
    ring = t.view(n * STACK, FRAME_BYTES)
    refs = torch.arange(n * STACK, dtype=torch.int32, device="cuda").view(n, STACK)
    return ring, refs, n


def forward(params: QNet, states):
    """Q-values for a batch of uint8 frame stacks, one row per state (nn.forward)."""
    torch = _torch()
    was_numpy = not hasattr(states, "is_cuda")
    ring, refs, n = _stage_states(states)
    ws, cap = workspace(n, params.actions)
    q = torch.empty((n, params.actions), dtype=torch.float32, device="cuda")
    N.check(N.load().pq_forward(params.struct(), ring.data_ptr(), refs.data_ptr(), None, 4, 0, n,
                                params.actions, q.data_ptr(), ws.data_ptr(), cap,
                                N.stream_ptr()), "forward")
    if was_numpy:
        return q.cpu().numpy().astype(np.float64)
    return q


def huber_arg(huber) -> float:
    """The C ABI's Huber knob: 0 = the reference's half-squared TD loss."""
    if huber is None or huber == float("inf"):
        return 0.0
    if not huber > 0:
        raise ValueError("huber delta must be positive (or None for the squared loss)")
    return float(huber)


def _learn(theta: QNet, opt: OptState, target: QNet | None, ring, records, idx, n,
           gamma=0.99, cfg: OptConfig | None = None, ext_targets=None, ext_actions=None,
           theta_out=None, opt_out=None, want_grad=False, want_q=False, flag=None,
           update_counter=None, idx_base=None, stream=None, huber=None):
    torch = _torch()
    cfg = cfg or OptConfig()
    A = theta.actions
    ws, cap = workspace(n, A)
    if theta_out is None:
        theta_out = QNet.empty(A)
    if opt_out is None:
        opt_out = OptState(torch.empty_like(opt.m), torch.empty_like(opt.v), opt.step)
    own_flag = flag is None
    if own_flag:
        flag = torch.full((1,), 2**31 - 1, dtype=torch.int32, device="cuda")
    grad = torch.empty_like(theta.master) if want_grad else None
    qout = torch.empty((2, n, A), dtype=torch.float32, device="cuda") if want_q else None
    td = torch.empty((n, 3), dtype=torch.float32, device="cuda") if want_q else None
    tgt = target if target is not None else theta
    a = N.PqLearnArgs(
        theta=theta.struct(), opt=opt.struct(), theta_out=theta_out.struct(),
        opt_out=opt_out.struct(), target=tgt.struct(), ring=N.ptr(ring), records=N.ptr(records),
        idx=N.ptr(idx), idx_base=N.ptr(idx_base), update_counter=N.ptr(update_counter),
        ext_targets=N.ptr(ext_targets), ext_actions=N.ptr(ext_actions), n=n, actions=A,
        gamma=gamma, lr=cfg.learning_rate, rho=cfg.rho, kappa=cfg.kappa,
        nonfinite=flag.data_ptr(), grad_out=N.ptr(grad), q_out=N.ptr(qout), td_out=N.ptr(td),
        ws=ws.data_ptr(), max_batch=cap, huber=huber_arg(huber))
    N.check(N.load().pq_learn_step(ctypes.byref(a), N.stream_ptr(stream)), "learn_step")
    if own_flag and int(flag.item()) != 2**31 - 1:
        raise ValueError("gradient contains non-finite entries")
    opt_out.step = opt.step + 1
    return theta_out, opt_out, grad, qout, td


def _check_batch(params, states, actions, targets):
    actions = np.ascontiguousarray(actions, dtype=np.int64).reshape(-1)
    targets = np.ascontiguousarray(targets, dtype=np.float64).reshape(-1)
    n = np.asarray(states).shape[0] if np.asarray(states).ndim == 4 else 1
    if actions.shape != (n,) or targets.shape != (n,):
        raise ValueError("states, actions and targets must have matching batch sizes")
    if actions.size and (actions.min() < 0 or actions.max() >= params.actions):
        raise ValueError("action index out of range")
    return actions, targets, n


def gradient(params: QNet, states, actions, targets) -> Gradients:
    """Gradient of the mean half-squared TD error (nn.gradient, nn.py:134-170)."""
    torch = _torch()
    actions, targets, n = _check_batch(params, states, actions, targets)
    ring, refs, _ = _stage_states(states)
    # records [n][8]: frames f0..f3 of state b; f4 unused (fixed-target mode)
    rec = torch.full((n, 8), -1, dtype=torch.int32, device="cuda")
    rec[:, :4] = refs
    at = torch.as_tensor(actions.astype(np.int32)).cuda()
    tt = torch.as_tensor(targets.astype(np.float32)).cuda()
    _, _, g, _, _ = _learn(params, OptState.zeros(params), None, ring, rec, None, n,
                           ext_targets=tt, ext_actions=at, want_grad=True)
    return Parameters.from_flat(g.cpu().numpy().astype(np.float64) / n, params.actions)


def rmsprop_step(opt: OptState, cfg: OptConfig, params: QNet, grad) -> tuple:
    """One centered-RMSProp update; returns fresh (QNet, OptState) (nn.py:173-203)."""
    torch = _torch()
    if isinstance(grad, Parameters):
        flat = grad.flat()
        if not np.all(np.isfinite(flat)):
            raise ValueError("gradient contains non-finite entries")
        g = torch.as_tensor(flat.astype(np.float32)).cuda()
    else:
        g = grad
    flag = torch.full((1,), 2**31 - 1, dtype=torch.int32, device="cuda")
    out = QNet.empty(params.actions)
    m2, v2 = torch.empty_like(opt.m), torch.empty_like(opt.v)
    N.check(N.load().pq_rmsprop_f32(params.master.data_ptr(), g.data_ptr(), opt.m.data_ptr(),
                                    opt.v.data_ptr(), params.master.numel(), cfg.learning_rate,
                                    cfg.rho, cfg.kappa, out.master.data_ptr(), m2.data_ptr(),
                                    v2.data_ptr(), flag.data_ptr(), N.stream_ptr()), "rmsprop")
    if int(flag.item()) != 2**31 - 1:
        raise ValueError("gradient contains non-finite entries")
    out.sync_shadow()
    return out, OptState(m2, v2, opt.step + 1)


def copy_parameters(source: QNet) -> QNet:
    """Deep, independent device copy (nn.py:206-211)."""
    return source.copy()


def copy_into(dst: QNet, src: QNet, stream=None) -> None:
    """theta-minus <- theta in place (the executor's per-epoch target sync)."""
    N.check(N.load().pq_net_copy(dst.struct(), src.struct(), src.actions, N.stream_ptr(stream)),
            "net_copy")


def parameter_bytes(params) -> bytes:
    """Little-endian float64 bytes in layer order, weights then bias (nn.py:214-220)."""
    flat = params.flat() if hasattr(params, "flat") else Parameters(*params).flat()
    return np.ascontiguousarray(flat, dtype="<f8").tobytes()


def theta_hash(params) -> str:
    """64-bit FNV-1a over parameter_bytes as 16 hex digits (nn.py:223-229), in C."""
    if not isinstance(params, np.ndarray):
        params = params.flat() if hasattr(params, "flat") else params
    flat = np.ascontiguousarray(params, dtype="<f8")
    h = N.load().pq_theta_hash_f64(flat.ctypes.data, flat.size)
    return f"{h:016x}"


PARAMS_MAGIC = b"PQNET1\x00\x00"


def save_parameters(path, params) -> None:
    """The reference PQNET1 format (nn.py:232-241)."""
    p = params.to_params() if isinstance(params, QNet) else params
    with open(path, "wb") as fh:
        fh.write(PARAMS_MAGIC)
        fh.write(np.uint32(p.n_layers).tobytes())
        for w in p.weights:
            fh.write(np.asarray(w.shape, dtype="<u4").tobytes())
        fh.write(parameter_bytes(p))


def load_parameters(path) -> Parameters:
    """nn.load_parameters (nn.py:244-259)."""
    with open(path, "rb") as fh:
        if fh.read(len(PARAMS_MAGIC)) != PARAMS_MAGIC:
            raise ValueError(f"{path}: not a parameter file")
        (n_layers,) = np.frombuffer(fh.read(4), dtype="<u4")
        shapes = [tuple(np.frombuffer(fh.read(8), dtype="<u4")) for _ in range(n_layers)]
        ws, bs = [], []
        for o, i in shapes:
            ws.append(np.frombuffer(fh.read(8 * o * i), dtype="<f8").reshape(o, i).copy())
            bs.append(np.frombuffer(fh.read(8 * o), dtype="<f8").copy())
    return Parameters(ws, bs)
