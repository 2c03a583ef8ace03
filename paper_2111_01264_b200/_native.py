"""ctypes binding of the sm_100a C-ABI library (include/paraq_b200.h).

The library is built in-tree by ``make`` (or ``__graft_entry__.build()``) into
``paper_2111_01264_b200/_lib/libparaq_b200.so``.  There is no fallback: if the
library or a CUDA device is missing, every device entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libparaq_b200.so")

_lib = None

u8p = C.POINTER(C.c_uint8)
vp = C.c_void_p


class PqNet(C.Structure):
    _fields_ = [("master", vp), ("shadow", vp)]


class PqOpt(C.Structure):
    _fields_ = [("m", vp), ("v", vp)]


class PqEnvs(C.Structure):
    _fields_ = [(n, vp) for n in ("pcg", "episode", "t", "stack", "ep_return", "key",
                                  "slot_next", "ep_count", "ep_label", "ep_ret", "actions",
                                  "reset_next", "reset_ep", "reset_slot")]


class PqHenv(C.Structure):
    _fields_ = [("pcg", C.c_uint64 * 6), ("key", C.c_uint64), ("episode", C.c_int64),
                ("t", C.c_int32), ("pad", C.c_int32), ("ep_return", C.c_double)]


class PqLearnArgs(C.Structure):
    _fields_ = [
        ("theta", PqNet), ("opt", PqOpt), ("theta_out", PqNet), ("opt_out", PqOpt),
        ("target", PqNet),
        ("ring", vp), ("records", vp), ("idx", vp), ("idx_base", vp), ("update_counter", vp),
        ("ext_targets", vp), ("ext_actions", vp),
        ("n", C.c_int), ("actions", C.c_int),
        ("gamma", C.c_float), ("lr", C.c_float), ("rho", C.c_float), ("kappa", C.c_float),
        ("nonfinite", vp), ("grad_out", vp), ("q_out", vp), ("td_out", vp),
        ("ws", vp), ("max_batch", C.c_int), ("huber", C.c_float),
    ]


class PqActArgs(C.Structure):
    _fields_ = [
        ("net", PqNet), ("envs", PqEnvs), ("ring", vp), ("staging", vp), ("step_counter", vp),
        ("W", C.c_int), ("steps", C.c_int), ("actions", C.c_int), ("episode_length", C.c_int),
        ("epoch_start", C.c_int64), ("frame_capacity", C.c_int64),
        ("eps_start", C.c_double), ("eps_end", C.c_double), ("eps_anneal", C.c_int64),
        ("terminal_p", C.c_double), ("q_out", vp), ("ws", vp), ("max_batch", C.c_int),
        ("max_episodes", C.c_int), ("sampler0", C.c_int), ("W_total", C.c_int),
    ]


EXPORTS = {
    "pq_abi_version": ([], C.c_int),
    "pq_last_error": ([], C.c_char_p),
    "pq_num_params": ([C.c_int], C.c_int64),
    "pq_num_shadow": ([], C.c_int64),
    "pq_timeline": ([C.c_int, vp, vp], C.c_int),
    "pq_timeline_tma": ([C.c_int, vp, vp], C.c_int),
    "pq_cta_trace": ([C.c_int, vp, vp], C.c_int),
    "pq_net_sync_shadow": ([PqNet, vp], C.c_int),
    "pq_net_copy": ([PqNet, PqNet, C.c_int, vp], C.c_int),
    "pq_l2_persist": ([vp, vp, C.c_size_t, C.c_float], C.c_int),
    "pq_sample_indices": ([vp, C.c_uint32, C.c_int64, vp, vp], C.c_int),
    "pq_replay_gather": ([vp, vp, vp, C.c_int64, vp, vp, vp, vp, vp, vp], C.c_int),
    "pq_replay_gather_tma": ([vp, vp, vp, C.c_int64, vp, vp, vp, vp, vp, vp], C.c_int),
    "pq_replay_gather_ldg": ([vp, vp, vp, C.c_int64, vp, vp, vp, vp, vp, vp], C.c_int),
    "pq_replay_flush": ([vp, C.c_int, C.c_int, vp, C.c_int64, C.c_int64, vp], C.c_int),
    "pq_replay_flush_range": ([vp, C.c_int, C.c_int, C.c_int, C.c_int, vp, C.c_int64, C.c_int64,
                               vp], C.c_int),
    "pq_env_reset": ([PqEnvs, C.c_int, vp, vp, vp], C.c_int),
    "pq_prepopulate": ([vp, C.c_uint64, C.c_int, C.c_int, C.c_double, C.c_int64, vp, C.c_int64,
                        C.c_int64, vp, vp, vp, vp], C.c_int),
    "pq_prepopulate_walk": ([vp, C.c_int, C.c_int, C.c_double, C.c_int64, C.c_int64, C.c_int64, vp, vp,
                             vp, vp], C.c_int),
    "pq_prepopulate_frames": ([C.c_uint64, vp, C.c_int64, C.c_int64, vp, vp, vp], C.c_int),
    "pq_prepopulate_scratch_bytes": ([C.c_int64], C.c_size_t),
    "pq_workspace_bytes": ([C.c_int, C.c_int], C.c_size_t),
    "pq_fc1_splits": ([C.c_int, C.c_int], C.c_int),
    "pq_workspace_layout": ([C.c_int, C.c_int, C.POINTER(C.c_int64)], C.c_int),
    "pq_forward": ([PqNet, vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, vp, vp, C.c_int, vp],
                   C.c_int),
    "pq_learn_step": ([C.POINTER(PqLearnArgs), vp], C.c_int),
    "pq_learn_step_pipelined": ([C.POINTER(PqLearnArgs), vp], C.c_int),
    "pq_learn_target_prologue": ([C.POINTER(PqLearnArgs), vp], C.c_int),
    "pq_act_step": ([C.POINTER(PqActArgs), vp], C.c_int),
    "pq_learn_grad": ([C.POINTER(PqLearnArgs), vp, vp], C.c_int),
    "pq_learn_grad_ev": ([C.POINTER(PqLearnArgs), vp, vp, vp], C.c_int),
    "pq_rmsprop_apply": ([PqNet, PqOpt, vp, C.c_int, C.c_float, C.c_float, C.c_float, vp, C.c_int, vp],
                         C.c_int),
    "pq_rmsprop_f32": ([vp, vp, vp, vp, C.c_int64, C.c_float, C.c_float, C.c_float, vp, vp, vp,
                        vp, vp], C.c_int),
    "pq_henv_reset": ([vp, C.c_int, vp, C.c_int64, vp, vp], C.c_int),
    "pq_henv_step": ([vp, C.c_int, vp, C.c_int, C.c_int, C.c_double, C.c_int64, C.c_double,
                      C.c_double, C.c_int64, vp, C.c_int64, vp, vp, vp, vp, vp, vp, vp], C.c_int),
    "pq64_affine_rows": ([vp, vp, vp, C.c_int64, C.c_int64, C.c_int64, vp, vp], C.c_int),
    "pq64_relu": ([vp, C.c_int64, vp, vp], C.c_int),
    "pq64_output_delta": ([vp, vp, vp, C.c_int64, C.c_int64, vp, vp], C.c_int),
    "pq64_weight_grad": ([vp, vp, C.c_int64, C.c_int64, C.c_int64, vp, vp], C.c_int),
    "pq64_bias_grad": ([vp, C.c_int64, C.c_int64, vp, vp], C.c_int),
    "pq64_hidden_delta": ([vp, vp, vp, C.c_int64, C.c_int64, C.c_int64, vp, vp], C.c_int),
    "pq64_rmsprop_flat": ([vp, vp, vp, vp, C.c_int64, C.c_double, C.c_double, C.c_double, vp,
                           vp, vp, vp], C.c_int),
    "pq_theta_hash_f32": ([vp, C.c_int64], C.c_uint64),
    "pq_theta_hash_f64": ([vp, C.c_int64], C.c_uint64),
    "pq_sm_partition_stream": ([C.c_int, C.POINTER(vp), C.POINTER(C.c_int)], C.c_int),
}


class NativeError(RuntimeError):
    pass


def load(path: str | None = None):
    """Load and type the library (no GPU needed to load it).  PQ_LIB overrides the path
    (profiling: the probe build from ``make probes``)."""
    global _lib
    if _lib is None:
        path = path or os.environ.get("PQ_LIB") or LIB_PATH
        if not os.path.exists(path):
            raise NativeError(
                f"{path} is missing: build the sm_100a library first (make, or "
                "python -c 'import __graft_entry__ as g; g.build()')")
        lib = C.CDLL(path)
        for name, (args, res) in EXPORTS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
    return _lib


def check(rc: int, what: str = "", value_error: bool = False) -> None:
    if rc != 0:
        msg = load().pq_last_error().decode(errors="replace")
        exc = ValueError if (value_error or rc == 1) else NativeError
        raise exc(f"{what}: {msg}" if what else msg)


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise NativeError("paper_2111_01264_b200 needs a CUDA device (sm_100a); none is visible")
    major, minor = torch.cuda.get_device_capability()
    if major != 10:
        raise NativeError(f"this build targets sm_100a; found compute capability {major}.{minor}")
    return torch


def sm_partition_stream(sm_count: int):
    """A torch stream whose kernels run on a green-context partition of >= sm_count SMs
    (multiples of 8 on sm_100a); kept alive for the process (pq_sm_partition_stream)."""
    import torch

    key = (torch.cuda.current_device(), int(sm_count))
    if key not in _PARTITIONS:  # one green context per (device, size) for the process
        p, got = vp(), C.c_int(0)
        check(load().pq_sm_partition_stream(int(sm_count), C.byref(p), C.byref(got)), "sm partition stream")
        s = torch.cuda.ExternalStream(p.value)
        s.sm_count = got.value
        _PARTITIONS[key] = s
    return _PARTITIONS[key]


_PARTITIONS: dict = {}


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


WS_BUFFERS = ("act1", "act2", "act3", "fc1part", "act1_t", "act2_t", "act3_t", "fc1part_t", "q",
              "h1", "dh1", "td", "dh1_bf", "dh1T", "act", "dY3", "dY2", "dY1", "part1", "part2",
              "part3", "grad4", "dY1p", "dY2p", "act1s2", "act1s2_t")


def workspace_layout(max_batch: int, actions: int) -> dict:
    offs = (C.c_int64 * len(WS_BUFFERS))()
    load().pq_workspace_layout(max_batch, actions, offs)
    return dict(zip(WS_BUFFERS, list(offs)))


def ptr(t) -> int:
    return 0 if t is None else t.data_ptr()
