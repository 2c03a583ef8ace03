"""B200-native fast-DQN hot path (arXiv 2111.01264: concurrent training +
synchronized execution), drop-in for the reference `paraq` agent / replay /
trainer API.  Hot ops are hand-written sm_100a kernels (tcgen05/TMEM implicit
GEMMs, numpy-exact PCG64 replay sampling, fused acting + env step, fused
centered RMSProp) behind the C ABI in include/paraq_b200.h.

Importing the package needs no GPU; every device entry point raises if the
in-tree library or a CUDA device is missing (no CPU fallback).
"""

from . import _native
from .agent import EpsilonSchedule, HyperParams, MODES, epsilon_at, select_action, \
    target_update, td_targets, train_minibatch
from .nn import OptConfig, OptState, Parameters, QNet, copy_parameters, forward, gradient, \
    init_network, load_parameters, network_sizes, num_params, parameter_bytes, rmsprop_step, \
    save_parameters, theta_hash

BACKEND = "b200"
__version__ = "0.1.0"


def __getattr__(name):
    # executor / replay / envs pull in torch lazily
    if name in ("ReplayMemory", "SampleBuffer", "Transition", "Batch"):
        from . import replay

        return getattr(replay, name)
    if name in ("run", "sequential_reference", "DeviceRun", "HostEnvRun", "InferenceWorker",
                "RunRecord", "batched_inference", "transaction_count", "transaction_breakdown",
                "rng_stream", "derived_seed"):
        from . import executor

        return getattr(executor, name)
    if name in ("FrameEnvSpec", "DeviceEnvs"):
        from . import envs

        return getattr(envs, name)
    raise AttributeError(name)
