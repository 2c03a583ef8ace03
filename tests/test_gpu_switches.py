"""The switch-selected GPU paths stay correct (each runs in a subprocess because the
switches are read once per process):

* PQ_TMA=1 — the warp-specialised TMA engine forced at batch 32 (default: from 128):
  Q-values bit-identical, one learner step within fp32 summation order (1e-5) of the
  cp.async engine;
* PQ_C1SHIFT=0 — the conv layers by TMA im2col / cp.async gathers instead of row-shifted
  descriptors (batch >= 128): the conv1/2/3 forward and the conv2 data gradient run the
  same MMA sequences, so Q-values are bit-identical; the conv1/conv2 weight gradients sum
  the padded grids in other K chunks and splits, so the learner update agrees to fp32
  summation order (1e-5);
* PQ_FUSED=0 — the multi-stream learner backward instead of the single-stream fused
  launches (batch < 128): the same GEMMs and reductions, bit-identical update."""

import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PROBE = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import torch
from paper_2111_01264_b200 import nn as dnn
from paper_2111_01264_b200.envs import FrameEnvSpec
from paper_2111_01264_b200.replay import ReplayMemory
W, B = int(sys.argv[3]), int(sys.argv[4])
net = dnn.init_network(dnn.network_sizes(), 5)
x = np.random.default_rng(1).integers(0, 256, size=(W, 4, 84, 84), dtype=np.uint8)
q = dnn.forward(net, x)
mem = ReplayMemory(4096)
mem.prepopulate(FrameEnvSpec(key=3), 2000, np.random.default_rng(2))
theta, target = dnn.init_network(dnn.network_sizes(), 6), dnn.init_network(dnn.network_sizes(), 7)
idx = mem.sample_indices(B, np.random.default_rng(4))
th2, _, _, _, _ = dnn._learn(theta, dnn.OptState.zeros(theta), target, mem.ring, mem.records, idx, B)
np.savez(sys.argv[2], q=q, theta=th2.master.cpu().numpy(), theta0=theta.master.cpu().numpy())
"""


def run_probe(tmp_path, name, env, W=24, B=32):
    out = tmp_path / f"{name}.npz"
    e = dict(os.environ)
    e.update(env)
    subprocess.run([sys.executable, "-c", PROBE, ROOT, str(out), str(W), str(B)], check=True, env=e, timeout=600)
    return np.load(out)


def test_forced_tma_matches_default(tmp_path):
    base = run_probe(tmp_path, "base", {"PQ_TMA": "0"})
    tma = run_probe(tmp_path, "tma", {"PQ_TMA": "1"})
    assert np.array_equal(tma["q"], base["q"])
    d = base["theta"] - base["theta0"]
    assert np.linalg.norm(tma["theta"] - base["theta"]) <= 1e-5 * np.linalg.norm(d)


def test_conv1_shift_matches_im2col(tmp_path):
    shift = run_probe(tmp_path, "shift", {"PQ_C1SHIFT": "1"}, W=200, B=256)
    im2col = run_probe(tmp_path, "im2col", {"PQ_C1SHIFT": "0"}, W=200, B=256)
    assert np.array_equal(shift["q"], im2col["q"])
    d = im2col["theta"] - im2col["theta0"]
    assert np.linalg.norm(shift["theta"] - im2col["theta"]) <= 1e-5 * np.linalg.norm(d)


def test_fused_backward_matches_multistream(tmp_path):
    fused = run_probe(tmp_path, "fused_bw", {"PQ_FUSED": "1"})
    multi = run_probe(tmp_path, "multi_bw", {"PQ_FUSED": "0"})
    assert np.array_equal(fused["q"], multi["q"])
    assert np.array_equal(fused["theta"], multi["theta"])


@pytest.mark.parametrize("graphs", [False, True])
def test_pipelined_target_forward_is_bit_identical(graphs, monkeypatch):
    """PQ_PIPE_TARGET (executor, default on): the target network's forward of step k+1 runs
    inside step k's backward launches; epoch after epoch the parameters must match the
    unpipelined learner bit for bit (theta hash per epoch and at the end)."""
    from paper_2111_01264_b200.agent import EpsilonSchedule, HyperParams
    from paper_2111_01264_b200.executor import run

    hp = HyperParams(C=400, F=4, N=2000, W=8, batch_size=32, total_steps=1200, capacity=5000, seed=3,
                     schedule=EpsilonSchedule(1.0, 0.1, 600), eval_period=0)
    recs = []
    for flag in ("0", "1"):
        monkeypatch.setenv("PQ_PIPE_TARGET", flag)
        recs.append(run(hp, use_graphs=graphs, graph_chunk=25))
    assert recs[0].epoch_hashes == recs[1].epoch_hashes
    assert recs[0].final_hash == recs[1].final_hash



@pytest.mark.parametrize("graphs", [False, True])
def test_sm_partitioned_acting_is_bit_identical(graphs, monkeypatch):
    """PQ_ACT_SMS (executor): the acting stream on a green-context SM partition
    (pq_sm_partition_stream) changes only where the acting blocks run -- replay records,
    episode log and parameters match the default run bit for bit."""
    from paper_2111_01264_b200.agent import EpsilonSchedule, HyperParams
    from paper_2111_01264_b200.executor import run

    hp = HyperParams(C=400, F=4, N=2000, W=8, batch_size=32, total_steps=1200, capacity=5000, seed=4,
                     schedule=EpsilonSchedule(1.0, 0.1, 600), eval_period=0)
    recs = []
    for sms in ("0", "16"):
        monkeypatch.setenv("PQ_ACT_SMS", sms)
        recs.append(run(hp, use_graphs=graphs, graph_chunk=25))
    assert recs[0].epoch_hashes == recs[1].epoch_hashes
    assert recs[0].final_hash == recs[1].final_hash
    assert recs[0].to_csv_text() == recs[1].to_csv_text()
