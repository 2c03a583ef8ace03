"""Host-side logic of the package (no GPU): configuration validation, the epsilon
schedule and select_action discipline, parameter files, run-record format, and the
multi-process plumbing (gloo, world_size 2)."""

import os

import numpy as np
import pytest

from paper_2111_01264_b200 import dist as pdist
from paper_2111_01264_b200.agent import EpsilonSchedule, HyperParams, epsilon_at, select_action
from paper_2111_01264_b200.executor import RunRecord, transaction_count
from paper_2111_01264_b200.nn import Parameters, layer_shapes, load_parameters, num_params, \
    save_parameters, theta_hash

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_select_action_matches_reference_golden():
    """agent.py:53-66 draw discipline, against the reference's recorded sequence."""
    g = np.load(os.path.join(GOLD, "pcg64.npz"))
    from paper_2111_01264_b200.replay import pcg_state_to_generator, pcg_state_from_generator

    rng = np.random.default_rng(0)
    pcg_state_to_generator(g["sel_s0"], rng)
    acts = [select_action(g["sel_q"][i], float(g["sel_eps"][i]), rng) for i in range(500)]
    assert np.array_equal(acts, g["sel_out"])
    assert np.array_equal(pcg_state_from_generator(rng), g["sel_s1"])


def test_epsilon_schedule():
    """pkg/tests/test_agent.py epsilon cases."""
    s = EpsilonSchedule(1.0, 0.1, 10)
    assert epsilon_at(1, s) == 1.0
    assert epsilon_at(10, s) == 0.1 and epsilon_at(1000, s) == 0.1
    assert abs(epsilon_at(5, s) - (1.0 + (0.1 - 1.0) * 4 / 9)) < 1e-15
    with pytest.raises(ValueError):
        epsilon_at(0, s)
    assert epsilon_at(3, EpsilonSchedule(0.5, 0.5, 1)) == 0.5


@pytest.mark.parametrize("kw", [dict(C=10, F=3), dict(C=10, W=3), dict(W=1),
                                dict(N=11, capacity=10), dict(total_steps=15, C=10),
                                dict(gamma=1.5), dict(action_count=40), dict(batch_size=0),
                                dict(env="gridworld"), dict(hidden=32), dict(state_dim=32),
                                dict(latency_s=1e-3)])
def test_hyperparams_validate_rejects(kw):
    base = dict(C=10, F=2, W=2, N=5, capacity=10, total_steps=20)
    base.update(kw)
    with pytest.raises(ValueError):
        HyperParams(**base).validate()


def test_hyperparams_modes_and_transactions():
    hp = HyperParams(C=40, F=4, W=4, total_steps=200, N=10, capacity=100, eval_period=0)
    assert hp.mode == "both"
    assert hp.with_mode("concurrent").mode == "concurrent"
    assert transaction_count(hp, 200) == 200 // 4 + 200 // 4
    assert transaction_count(hp.with_mode("concurrent"), 200) == 200 + 50


def test_parameter_file_roundtrip_and_layout(tmp_path):
    rng = np.random.default_rng(0)
    flat = rng.normal(size=num_params(18))
    p = Parameters.from_flat(flat, 18)
    assert [w.shape for w in p.weights] == [(o, i) for o, i in layer_shapes(18)]
    path = tmp_path / "net.params"
    save_parameters(path, p)
    q = load_parameters(path)
    assert np.array_equal(q.flat(), flat)
    assert theta_hash(p) == theta_hash(q)


def test_parameter_file_readable_by_reference(tmp_path, reference_paraq):
    """The PQNET1 file format is the reference's (nn.py:232-259)."""
    from paraq.nn import load_parameters as ref_load, theta_hash as ref_hash

    flat = np.random.default_rng(1).normal(size=num_params(4))
    p = Parameters.from_flat(flat, 4)
    path = tmp_path / "x.params"
    save_parameters(path, p)
    r = ref_load(path)
    assert ref_hash(r) == theta_hash(p)


def test_run_record_csv_format_matches_reference(reference_paraq):
    from paraq.executor import RunRecord as RefRecord

    kw = dict(config={"b": "2", "a": "1"}, seed=3, mode="both",
              events=[(40, "episode", "0.5"), (40, "theta_hash", "abcd")],
              final_hash="ffff", counters={"train_calls": 5, "flush_pushes": 7})
    assert RunRecord(**kw).to_csv_text() == RefRecord(**kw).to_csv_text()


def test_shard_covers_batch():
    for B in (32, 33, 1024):
        for G in (1, 2, 3, 8):
            parts = [pdist.shard(B, r, G) for r in range(G)]
            assert parts[0][0] == 0 and parts[-1][1] == B
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    seed = pdist.replica_seed(0, rank)
    mx = pdist.reduce_max(float(rank + 1.5))
    g = torch.full((8,), float(rank + 1))
    pdist.allreduce_sum_(g)
    seeds = [None] * world
    dist.all_gather_object(seeds, seed)
    out.put((rank, seeds, mx, g.tolist()))
    dist.destroy_process_group()


def test_multiprocess_replicas_and_gradient_allreduce_gloo():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 2000)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for rank, seeds, mx, g in res:
        assert len(set(seeds)) == 2          # distinct replica seeds
        assert mx == 2.5                     # max over ranks
        assert g == [3.0] * 8                # sum all-reduce of per-rank gradient shards


def test_api_signatures_match_reference(reference_paraq):
    """Drop-in surface: the reference's positional signatures and HyperParams fields
    (executor.py:591-596, nn.py:93, agent.py:115-147)."""
    import dataclasses
    import inspect

    from paraq import agent as ragent, executor as rexec, nn as rnn

    from paper_2111_01264_b200 import executor, nn

    for mine, ref in ((executor.run, rexec.run), (executor.sequential_reference,
                                                  rexec.sequential_reference),
                      (nn.init_network, rnn.init_network)):
        pm = list(inspect.signature(mine).parameters.values())
        pr = list(inspect.signature(ref).parameters.values())
        assert [p.name for p in pm[:len(pr)]] == [p.name for p in pr]
        assert all(p.kind == p.KEYWORD_ONLY or p.kind == p.VAR_KEYWORD for p in pm[len(pr):])
    ours = {f.name: f for f in dataclasses.fields(HyperParams)}
    for f in dataclasses.fields(ragent.HyperParams):
        assert f.name in ours, f.name
        if f.name not in ("env", "hidden", "latency_s", "state_dim", "action_count"):
            d_ref = f.default if f.default is not dataclasses.MISSING else f.default_factory()
            o = ours[f.name]
            d_me = o.default if o.default is not dataclasses.MISSING else o.default_factory()
            assert type(d_me).__name__ == type(d_ref).__name__, f.name
            if not dataclasses.is_dataclass(d_ref):
                assert d_me == d_ref, f.name
    hp = HyperParams()
    assert hp.actions == hp.action_count == 18 and hp.state_dim == 4 * 84 * 84


def test_init_network_takes_reference_layer_sizes():
    from paper_2111_01264_b200 import nn

    with pytest.raises(ValueError):
        nn.init_network([32, 256, 4], 0)   # the reference's MLP sizes have no conv stack here
    assert nn.network_sizes(18) == [4 * 84 * 84, 512, 18]


def _acting_worker(rank, world, port, out):
    """Sharded-acting plumbing on CPU tensors: pack each rank's epoch block, all-gather
    over gloo, renumber into one ring; rank 0 checks every stack against the originals."""
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = torch.Generator().manual_seed(rank)
    Wl, steps, fcap, F = 3, 4, 64, 16
    ring = torch.randint(0, 256, (fcap, F), dtype=torch.uint8, generator=g)
    hist = torch.tensor([[-1, -1, 5, 6], [-1, 7, 8, 9], [10, 11, 12, 13]], dtype=torch.int32)
    base = 20
    ep = (base + torch.arange(Wl * 2 * steps)) % fcap
    staging = torch.full((Wl, steps, 8), -1, dtype=torch.int32)
    for j in range(Wl):
        cur = hist[j].tolist()
        for b in range(steps):
            nxt = int(ep[j * 2 * steps + b])
            staging[j, b, :5] = torch.tensor(cur + [nxt])
            staging[j, b, 5] = 100 * rank + 10 * j + b
            cur = cur[1:] + [nxt]
    frames, rec = pdist.pack_epoch(ring, hist, ep, staging)
    fr = [torch.empty_like(frames) for _ in range(world)]
    rr = [torch.empty_like(rec) for _ in range(world)]
    dist.all_gather(fr, frames)
    dist.all_gather(rr, rec)
    st = [torch.empty_like(staging) for _ in range(world)]
    rings = [torch.empty_like(ring) for _ in range(world)]
    dist.all_gather(st, staging)
    dist.all_gather(rings, ring)
    ok = True
    if rank == 0:
        big_cap, first = 500, 470   # wraps around the big ring
        G, Fr = world, fr[0].shape[0]
        big = torch.zeros((big_cap, F), dtype=torch.uint8)
        slots = (first + torch.arange(G * Fr)) % big_cap
        big[slots] = torch.cat(fr)
        flat = pdist.remap_gathered(torch.stack(rr), Fr, first, big_cap)
        for r in range(G):
            for j in range(Wl):
                for b in range(steps):
                    orig, new = st[r][j, b], flat[r * Wl + j, b]
                    assert int(new[5]) == int(orig[5])
                    for c in range(5):
                        o, n = int(orig[c]), int(new[c])
                        assert (o < 0) == (n < 0)
                        if o >= 0:
                            ok &= torch.equal(big[n], rings[r][o])
    out.put((rank, ok))
    dist.destroy_process_group()


def test_sharded_acting_pack_gather_remap_gloo():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 30500 + (os.getpid() % 2000)
    procs = [ctx.Process(target=_acting_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok in res)


def test_reset_rate_bound():
    """Frame-ring sizing: twice the expected reset frames per step (1 / E[episode length])."""
    from paper_2111_01264_b200.agent import HyperParams
    from paper_2111_01264_b200.executor import reset_rate_bound

    hp = HyperParams()
    L, p = hp.episode_length, hp.terminal_p
    mean = (1 - (1 - p) ** L) / p
    assert abs(reset_rate_bound(hp) - 2 / mean) < 1e-12
    assert reset_rate_bound(HyperParams(episode_length=1)) == 1.0
    assert reset_rate_bound(HyperParams(episode_length=10, terminal_p=0.0)) == 0.2
