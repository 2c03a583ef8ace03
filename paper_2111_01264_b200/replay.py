"""GPU-resident replay memory with the reference ReplayMemory API (replay.py:30-143).

Layout in HBM:

* ``ring``    uint8 [frame_capacity, 7056]: every 84x84 frame stored once;
* ``records`` int32 [capacity, 8]: per transition {f0, f1, f2, f3, f4,
  action | bootstrap terminal << 16, reward (f64 bits: lo, hi)}; the state is frames
  f0..f3 and the next state f1..f4 (slot -1 = masked all-zero frame before an episode
  start).

Semantics kept from the reference: physical slot of the k-th push is k mod capacity
(append then overwrite, replay.py:53-59), ``version`` counts every push, ``sample``
draws ``rng.integers(0, len, size=B)`` -- here on the GPU, bit-exactly, advancing the
caller's numpy Generator (replay.py:61-66) -- and ``flush`` appends sampler buffers in
ascending owner id (replay.py:82-93).
"""

from __future__ import annotations

import threading
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .nn import FRAME, FRAME_BYTES, STACK

REC_INTS = 8
INT_MAX = 2**31 - 1


@dataclass
class Transition:
    """One experience tuple (replay.py:19-27) with uint8 [4, 84, 84] stacks."""

    state: np.ndarray
    action: int
    reward: float
    next_state: np.ndarray
    terminal: bool


def pcg_state_from_generator(rng: np.random.Generator) -> np.ndarray:
    st = rng.bit_generator.state
    if st["bit_generator"] != "PCG64":
        raise ValueError("replay sampling needs a PCG64 numpy Generator (np.random.default_rng)")
    s, inc = st["state"]["state"], st["state"]["inc"]
    m = (1 << 64) - 1
    return np.array([s >> 64, s & m, inc >> 64, inc & m, st["has_uint32"], st["uinteger"]],
                    dtype=np.uint64)


def pcg_state_to_generator(state, rng: np.random.Generator) -> None:
    s = [int(v) for v in np.asarray(state, dtype=np.uint64)]
    rng.bit_generator.state = {
        "bit_generator": "PCG64",
        "state": {"state": (s[0] << 64) | s[1], "inc": (s[2] << 64) | s[3]},
        "has_uint32": s[4],
        "uinteger": s[5],
    }


def device_pcg(rng: np.random.Generator):
    torch = N.require_cuda()
    return torch.from_numpy(pcg_state_from_generator(rng).view(np.int64)).cuda()


def sample_indices_device(pcg_dev, n: int, count: int, out=None, stream=None):
    """rng.integers(0, n, size=count) on the GPU; pcg_dev (int64[6] device) advances."""
    torch = N.require_cuda()
    if n < 1:
        raise ValueError("cannot sample from an empty replay memory")
    if n >= 2**32:
        raise ValueError("replay length must be < 2^32")
    if out is None:
        out = torch.empty(count, dtype=torch.int64, device="cuda")
    N.check(N.load().pq_sample_indices(pcg_dev.data_ptr(), n, count, out.data_ptr(),
                                       N.stream_ptr(stream)), "sample_indices")
    return out


@dataclass
class Batch:
    """A sampled minibatch: record slots into a device ReplayMemory.  It is also the
    reference's ``list[Transition]`` (replay.py:61-66): len(), indexing and iteration
    yield host Transitions (one gather of the whole batch on first use)."""

    memory: "ReplayMemory"
    idx: object  # torch.int64 [B] on the GPU

    def __len__(self):
        return int(self.idx.numel())

    def gather(self):
        return self.memory.gather(self.idx)

    def transitions(self) -> list:
        cached = self.__dict__.get("_host")
        if cached is None:
            s, a, r, s2, term = self.gather()
            s, s2 = s.cpu().numpy(), s2.cpu().numpy()
            a, r, term = a.cpu().numpy(), r.cpu().numpy(), term.cpu().numpy()
            cached = [Transition(s[i], int(a[i]), float(r[i]), s2[i], bool(term[i]))
                      for i in range(len(self))]
            self.__dict__["_host"] = cached
        return cached

    def __iter__(self):
        return iter(self.transitions())

    def __getitem__(self, i):
        return self.transitions()[i]


def as_batch(batch) -> Batch:
    """A Batch, or a reference-style list of frame-stack Transitions staged into a
    scratch device memory in order (so train_minibatch / td_targets accept both)."""
    if isinstance(batch, Batch):
        return batch
    items = list(batch)
    if not items:
        raise ValueError("empty batch")
    mem = ReplayMemory(len(items), frame_capacity=8 * len(items) + 64)
    for t in items:
        mem.push(t)
    torch = N.require_cuda()
    return Batch(mem, torch.arange(len(items), device="cuda"))


class ReplayMemory:
    """Ring buffer of frame-stacked transitions in HBM with uniform sampling."""

    def __init__(self, capacity: int, frame_capacity: int | None = None):
        if capacity < 1:
            raise ValueError("capacity must be at least 1")
        torch = N.require_cuda()
        self.capacity = int(capacity)
        self.frame_capacity = int(frame_capacity or (2 * capacity + 4096))
        self.ring = torch.zeros((self.frame_capacity, FRAME_BYTES), dtype=torch.uint8,
                                device="cuda")
        self.records = torch.full((self.capacity, REC_INTS), -1, dtype=torch.int32, device="cuda")
        self._len = 0
        self.push_count = 0
        self.version = 0
        self.frame_seq = 0            # frames ever allocated; slot = seq mod frame_capacity
        # oldest frame sequence number referenced by each record (host bookkeeping
        # that guarantees no live transition loses a frame to ring wrap-around)
        self._rec_min_seq = np.full(self.capacity, -1, dtype=np.int64)
        self._safe_until = self.frame_capacity
        self._prev = None             # (next_state bytes, slots f1..f4, seqs) of the last push

    def __len__(self) -> int:
        return self._len

    # -- frame allocation -----------------------------------------------------------
    def _reserve_frames(self, count: int) -> int:
        """Reserve `count` consecutive frame sequence numbers; returns the first."""
        first = self.frame_seq
        end = first + count
        if end > self._safe_until:
            live = self._rec_min_seq[: self._len]
            live = live[live >= 0]
            oldest = int(live.min()) if live.size else end
            self._safe_until = oldest + self.frame_capacity
            if end > self._safe_until:
                raise RuntimeError(
                    "frame ring too small: a live transition still references a frame that "
                    "would be overwritten; construct ReplayMemory with a larger frame_capacity")
        self.frame_seq = end
        return first

    def _advance(self, n: int, min_seqs) -> np.ndarray:
        """Account for n pushes; returns their physical slots (replay.py:53-59)."""
        slots = (self.push_count + np.arange(n)) % self.capacity
        self._rec_min_seq[slots] = min_seqs
        self.push_count += n
        self._len = min(self.capacity, self._len + n)
        self.version += n
        return slots

    # -- pushes ---------------------------------------------------------------------
    def push(self, t: Transition) -> None:
        """Store one transition.  Frames shared with the previous push (its next state
        is this state) are not stored twice; zero frames become masked slots."""
        torch = N.require_cuda()
        s = np.ascontiguousarray(t.state, dtype=np.uint8)
        s2 = np.ascontiguousarray(t.next_state, dtype=np.uint8)
        if s.shape != (STACK, FRAME, FRAME) or s2.shape != (STACK, FRAME, FRAME):
            raise ValueError("transitions must hold uint8 [4, 84, 84] frame stacks")
        if not np.array_equal(s2[:STACK - 1], s[1:]):
            raise ValueError("next_state must be the state shifted by one frame")
        refs = [-1] * 5
        seqs = [-1] * 5
        new_frames = []
        if self._prev is not None and self._prev[0] == s.tobytes():
            refs[:4], seqs[:4] = list(self._prev[1]), list(self._prev[2])
        else:
            for c in range(STACK):
                if s[c].any():
                    new_frames.append((c, s[c]))
        new_frames.append((4, s2[STACK - 1]))
        if new_frames:
            first = self._reserve_frames(len(new_frames))
            host = np.stack([f for _, f in new_frames]).reshape(len(new_frames), FRAME_BYTES)
            slots_dev = []
            for k, (c, _) in enumerate(new_frames):
                seq = first + k
                refs[c] = seq % self.frame_capacity
                seqs[c] = seq
                slots_dev.append(refs[c])
            idx = torch.as_tensor(np.array(slots_dev, dtype=np.int64)).cuda()
            self.ring.index_copy_(0, idx, torch.from_numpy(host).cuda())
        if not s2[STACK - 1].any():
            refs[4] = -1
        rec = np.array(refs + [int(t.action) | (1 << 16 if t.terminal else 0), 0, 0],
                       dtype=np.int32)
        rec[6:8] = np.array([float(t.reward)], dtype="<f8").view(np.int32)
        valid = [q for q in seqs if q >= 0]
        slot = int(self._advance(1, min(valid) if valid else -1)[0])
        self.records[slot] = torch.from_numpy(rec).cuda()
        self._prev = (s2.tobytes(), refs[1:5], seqs[1:5])

    def push_device_records(self, rec, n: int, min_seq, stream=None) -> None:
        """Append n device records [n, 8] (owner-major order already applied); min_seq:
        the oldest frame sequence number they reference (scalar or one per record)."""
        slots = self._advance(n, min_seq)
        start = int(slots[0])
        first = min(n, self.capacity - start)
        self.records[start:start + first].copy_(rec[:first], non_blocking=True)
        if first < n:
            self.records[: n - first].copy_(rec[first:n], non_blocking=True)
        self._prev = None

    # -- sampling -------------------------------------------------------------------
    def sample_indices(self, batch_size: int, rng: np.random.Generator):
        """batch_size uniform draws with replacement from rng only (replay.py:61-66)."""
        if self._len == 0:
            raise ValueError("cannot sample from an empty replay memory")
        st = device_pcg(rng)
        idx = sample_indices_device(st, self._len, batch_size)
        pcg_state_to_generator(st.cpu().numpy().view(np.uint64), rng)
        return idx

    def sample(self, batch_size: int, rng: np.random.Generator) -> Batch:
        return Batch(self, self.sample_indices(batch_size, rng))

    def gather(self, idx, stream=None):
        """Stack gather (agent.py:76, :100): states, actions, rewards, next states,
        terminals as device tensors."""
        torch = N.require_cuda()
        idx = torch.as_tensor(idx, dtype=torch.int64, device="cuda").contiguous()
        B = idx.numel()
        s = torch.empty((B, STACK, FRAME, FRAME), dtype=torch.uint8, device="cuda")
        s2 = torch.empty_like(s)
        a = torch.empty(B, dtype=torch.int32, device="cuda")
        r = torch.empty(B, dtype=torch.float64, device="cuda")
        term = torch.empty(B, dtype=torch.uint8, device="cuda")
        N.check(N.load().pq_replay_gather(self.ring.data_ptr(), self.records.data_ptr(),
                                          idx.data_ptr(), B, s.data_ptr(), s2.data_ptr(),
                                          a.data_ptr(), r.data_ptr(), term.data_ptr(),
                                          N.stream_ptr(stream)), "gather")
        return s, a, r, s2, term

    def snapshot(self):
        """Contents in insertion order as host Transitions (replay.py:45-51)."""
        torch = N.require_cuda()
        if self._len < self.capacity:
            order = np.arange(self._len)
        else:
            cur = self.push_count % self.capacity
            order = np.concatenate([np.arange(cur, self.capacity), np.arange(cur)])
        s, a, r, s2, term = self.gather(torch.as_tensor(order))
        s, s2 = s.cpu().numpy(), s2.cpu().numpy()
        a, r, term = a.cpu().numpy(), r.cpu().numpy(), term.cpu().numpy()
        return [Transition(s[i], int(a[i]), float(r[i]), s2[i], bool(term[i]))
                for i in range(len(order))]

    # -- prepopulation / flush ----------------------------------------------------------
    def prepopulate(self, env, n: int, rng: np.random.Generator) -> None:
        """Insert exactly n uniform-random-action transitions (replay.py:68-80).
        A device frame env (``FrameEnvSpec``) runs entirely on the GPU on the same
        PCG64 stream; any other env is stepped on the host and pushed."""
        if n > self.capacity:
            raise ValueError("prepopulation count exceeds capacity")
        if n == 0:
            return
        if hasattr(env, "key") and hasattr(env, "terminal_p") and getattr(env, "device", False):
            self._prepopulate_device(env, n, rng)
            return
        state = env.reset(rng)
        for _ in range(n):
            action = int(rng.integers(env.action_count))
            next_state, reward, terminal = env.step(action, rng)
            boot = terminal and not getattr(env, "truncated", False)
            self.push(Transition(state, action, reward, next_state, boot))
            state = env.reset(rng) if terminal else next_state

    def _prepopulate_device(self, env, n: int, rng) -> None:
        torch = N.require_cuda()
        lib = N.load()
        st = device_pcg(rng)
        rec = torch.empty((n, REC_INTS), dtype=torch.int32, device="cuda")
        used = torch.zeros(1, dtype=torch.int64, device="cuda")
        scratch = torch.empty(lib.pq_prepopulate_scratch_bytes(n), dtype=torch.uint8,
                              device="cuda")
        # the walk first (records + frame descriptors), then exactly the frames it used are
        # reserved -- the ring need not hold the worst case of 2 frames per transition
        first = self.frame_seq
        N.check(lib.pq_prepopulate_walk(st.data_ptr(), env.episode_length, env.action_count,
                                        env.terminal_p, n, first, self.frame_capacity, rec.data_ptr(),
                                        used.data_ptr(), scratch.data_ptr(), N.stream_ptr()),
                "prepopulate walk")
        if self._reserve_frames(int(used.item())) != first:
            raise RuntimeError("frame reservation moved during prepopulation")
        N.check(lib.pq_prepopulate_frames(env.key, self.ring.data_ptr(), first, self.frame_capacity,
                                          used.data_ptr(), scratch.data_ptr(), N.stream_ptr()),
                "prepopulate frames")
        pcg_state_to_generator(st.cpu().numpy().view(np.uint64), rng)
        # each record's oldest referenced frame, so the ring-wrap guard frees the prepopulated
        # frames as their records are overwritten (slot = seq mod frame_capacity, and the
        # walk's frames are the sequence numbers [first, first + used))
        fc = self.frame_capacity
        refs = rec[:, :5].to(torch.int64)
        seqs = first + torch.remainder(refs - first % fc, fc)
        seqs = torch.where(refs >= 0, seqs, torch.full_like(seqs, 1 << 62))
        self.push_device_records(rec, n, seqs.min(dim=1).values.cpu().numpy())
        env.episode += 1  # the device walk leaves the env mid-episode (state not kept)


class SampleBuffer:
    """Transitions one sampler collected since the last flush (replay.py:96-120)."""

    def __init__(self, owner_id: int):
        self.owner_id = owner_id
        self._items: list = []
        self._lock = threading.Lock()

    def __len__(self):
        return len(self._items)

    def append(self, t: Transition) -> None:
        with self._lock:
            self._items.append(t)

    def drain(self) -> list:
        with self._lock:
            items, self._items = self._items, []
        return items


def flush(memory: ReplayMemory, buffers) -> int:
    """ReplayMemory.flush (replay.py:82-93): ascending owner id, chronological."""
    moved = 0
    for buf in sorted(buffers, key=lambda b: b.owner_id):
        for t in buf.drain():
            memory.push(t)
            moved += 1
    return moved


ReplayMemory.flush = lambda self, buffers: flush(self, buffers)  # noqa: E731
