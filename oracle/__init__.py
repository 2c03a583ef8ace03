"""CPU parity oracle -- TEST INFRASTRUCTURE, not the product.

A restatement of the reference `paraq` hot path (/root/reference/pkg/src/paraq):

* ``kernels.c``  -- the fp64 kernel module (_kernels_numba.py:19-111) and numpy's
  PCG64 / Lemire draw discipline (replay.py:65, agent.py:63-66), bit-exact.
* ``natcnn.py``  -- Nature-CNN forward / gradient / RMSProp / train_minibatch,
  composed from those kernels through im2col exactly like nn.forward
  (nn.py:123-131), nn.gradient (nn.py:134-170) and agent.train_minibatch
  (agent.py:84-105).
* ``replay.py``  -- the ReplayMemory ring (replay.py:30-93) holding frame-stacked
  uint8 transitions, plus the batch stack gather (agent.py:76, :100).
* ``envs.py``    -- the synthetic 84x84 frame environment used on both sides.

Parity pinning: tests/test_oracle.py checks every kernel bit-exactly against
tests/golden/*.npz, which tests/golden/make_golden.py produced by running the
unmodified reference.  Only tests/, __graft_entry__.smoke() and bench.py's
CPU-baseline / reference arm may import this package.
"""
