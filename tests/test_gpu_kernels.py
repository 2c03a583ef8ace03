"""Stage-wise numerics of every tcgen05 GEMM / head / optimizer kernel of one learner
step, each checked against a plain PyTorch fp32 computation fed with the GPU's own
inputs of that stage (bf16 operands, fp32 accumulation), so accumulation order is
the only difference.  Tolerances: relative Frobenius error 2e-3 on bf16-stored
outputs (one bf16 rounding), 1e-4 on fp32 outputs."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2111_01264_b200 as pq  # noqa: E402
from paper_2111_01264_b200 import _native as N  # noqa: E402
from paper_2111_01264_b200 import nn as dnn  # noqa: E402
from paper_2111_01264_b200.replay import ReplayMemory, Transition  # noqa: E402

from oracle import natcnn  # noqa: E402

F = torch.nn.functional
A = 18


@pytest.fixture(autouse=True)
def _no_tf32():
    old = (torch.backends.cuda.matmul.allow_tf32, torch.backends.cudnn.allow_tf32)
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    yield
    torch.backends.cuda.matmul.allow_tf32, torch.backends.cudnn.allow_tf32 = old


def rel(a, b):
    a, b = a.double(), b.double()
    return float((a - b).norm() / max(b.norm(), 1e-30))


def bf16_of(t_int16):
    return t_int16.view(torch.bfloat16).float()


def make_memory(rng, n_frames=80, cap=128):
    mem = ReplayMemory(cap)
    frames = rng.integers(0, 256, size=(n_frames, 84, 84), dtype=np.uint8)
    for k in range(n_frames - 4):
        s, s2 = frames[k:k + 4].copy(), frames[k + 1:k + 5].copy()
        if k % 9 == 0:
            s[:2] = 0
            s2[:1] = 0
        mem.push(Transition(s, int(rng.integers(A)), float(rng.random()), s2, bool(k % 11 == 5)))
    return mem


def net_from(seed):
    spec = natcnn.nature_cnn(A)
    p = natcnn.init_params(spec, seed)
    # non-zero biases so the bias paths are exercised
    brng = np.random.default_rng(seed + 1)
    for b in p.biases:
        b[:] = brng.normal(scale=0.05, size=b.shape)
    flat = np.concatenate([np.r_[w.ravel(), b] for w, b in zip(p.weights, p.biases)])
    return spec, p, dnn.QNet.from_flat(flat, A)


def view(ws, off, shape, dtype):
    nbytes = int(np.prod(shape)) * torch.empty(0, dtype=dtype).element_size()
    return ws[off:off + nbytes].view(dtype).view(*shape)


def unpack(net):
    m = net.master
    sh = net.shadow
    P = dict(W1=m[0:8192].view(32, 256), b1=m[8192:8224], W2=m[8224:40992].view(64, 512),
             b2=m[40992:41056], W3=m[41056:77920].view(64, 576), b3=m[77920:77984],
             W4=m[77984:1683616].view(512, 3136), b4=m[1683616:1684128],
             W5=m[1684128:1684128 + A * 512].view(A, 512), b5=m[1684128 + A * 512:])
    S = dict(W1=bf16_of(sh[0:8192]).view(32, 256), W2=bf16_of(sh[8192:40960]).view(64, 512),
             W3=bf16_of(sh[40960:77824]).view(64, 576),
             W4=bf16_of(sh[77824:1683456]).view(512, 3136))
    return P, S


@pytest.mark.parametrize("B", [32, 8, 40, 256, 333, 1024])
def test_learner_step_stagewise(B):
    rng = np.random.default_rng(B)
    mem = make_memory(rng)
    spec, p, theta = net_from(3)
    _, _, target = net_from(4)
    batch = mem.sample(B, np.random.default_rng(7))
    opt = dnn.OptState.zeros(theta)
    # perturb the moments so the RMSProp check is not trivial
    opt.m.copy_(torch.randn_like(opt.m) * 1e-3)
    opt.v.copy_(opt.m * opt.m + torch.rand_like(opt.v) * 1e-4)
    th2, op2, grad, qout, td = dnn._learn(theta, opt, target, mem.ring, mem.records,
                                          batch.idx, B, gamma=0.99, want_grad=True, want_q=True)
    torch.cuda.synchronize()
    ws, cap = dnn.workspace(B, A)
    L = N.workspace_layout(cap, A)
    n8 = (cap + 7) // 8 * 8
    P, S = unpack(theta)
    PT, ST = unpack(target)
    s, a, r, s2, term = mem.gather(batch.idx)

    def act1_of(suffix):
        if B >= 128:   # TMA engine: conv1 writes only act1's 2x2 space-to-depth copy
            a = view(ws, L["act1s2" + suffix], (B, 10, 10, 2, 2, 32), torch.bfloat16).float()
            return a.permute(0, 1, 3, 2, 4, 5).reshape(B, 20, 20, 32)
        return view(ws, L["act1" + suffix], (B, 20, 20, 32), torch.bfloat16).float()

    def fwd_stage(x_u8, Pp, Sp, suffix):
        act1 = act1_of(suffix)
        x = x_u8.float()
        ref1 = F.relu(F.conv2d(x, Sp["W1"].view(32, 4, 8, 8), stride=4) / 255.0 +
                      Pp["b1"].view(1, -1, 1, 1)).permute(0, 2, 3, 1)
        assert rel(act1, ref1) < 2e-3, "conv1 forward"
        act2 = view(ws, L["act2" + suffix], (B, 9, 9, 64), torch.bfloat16).float()
        ref2 = F.relu(F.conv2d(act1.permute(0, 3, 1, 2), Sp["W2"].view(64, 4, 4, 32).permute(0, 3, 1, 2),
                               Pp["b2"], stride=2)).permute(0, 2, 3, 1)
        assert rel(act2, ref2) < 2e-3, "conv2 forward"
        act3 = view(ws, L["act3" + suffix], (B, 7, 7, 64), torch.bfloat16).float()
        ref3 = F.relu(F.conv2d(act2.permute(0, 3, 1, 2), Sp["W3"].view(64, 3, 3, 64).permute(0, 3, 1, 2),
                               Pp["b3"], stride=1)).permute(0, 2, 3, 1)
        assert rel(act3, ref3) < 2e-3, "conv3 forward"
        ns = N.load().pq_fc1_splits(B, 2)  # 1 when the forward reduced the splits in TMEM
        part = view(ws, L["fc1part" + suffix], (7, B, 512), torch.float32)[:ns].sum(0)
        ref4 = act3.reshape(B, 3136) @ Sp["W4"].T
        assert rel(part, ref4) < 1e-4, "fc1 forward"
        h1 = F.relu(part + Pp["b4"])
        q = h1 @ Pp["W5"].T + Pp["b5"]
        return act1, act2, act3, h1, q

    act1, act2, act3, h1, q = fwd_stage(s, P, S, "")
    _, _, _, _, qt = fwd_stage(s2, PT, ST, "_t")
    assert rel(qout[0], q) < 1e-5 and rel(qout[1], qt) < 1e-5, "fc2 head"
    rr, aa, tt = r.float(), a.long(), term.bool()
    target_ref = torch.where(tt, rr, rr + 0.99 * qout[1].max(1).values)
    d = qout[0][torch.arange(B), aa] - target_ref
    assert rel(td[:, 0], target_ref) < 1e-6 and rel(td[:, 1], d) < 1e-5, "TD head"
    dh1 = view(ws, L["dh1"], (B, 512), torch.float32)
    ref_dh1 = d[:, None] * P["W5"][aa] * (h1 > 0)
    assert rel(dh1, ref_dh1) < 1e-5, "fc2 back-prop"
    dh1_bf = view(ws, L["dh1_bf"], (B, 512), torch.bfloat16).float()
    # fc1 data gradient (MN-major W4 operand) with the conv3 ReLU mask
    dY3 = view(ws, L["dY3"], (B, 7, 7, 64), torch.bfloat16).float()
    ref = ((dh1_bf @ S["W4"]).view(B, 7, 7, 64)) * (act3 > 0)
    assert rel(dY3, ref) < 2e-3, "fc1 dgrad"
    # fc1 weight gradient (contraction over the batch)
    g4 = grad[77984:1683616].view(512, 3136)   # fused fc1 wgrad + RMSProp epilogue
    assert rel(g4, dh1_bf.T @ act3.reshape(B, 3136)) < 1e-4, "fc1 wgrad"
    # conv3 wgrad (+ bias row) and dgrad
    x2 = act2.permute(0, 3, 1, 2)
    dy3 = dY3.permute(0, 3, 1, 2)
    gw3 = torch.nn.grad.conv2d_weight(x2, (64, 64, 3, 3), dy3, stride=1).permute(0, 2, 3, 1)
    grad_w3 = grad[41056:77920].view(64, 576)
    assert rel(grad_w3, gw3.reshape(64, 576)) < 1e-4, "conv3 wgrad"
    assert rel(grad[77920:77984], dy3.sum((0, 2, 3))) < 1e-4, "conv3 bias grad"
    dY2 = view(ws, L["dY2"], (B, 9, 9, 64), torch.bfloat16).float()
    ref = torch.nn.grad.conv2d_input((B, 64, 9, 9), S["W3"].view(64, 3, 3, 64).permute(0, 3, 1, 2),
                                     dy3, stride=1).permute(0, 2, 3, 1) * (act2 > 0)
    assert rel(dY2, ref) < 2e-3, "conv3 dgrad"
    if B >= 128:   # TMA engine: the same rows on the zero-padded 11 x 11 grid (shifted conv2 dgrad)
        dY2p = view(ws, L["dY2p"], (B, 11, 11, 64), torch.bfloat16).float()
        assert torch.equal(dY2p[:, 1:10, 1:10], dY2)
        assert not dY2p[:, 0].any() and not dY2p[:, 10].any()
        assert not dY2p[:, :, 0].any() and not dY2p[:, :, 10].any()
    # conv2
    x1 = act1.permute(0, 3, 1, 2)
    dy2 = dY2.permute(0, 3, 1, 2)
    gw2 = torch.nn.grad.conv2d_weight(x1, (64, 32, 4, 4), dy2, stride=2).permute(0, 2, 3, 1)
    assert rel(grad[8224:40992].view(64, 512), gw2.reshape(64, 512)) < 1e-4, "conv2 wgrad"
    assert rel(grad[40992:41056], dy2.sum((0, 2, 3))) < 1e-4, "conv2 bias grad"
    if B >= 128:   # TMA engine: conv2's data gradient on the padded 21 x 21 grid (zero pad rows)
        dY1p = view(ws, L["dY1p"], (B, 21, 21, 32), torch.bfloat16).float()
        assert not dY1p[:, 20].any() and not dY1p[:, :, 20].any()
        dY1 = dY1p[:, :20, :20].contiguous()
    else:
        dY1 = view(ws, L["dY1"], (B, 20, 20, 32), torch.bfloat16).float()
    ref = torch.nn.grad.conv2d_input((B, 32, 20, 20), S["W2"].view(64, 4, 4, 32).permute(0, 3, 1, 2),
                                     dy2, stride=2).permute(0, 2, 3, 1) * (act1 > 0)
    assert rel(dY1, ref) < 2e-3, "conv2 dgrad"
    # conv1 wgrad straight from the uint8 frames of the replay ring
    dy1 = dY1.permute(0, 3, 1, 2)
    gw1 = torch.nn.grad.conv2d_weight(s.float(), (32, 4, 8, 8), dy1, stride=4) / 255.0
    assert rel(grad[0:8192].view(32, 256), gw1.reshape(32, 256)) < 1e-4, "conv1 wgrad"
    assert rel(grad[8192:8224], dy1.sum((0, 2, 3))) < 1e-4, "conv1 bias grad"
    # fc1 bias and fc2 grads (optimizer-side reductions)
    assert rel(grad[1683616:1684128], dh1.sum(0)) < 1e-5
    gw5 = torch.zeros(A, 512, device="cuda").index_add_(0, aa, d[:, None] * h1)
    assert rel(grad[1684128:1684128 + A * 512].view(A, 512), gw5) < 1e-5
    # centered RMSProp on the summed gradient (fp32)
    m2 = 0.95 * opt.m + 0.05 * grad
    v2 = 0.95 * opt.v + 0.05 * grad * grad
    p2 = theta.master - 2.5e-4 * grad / torch.sqrt(v2 - m2 * m2 + 0.01)
    assert rel(op2.m, m2) < 1e-6 and rel(op2.v, v2) < 1e-6
    assert float((th2.master - p2).abs().max()) < 1e-6
    S2 = unpack(th2)[1]
    assert torch.equal(S2["W4"], th2.master[77984:1683616].view(512, 3136).bfloat16().float())


def test_forward_rows_independent_bitexact():
    """nn.forward row independence (pkg/tests/test_nn.py:117-124), bit-exact."""
    _, _, net = net_from(11)
    rng = np.random.default_rng(0)
    x = rng.integers(0, 256, size=(16, 4, 84, 84), dtype=np.uint8)
    together = dnn.forward(net, x)
    for r in range(16):
        alone = dnn.forward(net, x[r:r + 1])
        assert together[r].tobytes() == alone[0].tobytes()


def test_forward_zero_network_gives_zero_rows():
    """pkg/tests/test_nn.py:108-114."""
    net = dnn.QNet.from_flat(np.zeros(dnn.num_params(A)), A)
    q = dnn.forward(net, np.ones((5, 4, 84, 84), dtype=np.uint8))
    assert q.shape == (5, A) and (q == 0).all()


@pytest.mark.parametrize("W", [128, 512])
def test_wide_acting_batch_rows_match_small_batches(W):
    """Synchronized-execution sweep (configs[2]): a W-row batched forward equals the
    forwards of its 8-row slices (row independence across tile / N-shape choices)."""
    _, _, net = net_from(12)
    x = np.random.default_rng(W).integers(0, 256, size=(W, 4, 84, 84), dtype=np.uint8)
    big = dnn.forward(net, x)
    small = np.concatenate([dnn.forward(net, x[i:i + 8]) for i in range(0, W, 8)])
    assert np.array_equal(big, small)
