"""The B200 fp64 kernel module (the reference's plugin API) is bit-exact with the
reference numba kernels: against the golden vectors made by running the reference,
and composed into the oracle's MLP restatement of nn.forward / gradient /
train_minibatch against the reference's own golden outputs."""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2111_01264_b200 import kernels as K  # noqa: E402

from oracle import natcnn  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.mark.parametrize("case", [0, 1, 2])
def test_plugin_kernels_bit_exact_vs_reference_golden(case):
    g = np.load(os.path.join(GOLD, "kernels.npz"))
    c = str(case)
    assert K.affine_rows(g[f"aff{c}_w"], g[f"aff{c}_b"], g[f"aff{c}_x"]).tobytes() == \
        g[f"aff{c}_out"].tobytes()
    assert K.relu(g[f"aff{c}_x"]).tobytes() == g[f"relu{c}_out"].tobytes()
    assert K.output_delta(g[f"od{c}_q"], g[f"od{c}_a"], g[f"od{c}_t"]).tobytes() == \
        g[f"od{c}_out"].tobytes()
    assert K.weight_grad(g[f"wg{c}_delta"], g[f"wg{c}_acts"]).tobytes() == g[f"wg{c}_out"].tobytes()
    assert K.bias_grad(g[f"wg{c}_delta"]).tobytes() == g[f"bg{c}_out"].tobytes()
    assert K.hidden_delta(g[f"wg{c}_delta"], g[f"hd{c}_w"], g[f"hd{c}_pre"]).tobytes() == \
        g[f"hd{c}_out"].tobytes()
    p, gg, m, v = g[f"rms{c}_in"]
    assert np.stack(K.rmsprop_flat(p, gg, m, v, 2.5e-4, 0.95, 0.01)).tobytes() == \
        g[f"rms{c}_out"].tobytes()


def test_reference_mlp_composition_on_b200_plugin_bit_exact(monkeypatch):
    """nn.forward / nn.gradient / 2 x agent.train_minibatch of the reference (golden
    mlp.npz) reproduced with the B200 kernel module swapped in for the kernels."""
    from oracle import natcnn as nc

    monkeypatch.setattr(nc, "_K_EXACT", K)
    g = np.load(os.path.join(GOLD, "mlp.npz"))
    spec = nc.mlp([6, 9, 5, 4])
    theta = nc.Params([g[f"theta_w{k}"] for k in range(3)], [g[f"theta_b{k}"] for k in range(3)])
    target = nc.Params([g[f"target_w{k}"] for k in range(3)], [g[f"target_b{k}"] for k in range(3)])
    assert nc.forward(spec, theta, g["states"]).tobytes() == g["q"].tobytes()
    gr = nc.gradient(spec, theta, g["states"], g["actions"], g["targets"])
    for k in range(3):
        assert gr.weights[k].tobytes() == g[f"grad_w{k}"].tobytes()
    batch = (g["states"], g["actions"], g["rewards"], g["next_states"], g["terminals"])
    p1, o1 = nc.train_minibatch(spec, theta, nc.Opt.zeros(theta), batch, target, 0.99)
    p2, o2 = nc.train_minibatch(spec, p1, o1, batch, target, 0.99)
    for k in range(3):
        assert p2.weights[k].tobytes() == g[f"p2_w{k}"].tobytes()
        assert o2.v_weights[k].tobytes() == g[f"v2_w{k}"].tobytes()


def test_plugin_matches_oracle_at_nature_cnn_shapes():
    """fc1-sized affine_rows / weight_grad / hidden_delta bit-exact with the oracle C
    restatement (itself pinned to numba)."""
    from oracle import _lib as OK

    rng = np.random.default_rng(0)
    w, b, x = rng.normal(size=(512, 3136)), rng.normal(size=512), rng.normal(size=(8, 3136))
    assert K.affine_rows(w, b, x).tobytes() == OK.affine_rows(w, b, x).tobytes()
    delta = rng.normal(size=(8, 512)) * (rng.random((8, 512)) < 0.5)
    assert K.weight_grad(delta, x).tobytes() == OK.weight_grad(delta, x).tobytes()
    pre = rng.normal(size=(8, 3136))
    assert K.hidden_delta(delta, w, pre).tobytes() == OK.hidden_delta(delta, w, pre).tobytes()
