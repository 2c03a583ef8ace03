"""Read the device learner's stored intermediates out of its workspace (test helper).

After one `pq_learn_step`, the workspace holds every tensor the step stored in bf16
(DESIGN.md §2): the conv activations of both networks, fc1's output h1 (fp32), the
fc1 output delta dh1 (bf16 copy) and the data gradients dY3 / dY2 / dY1.  They are
returned in the oracle's row layout (oracle/natcnn.py: NHWC pixels x channels,
flattened per sample) so `natcnn.Bf16Storage` can take them as the next stage's
inputs (teacher forcing) and the stage outputs can be compared one by one.
"""

from __future__ import annotations

import numpy as np


def _view(torch, ws, off, shape, dtype):
    nbytes = int(np.prod(shape)) * torch.empty(0, dtype=dtype).element_size()
    return ws[off:off + nbytes].view(dtype).view(*shape)


def learner_taps(B: int, A: int = 18) -> dict:
    import torch

    from paper_2111_01264_b200 import _native as N
    from paper_2111_01264_b200 import nn as dnn

    torch.cuda.synchronize()
    ws, cap = dnn.workspace(B, A)
    L = N.workspace_layout(cap, A)
    bf = torch.bfloat16

    def np64(t):
        return t.float().cpu().numpy().astype(np.float64).reshape(B, -1)

    def act1(suffix):
        if L["act1s2" + suffix] >= 0 and B >= 128:
            # the shifted-descriptor conv kernels keep act1 as its 2x2 space-to-depth copy
            a = _view(torch, ws, L["act1s2" + suffix], (B, 10, 10, 2, 2, 32), bf)
            return a.permute(0, 1, 3, 2, 4, 5).reshape(B, 20, 20, 32)
        return _view(torch, ws, L["act1" + suffix], (B, 20, 20, 32), bf)

    out = {}
    for suffix, name in (("", "online"), ("_t", "target")):
        out[name] = {
            0: np64(act1(suffix)),
            1: np64(_view(torch, ws, L["act2" + suffix], (B, 9, 9, 64), bf)),
            2: np64(_view(torch, ws, L["act3" + suffix], (B, 7, 7, 64), bf)),
        }
    out["h1"] = np64(_view(torch, ws, L["h1"], (B, 512), torch.float32))
    if B >= 128 and L["dY1p"] >= 0:
        dy1 = _view(torch, ws, L["dY1p"], (B, 21, 21, 32), bf)[:, :20, :20]
    else:
        dy1 = _view(torch, ws, L["dY1"], (B, 20, 20, 32), bf)
    # delta feeding layer k (natcnn.gradient): k=3 dh1, k=2 dY3, k=1 dY2, k=0 dY1
    out["deltas"] = {
        3: np64(_view(torch, ws, L["dh1_bf"], (B, 512), bf)),
        2: np64(_view(torch, ws, L["dY3"], (B, 7, 7, 64), bf)),
        1: np64(_view(torch, ws, L["dY2"], (B, 9, 9, 64), bf)),
        0: np64(dy1),
    }
    return out
