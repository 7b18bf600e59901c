"""GPU diagnostic: per-layer error of the tcgen05 generator against fp32
torch on the GPU's own bf16 inputs (isolates each layer), plus the
end-to-end drift.  Usage (on a B200): python tests/gen_layer_diag.py
"""
import ctypes as C
import os
import sys

import numpy as np
import torch
import torch.nn.functional as F

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from paper_2512_18318_b200 import generator  # noqa: E402
from paper_2512_18318_b200.api import Context  # noqa: E402
from test_generator import _inputs, _oracle  # noqa: E402


def main():
    gref = _oracle()
    w = generator.synthetic_weights(0)
    params = gref.split_blob(w)
    Ls = generator.layers()
    ctx = Context(0)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    eng = generator.LipsyncEngine(w, max_batch=max(B, 4), ctx=ctx)
    rows, chunk_row, target, refs, ref_index = _inputs(B, 7)
    d = [torch.from_numpy(np.ascontiguousarray(v)).cuda() for v in (rows, chunk_row, target, refs, ref_index)]
    fn = eng.lib.dll.lsgdbg_run_until
    buf = torch.empty(B * 96 * 96 * 1024, dtype=torch.float32, device="cuda")
    shape = (C.c_int32 * 4)()

    def dump(layer, which):
        rc = fn(eng.h, C.c_void_p(d[0].data_ptr()), C.c_void_p(d[1].data_ptr()), C.c_void_p(d[2].data_ptr()),
                C.c_void_p(d[3].data_ptr()), C.c_void_p(d[4].data_ptr()), B, layer, which,
                C.c_void_p(buf.data_ptr()), shape)
        assert rc == 0, eng.lib.dll.lsg_last_error()
        torch.cuda.synchronize()
        n = shape[0] * shape[1] * shape[2] * shape[3]
        return buf[:n].reshape(shape[0], shape[1], shape[2], shape[3]).permute(0, 3, 1, 2).cpu()

    worst = 0
    for i in range(len(Ls) - 1):
        L = Ls[i]
        x = dump(i, 0)
        y = dump(i, 1)
        wt, bt = (torch.from_numpy(np.ascontiguousarray(a)) for a in params[i])
        xc = x[:, :L.cin]
        if L.kind == 0:
            ref = F.conv2d(xc, wt, bt, (L.sh, L.sw), (L.ph, L.pw))
        else:
            ref = F.conv_transpose2d(xc, wt, bt, (L.sh, L.sw), (L.ph, L.pw), (L.oph, L.opw))
        if L.res:
            ref = ref + xc
        ref = torch.relu(ref)
        err = (y - ref).abs().max().item()
        scale = ref.abs().max().item() + 1e-6
        rel = err / scale
        worst = max(worst, rel)
        flag = "  <-- BAD" if rel > 0.02 else ""
        print(f"layer {i:2d} kind {L.kind} {L.cin:4d}->{L.cout:4d} k{L.kh} s{L.sh}{L.sw} out {tuple(y.shape)} "
              f"maxerr {err:.4g} scale {scale:.3g} rel {rel:.4g}{flag}")
    print("worst rel", worst)


if __name__ == "__main__":
    main()
