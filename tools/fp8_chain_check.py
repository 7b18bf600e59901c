"""Diagnostic: for each fp8 layer, the dequantised input it reads must equal
the dequantised output its producer wrote (same tensor, same scale).
    python tools/fp8_chain_check.py"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from paper_2512_18318_b200 import generator  # noqa: E402
from paper_2512_18318_b200.api import Context  # noqa: E402
from test_generator import _inputs  # noqa: E402


def main():
    ctx = Context(0)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    w = generator.synthetic_weights(0)
    B = 2
    eng = generator.LipsyncEngine(w, max_batch=B, ctx=ctx, precision=2)
    print("absmax", np.round(eng.act_absmax, 3).tolist())
    rows, chunk_row, target, refs, ref_index = _inputs(B, 77)
    d = [torch.from_numpy(np.ascontiguousarray(v)).cuda() for v in (rows, chunk_row, target, refs, ref_index)]
    buf = torch.empty(B * 96 * 96 * 1024, dtype=torch.float32, device="cuda")
    shape = (C.c_int32 * 4)()
    fn = eng.lib.dll.lsgdbg_run_until

    def dump(layer, which):
        rc = fn(eng.h, *[C.c_void_p(t.data_ptr()) for t in d], B, layer, which, C.c_void_p(buf.data_ptr()), shape)
        assert rc == 0
        torch.cuda.synchronize()
        n = shape[0] * shape[1] * shape[2] * shape[3]
        return buf[:n].reshape(*shape).permute(0, 3, 1, 2).cpu().clone()
    Ls = generator.layers()
    outs = {}
    for i in range(len(Ls) - 1):
        x = dump(i, 0)
        if i < len(Ls) - 2:
            outs[i] = dump(i, 1)
        L = Ls[i]
        # candidate producers: previous layer with matching shape
        best = None
        for j in range(i - 1, -1, -1):
            if j in outs and outs[j].shape[2:] == x.shape[2:]:
                o = outs[j]
                for off in range(0, x.shape[1] - o.shape[1] + 1, 16):
                    seg = x[:, off:off + o.shape[1]]
                    if seg.shape == o.shape:
                        err = (seg - o).abs().max().item() / (o.abs().max().item() + 1e-9)
                        if best is None or err < best[0]:
                            best = (err, j, off)
        print(f"layer {i:2d} in {tuple(x.shape)} absmax {x.abs().max():.4g}  best producer match "
              f"{best}")


if __name__ == "__main__" and not os.environ.get("OUT0"):
    main()


def check_out0():
    """fused out0+out1 (fp8) vs fp32 math on the GPU's own cat6 input."""
    import torch.nn.functional as F
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
    import generator_ref as gref
    from test_generator_fp8 import _wq
    ctx = Context(0)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    w = generator.synthetic_weights(0)
    B = 2
    for prec in (1, 2):
        eng = generator.LipsyncEngine(w, max_batch=B, ctx=ctx, precision=prec)
        rows, chunk_row, target, refs, ref_index = _inputs(B, 77)
        d = [torch.from_numpy(np.ascontiguousarray(v)).cuda() for v in (rows, chunk_row, target, refs, ref_index)]
        buf = torch.empty(B * 96 * 96 * 1024, dtype=torch.float32, device="cuda")
        shape = (C.c_int32 * 4)()
        fn = eng.lib.dll.lsgdbg_run_until

        def dump(layer, which):
            rc = fn(eng.h, *[C.c_void_p(t.data_ptr()) for t in d], B, layer, which, C.c_void_p(buf.data_ptr()), shape)
            assert rc == 0
            torch.cuda.synchronize()
            n = shape[0] * shape[1] * shape[2] * shape[3]
            return buf[:n].reshape(*shape).permute(0, 3, 1, 2).cpu().clone()
        cat6 = torch.cat([dump(48, 1), dump(0, 1)], 1)
        lg = torch.empty(B, 3, 96, 96, dtype=torch.float32, device="cuda")
        eng.forward_device(*[t.data_ptr() for t in d], lg.data_ptr(), 2, B)
        torch.cuda.synchronize()
        params = gref.split_blob(w)
        w0 = _wq(torch, params[49][0], 0) if prec == 2 else torch.from_numpy(np.ascontiguousarray(params[49][0]))
        y = torch.relu(F.conv2d(cat6, w0, torch.from_numpy(np.ascontiguousarray(params[49][1])), 1, 1))
        ref = F.conv2d(y, torch.from_numpy(np.ascontiguousarray(params[50][0])),
                       torch.from_numpy(np.ascontiguousarray(params[50][1])))
        err = (lg.cpu() - ref).abs().max().item()
        print(f"prec {prec}: out0+1 logits max err {err:.4g} (ref absmax {ref.abs().max():.4g})")
        # face input check: GPU x_face vs the oracle's
        xf = dump(0, 0)[:, :6]
        want = torch.from_numpy(np.stack([gref.face_input(target[b], refs[ref_index[b]]) for b in range(B)]))
        print(f"prec {prec}: face input max err {(xf - want).abs().max().item():.4g}")
        eng.close()


if __name__ == "__main__" and os.environ.get("OUT0"):
    check_out0()
