"""Per-layer divergence of an 8-bit tail engine from the fp16 engine on the
same inputs (lsgdbg_run_until dumps): relative error of every tail layer's
input and output, then of the final frames.

    python tools/i8_debug.py [prec]     (prec: 4 = INT8_TAIL (default), 3 = FP8_TAIL)
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_2512_18318_b200 import generator  # noqa: E402
from paper_2512_18318_b200.api import Context  # noqa: E402
from test_generator import _inputs  # noqa: E402


def main():
    prec = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    ctx = Context(0)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    w = generator.synthetic_weights(0)
    B = 4
    E = generator.LipsyncEngine
    e16 = E(w, max_batch=B, ctx=ctx, precision=E.PREC_FP16)
    eq = E(w, max_batch=B, ctx=ctx, precision=prec)
    rows, chunk_row, target, refs, ref_index = _inputs(B, 78)
    d = [torch.from_numpy(np.ascontiguousarray(v)).cuda() for v in (rows, chunk_row, target, refs, ref_index)]
    buf = torch.empty(B * 96 * 96 * 1024, dtype=torch.float32, device="cuda")
    shape = (C.c_int32 * 4)()

    def dump(eng, layer, which):
        rc = eng.lib.dll.lsgdbg_run_until(eng.h, *[C.c_void_p(t.data_ptr()) for t in d], B, layer, which,
                                          C.c_void_p(buf.data_ptr()), shape)
        assert rc == 0, eng.lib.dll.lsg_last_error()
        torch.cuda.synchronize()
        n = shape[0] * shape[1] * shape[2] * shape[3]
        return buf[:n].reshape(*shape).clone().cpu()
    t0 = 37 if prec == 4 else 46
    a, b = dump(e16, t0, 0), dump(eq, t0, 0)
    for c0, c1 in ((0, 64), (64, 256), (256, 512), (512, a.shape[-1])):
        if c0 >= a.shape[-1]:
            break
        x, y = a[..., c0:c1], b[..., c0:c1]
        print(f"  input channels [{c0},{c1}): rel {((x - y).norm() / x.norm()).item():.4f}")
    print("  fp16:", a[0, 2, 3, :12].numpy().round(3))
    print("  q   :", b[0, 2, 3, :12].numpy().round(3))
    print("  absmax cat0..6:", eq.act_absmax[2:9])
    s4 = eq.act_absmax[2 + (3 if prec == 4 else 6) - 1] / (255.0 if prec == 4 else 448.0 / 1.1)
    print("  q / s:", (b[0, 2, 3, :12] / s4).numpy().round(3))
    print("  fp16:", a[1, 4, 1, 600:612].numpy().round(3))
    print("  q   :", b[1, 4, 1, 600:612].numpy().round(3))
    for l in range(t0, 49):
        for which in (0, 1):
            a, b = dump(e16, l, which), dump(eq, l, which)
            b = b[..., :a.shape[-1]]
            rel = ((a - b).norm() / a.norm()).item()
            print(f"layer {l} {'in ' if which == 0 else 'out'} shape {tuple(a.shape)} rel {rel:.4f} "
                  f"max16 {a.abs().max():.3f} maxq {b.abs().max():.3f}", flush=True)
    outs = []
    for eng in (e16, eq):
        o = torch.empty(B, 3, 96, 96, dtype=torch.float32, device="cuda")
        eng.forward_device(*[t.data_ptr() for t in d], o.data_ptr(), 0, B)
        torch.cuda.synchronize()
        outs.append(o.cpu().numpy())
    mse = float(np.mean((outs[0] - outs[1]) ** 2))
    print(f"final frames: PSNR q vs fp16 {10 * np.log10(1 / mse):.2f} dB")
    # same through the eager path (B < max_batch: no graph)
    outs = []
    for eng in (e16, eq):
        o = torch.empty(B - 1, 3, 96, 96, dtype=torch.float32, device="cuda")
        eng.forward_device(*[t.data_ptr() for t in d], o.data_ptr(), 0, B - 1)
        torch.cuda.synchronize()
        outs.append(o.cpu().numpy())
    mse = float(np.mean((outs[0] - outs[1]) ** 2))
    print(f"final frames (eager, B-1): PSNR q vs fp16 {10 * np.log10(1 / mse):.2f} dB")


if __name__ == "__main__":
    main()
