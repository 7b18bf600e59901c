"""Where each conv_halo layer's time goes, per warp role: cycles the
producer, the MMA issuer and the epilogue groups spend waiting on each
barrier, from an instrumented library (-DLSG_TRACE: conv_halo.cuh LSG_HW).

    python -c "from paper_2512_18318_b200 import build; build.build(lib='abtest/trace/liblsg.so', \\
        obj_dir='abtest/trace/_build', extra=['-DLSG_TRACE'])"
    LSG_LIB=abtest/trace/liblsg.so python tools/halo_waits.py [B] [precision]

Per layer (CTA average, % of that role's own loop time): producer waits on
hempty; MMA waits on tempty / hfull / bfull (streamed weights); epilogue waits on the staging
drain + group barrier, rfull, tfull, and its math + staging share."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_18318_b200 import api, generator  # noqa: E402
from layer_inc import NAMES  # noqa: E402

EV, CTAS, LAYERS = 16, 160, 64


def main():
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    prec = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    ctx = api.Context(0)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    eng = generator.LipsyncEngine(generator.synthetic_weights(0), max_batch=B, ctx=ctx, precision=prec)
    rng = np.random.default_rng(1)
    face = generator.synthetic_face(1)
    d = [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (
        rng.normal(-5, 2.5, (B + 16, 80)).astype(np.float32), rng.integers(0, B, B).astype(np.int32),
        np.stack([face] * B), face[None], np.zeros(B, np.int32))]
    out = torch.empty(B, 96, 96, 3, dtype=torch.uint8, device="cuda")
    lib = eng.lib.dll
    eng.forward_device(*[t.data_ptr() for t in d], out.data_ptr(), 1, B)
    torch.cuda.synchronize()
    lib.lsgdbg_trace_read(None, C.c_int64(0))  # clear
    eng.forward_device(*[t.data_ptr() for t in d], out.data_ptr(), 1, B)
    torch.cuda.synchronize()
    buf = np.zeros(LAYERS * CTAS * EV, np.uint64)
    lib.lsgdbg_trace_read(C.c_void_p(buf.ctypes.data), C.c_int64(buf.size))
    t = buf.reshape(LAYERS, CTAS, EV).astype(np.float64)
    print(f"B={B} precision={prec}: per-CTA averages, % of the role's loop time")
    print("layer     | producer: loop us  hempty | MMA: loop us  tempty hfull bfull | "
          "epilogue: loop us  drain  rfull  tfull  math")
    for l in range(LAYERS):
        x = t[l]
        act = x[:, 2] > 0
        if not act.any():
            continue
        m = x[act].mean(axis=0)
        ghz = 1.9e3  # cycles per us (nominal; ratios are clock-free)
        pr, mm, ep = m[2], m[5], m[10] / 2  # epilogue: two groups summed

        def pc(v, tot):
            return 100.0 * v / tot if tot else 0.0
        name = NAMES[l] if l < len(NAMES) else str(l)
        print(f"{l:2d} {name:6s} | {pr / ghz:8.1f} {pc(m[0], pr):7.1f} | "
              f"{mm / ghz:8.1f} {pc(m[3], mm):7.1f} {pc(m[4], mm):5.1f} {pc(m[1], mm):5.1f} | "
              f"{ep / ghz:8.1f} {pc(m[6] / 2, ep):6.1f} {pc(m[7] / 2, ep):6.1f} {pc(m[8] / 2, ep):6.1f} "
              f"{pc(m[9] / 2, ep):5.1f}")


if __name__ == "__main__":
    main()
