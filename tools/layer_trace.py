"""Phase timeline of every conv_tc layer of one generator forward, from an
instrumented library (-DLSG_TRACE: globaltimer stamps per CTA, conv_kernel.cuh
LSG_TR).  Build the variant and run:

    python -c "from paper_2512_18318_b200 import build; build.build(lib='abtest/trace/liblsg.so', \
        obj_dir='abtest/trace/_build', extra=['-DLSG_TRACE'])"
    LSG_LIB=abtest/trace/liblsg.so python tools/layer_trace.py [B] [precision]

Columns (us, relative to the layer's first CTA entry): entry spread, setup
done, griddep release (previous layer complete), first stage landed, MMA done,
accumulator ready, split partial stored, split meeting done, split reduce
done, epilogue done, last CTA exit; `gap` = release - previous layer's exit."""
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
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    prec = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    ctx = api.Context(0)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    eng = generator.LipsyncEngine(generator.synthetic_weights(0), max_batch=B, ctx=ctx, precision=prec)
    rng = np.random.default_rng(1)
    face = generator.synthetic_face(1)
    d = [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (
        rng.normal(-5, 2.5, (B + 16, 80)).astype(np.float32), rng.integers(0, B, B).astype(np.int32),
        np.stack([face] * B), face[None], np.zeros(B, np.int32))]
    out = torch.empty(B, 96, 96, 3, dtype=torch.uint8, device="cuda")
    rd = eng.lib.dll.lsgdbg_trace_read
    for _ in range(3):
        eng.forward_device(*[t.data_ptr() for t in d], out.data_ptr(), 1, B)
    torch.cuda.synchronize()
    assert rd(None, C.c_int64(0)) == 0
    torch.cuda.synchronize()
    eng.forward_device(*[t.data_ptr() for t in d], out.data_ptr(), 1, B)
    torch.cuda.synchronize()
    buf = np.zeros(LAYERS * CTAS * EV, np.uint64)
    assert rd(C.c_void_p(buf.ctypes.data), C.c_int64(buf.size)) == 0
    tr = buf.reshape(LAYERS, CTAS, EV).astype(np.float64)
    t0 = None
    prev_exit = None
    cols = ["entry", "setup", "release", "data", "mma", "acc", "stored", "met", "reduced", "epi", "exit"]
    evs = [0, 1, 2, 4, 5, 6, 7, 8, 9, 10, 11]
    print(f"B={B} precision={prec}   (us; columns relative to the layer's first CTA entry; max over CTAs)")
    print(f"{'layer':8} {'start':>8} {'ctas':>4} " + " ".join(f"{c:>7}" for c in cols) + f" {'gap':>6}")
    for li in range(len(NAMES)):
        x = tr[li]
        live = x[:, 0] > 0
        if not live.any():
            prev_exit = None
            print(f"{NAMES[li]:8} (halo kernel: not traced)")
            continue
        x = x[live]
        base = x[:, 0].min()
        if t0 is None:
            t0 = base
        row = []
        for e in evs:
            v = x[:, e]
            v = v[v > 0]
            row.append((v.max() - base) / 1e3 if len(v) else float("nan"))
        gap = (x[:, 2].min() - prev_exit) / 1e3 if prev_exit is not None else float("nan")
        prev_exit = x[:, 11].max()
        print(f"{NAMES[li]:8} {(base - t0) / 1e3:8.1f} {int(live.sum()):4d} " + " ".join(f"{v:7.2f}" for v in row)
              + f" {gap:6.2f}")


if __name__ == "__main__":
    main()
