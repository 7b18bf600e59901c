"""Real (PDL-overlapped) per-layer cost of the generator forward: time the
prefix of the layer chain ending at each layer (lsgdbg_run_until without the
readback) and difference consecutive prefixes.  ncu launch lists serialise
kernels and add per-launch overhead; this is what the forward actually pays.

    python tools/layer_inc.py [B] [precision 0 bf16 | 1 fp16 | 2 fp8] [reps]"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_18318_b200 import api, generator  # noqa: E402

NAMES = ("fe0 fe1.0 fe1.1 fe1.2 fe2.0 fe2.1 fe2.2 fe2.3 fe3.0 fe3.1 fe3.2 fe4.0 fe4.1 fe4.2 fe5.0 fe5.1 fe6.0 fe6.1 "
         "ae0 ae1 ae2 ae3 ae4 ae5 ae6 ae7 ae8 ae9 ae10 ae11 ae12 fd0 fd1.0 fd1.1 fd2.0 fd2.1 fd2.2 fd3.0 fd3.1 fd3.2 "
         "fd4.0 fd4.1 fd4.2 fd5.0 fd5.1 fd5.2 fd6.0 fd6.1 fd6.2 out0+1").split()


def main():
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    prec = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    ctx = api.Context(0)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    eng = generator.LipsyncEngine(generator.synthetic_weights(0), max_batch=B, ctx=ctx, precision=prec)
    rng = np.random.default_rng(1)
    face = generator.synthetic_face(1)
    d = [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (
        rng.normal(-5, 2.5, (B + 16, 80)).astype(np.float32), rng.integers(0, B, B).astype(np.int32),
        np.stack([face] * B), face[None], np.zeros(B, np.int32))]
    out = torch.empty(B, 96, 96, 3, dtype=torch.uint8, device="cuda")
    fn = eng.lib.dll.lsgdbg_run_until
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timed(call):
        ts = []
        for _ in range(reps):
            e0.record()
            call()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        return float(np.median(ts))

    def prefix(stop):
        return lambda: fn(eng.h, *[C.c_void_p(t.data_ptr()) for t in d], B, stop, 1, None, None)

    def full():
        eng.forward_device(*[t.data_ptr() for t in d], out.data_ptr(), 1, B)

    timed(full)
    nL = len(NAMES)
    t = [timed(prefix(i)) for i in range(nL - 1)] + [timed(full)]
    prev = 0.0
    print(f"B={B} precision={prec}: per-layer increments of the PDL-overlapped chain (us)")
    for i, name in enumerate(NAMES):
        print(f"{i:3d} {name:8} {t[i] - prev:8.1f}   prefix {t[i]:8.1f}")
        prev = t[i]
    print(f"full forward {t[-1]:.1f} us")


if __name__ == "__main__":
    main()
