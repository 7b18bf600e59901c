"""Run the generator forward `reps` times at batch B on device-resident
inputs (profiling driver: ncu launch lists / --set full captures)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_18318_b200 import api, generator  # noqa: E402


def main():
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    prec = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    ctx = api.Context(0)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    eng = generator.LipsyncEngine(generator.synthetic_weights(0), max_batch=B, ctx=ctx, precision=prec)
    rng = np.random.default_rng(1)
    face = generator.synthetic_face(1)
    d = [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (
        rng.normal(-5, 2.5, (B + 16, 80)).astype(np.float32), rng.integers(0, B, B).astype(np.int32),
        np.stack([face] * B), face[None], np.zeros(B, np.int32))]
    out = torch.empty(B, 96, 96, 3, dtype=torch.uint8, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for r in range(reps):
        e0.record()
        eng.forward_device(*[t.data_ptr() for t in d], out.data_ptr(), 1, B)
        e1.record()
        torch.cuda.synchronize()
        print(f"forward B={B}: {e0.elapsed_time(e1):.3f} ms")


if __name__ == "__main__":
    main()
