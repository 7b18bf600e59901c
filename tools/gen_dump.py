"""Render a seeded batch through the generator and save the u8 frames
(tests/test_generator_paths.py: the same batch under different launch knobs
-- LSG_GEN_KNOBS -- and across repeated runs).

    python tools/gen_dump.py B precision out.npy [reps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_18318_b200 import api, generator  # noqa: E402


def main():
    B, prec, path = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
    reps = int(sys.argv[4]) if len(sys.argv) > 4 else 1
    ctx = api.Context(0)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    eng = generator.LipsyncEngine(generator.synthetic_weights(0), max_batch=B, ctx=ctx, precision=prec)
    rng = np.random.default_rng(11)
    faces = np.stack([np.roll(generator.synthetic_face(1 + (i % 5)), i % 7, axis=1) for i in range(B)])
    d = [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (
        rng.normal(-5, 2.5, (B + 16, 80)).astype(np.float32), rng.integers(0, B, B).astype(np.int32),
        faces, generator.synthetic_face(9)[None], np.zeros(B, np.int32))]
    outs = []
    for _ in range(reps):
        out = torch.empty(B, 96, 96, 3, dtype=torch.uint8, device="cuda")
        eng.forward_device(*[t.data_ptr() for t in d], out.data_ptr(), 1, B)
        torch.cuda.synchronize()
        outs.append(out.cpu().numpy())
    np.save(path, np.stack(outs))


if __name__ == "__main__":
    main()
