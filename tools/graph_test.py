"""Eager vs CUDA-graph replay of the generator forward (is the host's launch
rate part of the small-layer cost?).   python tools/graph_test.py [B] [prec]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_18318_b200 import api, generator  # noqa: E402


def main():
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    prec = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    st = torch.cuda.Stream()
    ctx = api.Context(0)
    ctx.set_stream(st.cuda_stream)
    eng = generator.LipsyncEngine(generator.synthetic_weights(0), max_batch=B, ctx=ctx, precision=prec)
    rng = np.random.default_rng(1)
    face = generator.synthetic_face(1)
    d = [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (
        rng.normal(-5, 2.5, (B + 16, 80)).astype(np.float32), rng.integers(0, B, B).astype(np.int32),
        np.stack([face] * B), face[None], np.zeros(B, np.int32))]
    out = torch.empty(B, 96, 96, 3, dtype=torch.uint8, device="cuda")
    args = [t.data_ptr() for t in d] + [out.data_ptr(), 1, B]
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timed(fn, reps=20):
        ts = []
        for _ in range(reps):
            with torch.cuda.stream(st):
                e0.record(st)
                fn()
                e1.record(st)
            st.synchronize()
            ts.append(e0.elapsed_time(e1))
        return min(ts)

    eager = timed(lambda: eng.forward_device(*args))
    ref = out.clone()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        eng.forward_device(*args)
    g.replay()
    st.synchronize()
    same = torch.equal(out, ref)
    graph = timed(lambda: g.replay())
    print(f"B={B} prec={prec}: eager {eager:.3f} ms, graph replay {graph:.3f} ms, identical={same}")


if __name__ == "__main__":
    main()
