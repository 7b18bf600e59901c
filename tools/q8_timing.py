"""Generator forward time per precision (B = 128 and 512, CUDA events on the
launching stream, device-resident inputs, bench.measure_generator):
fp16, the fp8 tail, the int8 tail, all-fp8.

    python tools/q8_timing.py
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2512_18318_b200 import generator  # noqa: E402
from paper_2512_18318_b200.api import Context  # noqa: E402


def main():
    ctx = Context(0)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    w = generator.synthetic_weights(0)
    E = generator.LipsyncEngine
    res = {}
    for B in (128, 512):
        for name, prec in (("fp16", E.PREC_FP16), ("fp8_tail", E.PREC_FP8_TAIL), ("int8_tail", E.PREC_INT8_TAIL),
                           ("fp8_all", E.PREC_FP8)):
            eng = E(w, max_batch=B, ctx=ctx, precision=prec)
            ms = bench.measure_generator(eng, torch, stream, 0, B, reps=20)
            eng.close()
            res[f"{name}_b{B}"] = ms
            print(f"B={B:4d} {name:10s} {ms:7.3f} ms  {B / ms * 1e3:9.0f} frames/s", flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
