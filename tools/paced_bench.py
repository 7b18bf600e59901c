"""bench.py's config-5 paced leg alone (lsg_paced, real time):
    python tools/paced_bench.py [streams] [seconds] [deadline_ms]"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2512_18318_b200 import api, generator  # noqa: E402


def main():
    S = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    secs = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    args = argparse.Namespace(paced_streams=S, paced_seconds=secs)
    ctx = api.Context(0)
    st = torch.cuda.Stream()
    ctx.set_stream(st.cuda_stream)
    eng = generator.LipsyncEngine(generator.synthetic_weights(0), max_batch=512, ctx=ctx, precision=1)
    out = bench.paced_leg(args, 0, 1, 0, None, torch, ctx, eng, api, generator, 25.0)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
