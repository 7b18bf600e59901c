"""Segmenter / mel stage rooflines alone (bench.py's scaled leg), for
iterating on those kernels and for ncu launch lists:
    python tools/stage_bench.py [streams]"""
import json
import os
import sys
import types

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    import torch
    from paper_2512_18318_b200 import api
    streams = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    ctx = api.Context(0)
    s = torch.cuda.Stream()
    args = types.SimpleNamespace(scaled_streams=streams)
    print(json.dumps(bench.scaled_leg(args, 0, torch, ctx, s, api), indent=1))


if __name__ == "__main__":
    main()
