"""Mel on many segments, device-resident (profiling driver for the mel kernel):
    python tools/mel_bench.py [n_segments] [seconds]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_18318_b200 import api  # noqa: E402


def main():
    nseg = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    secs = float(sys.argv[2]) if len(sys.argv) > 2 else 2.0
    n = int(secs * 16000)
    ctx = api.Context(0)
    st = torch.cuda.Stream()
    ctx.set_stream(st.cuda_stream)
    pcm = torch.randint(-8000, 8000, (nseg * n,), dtype=torch.int16, device="cuda")
    F = 1 + (n - 1024) // 256
    rows = torch.empty((nseg * F, 80), dtype=torch.float32, device="cuda")
    mel = api.MelExtractor(ctx=ctx, max_frames=1 << 22)
    offs = [s * n for s in range(nseg)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for rep in range(3):
        with torch.cuda.stream(st):
            e0.record(st)
            mel.batch_device(pcm.data_ptr(), offs, [n] * nseg, rows.data_ptr(), [s * F for s in range(nseg)])
            e1.record(st)
        st.synchronize()
        ms = e0.elapsed_time(e1)
        print(f"mel {nseg} x {secs} s: {ms:.3f} ms, {nseg * F / ms / 1e3:.1f} M frames/s, "
              f"{nseg * F * 25600 / ms / 1e9:.2f} TFLOP/s fp64")


if __name__ == "__main__":
    main()
