"""Segmenter on the scaled set (bench.py's stage_rooflines.segmenter): S
streams x 60 s of synthetic speech, device-resident, one push + finish per
stream, L2 flushed before each timed call.  Prints the call time, K1's time
and the cut count; under ncu it is the launch-list driver.
    python tools/seg_bench.py [streams] [reps]"""
import ctypes as C
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import stream_pattern  # noqa: E402
from paper_2512_18318_b200 import api  # noqa: E402


def main():
    S = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    peak_mode = int(sys.argv[3]) if len(sys.argv) > 3 else 0  # 0 Decay, 1 MaxHold, 2 Absolute
    secs, n = 60, 60 * 16000
    ctx = api.Context(0)
    st = torch.cuda.Stream()
    ctx.set_stream(st.cuda_stream)
    pcm = torch.empty((S, n), dtype=torch.int16, device="cuda")
    for s in range(S):
        lead, bursts, hz, amp = stream_pattern(5000 + s)
        pcm[s] = torch.from_numpy(api.synth_pattern(lead, bursts, hz, amp, secs * 1000)[:n])
    cfg = api.SegmenterConfig(vad=api.VadConfig(peak_mode=api.PeakMode(peak_mode)))
    seg = api.MultiStreamSegmenter(cfg, S, n, ctx=ctx)
    base = pcm.data_ptr()
    chunks = [(base + s * n * 2, n) for s in range(S)]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    args = seg.push_args(list(range(S)), chunks, [0] * S)
    for rep in range(reps):
        with torch.cuda.stream(st):
            ctx.lib.call("lsg_seg_reset", seg.h)
            flush.zero_()
            e0.record(st)
            import time
            th0 = time.perf_counter()
            ctx.lib.call("lsg_seg_push", *args[0])
            thp = time.perf_counter()
            ctx.lib.call("lsg_seg_finish", *args[1])
            th1 = time.perf_counter()
            e1.record(st)
        st.synchronize()
        cuts = seg.take_all_cuts()
        k1 = C.c_float()
        ctx.lib.check(ctx.lib.dll.lsgdbg_seg_k1_ms(seg.h, C.byref(k1)))
        cw, chh = C.c_double(), C.c_double()
        ctx.lib.check(ctx.lib.dll.lsgdbg_seg_collect_ms(seg.h, C.byref(cw), C.byref(chh)))
        ms = e0.elapsed_time(e1)
        print(f"segmenter {S} x {secs} s: host push {1e3 * (thp - th0):.3f} ms (+finish {1e3 * (th1 - thp):.3f}); call {ms:.3f} ms = {S * n * 2 / ms / 1e6:.0f} GB/s, "
              f"K1 {k1.value:.3f} ms = {S * n * 2 / k1.value / 1e6:.0f} GB/s, {len(cuts)} cuts; "
              f"finish: sync wait {cw.value:.3f} ms, host distribution {chh.value:.3f} ms")


if __name__ == "__main__":
    main()
