"""Where the paced driver's render-latency tail comes from: the 20 slowest
segments (decided time, frames, stream) of a 256-stream real-time run."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2512_18318_b200 import api, generator  # noqa: E402
from paper_2512_18318_b200.paced import LibPacedRunner  # noqa: E402


def main():
    S, secs = int(sys.argv[1]) if len(sys.argv) > 1 else 256, 20
    dl = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    ctx = api.Context(0)
    eng = generator.LipsyncEngine(generator.synthetic_weights(0), max_batch=512, ctx=ctx, precision=1)
    pcm, video, refs = bench.make_workload(0, S, secs + 1, 25.0, api, generator, 1, seed_base=1000)
    ms = max(len(p) for p in pcm)
    pcm_dev = torch.zeros((S, ms), dtype=torch.int16, device="cuda")
    for s, p in enumerate(pcm):
        pcm_dev[s, :len(p)] = torch.from_numpy(p)
    mv = max(len(v) for v in video)
    vid_dev = torch.zeros((S, mv, 96, 96, 3), dtype=torch.uint8, device="cuda")
    for s, v in enumerate(video):
        vid_dev[s, :len(v)] = torch.from_numpy(v)
    refs_dev = torch.from_numpy(refs).cuda()
    ns = [(secs * 1000 - (g % 10) * 400) * 16 for g in range(S)]
    r = LibPacedRunner(eng, S, ms, mv, max_batch=int(sys.argv[3]) if len(sys.argv) > 3 else 512, deadline_ms=dl)
    r.run(pcm_dev, ns, vid_dev, [len(v) for v in video], refs_dev, seconds=2)
    res, segs, _ = r.run(pcm_dev, ns, vid_dev, [len(v) for v in video], refs_dev, seconds=secs)
    ren = np.array([g["rendered_ms"] - g["decided_ms"] for g in segs])
    print("render p50 %.1f p90 %.1f p99 %.1f max %.1f ms; late ticks %d" % (np.percentile(ren, 50),
          np.percentile(ren, 90), np.percentile(ren, 99), ren.max(), res.late_ticks))
    for i in np.argsort(-ren)[:20]:
        g = segs[i]
        print(f"  render {ren[i]:7.1f} ms  decided {g['decided_ms']:8.1f}  end {g['end']:6d}  frames {g['frames']:3d}  "
              f"stream {g['stream']}  cause {g['cause']}")
    # decided-time histogram of the slow ones
    slow = [segs[i]["decided_ms"] for i in np.flatnonzero(ren > 30)]
    print("slow (>30 ms) count", len(slow), "decided-time quantiles", np.percentile(slow, [0, 25, 50, 75, 100]) if slow else None)


if __name__ == "__main__":
    main()
