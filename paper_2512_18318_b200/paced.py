"""Paced (real-time) streaming driver: config 5 "paced" of BASELINE.json.

Audio and video of every stream are released in real time (media time T is
available at wall time t0 + T).  Each tick pushes the newly released PCM of
all streams into the device segmenter (lsg_seg_push, device pointers), takes
the cuts it decided, and renders every segment whose frame window
[begin - margin, end + margin] (orchestrator.cpp:90-91, frame_ring.cpp:36-55)
has been released: 80-bin log-mel of the segment audio (lsg_mel_compute_batch,
device-resident), frame -> mel-chunk rule a8 (same rule as
csrc/pipeline.cu), generator forward (lsg_gen_forward) on the gathered crops.

The per-segment latency is (wall time the segment's last rendered frame is
complete on the device) - (wall time media time reached the segment's end),
so it contains the segmenter's own decision delay (a pause cut is only known
once the silence run is long enough, segmenter.cpp:51-99) plus our render
time; both parts are reported.

Host code only orchestrates (the reference's orchestrator is host code too);
every stage runs in the CUDA library.  torch is used for device buffers and
the index gather of face crops."""
from __future__ import annotations

import math
import time
from dataclasses import dataclass

import numpy as np

from .api import MelConfig, MelExtractor, MultiStreamSegmenter, SegmenterConfig

CROP = 96 * 96 * 3


@dataclass
class PacedResult:
    latencies_ms: np.ndarray   # per segment: render complete - media end
    decision_ms: np.ndarray    # per segment: cut known - media end
    render_ms: np.ndarray      # per segment: render complete - cut known
    frames: int
    segments: int
    ticks: int
    late_ticks: int            # ticks whose work overran the tick period


def _pct(a: np.ndarray, q: float) -> float:
    return float(np.percentile(a, q)) if len(a) else float("nan")


class PacedRunner:
    def __init__(self, engine, ctx, torch, n_streams: int, fps: float = 25.0, margin_ms: int = 50,
                 tick_ms: int = 40, seg_cfg: SegmenterConfig | None = None, mel_cfg: MelConfig | None = None):
        self.eng, self.ctx, self.torch = engine, ctx, torch
        self.S, self.fps, self.margin, self.tick = n_streams, fps, margin_ms, tick_ms
        self.seg_cfg = seg_cfg or SegmenterConfig()
        self.mel_cfg = mel_cfg or MelConfig()
        self.rate = self.seg_cfg.sample_rate
        self.hop_ms = self.mel_cfg.hop * 1000.0 / self.mel_cfg.sample_rate
        self.seg = MultiStreamSegmenter(self.seg_cfg, n_streams, self.rate * tick_ms // 1000 + 16, ctx=ctx)
        self.mel = MelExtractor(self.mel_cfg, max_frames=1 << 20, ctx=ctx)
        self.floor = float(math.log(1e-10))

    def run(self, pcm_dev, n_samples, video_dev, n_video, refs_dev, dev: str, seconds: float | None = None
            ) -> PacedResult:
        """pcm_dev: int16 [S, max_samples]; video_dev: uint8 [S, max_video, 96, 96, 3]; refs_dev [S, 96,96,3].
        Runs `seconds` of media (default: all of it); the segmenter starts fresh."""
        torch = self.torch
        self.ctx.lib.call("lsg_seg_reset", self.seg.h)
        S, tick = self.S, self.tick
        max_samples, max_video = pcm_dev.shape[1], video_dev.shape[1]
        vid_flat = video_dev.view(S * max_video, CROP)
        spt = self.rate * tick // 1000                     # samples per tick
        total_ms = int(min(n_samples) * 1000 // self.rate)
        if seconds is not None:
            total_ms = min(total_ms, int(seconds * 1000))
        n_ticks = total_ms // tick
        pending = []                                       # (cut, wall time the cut became known)
        lat, dec, ren = [], [], []
        frames = late = 0
        stream = torch.cuda.current_stream()
        t0 = time.perf_counter()
        for i in range(n_ticks + 1):
            final = i == n_ticks
            media_now = min((i + 1) * tick, total_ms)
            wait = t0 + media_now / 1000.0 - time.perf_counter()
            if wait > 0:
                time.sleep(wait)
            elif i > 0:
                late += 1
            # ---- release this tick's audio to the segmenter (device pointers)
            a, b = i * spt, min((i + 1) * spt, total_ms * self.rate // 1000)
            if b > a:
                base = pcm_dev.data_ptr()
                chunks = [(base + (s * max_samples + a) * 2, b - a) for s in range(S)]
                self.seg.push(list(range(S)), chunks, [a * 1000 // self.rate] * S, on_device=True)
            if final:
                self.seg.finish(list(range(S)))
            now = time.perf_counter()
            for c in self.seg.take_all_cuts():
                pending.append((c, now))
            # ---- segments whose whole frame window is released
            ready = [(c, tk) for c, tk in pending if final or c.end + self.margin <= media_now]
            pending = [(c, tk) for c, tk in pending if not (final or c.end + self.margin <= media_now)]
            if not ready:
                continue
            n_frames = self._render(ready, pcm_dev, max_samples, vid_flat, max_video, n_video, refs_dev, dev)
            stream.synchronize()
            done = time.perf_counter()
            frames += n_frames
            for c, tk in ready:
                media_end = t0 + c.end / 1000.0
                lat.append((done - media_end) * 1000.0)
                dec.append((tk - media_end) * 1000.0)
                ren.append((done - tk) * 1000.0)
        return PacedResult(np.array(lat), np.array(dec), np.array(ren), frames, len(lat), n_ticks + 1, late)

    def _render(self, ready, pcm_dev, max_samples, vid_flat, max_video, n_video, refs_dev, dev) -> int:
        torch = self.torch
        N, hop = self.mel_cfg.fft_size, self.mel_cfg.hop
        offs, lens, row0, jobs_row, jobs_frame, jobs_ref, pads = [], [], [], [], [], [], []
        rows = 0
        for c, _ in ready:
            F = 0 if c.sample_len < N else 1 + (c.sample_len - N) // hop
            R = max(F, 16)
            offs.append(c.stream * max_samples + c.sample_off)
            lens.append(c.sample_len)
            row0.append(rows)
            if F < 16:
                pads.append((rows, F, R))
            lo, hi = c.begin - self.margin, c.end + self.margin
            f = max(0, int(math.floor(lo * self.fps / 1000.0)) - 1)
            while f < n_video[c.stream]:
                ts = int(np.floor(f * 1000.0 / self.fps + 0.5))  # llround (synth.cpp:79)
                if ts > hi:
                    break
                if ts >= lo:
                    k = int(math.floor((ts - c.begin) / self.hop_ms))
                    k = min(max(k, 0), max(0, F - 16))
                    jobs_row.append(rows + k)
                    jobs_frame.append(c.stream * max_video + f)
                    jobs_ref.append(c.stream)
                f += 1
            rows += R
        mel_rows = torch.empty((max(rows, 1), 80), dtype=torch.float32, device=dev)
        self.mel.batch_device(pcm_dev.data_ptr(), offs, lens, mel_rows.data_ptr(), row0)
        for r0, F, R in pads:  # edge-replicate (log floor if F == 0), as pipeline.cu pad_mel
            if F > 0:
                mel_rows[r0 + F:r0 + R] = mel_rows[r0 + F - 1]
            else:
                mel_rows[r0:r0 + R] = self.floor
        J = len(jobs_row)
        if J == 0:
            return 0
        chunk = torch.tensor(jobs_row, dtype=torch.int32, device=dev)
        ref_idx = torch.tensor(jobs_ref, dtype=torch.int32, device=dev)
        target = vid_flat.index_select(0, torch.tensor(jobs_frame, dtype=torch.int64, device=dev))
        out = torch.empty((J, CROP), dtype=torch.uint8, device=dev)
        B = self.eng.max_batch
        for b0 in range(0, J, B):
            nb = min(B, J - b0)
            self.eng.forward_device(mel_rows.data_ptr(), chunk[b0:].data_ptr(), target[b0:].data_ptr(),
                                    refs_dev.data_ptr(), ref_idx[b0:].data_ptr(), out[b0:].data_ptr(), 1, nb)
        return J


class LibPacedRunner:
    """The paced driver in the library (lsg_paced, csrc/paced.cu): the same
    real-time release as PacedRunner, but the tick loop, the segment-ready
    rule, the deadline batcher (a generator batch as soon as max_batch
    frames are queued, or when the oldest has waited deadline_ms) and the
    completion stamps (cudaLaunchHostFunc) all run in C++; generator batches
    never block the tick loop, and the segmenter works on its own context."""

    def __init__(self, engine, n_streams: int, max_stream_samples: int, max_video: int, fps: float = 25.0,
                 margin_ms: int = 50, tick_ms: int = 40, max_batch: int | None = None, deadline_ms: int = 20,
                 seg_cfg: SegmenterConfig | None = None, mel_cfg: MelConfig | None = None):
        import ctypes as C
        from ._lib import PacedCfg, lib
        self.lib = lib()
        self.S = n_streams
        cfg = PacedCfg(n_streams, fps, margin_ms, tick_ms, max_batch or engine.max_batch, deadline_ms,
                       max_stream_samples, max_video)
        h = C.c_void_p()
        self.lib.call("lsg_paced_create", engine.h, C.byref(cfg), C.byref((seg_cfg or SegmenterConfig()).to_c()),
                      C.byref((mel_cfg or MelConfig()).to_c()), C.byref(h))
        self.h = h

    def close(self):
        if self.h:
            self.lib.lsg_paced_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def run(self, pcm_dev, n_samples, video_dev, n_video, refs_dev, seconds: float = 0.0, frames_out=None,
            frames_cap: int = 0):
        """Device tensors as PacedRunner.run; returns (PacedResult, segments
        [dicts], records [dicts] when frames_out is given)."""
        import ctypes as C
        from ._lib import FrameRec, PacedSeg
        S = self.S
        cap = S * 4096
        segs = (PacedSeg * cap)()
        ns = (C.c_int64 * S)(*n_samples)
        nv = (C.c_int64 * S)(*n_video)
        n_seg, n_fr, late = C.c_int64(), C.c_int64(), C.c_int32()
        recs = (FrameRec * max(frames_cap, 1))() if frames_out is not None else None
        self.lib.call("lsg_paced_run", self.h, C.c_void_p(pcm_dev.data_ptr()), ns, C.c_void_p(video_dev.data_ptr()),
                      nv, C.c_void_p(refs_dev.data_ptr()), float(seconds), segs, cap, C.byref(n_seg),
                      C.c_void_p(frames_out.data_ptr()) if frames_out is not None else None, recs, frames_cap,
                      C.byref(n_fr), C.byref(late))
        k = min(n_seg.value, cap)
        out = [dict(stream=segs[i].stream, segment=segs[i].segment, begin=segs[i].begin, end=segs[i].end,
                    cause=segs[i].cause, frames=segs[i].frames, decided_ms=segs[i].decided_ms,
                    rendered_ms=segs[i].rendered_ms) for i in range(k)]
        lat = np.array([s["rendered_ms"] - s["end"] for s in out])
        dec = np.array([s["decided_ms"] - s["end"] for s in out])
        ren = np.array([s["rendered_ms"] - s["decided_ms"] for s in out])
        total_ms = int(max(n_samples) * 1000 // 16000) if seconds <= 0 else int(seconds * 1000)
        res = PacedResult(lat, dec, ren, int(n_fr.value), k, total_ms // 40 + 1, int(late.value))
        rec = None
        if recs is not None:
            rec = [dict(stream=recs[i].stream, segment=recs[i].segment, frame_index=recs[i].frame_index,
                        ts_ms=recs[i].ts_ms, mel_row=recs[i].mel_row) for i in range(min(n_fr.value, frames_cap))]
        return res, out, rec


def summarize(r: PacedResult, streams_total: int, seconds: float) -> dict:
    return {"streams": streams_total, "seconds": seconds, "segments": r.segments, "frames": r.frames,
            "p50_ms": _pct(r.latencies_ms, 50), "p99_ms": _pct(r.latencies_ms, 99),
            "decision_p50_ms": _pct(r.decision_ms, 50), "render_p50_ms": _pct(r.render_ms, 50),
            "render_p99_ms": _pct(r.render_ms, 99), "late_ticks": r.late_ticks, "ticks": r.ticks}
