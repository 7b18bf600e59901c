"""Multi-stream lip-sync driver over lsg_pipe (the GPU stages of
run_pipeline_input, runner.cpp:239-351): segment -> mel -> gather -> render."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from ._lib import FrameRec, MelCfg, PipeCfg, PipeStats, SegCfg
from .api import MelConfig, SegmenterConfig, default_context

CROP = 96 * 96 * 3


@dataclass
class PipelineConfig:
    n_streams: int
    max_stream_ms: int
    fps: float = 25.0
    gather_margin_ms: int = 50
    max_batch: int = 128
    out_u8: bool = True


class Pipeline:
    def __init__(self, cfg: PipelineConfig, engine, seg: SegmenterConfig | None = None,
                 mel: MelConfig | None = None, ctx=None):
        self.ctx = ctx or engine.ctx or default_context()
        self.lib = self.ctx.lib
        self.cfg = cfg
        pc = PipeCfg(cfg.n_streams, cfg.max_stream_ms, cfg.fps, cfg.gather_margin_ms, cfg.max_batch,
                     1 if cfg.out_u8 else 0)
        sc: SegCfg = (seg or SegmenterConfig()).to_c()
        mc: MelCfg = (mel or MelConfig()).to_c()
        h = C.c_void_p()
        self.lib.call("lsg_pipe_create", self.ctx.h, C.byref(pc), C.byref(sc), C.byref(mc), engine.h, C.byref(h))
        self.h = h
        self.engine = engine

    def close(self):
        if self.h:
            self.lib.lsg_pipe_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def run_ptrs(self, pcm_ptrs, n_samples, video_ptrs, n_video, refs_ptr, frames_ptr=0, cap=0, recs=None):
        """Raw pointers (host or device).  Returns (n_frames, stats dict)."""
        S = self.cfg.n_streams
        pp = (C.c_void_p * S)(*pcm_ptrs)
        ns = (C.c_int64 * S)(*n_samples)
        vp = (C.c_void_p * S)(*video_ptrs)
        nv = (C.c_int64 * S)(*n_video)
        n = C.c_int64()
        st = PipeStats()
        self.lib.call("lsg_pipe_run", self.h, pp, ns, vp, nv, C.c_void_p(refs_ptr), recs, C.c_void_p(frames_ptr),
                      cap, C.byref(n), C.byref(st))
        return n.value, {k: getattr(st, k) for k, _ in PipeStats._fields_}

    def run(self, pcm: list[np.ndarray], video: list[np.ndarray], refs: np.ndarray, cap: int | None = None):
        """Host numpy arrays; returns (records, frames[n,96,96,3] u8, stats)."""
        pcm = [np.ascontiguousarray(p, np.int16) for p in pcm]
        video = [np.ascontiguousarray(v, np.uint8) for v in video]
        refs = np.ascontiguousarray(refs, np.uint8)
        if cap is None:
            cap = sum(len(v) for v in video) * 2 + 64
        px = CROP if self.cfg.out_u8 else CROP * 4
        out = np.zeros(cap * px, np.uint8)
        recs = (FrameRec * max(cap, 1))()
        n, st = self.run_ptrs([p.ctypes.data for p in pcm], [len(p) for p in pcm], [v.ctypes.data for v in video],
                              [len(v) for v in video], refs.ctypes.data, out.ctypes.data, cap, recs)
        k = min(n, cap)
        rec = [dict(stream=recs[i].stream, segment=recs[i].segment, frame_index=recs[i].frame_index,
                    ts_ms=recs[i].ts_ms, mel_row=recs[i].mel_row) for i in range(k)]
        frames = out[: k * px].view(np.uint8 if self.cfg.out_u8 else np.float32)
        frames = frames.reshape(k, 96, 96, 3) if self.cfg.out_u8 else frames.reshape(k, 3, 96, 96)
        return rec, frames, st


class MultiPipeline:
    """lsg_mpipe: the pipeline over several GPUs of ONE process, one host
    thread + context + generator per device, stream s on devices[s % G]
    (SURVEY.md §8 e, no collective).  Same run() contract as Pipeline; the
    records and frames come back in global stream order."""

    def __init__(self, cfg: PipelineConfig, weights: np.ndarray, devices, precision: int = 1,
                 seg: SegmenterConfig | None = None, mel: MelConfig | None = None, act_absmax=None):
        from ._lib import lib
        self.lib = lib()
        self.cfg = cfg
        self.devices = list(devices)
        pc = PipeCfg(cfg.n_streams, cfg.max_stream_ms, cfg.fps, cfg.gather_margin_ms, cfg.max_batch,
                     1 if cfg.out_u8 else 0)
        sc: SegCfg = (seg or SegmenterConfig()).to_c()
        mc: MelCfg = (mel or MelConfig()).to_c()
        w = np.ascontiguousarray(weights, np.float32)
        a = None if act_absmax is None else np.ascontiguousarray(act_absmax, np.float32)
        devs = (C.c_int32 * len(self.devices))(*self.devices)
        h = C.c_void_p()
        self.lib.call("lsg_mpipe_create", devs, len(self.devices), C.byref(pc), C.byref(sc), C.byref(mc),
                      C.c_void_p(w.ctypes.data), w.size, precision,
                      None if a is None else C.c_void_p(a.ctypes.data), 0 if a is None else a.size, C.byref(h))
        self.h = h

    def close(self):
        if self.h:
            self.lib.lsg_mpipe_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def run(self, pcm: list[np.ndarray], video: list[np.ndarray], refs: np.ndarray, cap: int | None = None):
        """Host numpy arrays; returns (records, frames, per-device stats)."""
        S = self.cfg.n_streams
        pcm = [np.ascontiguousarray(p, np.int16) for p in pcm]
        video = [np.ascontiguousarray(v, np.uint8) for v in video]
        refs = np.ascontiguousarray(refs, np.uint8)
        if cap is None:
            cap = sum(len(v) for v in video) * 2 + 64
        px = CROP if self.cfg.out_u8 else CROP * 4
        out = np.zeros(cap * px, np.uint8)
        recs = (FrameRec * max(cap, 1))()
        st = (PipeStats * len(self.devices))()
        n = C.c_int64()
        self.lib.call("lsg_mpipe_run", self.h, (C.c_void_p * S)(*[p.ctypes.data for p in pcm]),
                      (C.c_int64 * S)(*[len(p) for p in pcm]), (C.c_void_p * S)(*[v.ctypes.data for v in video]),
                      (C.c_int64 * S)(*[len(v) for v in video]), C.c_void_p(refs.ctypes.data), recs,
                      C.c_void_p(out.ctypes.data), cap, C.byref(n), st)
        k = min(n.value, cap)
        rec = [dict(stream=recs[i].stream, segment=recs[i].segment, frame_index=recs[i].frame_index,
                    ts_ms=recs[i].ts_ms, mel_row=recs[i].mel_row) for i in range(k)]
        frames = out[: k * px].view(np.uint8 if self.cfg.out_u8 else np.float32)
        frames = frames.reshape(k, 96, 96, 3) if self.cfg.out_u8 else frames.reshape(k, 3, 96, 96)
        return rec, frames, [{f: getattr(s, f) for f, _ in PipeStats._fields_} for s in st]
