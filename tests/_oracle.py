"""ctypes bindings for the checkers under oracle/ (test infrastructure only).

* ``Restated``  -- oracle/_build/liblsg_oracle.so, the plain-C restatement.
* ``Reference`` -- oracle/_ref/libref_lipstream.so, the reference's own
  sources (vad.cpp, segmenter.cpp, mel.cpp, synth.cpp, audio.cpp) compiled
  unmodified by oracle/Makefile.

Also the deterministic fixture generators the reference tests use
(splitmix64 streams, random_pattern from segmenter_tests.cpp:64-76).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "_build", "liblsg_oracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libref_lipstream.so")

M64 = (1 << 64) - 1


def splitmix64(state: list[int]) -> int:
    """include/lipstream/rng.hpp:14-19; ``state`` is a one-element list."""
    state[0] = (state[0] + 0x9E3779B97F4A7C15) & M64
    z = state[0]
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


@dataclass
class Pattern:
    """SpeechPattern (include/lipstream/synth.hpp:21-26)."""
    lead_silence_ms: int = 600
    bursts: list = field(default_factory=lambda: [(1400, 600)])
    tone_hz: float = 220.0
    amplitude: float = 0.3


def random_pattern(state: list[int]) -> Pattern:
    """segmenter_tests.cpp:64-76."""
    def pick(lo, hi, step):
        return lo + step * (splitmix64(state) % ((hi - lo) // step + 1))
    p = Pattern()
    p.lead_silence_ms = pick(0, 600, 20)
    n = pick(1, 3, 1)
    p.bursts = []
    for _ in range(n):
        s = pick(600, 2000, 20)
        q = pick(520, 960, 40)
        p.bursts.append((s, q))
    return p


class CCut(C.Structure):
    _fields_ = [("begin", C.c_int64), ("end", C.c_int64), ("confidence", C.c_double),
                ("cause", C.c_int32), ("pad", C.c_int32),
                ("sample_off", C.c_int64), ("sample_len", C.c_int64)]


SCORER = C.CFUNCTYPE(None, C.c_void_p, C.c_int64, C.c_int64, C.c_int64,
                     C.POINTER(C.c_int), C.POINTER(C.c_double), C.POINTER(C.c_double))


def _i64arr(xs):
    return (C.c_int64 * max(1, len(xs)))(*xs)


class Reference:
    """The reference's own code path (oracle/_ref)."""

    def __init__(self, path: str = REF_SO):
        self.lib = C.CDLL(path)
        L = self.lib
        L.ref_render_pattern.restype = C.c_int
        L.ref_segment.restype = C.c_int
        L.ref_compute_mel.restype = C.c_int64
        L.ref_mel_frame_count.restype = C.c_int64
        L.ref_mel_frame_count.argtypes = [C.c_int64]
        L.ref_splitmix64.restype = C.c_uint64

    def render_pattern(self, p: Pattern, total_ms: int, rate: int = 16000) -> np.ndarray:
        cap = total_ms * rate // 1000 + 16
        out = np.zeros(cap, np.int16)
        n = C.c_int64()
        sp = _i64arr([b[0] for b in p.bursts])
        pa = _i64arr([b[1] for b in p.bursts])
        rc = self.lib.ref_render_pattern(C.c_int64(p.lead_silence_ms), C.c_int(len(p.bursts)), sp, pa,
                                         C.c_double(p.tone_hz), C.c_double(p.amplitude),
                                         C.c_int64(total_ms), C.c_int(rate),
                                         out.ctypes.data_as(C.c_void_p), C.c_int64(cap), C.byref(n))
        if rc:
            raise ValueError(f"render_pattern rc={rc}")
        return out[: n.value].copy()

    # ---- A/V alignment (align.cpp)
    def energy_envelope(self, pcm: np.ndarray, rate: int = 16000) -> np.ndarray:
        pcm = np.ascontiguousarray(pcm, np.int16)
        f = self.lib.ref_energy_envelope
        f.restype = C.c_int64
        n = f(pcm.ctypes.data_as(C.c_void_p), C.c_int64(len(pcm)), C.c_int(rate), None, C.c_int64(0))
        out = np.zeros(max(n, 1), np.float64)
        f(pcm.ctypes.data_as(C.c_void_p), C.c_int64(len(pcm)), C.c_int(rate), out.ctypes.data_as(C.c_void_p),
          C.c_int64(n))
        return out[:n]

    def motion_envelope(self, frames, t0: int, span: int) -> np.ndarray:
        ts = np.ascontiguousarray([f[0] for f in frames] or [0], np.int64)
        mo = np.ascontiguousarray([f[1] for f in frames] or [0.0], np.float64)
        out = np.zeros(max(span, 1), np.float64)
        rc = self.lib.ref_motion_envelope(ts.ctypes.data_as(C.c_void_p), mo.ctypes.data_as(C.c_void_p),
                                          C.c_int64(len(frames)), C.c_int64(t0), C.c_int64(span),
                                          out.ctypes.data_as(C.c_void_p))
        if rc:
            raise ValueError("motion_envelope")
        return out[:span]

    def align(self, e, m, max_lag: int = 50):
        e = np.ascontiguousarray(e, np.float64)
        m = np.ascontiguousarray(m, np.float64)
        off, corr, low = C.c_int64(), C.c_double(), C.c_int()
        rc = self.lib.ref_align_envelopes(e.ctypes.data_as(C.c_void_p), C.c_int64(len(e)),
                                          m.ctypes.data_as(C.c_void_p), C.c_int64(len(m)), C.c_int64(max_lag),
                                          C.byref(off), C.byref(corr), C.byref(low))
        if rc:
            raise ValueError("align_envelopes")
        return off.value, corr.value, bool(low.value)

    def u64_to_unit(self, v: int) -> float:
        f = self.lib.ref_u64_to_unit
        f.restype = C.c_double
        f.argtypes = [C.c_uint64]
        return f(v)

    def ends_in_speech(self, p: Pattern, total_ms: int) -> bool:
        sp = _i64arr([b[0] for b in p.bursts])
        pa = _i64arr([b[1] for b in p.bursts])
        return bool(self.lib.ref_pattern_ends_in_speech(C.c_int64(p.lead_silence_ms), C.c_int(len(p.bursts)),
                                                        sp, pa, C.c_int64(total_ms)))

    def expected_durations(self, p: Pattern, total_ms: int, min_sil=500, min_seg=1500, max_seg=10000):
        sp = _i64arr([b[0] for b in p.bursts])
        pa = _i64arr([b[1] for b in p.bursts])
        out = (C.c_int64 * 4096)()
        n = C.c_int64()
        rc = self.lib.ref_expected_durations(C.c_int64(p.lead_silence_ms), C.c_int(len(p.bursts)), sp, pa,
                                             C.c_int64(total_ms), C.c_int64(min_sil), C.c_int64(min_seg),
                                             C.c_int64(max_seg), out, C.c_int64(4096), C.byref(n))
        if rc:
            raise ValueError(f"expected_durations rc={rc}")
        return [out[i] for i in range(n.value)]

    def segment(self, pcm: np.ndarray, cfg: dict | None = None, chunk_seed: int = 0, start_ms: int = 0,
                scorer=None):
        """Returns (cuts as list of dicts, metrics dict, rc)."""
        c = seg_cfg(cfg)
        pcm = np.ascontiguousarray(pcm, np.int16)
        cap = 1 << 16
        out = (CCut * cap)()
        n = C.c_int64()
        met = (C.c_double * 7)()
        cb = SCORER(scorer) if scorer is not None else SCORER()
        rc = self.lib.ref_segment(pcm.ctypes.data_as(C.c_void_p), C.c_int64(len(pcm)), C.c_int64(start_ms),
                                  C.c_int(c["mode"]), C.c_int(c["peak_mode"]), C.c_double(c["half_life"]),
                                  C.c_double(c["thr"]), C.c_int64(c["frame_ms"]), C.c_int64(c["min_sil"]),
                                  C.c_int64(c["min_seg"]), C.c_int64(c["max_seg"]), C.c_int(c["rate"]),
                                  C.c_uint64(chunk_seed), cb, None, out, C.c_int64(cap), C.byref(n), met)
        cuts = [cut_dict(out[i]) for i in range(min(n.value, cap))] if rc == 0 else []
        metrics = dict(zip(METRIC_KEYS, [met[i] for i in range(7)]))
        return cuts, metrics, rc

    def vad_frames(self, pcm: np.ndarray, cfg: dict | None = None):
        c = seg_cfg(cfg)
        fs = c["rate"] * c["frame_ms"] // 1000
        nf = len(pcm) // fs
        sp = np.zeros(max(nf, 1), np.uint8)
        db = np.zeros(max(nf, 1), np.float64)
        pcm = np.ascontiguousarray(pcm, np.int16)
        rc = self.lib.ref_vad_frames(pcm.ctypes.data_as(C.c_void_p), C.c_int64(len(pcm)), C.c_int(c["peak_mode"]),
                                     C.c_double(c["half_life"]), C.c_double(c["thr"]), C.c_int64(c["frame_ms"]),
                                     C.c_int(c["rate"]), sp.ctypes.data_as(C.c_void_p),
                                     db.ctypes.data_as(C.c_void_p))
        assert rc == 0
        return sp[:nf], db[:nf]

    def compute_mel(self, pcm: np.ndarray, rate=16000, fft=1024, hop=256, n_mels=80, fmin=0.0, fmax=8000.0):
        pcm = np.ascontiguousarray(pcm, np.int16)
        frames = 0 if len(pcm) < fft else 1 + (len(pcm) - fft) // hop
        out = np.zeros(max(frames, 1) * n_mels, np.float32)
        f = self.lib.ref_compute_mel(pcm.ctypes.data_as(C.c_void_p), C.c_int64(len(pcm)), C.c_int(rate),
                                     C.c_int(fft), C.c_int(hop), C.c_int(n_mels), C.c_double(fmin),
                                     C.c_double(fmax), out.ctypes.data_as(C.c_void_p), C.c_int64(out.size))
        if f < 0:
            raise ValueError("compute_mel rejected the config")
        return out[: f * n_mels].reshape(f, n_mels)

    def mel_frame_count(self, n: int) -> int:
        return self.lib.ref_mel_frame_count(n)

    def fft(self, z: np.ndarray) -> np.ndarray:
        buf = np.empty(2 * len(z), np.float64)
        buf[0::2] = z.real
        buf[1::2] = z.imag
        rc = self.lib.ref_fft(buf.ctypes.data_as(C.c_void_p), C.c_int64(len(z)))
        if rc:
            raise ValueError("fft rejected the size")
        return buf[0::2] + 1j * buf[1::2]

    def write_mel(self, path: str, mel: np.ndarray):
        mel = np.ascontiguousarray(mel, np.float32)
        rc = self.lib.ref_write_mel(path.encode(), mel.ctypes.data_as(C.c_void_p), C.c_int64(mel.shape[0]),
                                    C.c_int(mel.shape[1]))
        assert rc == 0


METRIC_KEYS = ["frames", "speech_frames", "cuts_pause", "cuts_forced", "cuts_eos", "scorer_calls",
               "scorer_cost_ms"]


def seg_cfg(cfg: dict | None) -> dict:
    """SegmenterConfig defaults (segmenter.hpp:51-58, vad.hpp:19-24)."""
    c = dict(mode=1, peak_mode=0, half_life=10000.0, thr=-40.0, frame_ms=20, min_sil=500, min_seg=1500,
             max_seg=10000, rate=16000)
    if cfg:
        c.update(cfg)
    return c


def cut_dict(c) -> dict:
    return dict(begin=c.begin, end=c.end, confidence=c.confidence, cause=c.cause,
                sample_off=c.sample_off, sample_len=c.sample_len)


class OrVadCfg(C.Structure):
    _fields_ = [("peak_mode", C.c_int), ("peak_half_life_ms", C.c_double),
                ("speech_threshold_db", C.c_double), ("frame_ms", C.c_int64)]


class OrSegCfg(C.Structure):
    _fields_ = [("mode", C.c_int), ("vad", OrVadCfg), ("min_silence_ms", C.c_int64),
                ("min_segment_ms", C.c_int64), ("max_segment_ms", C.c_int64), ("sample_rate", C.c_int)]


class OrCut(C.Structure):
    _fields_ = [("begin", C.c_int64), ("end", C.c_int64), ("confidence", C.c_double), ("cause", C.c_int),
                ("sample_off", C.c_int64), ("sample_len", C.c_int64)]


class OrMelCfg(C.Structure):
    _fields_ = [("sample_rate", C.c_int), ("fft_size", C.c_int), ("hop", C.c_int), ("n_mels", C.c_int),
                ("fmin", C.c_double), ("fmax", C.c_double)]


class Restated:
    """The plain-C restatement (oracle/lsg_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        self.lib = C.CDLL(path)
        self.lib.or_seg_sizeof.restype = C.c_int64
        self.SEG_BYTES = self.lib.or_seg_sizeof()
        self.lib.or_compute_mel.restype = C.c_int64
        self.lib.or_mel_frame_count.restype = C.c_int64

    # ---- A/V alignment (lsg_oracle.c or_*align*)
    def energy_envelope(self, pcm: np.ndarray, rate: int = 16000) -> np.ndarray:
        pcm = np.ascontiguousarray(pcm, np.int16)
        f = self.lib.or_energy_envelope
        f.restype = C.c_int64
        n = f(pcm.ctypes.data_as(C.c_void_p), C.c_int64(len(pcm)), C.c_int(rate), None, C.c_int64(0))
        out = np.zeros(max(n, 1), np.float64)
        f(pcm.ctypes.data_as(C.c_void_p), C.c_int64(len(pcm)), C.c_int(rate), out.ctypes.data_as(C.c_void_p),
          C.c_int64(n))
        return out[:n]

    def motion_envelope(self, frames, t0: int, span: int) -> np.ndarray:
        ts = np.ascontiguousarray([f[0] for f in frames] or [0], np.int64)
        mo = np.ascontiguousarray([f[1] for f in frames] or [0.0], np.float64)
        out = np.zeros(max(span, 1), np.float64)
        rc = self.lib.or_motion_envelope(ts.ctypes.data_as(C.c_void_p), mo.ctypes.data_as(C.c_void_p),
                                         C.c_int64(len(frames)), C.c_int64(t0), C.c_int64(span),
                                         out.ctypes.data_as(C.c_void_p))
        if rc:
            raise ValueError("motion_envelope")
        return out[:span]

    def align(self, e, m, max_lag: int = 50):
        class R(C.Structure):
            _fields_ = [("offset_ms", C.c_int64), ("peak_corr", C.c_double), ("low", C.c_int)]
        e = np.ascontiguousarray(e, np.float64)
        m = np.ascontiguousarray(m, np.float64)
        r = R()
        rc = self.lib.or_align_envelopes(e.ctypes.data_as(C.c_void_p), C.c_int64(len(e)),
                                         m.ctypes.data_as(C.c_void_p), C.c_int64(len(m)), C.c_int64(max_lag),
                                         C.byref(r))
        if rc:
            raise ValueError("align_envelopes")
        return r.offset_ms, r.peak_corr, bool(r.low)

    def segment(self, pcm: np.ndarray, cfg: dict | None = None, chunks=None, start_ms: int = 0, scorer=None):
        c = seg_cfg(cfg)
        sc = OrSegCfg(c["mode"], OrVadCfg(c["peak_mode"], c["half_life"], c["thr"], c["frame_ms"]), c["min_sil"],
                      c["min_seg"], c["max_seg"], c["rate"])
        state = C.create_string_buffer(self.SEG_BYTES)
        cb = SCORER(scorer) if scorer is not None else SCORER()
        rc = self.lib.or_seg_init(state, C.byref(sc), cb, None)
        if rc:
            return [], {}, rc
        pcm = np.ascontiguousarray(pcm, np.int16)
        cap = 1 << 14
        out = (OrCut * cap)()
        n = C.c_int64()
        cuts = []
        if chunks is None:
            chunks = [len(pcm)] if len(pcm) else []
        off = 0
        try:
            for ln in chunks:
                st = start_ms + off * 1000 // c["rate"]
                rc = self.lib.or_seg_push(state, pcm[off:].ctypes.data_as(C.c_void_p), C.c_int64(ln), C.c_int64(st),
                                          C.c_int(c["rate"]), out, C.c_int64(cap), C.byref(n))
                if rc:
                    return cuts, {}, rc
                cuts += [_orcut(out[i]) for i in range(n.value)]
                off += ln
            rc = self.lib.or_seg_finish(state, out, C.c_int64(cap), C.byref(n))
            cuts += [_orcut(out[i]) for i in range(n.value)]
            m = OrMetrics()
            self.lib.or_seg_get_metrics(state, C.byref(m))
            metrics = dict(zip(METRIC_KEYS, [float(m.v[i]) for i in range(6)] + [m.cost]))
        finally:
            self.lib.or_seg_free(state)
        return cuts, metrics, rc

    def compute_mel(self, pcm: np.ndarray, **kw) -> np.ndarray:
        cfg = OrMelCfg(kw.get("rate", 16000), kw.get("fft", 1024), kw.get("hop", 256), kw.get("n_mels", 80),
                       kw.get("fmin", 0.0), kw.get("fmax", 8000.0))
        pcm = np.ascontiguousarray(pcm, np.int16)
        f = self.lib.or_mel_frame_count(C.c_int64(len(pcm)), C.byref(cfg))
        if f < 0:
            raise ValueError("bad mel config")
        out = np.zeros(max(f, 1) * cfg.n_mels, np.float32)
        self.lib.or_compute_mel(pcm.ctypes.data_as(C.c_void_p), C.c_int64(len(pcm)), C.byref(cfg),
                                out.ctypes.data_as(C.c_void_p))
        return out[: f * cfg.n_mels].reshape(f, cfg.n_mels)

    def filterbank(self, **kw) -> np.ndarray:
        cfg = OrMelCfg(kw.get("rate", 16000), kw.get("fft", 1024), kw.get("hop", 256), kw.get("n_mels", 80),
                       kw.get("fmin", 0.0), kw.get("fmax", 8000.0))
        w = np.zeros((cfg.n_mels, cfg.fft_size // 2 + 1), np.float64)
        assert self.lib.or_mel_filterbank(C.byref(cfg), w.ctypes.data_as(C.c_void_p)) == 0
        return w

    def fft(self, z: np.ndarray) -> np.ndarray:
        buf = np.empty(2 * len(z), np.float64)
        buf[0::2] = z.real
        buf[1::2] = z.imag
        if self.lib.or_fft_radix2(buf.ctypes.data_as(C.c_void_p), C.c_int64(len(z))):
            raise ValueError("fft rejected the size")
        return buf[0::2] + 1j * buf[1::2]


def _orcut(c) -> dict:
    return dict(begin=c.begin, end=c.end, confidence=c.confidence, cause=c.cause,
                sample_off=c.sample_off, sample_len=c.sample_len)


class OrMetrics(C.Structure):
    _fields_ = [("v", C.c_int64 * 6), ("cost", C.c_double)]


def random_chunks(n: int, seed: int) -> list[int]:
    """Chunk lengths 37..4037 drawn like segmenter_tests.cpp:34-47."""
    st = [seed]
    out, off = [], 0
    while off < n:
        ln = 37 + splitmix64(st) % 4001
        ln = min(ln, n - off)
        out.append(ln)
        off += ln
    return out
