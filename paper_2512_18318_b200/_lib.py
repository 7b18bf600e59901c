"""ctypes binding of liblsg.so (include/lsg.h).  No fallback: if the library
is missing or no sm_100 device is present, calls fail loudly."""
from __future__ import annotations

import ctypes as C
import os
import re

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LSG_LIB", os.path.join(PKG, "liblsg.so"))  # override: A/B builds in tools/
HEADER = os.path.join(os.path.dirname(PKG), "include", "lsg.h")

LSG_OK, LSG_EINVAL, LSG_ELOGIC, LSG_ERUNTIME, LSG_ECUDA = 0, 1, 2, 3, 4


class LsgError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class InvalidArgument(LsgError, ValueError):
    """std::invalid_argument in the reference."""


class LogicError(LsgError):
    """std::logic_error in the reference."""


class SegCfg(C.Structure):
    _fields_ = [("mode", C.c_int32), ("peak_mode", C.c_int32), ("peak_half_life_ms", C.c_double),
                ("speech_threshold_db", C.c_double), ("frame_ms", C.c_int64), ("min_silence_ms", C.c_int64),
                ("min_segment_ms", C.c_int64), ("max_segment_ms", C.c_int64), ("sample_rate", C.c_int32),
                ("flags_only", C.c_int32)]


class Cut(C.Structure):
    _fields_ = [("begin", C.c_int64), ("end", C.c_int64), ("confidence", C.c_double), ("cause", C.c_int32),
                ("stream", C.c_int32), ("sample_off", C.c_int64), ("sample_len", C.c_int64)]


class SegMetrics(C.Structure):
    _fields_ = [("frames", C.c_int64), ("speech_frames", C.c_int64), ("cuts_pause", C.c_int64),
                ("cuts_forced", C.c_int64), ("cuts_eos", C.c_int64), ("scorer_calls", C.c_int64),
                ("scorer_cost_ms", C.c_double)]


class MelCfg(C.Structure):
    _fields_ = [("sample_rate", C.c_int32), ("fft_size", C.c_int32), ("hop", C.c_int32), ("n_mels", C.c_int32),
                ("fmin", C.c_double), ("fmax", C.c_double)]


class PipeCfg(C.Structure):
    _fields_ = [("n_streams", C.c_int32), ("max_stream_ms", C.c_int32), ("fps", C.c_double),
                ("gather_margin_ms", C.c_int64), ("max_batch", C.c_int32), ("out_format", C.c_int32)]


class FrameRec(C.Structure):
    _fields_ = [("stream", C.c_int32), ("segment", C.c_int32), ("frame_index", C.c_int64), ("ts_ms", C.c_int64),
                ("mel_row", C.c_int32), ("pad", C.c_int32)]


class PacedCfg(C.Structure):
    _fields_ = [("n_streams", C.c_int32), ("fps", C.c_double), ("gather_margin_ms", C.c_int32),
                ("tick_ms", C.c_int32), ("max_batch", C.c_int32), ("deadline_ms", C.c_int32),
                ("max_stream_samples", C.c_int64), ("max_video", C.c_int64)]


class PacedSeg(C.Structure):
    _fields_ = [("stream", C.c_int32), ("segment", C.c_int32), ("begin", C.c_int64), ("end", C.c_int64),
                ("cause", C.c_int32), ("frames", C.c_int32), ("decided_ms", C.c_double), ("rendered_ms", C.c_double)]


class DevRef(C.Structure):
    """lsg_devref: a registry reference (uuid, kind, device, generation, offset, bytes)."""
    _fields_ = [("uuid", C.c_uint8 * 16), ("kind", C.c_int32), ("device", C.c_int32), ("generation", C.c_uint64),
                ("offset", C.c_int64), ("bytes", C.c_int64)]


class PipeStats(C.Structure):
    _fields_ = [("segments", C.c_int64), ("mel_frames", C.c_int64), ("frames_rendered", C.c_int64),
                ("unique_frames", C.c_int64), ("ms_segment", C.c_double), ("ms_mel", C.c_double),
                ("ms_generator", C.c_double), ("ms_total", C.c_double)]


P = C.c_void_p
I32, I64, F64, SZ = C.c_int32, C.c_int64, C.c_double, C.c_size_t
PI32, PI64, PP = C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.POINTER(C.c_void_p)

# name -> argtypes (every function returns lsg_status unless listed in _RESTYPE)
_SIGS = {
    "lsg_abi_version": [],
    "lsg_last_error": [],
    "lsg_device_count": [PI32],
    "lsg_ctx_create": [I32, PP],
    "lsg_ctx_destroy": [P],
    "lsg_ctx_set_stream": [P, P],
    "lsg_ctx_get_stream": [P, PP],
    "lsg_ctx_sync": [P],
    "lsg_ctx_launch_count": [P, PI64],
    "lsg_dev_alloc": [P, SZ, PP],
    "lsg_dev_free": [P, P],
    "lsg_host_alloc": [SZ, PP],
    "lsg_host_free": [P],
    "lsg_copy": [P, P, P, SZ],
    "lsg_seg_cfg_default": [C.POINTER(SegCfg)],
    "lsg_seg_create": [P, C.POINTER(SegCfg), I32, I64, PP],
    "lsg_seg_destroy": [P],
    "lsg_seg_reset": [P],
    "lsg_seg_push": [P, I32, PI32, PP, PI64, PI64, I32, I32],
    "lsg_seg_finish": [P, I32, PI32],
    "lsg_seg_take_cuts": [P, I32, C.POINTER(Cut), I64, PI64],
    "lsg_seg_take_all_cuts": [P, C.POINTER(Cut), I64, PI64],
    "lsg_seg_get_metrics": [P, I32, C.POINTER(SegMetrics)],
    "lsg_seg_take_flags": [P, I32, P, I64, PI64],
    "lsg_mel_cfg_default": [C.POINTER(MelCfg)],
    "lsg_mel_frames": [I64, C.POINTER(MelCfg), PI64],
    "lsg_mel_create": [P, C.POINTER(MelCfg), I64, PP],
    "lsg_mel_destroy": [P],
    "lsg_mel_compute": [P, P, I64, P, PI64],
    "lsg_mel_compute_batch": [P, I32, P, PI64, PI64, P, PI64],
    "lsg_fft_radix2": [P, P, I64, I32],
    "lsg_gen_param_count": [PI64],
    "lsg_gen_layer_info": [PI32, I32, PI32],
    "lsg_gen_create": [P, P, I64, I32, I32, PP],
    "lsg_gen_create_q": [P, P, I64, I32, P, I32, I32, PP],
    "lsg_gen_calibrate": [P, P, P, P, P, P, I32, P, I32, PI32],
    "lsg_gen_destroy": [P],
    "lsg_gen_forward": [P, P, P, P, P, P, P, I32, I32],
    "lsg_lipsync_validate": [I64, I64, I64],
    "lsg_align_energy": [P, I32, P, PI64, PI64, I32, P, PI64, PI64],
    "lsg_kalman_cfg_default": [P],
    "lsg_face_mock_detect": [I64, C.c_uint64, P],
    "lsg_face_track": [P, I32, PI64, PI64, P, P, P, P, C.c_uint64, P, P, P, PI32],
    "lsg_face_crop": [P, I32, P, I32, I32, P, P, P],
    "lsg_align_motion": [P, I32, P, P, PI64, PI64, PI64, PI64, P, PI64],
    "lsg_align_batch": [P, I32, P, PI64, PI64, P, PI64, PI64, I64, P],
    "lsg_pipe_create": [P, C.POINTER(PipeCfg), C.POINTER(SegCfg), C.POINTER(MelCfg), P, PP],
    "lsg_pipe_destroy": [P],
    "lsg_pipe_run": [P, PP, PI64, PP, PI64, P, C.POINTER(FrameRec), P, I64, PI64, C.POINTER(PipeStats)],
    "lsg_mpipe_create": [PI32, I32, C.POINTER(PipeCfg), C.POINTER(SegCfg), C.POINTER(MelCfg), P, I64, I32, P, I32,
                         PP],
    "lsg_mpipe_destroy": [P],
    "lsg_paced_create": [P, C.POINTER(PacedCfg), C.POINTER(SegCfg), C.POINTER(MelCfg), PP],
    "lsg_paced_destroy": [P],
    "lsg_paced_run": [P, P, PI64, P, PI64, P, F64, C.POINTER(PacedSeg), I64, PI64, P, C.POINTER(FrameRec), I64, PI64,
                      PI32],
    "lsg_mpipe_run": [P, PP, PI64, PP, PI64, P, C.POINTER(FrameRec), P, I64, PI64, C.POINTER(PipeStats)],
    "lsg_synth_pattern": [I64, I32, PI64, PI64, F64, F64, I64, I32, P, I64, PI64],
    "lsg_reg_create": [P, I64, PP],
    "lsg_reg_destroy": [P],
    "lsg_reg_put": [P, P, I32, P, I64, C.POINTER(DevRef)],
    "lsg_reg_put_view": [P, P, I32, P, I64, C.POINTER(DevRef)],
    "lsg_reg_alloc": [P, P, I32, I64, PP, C.POINTER(DevRef)],
    "lsg_reg_resolve": [P, C.POINTER(DevRef), PP, PI64],
    "lsg_reg_find": [P, P, I32, C.POINTER(DevRef)],
    "lsg_reg_retain": [P, C.POINTER(DevRef)],
    "lsg_reg_release": [P, C.POINTER(DevRef)],
    "lsg_reg_stats": [P, PI64, PI64, PI64],
    "lsg_devref_encode": [C.POINTER(DevRef), P],
    "lsg_devref_decode": [P, C.POINTER(DevRef)],
}
_RESTYPE = {"lsg_abi_version": C.c_int32, "lsg_last_error": C.c_char_p}


def header_symbols() -> list[str]:
    """Every function declared in include/lsg.h."""
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(lsg_[a-z0-9_]+)\s*\(", txt)) - {"lsg_status"})


class Lib:
    def __init__(self, path: str = LIB_PATH):
        if not os.path.exists(path):
            raise ImportError(f"{path} is not built; run `python -m paper_2512_18318_b200.build` "
                              "(there is no CPU fallback)")
        self.path = path
        self.dll = C.CDLL(path)
        self.missing = []
        for name, args in _SIGS.items():
            if not hasattr(self.dll, name):
                self.missing.append(name)
                continue
            fn = getattr(self.dll, name)
            fn.argtypes = args
            fn.restype = _RESTYPE.get(name, C.c_int)

    def __getattr__(self, name):
        return getattr(self.dll, name)

    def check(self, rc: int):
        if rc == LSG_OK:
            return
        msg = (self.dll.lsg_last_error() or b"").decode()
        cls = {LSG_EINVAL: InvalidArgument, LSG_ELOGIC: LogicError}.get(rc, LsgError)
        raise cls(rc, msg)

    def call(self, name: str, *args):
        self.check(getattr(self.dll, name)(*args))


_LIB: Lib | None = None


def lib() -> Lib:
    global _LIB
    if _LIB is None:
        _LIB = Lib()
    return _LIB
