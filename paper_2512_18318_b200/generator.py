"""Wav2Lip generator host side: layer table (from liblsg), synthetic
BN-calibrated weights, synthetic face crops, and the LipsyncEngine wrapper
over lsg_gen (the GPU forward).

The reference has no generator (mock_lipsync is a cost model,
visual_mocks.cpp:40-51) and no checkpoint is available offline, so weights
are synthetic: He-normal convolutions whose BatchNorm running statistics are
calibrated on a seeded batch (pre-activations ~N(0,1), output logits
~N(0,1)) and then folded -- random weights otherwise saturate the sigmoid and
make any precision comparison meaningless.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from ._lib import lib

CONV, CONVT = 0, 1


@dataclass(frozen=True)
class Layer:
    kind: int
    cin: int
    cout: int
    kh: int
    kw: int
    sh: int
    sw: int
    ph: int
    pw: int
    oph: int
    opw: int
    res: int

    @property
    def n_params(self) -> int:
        return self.cin * self.cout * self.kh * self.kw + self.cout


def layers() -> list[Layer]:
    L = lib()
    info = (C.c_int32 * (12 * 64))()
    n = C.c_int32()
    L.call("lsg_gen_layer_info", info, 64, C.byref(n))
    return [Layer(*[info[12 * i + j] for j in range(12)]) for i in range(n.value)]


def param_count() -> int:
    n = C.c_int64()
    lib().call("lsg_gen_param_count", C.byref(n))
    return n.value


# face encoder blocks / decoder blocks as [first, last] layer indices
FACE_BLOCKS = [(0, 0), (1, 3), (4, 7), (8, 10), (11, 13), (14, 15), (16, 17)]
AUDIO = (18, 30)
DEC_BLOCKS = [(31, 31), (32, 33), (34, 36), (37, 39), (40, 42), (43, 45), (46, 48)]
OUT0, OUT1 = 49, 50


def layer_shapes() -> list[tuple[int, int, int, int]]:
    """(H_in, W_in, H_out, W_out) per layer, walking the Wav2Lip graph."""
    Ls = layers()
    shapes = [None] * len(Ls)

    def out_hw(L, h, w):
        if L.kind == CONV:
            return (h + 2 * L.ph - L.kh) // L.sh + 1, (w + 2 * L.pw - L.kw) // L.sw + 1
        return (h - 1) * L.sh - 2 * L.ph + L.kh + L.oph, (w - 1) * L.sw - 2 * L.pw + L.kw + L.opw

    def run(a, b, h, w):
        for i in range(a, b + 1):
            oh, ow = out_hw(Ls[i], h, w)
            shapes[i] = (h, w, oh, ow)
            h, w = oh, ow
        return h, w
    h, w = 96, 96
    for a, b in FACE_BLOCKS:
        h, w = run(a, b, h, w)
    h, w = run(AUDIO[0], AUDIO[1], 80, 16)
    for a, b in DEC_BLOCKS:
        h, w = run(a, b, h, w)
    run(OUT0, OUT1, h, w)
    return shapes


def flops_per_frame() -> float:
    """Algorithmic FLOPs of one forward (2 x MAC; convT counted on its input
    grid, Hin*Win*Cin*Cout*k*k, i.e. no zero-insertion work)."""
    tot = 0
    for L, (hi, wi, ho, wo) in zip(layers(), layer_shapes()):
        pix = ho * wo if L.kind == CONV else hi * wi
        tot += 2 * pix * L.cin * L.cout * L.kh * L.kw
    return float(tot)


def synthetic_face(seed: int, size: int = 96) -> np.ndarray:
    """Smooth synthetic face crop [96,96,3] u8: gradient background, skin
    ellipse, darker eyes and mouth, seeded colours and mild noise."""
    rng = np.random.default_rng(seed)
    y, x = np.mgrid[0:size, 0:size].astype(np.float32) / size
    bg = rng.uniform(40, 200, 3)
    img = bg[None, None, :] * (0.6 + 0.4 * y[..., None])
    skin = rng.uniform([150, 100, 80], [240, 190, 160])
    face = ((x - 0.5) / 0.36) ** 2 + ((y - 0.52) / 0.45) ** 2 < 1.0
    img[face] = skin
    for ex in (0.35, 0.65):
        eye = ((x - ex) / 0.07) ** 2 + ((y - 0.4) / 0.04) ** 2 < 1.0
        img[eye] = skin * 0.3
    mouth = ((x - 0.5) / (0.14 + 0.04 * rng.random())) ** 2 + ((y - 0.72) / 0.05) ** 2 < 1.0
    img[mouth] = [120, 30, 40]
    img += rng.normal(0, 4, img.shape)
    return np.clip(img, 0, 255).astype(np.uint8)


def jitter_face(ref: np.ndarray, frame_index: int, seed: int) -> np.ndarray:
    """Per-frame target: the reference crop shifted by a seeded +-3 px wobble
    (mock_face_detect's jitter, visual_mocks.cpp:10-22)."""
    rng = np.random.default_rng((seed * 1000003 + frame_index) & 0xFFFFFFFF)
    dy, dx = rng.integers(-3, 4, 2)
    return np.roll(ref, (int(dy), int(dx)), axis=(0, 1))


def _forward_calibrate(blob_layers, mel, faces, rng):
    """fp32 forward that sets each BN layer's statistics from its own
    pre-activations (batch statistics, gamma=1, beta=0) and folds them."""
    import torch
    import torch.nn.functional as F
    Ls = layers()
    out = []

    def conv(i, x):
        L = Ls[i]
        fan_in = L.cin * L.kh * L.kw / (L.sh * L.sw if L.kind == CONVT else 1)
        std = np.sqrt(2.0 / fan_in)
        if L.kind == CONV:
            w = rng.normal(0, std, (L.cout, L.cin, L.kh, L.kw)).astype(np.float32)
            y = F.conv2d(x, torch.from_numpy(w), None, (L.sh, L.sw), (L.ph, L.pw))
        else:
            w = rng.normal(0, std, (L.cin, L.cout, L.kh, L.kw)).astype(np.float32)
            y = F.conv_transpose2d(x, torch.from_numpy(w), None, (L.sh, L.sw), (L.ph, L.pw), (L.oph, L.opw))
        if i == OUT1:
            mu = y.mean(dim=(0, 2, 3)).numpy()
            sd = y.std(dim=(0, 2, 3)).numpy() + 1e-6
            w = w / sd[:, None, None, None]
            b = (-mu / sd).astype(np.float32)
            out.append((w.astype(np.float32), b))
            return (y - torch.from_numpy(mu)[None, :, None, None]) / torch.from_numpy(sd)[None, :, None, None]
        mu = y.mean(dim=(0, 2, 3))
        var = y.var(dim=(0, 2, 3), unbiased=False)
        inv = 1.0 / torch.sqrt(var + 1e-5)
        shape = (-1, 1, 1, 1) if L.kind == CONV else (1, -1, 1, 1)
        wf = (torch.from_numpy(w) * inv.reshape(shape)).numpy().astype(np.float32)
        bf = (-mu * inv).numpy().astype(np.float32)
        out.append((wf, bf))
        y = (y - mu[None, :, None, None]) * inv[None, :, None, None]
        if L.res:
            y = y + x
        return torch.relu(y)

    feats = []
    x = faces
    for a, b in FACE_BLOCKS:
        for i in range(a, b + 1):
            x = conv(i, x)
        feats.append(x)
    a_out = mel
    for i in range(AUDIO[0], AUDIO[1] + 1):
        a_out = conv(i, a_out)
    # weights must be appended in layer order: audio layers were generated
    # after the face layers, matching the blob order (face, audio, decoder)
    x = a_out
    for a, b in DEC_BLOCKS:
        for i in range(a, b + 1):
            x = conv(i, x)
        x = torch.cat([x, feats.pop()], dim=1)
    x = conv(OUT0, x)
    conv(OUT1, x)
    return out


def synthetic_weights(seed: int = 0, calib: int = 16) -> np.ndarray:
    """Folded fp32 weight blob in lsg_gen's layer order (deterministic)."""
    import torch
    torch.set_num_threads(max(1, torch.get_num_threads()))
    rng = np.random.default_rng(seed)
    crng = np.random.default_rng(seed + 12345)
    mel = torch.from_numpy(crng.normal(-5.0, 2.5, (calib, 1, 80, 16)).astype(np.float32))
    faces = np.stack([face_input(synthetic_face(seed * 100 + i), synthetic_face(seed * 100 + i + 50))
                      for i in range(calib)])
    with torch.no_grad():
        folded = _forward_calibrate(None, mel, torch.from_numpy(faces), rng)
    blob = np.concatenate([np.concatenate([w.ravel(), b.ravel()]) for w, b in folded]).astype(np.float32)
    assert blob.size == param_count(), (blob.size, param_count())
    return blob


def face_input(target_u8: np.ndarray, ref_u8: np.ndarray) -> np.ndarray:
    """[6,96,96] f32 network input: lower half of the target masked, then the
    reference, /255 (Wav2Lip's preprocessing)."""
    t = target_u8.astype(np.float32) / 255.0
    t[48:] = 0.0
    r = ref_u8.astype(np.float32) / 255.0
    return np.concatenate([t, r], axis=2).transpose(2, 0, 1).copy()


def calibration_batch(seed: int = 7, frames: int = 64):
    """Seeded calibration inputs for the fp8 activation ranges (SURVEY §8 d:
    a 64-frame seeded batch): mel rows of synthetic speech through the
    library's own mel stage (silence included, so the log floor is in range),
    jittered synthetic faces.  Returns host arrays
    (mel_rows [R,80] f32, chunk_row [B] i32, target [B,96,96,3] u8,
     refs [R,96,96,3] u8, ref_index [B] i32)."""
    from .api import AudioBuffer, compute_mel, synth_pattern
    rng = np.random.default_rng(seed)
    pcm = synth_pattern(300, [(900, 500), (1200, 700), (800, 600)], 220.0, 0.3, 6000)
    mel = compute_mel(AudioBuffer(samples=pcm)).data.reshape(-1, 80).astype(np.float32)
    chunk = rng.integers(0, mel.shape[0] - 16, frames).astype(np.int32)
    refs = np.stack([synthetic_face(seed * 1000 + i) for i in range(4)])
    ridx = rng.integers(0, 4, frames).astype(np.int32)
    target = np.stack([np.roll(refs[r], (int(a), int(b)), axis=(0, 1))
                       for r, a, b in zip(ridx, rng.integers(-3, 4, frames), rng.integers(-3, 4, frames))])
    return mel, chunk, target.astype(np.uint8), refs.astype(np.uint8), ridx


class _Dev:
    """Device copies of host arrays through the library's allocator."""

    def __init__(self, ctx, arrays):
        self.ctx, self.ptrs = ctx, []
        for a in arrays:
            a = np.ascontiguousarray(a)
            p = C.c_void_p()
            ctx.lib.call("lsg_dev_alloc", ctx.h, max(a.nbytes, 1), C.byref(p))
            ctx.lib.call("lsg_copy", ctx.h, p, C.c_void_p(a.ctypes.data), a.nbytes)
            self.ptrs.append(p)
        ctx.sync()

    def free(self):
        for p in self.ptrs:
            self.ctx.lib.lsg_dev_free(self.ctx.h, p)
        self.ptrs = []


def calibrate(weights: np.ndarray, ctx, batch=None) -> np.ndarray:
    """max |x| per fp8 scale group (lsg_gen_calibrate on an fp16 engine)."""
    mel, chunk, target, refs, ridx = batch or calibration_batch()
    B = len(chunk)
    eng = LipsyncEngine(weights, max_batch=B, ctx=ctx, precision=LipsyncEngine.PREC_FP16)
    dev = _Dev(ctx, [mel, chunk, target, refs, ridx])
    try:
        n = C.c_int32()
        eng.lib.call("lsg_gen_calibrate", eng.h, *dev.ptrs[:5], B, None, 0, C.byref(n))
        out = np.zeros(n.value, np.float32)
        eng.lib.call("lsg_gen_calibrate", eng.h, *dev.ptrs[:5], B, C.c_void_p(out.ctypes.data), n.value, C.byref(n))
    finally:
        dev.free()
        eng.close()
    return out


class LipsyncEngine:
    """The lip-sync stage on the GPU (lsg_gen): replaces mock_lipsync's cost
    model (visual_mocks.hpp:41-43) with the generator forward.  precision
    The 8-bit precisions calibrate per-tensor activation ranges first
    (calibrate()); PREC_FP8_TAIL runs fp16 up to fd5.2 and e4m3 from fd6.0
    on, PREC_INT8_TAIL fp16 up to fd0 and u8 x s8 (kind::i8) from fd1.0 on
    (the splits that keep >= 30 dB vs the fp32 oracle)."""

    PREC_BF16, PREC_FP16, PREC_FP8, PREC_FP8_TAIL, PREC_INT8_TAIL = 0, 1, 2, 3, 4
    int8_headroom = 1.0  # u8 activation scale = calibrated max |x| * headroom / 255 (generator.cu)

    def __init__(self, weights: np.ndarray, max_batch: int = 128, ctx=None, precision: int = 1, calib=None):
        from .api import default_context
        self.ctx = ctx or default_context()
        self.lib = self.ctx.lib
        w = np.ascontiguousarray(weights, np.float32)
        h = C.c_void_p()
        self.precision = precision
        self.act_absmax = None
        if precision in (self.PREC_FP8, self.PREC_FP8_TAIL, self.PREC_INT8_TAIL):
            self.act_absmax = calibrate(w, self.ctx, calib)
            a = self.act_absmax
            self.lib.call("lsg_gen_create_q", self.ctx.h, C.c_void_p(w.ctypes.data), w.size, precision,
                          C.c_void_p(a.ctypes.data), a.size, max_batch, C.byref(h))
        else:
            self.lib.call("lsg_gen_create", self.ctx.h, C.c_void_p(w.ctypes.data), w.size, precision, max_batch,
                          C.byref(h))
        self.h = h
        self.max_batch = max_batch

    def close(self):
        if self.h:
            self.lib.lsg_gen_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def forward_device(self, mel_rows: int, chunk_row: int, target: int, refs: int, ref_index: int, out: int,
                       out_format: int, B: int):
        """All arguments are device pointers (ints)."""
        self.lib.call("lsg_gen_forward", self.h, C.c_void_p(mel_rows), C.c_void_p(chunk_row), C.c_void_p(target),
                      C.c_void_p(refs), C.c_void_p(ref_index), C.c_void_p(out), out_format, B)

    @staticmethod
    def validate(audio_span_ms: int, frame_span_ms: int, n_frames: int):
        lib().call("lsg_lipsync_validate", audio_span_ms, frame_span_ms, n_frames)
