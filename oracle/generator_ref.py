"""fp32 CPU restatement of the Wav2Lip generator forward -- the oracle for
the GPU lip-sync stage.  TEST INFRASTRUCTURE ONLY (tests/, smoke(),
bench.py's cpu_baseline leg).

The reference repository has no generator: its lip-sync stage is the cost
model mock_lipsync (proj/core/src/visual_mocks.cpp:24-51), so GENERATOR
PARITY IS UNPINNED BY THE REFERENCE.  The topology restated here is the
public Wav2Lip generator (models/wav2lip.py of Wav2Lip, referenced by name in
PAPER.md:57, :190-194, :246), as tabulated in SURVEY.md Appendix B:

  Conv block  = Conv2d -> BatchNorm (folded into the weights) -> (+x) -> ReLU
  ConvT block = ConvTranspose2d -> BatchNorm (folded) -> ReLU
  audio_embedding = audio_encoder(mel[B,1,80,16])            -> [B,512,1,1]
  feats = outputs of the 7 face-encoder blocks on face[B,6,96,96]
  x = audio_embedding; for each decoder block: x = cat(block(x), feats.pop())
  out = sigmoid(conv1x1_32->3(Conv(80->32)(x)))

It is written in NCHW with torch.nn.functional (fp32, CPU), independently
of the GPU's NHWC implicit-GEMM / phase-decomposed formulation.  The layer
table below is restated from Wav2Lip and checked against the library's
lsg_gen_layer_info by tests/test_generator.py.
"""
from __future__ import annotations

import numpy as np

# (kind, cin, cout, k, stride(h,w), pad, output_padding, residual)
C_, T_ = 0, 1
FACE = [
    [(C_, 6, 16, 7, (1, 1), 3, 0, 0)],
    [(C_, 16, 32, 3, (2, 2), 1, 0, 0), (C_, 32, 32, 3, (1, 1), 1, 0, 1), (C_, 32, 32, 3, (1, 1), 1, 0, 1)],
    [(C_, 32, 64, 3, (2, 2), 1, 0, 0)] + [(C_, 64, 64, 3, (1, 1), 1, 0, 1)] * 3,
    [(C_, 64, 128, 3, (2, 2), 1, 0, 0)] + [(C_, 128, 128, 3, (1, 1), 1, 0, 1)] * 2,
    [(C_, 128, 256, 3, (2, 2), 1, 0, 0)] + [(C_, 256, 256, 3, (1, 1), 1, 0, 1)] * 2,
    [(C_, 256, 512, 3, (2, 2), 1, 0, 0), (C_, 512, 512, 3, (1, 1), 1, 0, 1)],
    [(C_, 512, 512, 3, (1, 1), 0, 0, 0), (C_, 512, 512, 1, (1, 1), 0, 0, 0)],
]
AUDIO = [
    (C_, 1, 32, 3, (1, 1), 1, 0, 0), (C_, 32, 32, 3, (1, 1), 1, 0, 1), (C_, 32, 32, 3, (1, 1), 1, 0, 1),
    (C_, 32, 64, 3, (3, 1), 1, 0, 0), (C_, 64, 64, 3, (1, 1), 1, 0, 1), (C_, 64, 64, 3, (1, 1), 1, 0, 1),
    (C_, 64, 128, 3, (3, 3), 1, 0, 0), (C_, 128, 128, 3, (1, 1), 1, 0, 1), (C_, 128, 128, 3, (1, 1), 1, 0, 1),
    (C_, 128, 256, 3, (3, 2), 1, 0, 0), (C_, 256, 256, 3, (1, 1), 1, 0, 1),
    (C_, 256, 512, 3, (1, 1), 0, 0, 0), (C_, 512, 512, 1, (1, 1), 0, 0, 0),
]
DECODER = [
    [(C_, 512, 512, 1, (1, 1), 0, 0, 0)],
    [(T_, 1024, 512, 3, (1, 1), 0, 0, 0), (C_, 512, 512, 3, (1, 1), 1, 0, 1)],
    [(T_, 1024, 512, 3, (2, 2), 1, 1, 0)] + [(C_, 512, 512, 3, (1, 1), 1, 0, 1)] * 2,
    [(T_, 768, 384, 3, (2, 2), 1, 1, 0)] + [(C_, 384, 384, 3, (1, 1), 1, 0, 1)] * 2,
    [(T_, 512, 256, 3, (2, 2), 1, 1, 0)] + [(C_, 256, 256, 3, (1, 1), 1, 0, 1)] * 2,
    [(T_, 320, 128, 3, (2, 2), 1, 1, 0)] + [(C_, 128, 128, 3, (1, 1), 1, 0, 1)] * 2,
    [(T_, 160, 64, 3, (2, 2), 1, 1, 0)] + [(C_, 64, 64, 3, (1, 1), 1, 0, 1)] * 2,
]
OUTPUT = [(C_, 80, 32, 3, (1, 1), 1, 0, 0), (C_, 32, 3, 1, (1, 1), 0, 0, 0)]


def layer_table():
    """Flat table in blob order: face encoder, audio encoder, decoder, output."""
    flat = [l for blk in FACE for l in blk] + AUDIO + [l for blk in DECODER for l in blk] + OUTPUT
    return flat


def split_blob(blob: np.ndarray):
    """-> list of (weight, bias) fp32 arrays in layer order."""
    out, off = [], 0
    for kind, cin, cout, k, s, p, op, res in layer_table():
        shape = (cout, cin, k, k) if kind == C_ else (cin, cout, k, k)
        n = int(np.prod(shape))
        w = blob[off:off + n].reshape(shape)
        off += n
        b = blob[off:off + cout]
        off += cout
        out.append((w, b))
    assert off == blob.size
    return out


def forward(blob: np.ndarray, mel_chunks: np.ndarray, faces: np.ndarray, logits: bool = False) -> np.ndarray:
    """mel_chunks [B,1,80,16] f32, faces [B,6,96,96] f32 -> [B,3,96,96] f32."""
    import torch
    import torch.nn.functional as F
    params = split_blob(np.asarray(blob, np.float32))
    it = iter(zip(layer_table(), params))

    def block(x, last_relu=True):
        (kind, cin, cout, k, s, p, op, res), (w, b) = next(it)
        wt, bt = torch.from_numpy(np.ascontiguousarray(w)), torch.from_numpy(np.ascontiguousarray(b))
        if kind == C_:
            y = F.conv2d(x, wt, bt, s, p)
        else:
            y = F.conv_transpose2d(x, wt, bt, s, p, op)
        if res:
            y = y + x
        return torch.relu(y) if last_relu else y

    with torch.no_grad():
        x = torch.from_numpy(np.ascontiguousarray(faces, np.float32))
        feats = []
        for blk in FACE:
            for _ in blk:
                x = block(x)
            feats.append(x)
        a = torch.from_numpy(np.ascontiguousarray(mel_chunks, np.float32))
        for _ in AUDIO:
            a = block(a)
        x = a
        for blk in DECODER:
            for _ in blk:
                x = block(x)
            x = torch.cat([x, feats.pop()], dim=1)
        x = block(x)                      # out0: conv + BN + ReLU
        y = block(x, last_relu=False)     # out1: 1x1 conv with bias
        return (y if logits else torch.sigmoid(y)).numpy()


def mel_chunk(mel_rows: np.ndarray, row0: int) -> np.ndarray:
    """[80,16] window: chunk[h][w] = mel_rows[row0 + w][h] (Wav2Lip's
    spec[:, start:start+16] on a [80, T] spectrogram)."""
    return mel_rows[row0:row0 + 16].T.copy()


def face_input(target_u8: np.ndarray, ref_u8: np.ndarray) -> np.ndarray:
    """[6,96,96]: target with rows >= 48 zeroed, then reference, /255."""
    t = target_u8.astype(np.float32) / 255.0
    t[48:] = 0.0
    r = ref_u8.astype(np.float32) / 255.0
    return np.concatenate([t, r], axis=2).transpose(2, 0, 1).copy()


def psnr(a: np.ndarray, b: np.ndarray) -> float:
    mse = float(np.mean((np.asarray(a, np.float64) - np.asarray(b, np.float64)) ** 2))
    return float("inf") if mse == 0 else 10.0 * np.log10(1.0 / mse)


def he_weights(seed: int = 0) -> np.ndarray:
    """He-normal weight blob in layer order, zero biases: for TIMING the CPU
    restatement (bench.py's reference arm), where values do not matter; the
    parity tests use the library's BN-calibrated synthetic weights."""
    rng = np.random.default_rng(seed)
    parts = []
    for kind, cin, cout, k, s, p, op, res in layer_table():
        fan_in = cin * k * k / (s[0] * s[1] if kind == T_ else 1)
        parts.append(rng.normal(0.0, np.sqrt(2.0 / fan_in), cin * cout * k * k).astype(np.float32))
        parts.append(np.zeros(cout, np.float32))
    return np.concatenate(parts)
