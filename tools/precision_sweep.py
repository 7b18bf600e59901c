"""Where the 16-bit / fp8 error of the synthetic generator comes from (CPU,
fp32 oracle = oracle/generator_ref.py, synthetic_weights(0), 4 seeded frames):

  1. per-layer relative error growth of the bf16 and fp16 rounding models
     (weights + every stored activation rounded);
  2. bf16 with only the weights / only the activations rounded;
  3. fp8 (e4m3: per-output-channel weight scales, per-tensor activation
     scales, as lsg_gen_create_q packs them) one layer at a time, rest fp16:
     the sensitivity of each layer, and fp8 tails (layers t0.. in fp8) with
     their share of the FLOPs -- the sweep behind LSG_PREC_FP8_TAIL.

    python tools/precision_sweep.py            (~1 min on 8 cores)
"""
import importlib.util
import os
import sys

import numpy as np
import torch
import torch.nn.functional as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2512_18318_b200 import generator  # noqa: E402

spec = importlib.util.spec_from_file_location("g", os.path.join(ROOT, "oracle", "generator_ref.py"))
gref = importlib.util.module_from_spec(spec)
spec.loader.exec_module(gref)

ident = lambda t: t  # noqa: E731
bf = lambda t: t.to(torch.bfloat16).float()  # noqa: E731
fh = lambda t: t.to(torch.float16).float()  # noqa: E731


def wq8(t, kind):
    co = 0 if kind == 0 else 1
    m = t.abs().amax(dim=[d for d in range(4) if d != co], keepdim=True)
    s = torch.where(m > 0, m / 448.0, torch.ones_like(m))
    return (t / s).to(torch.float8_e4m3fn).float() * s


def aq8(t):
    s = t.abs().max() * 1.1 / 448.0
    return (t / s).clamp(-448, 448).to(torch.float8_e4m3fn).float() * s


def run(w, mel, faces, qw, qa, prec=None, taps=None):
    """qw/qa: weight / stored-activation rounding; prec[i] in {8, 16} overrides per layer."""
    table, params = gref.layer_table(), gref.split_blob(w)
    li = [0]

    def block(x, last=True):
        i = li[0]
        li[0] += 1
        (kind, cin, cout, k, s, p, op, res), (wt, b) = table[i], params[i]
        wt, b = torch.from_numpy(np.ascontiguousarray(wt)), torch.from_numpy(np.ascontiguousarray(b))
        if prec is not None:
            x, wt = (aq8(x), wq8(wt, kind)) if prec[i] == 8 else (fh(x), fh(wt))
        else:
            wt = qw(wt)
        y = F.conv2d(x, wt, b, s, p) if kind == 0 else F.conv_transpose2d(x, wt, b, s, p, op)
        if res:
            y = y + x
        out = (torch.relu(y) if prec is not None else qa(torch.relu(y))) if last else y
        if taps is not None:
            taps.append(out)
        return out
    with torch.no_grad():
        x = qa(torch.from_numpy(faces))
        feats = []
        for blk in gref.FACE:
            for _ in blk:
                x = block(x)
            feats.append(x)
        a = qa(torch.from_numpy(mel))
        for _ in gref.AUDIO:
            a = block(a)
        x = a
        for blk in gref.DECODER:
            for _ in blk:
                x = block(x)
            x = torch.cat([x, feats.pop()], 1)
        x = block(x)
        return torch.sigmoid(block(x, last=False)).numpy()


def main():
    torch.set_num_threads(os.cpu_count() or 1)
    w = generator.synthetic_weights(0)
    B = 4
    rng = np.random.default_rng(5)
    refs = [generator.synthetic_face(300 + i) for i in range(B)]
    faces = np.stack([gref.face_input(generator.jitter_face(refs[i], i, 3), refs[i]) for i in range(B)])
    rows = rng.normal(-5, 2.5, (B + 40, 80)).astype(np.float32)
    mel = np.stack([gref.mel_chunk(rows, i)[None] for i in range(B)])
    ref = gref.forward(w, mel, faces)
    t32, tbf, tfh = [], [], []
    run(w, mel, faces, ident, ident, taps=t32)
    pbf = gref.psnr(run(w, mel, faces, bf, bf, taps=tbf), ref)
    pfh = gref.psnr(run(w, mel, faces, fh, fh, taps=tfh), ref)
    print(f"rounding models vs fp32: bf16 {pbf:.2f} dB, fp16 {pfh:.2f} dB")
    print("layer  rel.err bf16  rel.err fp16   (||y_q - y|| / ||y||, stored output of each layer)")
    for i, (a, b, c) in enumerate(zip(t32, tbf, tfh)):
        print(f"{i:5d}  {((b - a).norm() / a.norm()).item():.2e}      {((c - a).norm() / a.norm()).item():.2e}")
    print(f"bf16 weights only: {gref.psnr(run(w, mel, faces, bf, ident), ref):.2f} dB; "
          f"bf16 activations only: {gref.psnr(run(w, mel, faces, ident, bf), ref):.2f} dB")
    fl = []
    for L, (hi, wi, ho, wo) in zip(generator.layers(), generator.layer_shapes()):
        fl.append(2 * (ho * wo if L.kind == 0 else hi * wi) * L.cin * L.cout * L.kh * L.kw)
    fl = np.array(fl, float)
    print("fp8 one layer at a time (rest fp16): layer, PSNR, FLOP share")
    for i in range(50):
        pr = [16] * 51
        pr[i] = 8
        print(f"{i:5d}  {gref.psnr(run(w, mel, faces, None, ident, prec=pr), ref):6.2f} dB  {fl[i] / fl.sum():.3f}")
    print("fp8 tails: first fp8 layer, FLOP share, PSNR")
    for t0 in (43, 46, 47, 48, 49):
        pr = [16] * t0 + [8] * (50 - t0) + [16]
        print(f"{t0:5d}  {fl[t0:50].sum() / fl.sum():.3f}  {gref.psnr(run(w, mel, faces, None, ident, prec=pr), ref):6.2f} dB")


if __name__ == "__main__":
    main()
