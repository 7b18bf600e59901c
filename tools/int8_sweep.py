"""INT8 tails of the synthetic generator (CPU, fp32 oracle =
oracle/generator_ref.py, synthetic_weights(0)): layers t0.. run as u8
activations x s8 weights (per-output-channel weight scales, per-tensor
activation scales, int32 accumulation), layers before t0 as fp16, out1 f32 --
the sweep behind LSG_PREC_INT8_TAIL.  Activation ranges come from the fp32
oracle on a separate 16-frame calibration batch (the engine calibrates on its
own fp16 forward, tests/test_generator_int8.py).

    python tools/int8_sweep.py            (~2 min on 8 cores)
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


def inputs(B, seed):
    rng = np.random.default_rng(seed)
    refs = [generator.synthetic_face(seed * 100 + i) for i in range(B)]
    faces = np.stack([gref.face_input(generator.jitter_face(refs[i], i, 3), refs[i]) for i in range(B)])
    rows = rng.normal(-5, 2.5, (B + 40, 80)).astype(np.float32)
    mel = np.stack([gref.mel_chunk(rows, i)[None] for i in range(B)])
    return mel, faces


def main():
    torch.set_num_threads(os.cpu_count() or 1)
    w = generator.synthetic_weights(0)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from test_generator_int8 import int8_tail_rounding_model, oracle_absmax
    absmax = oracle_absmax(gref, w, *inputs(16, 9))
    mel, faces = inputs(8, 5)
    ref = gref.forward(w, mel, faces)
    fl = []
    for L, (hi, wi, ho, wo) in zip(generator.layers(), generator.layer_shapes()):
        fl.append(2 * (ho * wo if L.kind == 0 else hi * wi) * L.cin * L.cout * L.kh * L.kw)
    fl = np.array(fl, float)
    print("int8 tails: first int8 layer, FLOP share, PSNR (headroom 1.0 / 1.1)")
    for t0 in (31, 34, 37, 40, 43, 46):
        p = [gref.psnr(int8_tail_rounding_model(gref, w, mel, faces, absmax, t0, hr), ref) for hr in (1.0, 1.1)]
        print(f"{t0:5d}  {fl[t0:50].sum() / fl.sum():.3f}  {p[0]:6.2f} dB  {p[1]:6.2f} dB")


if __name__ == "__main__":
    main()
