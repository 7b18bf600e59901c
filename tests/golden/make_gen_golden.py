"""Config-1 generator goldens: one stream, 10 s of
the stock synthetic speech + 25 fps 96x96 face crops, generator batch 16,
fp32 -- the CPU oracle workload -- written by the fp32 oracle
(oracle/generator_ref.py) from inputs that the REFERENCE's own code produced
(render_pattern, Segmenter, compute_mel from oracle/_ref).

    python tests/golden/make_gen_golden.py          (build container; ~3 min CPU)

Writes gen_config1.npz:
  pcm_sha256            the stream (= stock10s.s16)
  records [J, 5] i64    (segment, frame index, ts_ms, chunk row k, segment row0) per rendered
                        frame: FrameRing window [begin-50, end+50] (frame_ring.cpp:36-55,
                        orchestrator.cpp:90-91), chunk rule a8 k = clamp(floor((ts-begin)/16),
                        0, max(0, F-16)); J = 258
  mel_rows [R, 80] f32  every segment's reference compute_mel, segments back to back, each
                        edge-padded to >= 16 rows (the layout the pipeline builds)
  ref_face [96,96,3] u8 synthetic_face(77); target f = jitter_face(ref, f, 1)
  out_f32_b0 [16,3,96,96] f32   oracle frames of the first generator batch
  out_u8 [J,96,96,3] u8          round(255 x) of every frame, batches of 16
  w_layer_sums [51, 2] f64       sum / sum of squares of each layer's folded weights (pins
                                 synthetic_weights(0) up to fp32 summation order)
  sha256 of out_f32_b0 / out_u8 in gen_config1.json
"""
import hashlib
import importlib.util
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from _oracle import Pattern, Reference  # noqa: E402

FPS = 25.0
SECONDS = 10


def gref():
    spec = importlib.util.spec_from_file_location("generator_ref", os.path.join(ROOT, "oracle", "generator_ref.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def workload(ref):
    """(pcm, records, mel_rows) of config 1 from the reference build."""
    pcm = ref.render_pattern(Pattern(), SECONDS * 1000)
    cuts, _, _ = ref.segment(pcm)
    nvid = int(np.ceil(len(pcm) / 16000 * FPS))
    recs, rows, row0 = [], [], 0
    for j, c in enumerate(cuts):
        audio = pcm[c["sample_off"]:c["sample_off"] + c["sample_len"]]
        mel = ref.compute_mel(audio)
        F = mel.shape[0]
        r = np.zeros((max(F, 16), 80), np.float32)
        r[:F] = mel
        r[F:] = mel[-1] if F else np.float32(np.log(1e-10))
        for f in range(nvid):
            ts = int(round(f * 1000.0 / FPS))
            if c["begin"] - 50 <= ts <= c["end"] + 50:
                k = min(max((ts - c["begin"]) // 16, 0), max(0, F - 16))
                recs.append((j, f, ts, k, row0))
        rows.append(r)
        row0 += r.shape[0]
    return pcm, np.array(recs, np.int64), np.concatenate(rows)


def main():
    import torch
    torch.set_num_threads(os.cpu_count() or 1)
    from paper_2512_18318_b200 import generator
    g = gref()
    ref = Reference()
    pcm, recs, mel_rows = workload(ref)
    face = generator.synthetic_face(77)
    w = generator.synthetic_weights(0)
    sums = np.array([(float(np.sum(wt, dtype=np.float64)), float(np.sum(wt.astype(np.float64) ** 2)))
                     for wt, _ in g.split_blob(w)])
    J = len(recs)
    outs = []
    for b0 in range(0, J, 16):
        rr = recs[b0:b0 + 16]
        mel = np.stack([g.mel_chunk(mel_rows, int(r[4] + r[3]))[None] for r in rr])
        faces = np.stack([g.face_input(generator.jitter_face(face, int(r[1]), 1), face) for r in rr])
        outs.append(g.forward(w, mel, faces))
        print(f"batch {b0 // 16 + 1}/{(J + 15) // 16}", flush=True)
    out = np.concatenate(outs)
    u8 = np.round(np.clip(out.transpose(0, 2, 3, 1), 0, 1) * 255.0).astype(np.uint8)
    np.savez_compressed(os.path.join(HERE, "gen_config1.npz"), records=recs, mel_rows=mel_rows, ref_face=face,
                        out_f32_b0=out[:16].astype(np.float32), out_u8=u8, w_layer_sums=sums)
    meta = {"pcm_sha256": hashlib.sha256(pcm.tobytes()).hexdigest(), "frames": int(J),
            "segments": int(recs[:, 0].max() + 1),
            "out_f32_b0_sha256": hashlib.sha256(out[:16].astype(np.float32).tobytes()).hexdigest(),
            "out_u8_sha256": hashlib.sha256(u8.tobytes()).hexdigest(),
            "generator": "oracle/generator_ref.py fp32, synthetic_weights(0), batches of 16"}
    json.dump(meta, open(os.path.join(HERE, "gen_config1.json"), "w"), indent=1)
    print(meta)


if __name__ == "__main__":
    main()
