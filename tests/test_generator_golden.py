"""Config-1 goldens (tests/golden/gen_config1.npz, make_gen_golden.py): the
stock 10 s stream's 258 rendered frames, fp32 oracle, batches of 16, from
inputs the reference build produced.

CPU: the oracle and synthetic_weights(0) reproduce the committed goldens on
this machine (the oracle is pinned to its committed output, not only to
itself).  GPU: the whole path (lsg_pipe: segmenter -> mel -> gather ->
generator, fp16, batches of 16) on the same stream returns exactly the
golden frame records and frames within PSNR >= 40 dB (u8, all 258 frames;
f32 frames of the first batch through lsg_gen_forward)."""
import importlib.util
import json
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


@pytest.fixture(scope="module")
def gold():
    d = np.load(os.path.join(GOLD, "gen_config1.npz"))
    return {k: d[k] for k in d.files} | json.load(open(os.path.join(GOLD, "gen_config1.json")))


@pytest.fixture(scope="module")
def gref():
    spec = importlib.util.spec_from_file_location("generator_ref", os.path.join(ROOT, "oracle", "generator_ref.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


@pytest.fixture(scope="module")
def weights(lsg):
    from paper_2512_18318_b200 import generator
    return generator.synthetic_weights(0)


def _batch0(gold, gref):
    from paper_2512_18318_b200 import generator
    recs, rows, face = gold["records"][:16], gold["mel_rows"], gold["ref_face"]
    mel = np.stack([gref.mel_chunk(rows, int(r[4] + r[3]))[None] for r in recs])
    faces = np.stack([gref.face_input(generator.jitter_face(face, int(r[1]), 1), face) for r in recs])
    return mel, faces


def test_golden_stream_and_weights(gold, weights, gref):
    stock = np.fromfile(os.path.join(GOLD, "stock10s.s16"), np.int16)
    import hashlib
    assert hashlib.sha256(stock.tobytes()).hexdigest() == gold["pcm_sha256"]
    assert gold["frames"] == 258 and gold["segments"] == 5
    sums = np.array([(np.sum(w, dtype=np.float64), np.sum(w.astype(np.float64) ** 2))
                     for w, _ in gref.split_blob(weights)])
    assert np.allclose(sums, gold["w_layer_sums"], rtol=1e-5, atol=1e-6)


def test_oracle_reproduces_golden(gold, weights, gref):
    mel, faces = _batch0(gold, gref)
    out = gref.forward(weights, mel, faces)
    assert np.abs(out - gold["out_f32_b0"]).max() < 1e-4
    assert gref.psnr(out, gold["out_f32_b0"]) > 80.0


@pytest.mark.gpu
def test_pipeline_on_config1_matches_golden(gold, weights, gref):
    torch = pytest.importorskip("torch")
    from paper_2512_18318_b200 import api, generator
    from paper_2512_18318_b200.pipeline import Pipeline, PipelineConfig
    pcm = np.fromfile(os.path.join(GOLD, "stock10s.s16"), np.int16)
    face = gold["ref_face"]
    nvid = int(np.ceil(len(pcm) / 16000 * 25.0))
    video = np.stack([generator.jitter_face(face, f, 1) for f in range(nvid)])
    ctx = api.Context(0)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    eng = generator.LipsyncEngine(weights, max_batch=16, ctx=ctx, precision=1)
    pipe = Pipeline(PipelineConfig(1, 10000, 25.0, 50, 16, True), eng, ctx=ctx)
    recs, frames, st = pipe.run([pcm], [video], face[None])
    got = [(r["segment"], r["frame_index"], r["ts_ms"]) for r in recs]
    assert got == [tuple(int(x) for x in r[:3]) for r in gold["records"]]
    p = gref.psnr(frames.astype(np.float64) / 255.0, gold["out_u8"].astype(np.float64) / 255.0)
    worst = min(gref.psnr(frames[i] / 255.0, gold["out_u8"][i] / 255.0) for i in range(len(frames)))
    print(f"config 1 through lsg_pipe: {len(frames)} frames, u8 PSNR {p:.2f} dB (worst frame {worst:.2f})")
    assert p >= 40.0 and worst >= 36.0
    # first batch as f32 through lsg_gen_forward
    mel, faces = _batch0(gold, gref)
    recs16 = gold["records"][:16]
    rows = torch.from_numpy(np.ascontiguousarray(gold["mel_rows"])).cuda()
    chunk = torch.from_numpy((recs16[:, 4] + recs16[:, 3]).astype(np.int32)).cuda()
    tgt = torch.from_numpy(video[recs16[:, 1]]).cuda()
    refs = torch.from_numpy(face[None].copy()).cuda()
    ridx = torch.zeros(16, dtype=torch.int32, device="cuda")
    out = torch.empty(16, 3, 96, 96, dtype=torch.float32, device="cuda")
    eng.forward_device(rows.data_ptr(), chunk.data_ptr(), tgt.data_ptr(), refs.data_ptr(), ridx.data_ptr(),
                       out.data_ptr(), 0, 16)
    torch.cuda.synchronize()
    pf = gref.psnr(out.cpu().numpy(), gold["out_f32_b0"])
    print(f"config 1 batch 0 f32: PSNR {pf:.2f} dB vs the golden fp32 oracle frames")
    assert pf >= 40.0
    pipe.close()
    eng.close()
    ctx.set_stream(None)
