"""The library's paced driver (lsg_paced, csrc/paced.cu; BASELINE.json
config 5 paced): audio and video released in real time over 40 ms ticks,
deadline-batched generator launches, completion stamps from
cudaLaunchHostFunc.  Checks: the segments are the reference Segmenter's
(chunked pushes, chunk invariance); every segment's gathered frames and
chunk rows equal lsg_pipe's for the same streams; the rendered frames match
lsg_pipe's (PSNR >= 40 dB: different batch compositions); the timeline is
causal (cut decided after the segment end, rendered after the decision)."""
import numpy as np
import pytest

from streams import random_scenario_pattern

pytestmark = pytest.mark.gpu


def test_paced_driver_matches_pipeline(reference):
    torch = pytest.importorskip("torch")
    from paper_2512_18318_b200 import api, generator
    from paper_2512_18318_b200.paced import LibPacedRunner
    from paper_2512_18318_b200.pipeline import Pipeline, PipelineConfig
    S, secs, fps = 6, 8, 25.0
    pcm = [reference.render_pattern(random_scenario_pattern(40 + i), secs * 1000) for i in range(S)]
    refs = np.stack([generator.synthetic_face(90 + s) for s in range(S)])
    nvid = [int(np.ceil(len(p) / 16000 * fps)) for p in pcm]
    video = [np.stack([generator.jitter_face(refs[s], f, s) for f in range(nvid[s])]) for s in range(S)]
    w = generator.synthetic_weights(0)
    ctx = api.Context(0)
    eng = generator.LipsyncEngine(w, max_batch=64, ctx=ctx, precision=1)
    # lsg_pipe over the same streams (the non-paced path) as the expectation
    pipe = Pipeline(PipelineConfig(S, secs * 1000, fps, 50, 64, True), eng, ctx=ctx)
    r_pipe, f_pipe, _ = pipe.run(pcm, video, refs)
    pipe.close()
    ms = secs * 16000
    dev = "cuda"
    pcm_dev = torch.from_numpy(np.stack([p[:ms] for p in pcm])).to(dev)
    vid_dev = torch.from_numpy(np.stack(video)).to(dev)
    refs_dev = torch.from_numpy(refs).to(dev)
    runner = LibPacedRunner(eng, S, ms, max(nvid), fps=fps, deadline_ms=20)
    J = len(r_pipe)
    frames = torch.empty((J + 64, 96, 96, 3), dtype=torch.uint8, device=dev)
    res, segs, recs = runner.run(pcm_dev, [ms] * S, vid_dev, nvid, refs_dev, 0.0, frames_out=frames,
                                 frames_cap=J + 64)
    # segments = the reference's cuts, stream by stream
    for s in range(S):
        want, _, _ = reference.segment(pcm[s][:ms])
        got = [(g["begin"], g["end"], g["cause"]) for g in segs if g["stream"] == s]
        assert got == [(c["begin"], c["end"], c["cause"]) for c in want], s
    # frames and chunk rows = lsg_pipe's (render order differs)
    key = lambda r: (r["stream"], r["segment"], r["frame_index"])  # noqa: E731
    assert sorted((key(r), r["mel_row"]) for r in recs) == sorted((key(r), r["mel_row"]) for r in r_pipe)
    pos = {key(r): i for i, r in enumerate(r_pipe)}
    f_paced = frames[:len(recs)].cpu().numpy()
    order = [pos[key(r)] for r in recs]
    mse = float(np.mean((f_paced.astype(np.float64) - f_pipe[order].astype(np.float64)) ** 2)) / 255.0 ** 2
    assert mse == 0 or 10 * np.log10(1 / mse) >= 40.0, mse
    # causality and completeness
    assert all(g["rendered_ms"] >= g["decided_ms"] >= 0 for g in segs)
    assert sum(g["frames"] for g in segs) == res.frames == J
    runner.close()
    eng.close()
