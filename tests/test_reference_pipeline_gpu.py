"""The reference's OWN pipeline on the GPU stages (SURVEY.md §8 b, a10).

integration/Makefile builds the reference's proj/core sources twice: stock
(ref_cpu_pipeline) and with Segmenter / compute_mel / mel_frame_count /
fft_radix2 / mock_lipsync resolved at link time to integration/
lipstream_gpu.cpp, i.e. to liblsg.so (ref_gpu_pipeline).  The same driver
(integration/pipeline_driver.cpp) runs run_pipeline_input (runner.cpp:
239-351) over the paper scenario and four random scenarios at 3-30 s and the
reference's known answers; the GPU build's dump must equal the stock build's
line for line (segments, uuids, segmenter metrics, orchestrator stats, every
event), the orchestrator's pair must carry mel_frames 140 / 40
(pipeline_tests.cpp:417-418), and the GPU mel must match the reference's CPU
mel (linked into the same binary under another name) within 1e-4."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "integration", "_build")
CPU_BIN = os.path.join(BUILD, "ref_cpu_pipeline")
GPU_BIN = os.path.join(BUILD, "ref_gpu_pipeline")


def _run(path, env=None):
    r = subprocess.run([path], capture_output=True, text=True, timeout=600, env=env)
    return r.returncode, r.stdout, r.stderr


@pytest.fixture(scope="module")
def cpu_dump():
    if not os.path.exists(CPU_BIN):
        pytest.skip("integration/_build not built (needs /root/reference at build time)")
    rc, out, err = _run(CPU_BIN)
    assert rc == 0, err
    return out


def test_stock_reference_pipeline_known_answers(cpu_dump):
    lines = cpu_dump.splitlines()
    assert "stock8s begins 0 2300 4300 6300" in lines
    assert "mel [0,2300) frames=140 mels=80" in lines and "mel [2300,3000) frames=40 mels=80" in lines
    assert "fft16 ok bad12_throws=1" in lines
    assert sum(1 for l in lines if l.startswith("run ")) == 17


@pytest.mark.gpu
def test_reference_pipeline_on_gpu_stages_matches_stock(cpu_dump, tmp_path):
    if not os.path.exists(GPU_BIN):
        pytest.skip("integration/_build/ref_gpu_pipeline not built")
    from paper_2512_18318_b200 import generator
    w = tmp_path / "weights.f32"
    generator.synthetic_weights(0).astype(np.float32).tofile(w)
    env = dict(os.environ, LSG_GEN_WEIGHTS=str(w))
    rc, out, err = _run(GPU_BIN, env)
    assert rc == 0, err
    assert err.count("vs reference cpu") == 2 and "FAIL" not in err, err
    want, got = cpu_dump.splitlines(), out.splitlines()
    diff = [(a, b) for a, b in zip(want, got) if a != b]
    assert len(want) == len(got) and not diff, diff[:5]
    # liblsg.so is what served those symbols
    maps = subprocess.run(["ldd", GPU_BIN], capture_output=True, text=True).stdout
    assert "liblsg.so" in maps
