"""C++ drop-in classes (include/lsg/lipstream_b200.hpp) on the reference's
own known-answer cases (tests/cpp/dropin_test.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CPP = os.path.join(ROOT, "tests", "cpp")


def _build():
    subprocess.run(["make", "-C", CPP], check=True, capture_output=True)
    return os.path.join(CPP, "_build", "dropin_test")


def test_dropin_header_compiles(lsg):
    assert os.path.exists(_build())


@pytest.mark.gpu
def test_dropin_known_answers(tmp_path):
    from paper_2512_18318_b200 import generator
    exe = _build()
    wfile = tmp_path / "weights.f32"
    generator.synthetic_weights(0).astype("<f4").tofile(wfile)  # the LipsyncStage checks' blob
    r = subprocess.run([exe, os.path.join(ROOT, "tests", "golden"), str(wfile)], capture_output=True, text=True,
                       timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all drop-in checks passed" in r.stdout
    assert "INT8-tail stage vs fp16 stage" in r.stdout
