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
def test_dropin_known_answers():
    exe = _build()
    r = subprocess.run([exe, os.path.join(ROOT, "tests", "golden")], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all drop-in checks passed" in r.stdout
