"""CPU-only checks of the product library: it loads, exports every entry
point include/lsg.h declares, and its host-only functions (config checks,
frame counts, workload synthesis) behave like the reference."""
import ctypes as C

import numpy as np
import pytest

from _oracle import Pattern, random_pattern


def test_exports_every_declared_symbol(lsg):
    from paper_2512_18318_b200._lib import _SIGS, header_symbols
    declared = header_symbols()
    assert len(declared) >= 35
    missing = [s for s in declared if not hasattr(lsg.dll, s)]
    assert not missing, f"liblsg.so lacks {missing}"
    assert set(declared) == set(_SIGS), "ctypes table out of sync with include/lsg.h"
    assert lsg.lsg_abi_version() == 1


def test_no_gpu_is_a_loud_failure(lsg):
    n = C.c_int32(-1)
    assert lsg.lsg_device_count(C.byref(n)) == 0
    if n.value == 0:
        h = C.c_void_p()
        rc = lsg.lsg_ctx_create(0, C.byref(h))
        assert rc != 0 and h.value is None


def test_mel_frame_count_host(lsg):
    from paper_2512_18318_b200 import api
    for n, want in ((0, 0), (1023, 0), (1024, 1), (1279, 1), (1280, 2), (160000, 622)):
        assert api.mel_frame_count(n) == want
    with pytest.raises(api.InvalidArgument):
        api.mel_frame_count(100, api.MelConfig(fft_size=1000))


def test_synth_matches_reference_render_pattern(lsg, reference):
    from paper_2512_18318_b200 import api
    state = [31]
    for i in range(20):
        p = random_pattern(state)
        p.tone_hz = 150.0 + 13 * i
        p.amplitude = 0.1 + 0.04 * i
        for total in (1000, 7777, 60000):
            want = reference.render_pattern(p, total)
            got = api.synth_pattern(p.lead_silence_ms, p.bursts, p.tone_hz, p.amplitude, total)
            assert np.array_equal(got, want)
    assert np.array_equal(api.synth_pattern(600, [(1400, 600)], 220.0, 0.3, 8000),
                          reference.render_pattern(Pattern(), 8000))


def test_lipsync_validate_contract(lsg):
    # mock_lipsync (visual_mocks.cpp:40-51): >=2 frames, |span diff| <= 150 ms
    assert lsg.lsg_lipsync_validate(2000, 2020, 61) == 0
    assert lsg.lsg_lipsync_validate(2000, 2020, 1) == 1
    assert lsg.lsg_lipsync_validate(2000, 2400, 61) == 1
    assert lsg.lsg_lipsync_validate(2000, 2150, 2) == 0
