"""Zero-copy stage hand-off, host side: the wire codecs of
the path's stage messages.

CPU: our encoders reproduce the reference's bytes exactly (stage.cpp:176-301,
built from the reference sources into oracle/_ref) for seeded messages, the
reference decodes our bytes and we decode its bytes, malformed payloads fail
the same way (WireReader: truncated / wrong tag / trailing bytes), the *Ref
variants round-trip, and the 48-byte device reference matches the library's
lsg_devref_encode/decode."""
import ctypes as C

import numpy as np
import pytest

from _oracle import REF_SO  # noqa: F401
from paper_2512_18318_b200 import wire


def _ref():
    lib = C.CDLL(REF_SO)
    for f in ("ref_encode_segment", "ref_decode_segment", "ref_encode_aligned_pair", "ref_decode_aligned_pair",
              "ref_encode_final", "ref_wire_tag"):
        getattr(lib, f).restype = C.c_int
    return lib


def _uuid(rng):
    return rng.integers(0, 256, 16, dtype=np.uint8).tobytes()


def _i64(rng):
    return int(rng.integers(-2 ** 62, 2 ** 62))


def _buf(n=1 << 16):
    return (C.c_uint8 * n)(), C.c_int64()


def test_codecs_match_reference_bytes(reference):
    lib = _ref()
    rng = np.random.default_rng(2024)
    for k in range(60):
        u = _uuid(rng)
        # SegmentMsg: header + samples (empty, short, with extreme values)
        n = [0, 1, 37, 4000][k % 4]
        s = rng.integers(-32768, 32768, n, dtype=np.int16)
        if n:
            s[0] = -32768
        m = wire.SegmentMsg(u, _i64(rng), _i64(rng), _i64(rng), float(rng.normal()), int(rng.integers(1, 96000)), s)
        out, nb = _buf()
        assert lib.ref_encode_segment(C.c_char_p(u), C.c_int64(m.birth), C.c_int64(m.begin), C.c_int64(m.end),
                                      C.c_double(m.confidence), C.c_int32(m.sample_rate),
                                      s.ctypes.data_as(C.c_void_p), C.c_int64(n), out, C.c_int64(len(out)),
                                      C.byref(nb)) == 0
        mine = wire.encode_segment(m)
        assert mine == bytes(out[:nb.value])
        # the reference decodes our bytes
        f3, conf, rate, got, ns = (C.c_int64 * 3)(), C.c_double(), C.c_int32(), np.zeros(max(n, 1), np.int16), C.c_int64()
        assert lib.ref_decode_segment(C.c_char_p(mine), C.c_int64(len(mine)), f3, C.byref(conf), C.byref(rate),
                                      got.ctypes.data_as(C.c_void_p), C.c_int64(len(got)), C.byref(ns)) == 0
        assert list(f3) == [m.birth, m.begin, m.end] and conf.value == m.confidence and rate.value == m.sample_rate
        np.testing.assert_array_equal(got[:ns.value], s)
        back = wire.decode_segment(bytes(out[:nb.value]))
        assert (back.uuid, back.birth, back.begin, back.end, back.confidence, back.sample_rate) == \
            (u, m.birth, m.begin, m.end, m.confidence, m.sample_rate)
        np.testing.assert_array_equal(back.samples, s)

        # AlignedPairMsg
        f9 = [_i64(rng) for _ in range(9)]
        low = int(k % 3 == 0)
        p = wire.AlignedPairMsg(u, f9[0], f9[1], f9[2], f9[3], f9[4], bool(low), f9[5], f9[6], f9[7], f9[8])
        out, nb = _buf()
        assert lib.ref_encode_aligned_pair(C.c_char_p(u), (C.c_int64 * 9)(*f9), C.c_int32(low), out,
                                           C.c_int64(len(out)), C.byref(nb)) == 0
        mine = wire.encode_aligned_pair(p)
        assert mine == bytes(out[:nb.value])
        ub, g9, gl = (C.c_uint8 * 16)(), (C.c_int64 * 9)(), C.c_int32()
        assert lib.ref_decode_aligned_pair(C.c_char_p(mine), C.c_int64(len(mine)), ub, g9, C.byref(gl)) == 0
        assert bytes(ub) == u and list(g9) == f9 and gl.value == low
        assert wire.decode_aligned_pair(mine) == p

        # FinalMsg
        f6 = [_i64(rng) for _ in range(6)]
        fm = wire.FinalMsg(u, *f6)
        out, nb = _buf()
        assert lib.ref_encode_final(C.c_char_p(u), (C.c_int64 * 6)(*f6), out, C.c_int64(len(out)), C.byref(nb)) == 0
        assert wire.encode_final(fm) == bytes(out[:nb.value])
        assert wire.decode_final(bytes(out[:nb.value])) == fm


def test_malformed_payloads_fail_like_the_reference(reference):
    lib = _ref()
    u = bytes(range(16))
    good = wire.encode_aligned_pair(wire.AlignedPairMsg(u, 1, 2, 3, 4, 5, True, 6, 7, 8, 9))
    ub, g9, gl = (C.c_uint8 * 16)(), (C.c_int64 * 9)(), C.c_int32()
    for bad, msg in ((good[:-1], "truncated"), (good + b"\0", "trailing"), (good[:3], "truncated"),
                     (wire.encode_final(wire.FinalMsg(u)), "expected tag 5, got 6")):
        assert lib.ref_decode_aligned_pair(C.c_char_p(bad), C.c_int64(len(bad)), ub, g9, C.byref(gl)) == -1
        with pytest.raises(wire.WireError, match=msg):
            wire.decode_aligned_pair(bad)
    tag = C.c_uint32()
    assert lib.ref_wire_tag(C.c_char_p(good), C.c_int64(len(good)), C.byref(tag)) == 0
    assert wire.wire_tag(good) == tag.value == wire.TAG_ALIGNED_PAIR
    assert lib.ref_wire_tag(C.c_char_p(b"ab"), C.c_int64(2), C.byref(tag)) == -1
    with pytest.raises(wire.WireError, match="truncated"):
        wire.wire_tag(b"ab")


def test_ref_messages_round_trip():
    rng = np.random.default_rng(7)
    u = _uuid(rng)
    mel = wire.Ref(u, wire.BUF_MEL, 0, 17, 4096, 140 * 80 * 4)
    frames = wire.Ref(u, wire.BUF_FRAMES, 0, 18, -1, 59 * 96 * 96 * 3)
    p = wire.AlignedPairRefMsg(u, 5, 0, 2300, 2300, -20, False, 59, 0, 2320, 140, refs=[mel, frames])
    b = wire.encode_aligned_pair_ref(p)
    # the reference header fields are laid out exactly as encode_aligned_pair's, then the refs
    plain = wire.encode_aligned_pair(wire.AlignedPairMsg(*[getattr(p, f) for f in (
        "uuid", "birth", "begin", "end", "source_duration_ms", "offset_ms", "low_confidence", "n_frames",
        "first_frame_ts", "last_frame_ts", "mel_frames")]))
    assert b[4:len(plain)] == plain[4:] and wire.wire_tag(b) == wire.TAG_ALIGNED_PAIR_REF
    assert len(b) == len(plain) + 4 + 2 * wire.DEVREF_BYTES
    q = wire.decode_aligned_pair_ref(b)
    assert q == p and q.ref(wire.BUF_MEL) == mel and q.ref(wire.BUF_RENDER) is None
    s = wire.SegmentRefMsg(u, 1, 2300, 4300, 0.75, 16000, wire.Ref(u, wire.BUF_AUDIO, 0, 3, -1, 64000))
    assert wire.decode_segment_ref(wire.encode_segment_ref(s)) == s
    f = wire.FinalRefMsg(u, 1, 2, 3, 4, 59, -20, refs=[wire.Ref(u, wire.BUF_RENDER, 0, 9, 0, 59 * 27648)])
    assert wire.decode_final_ref(wire.encode_final_ref(f)) == f
    with pytest.raises(wire.WireError, match="truncated"):
        wire.decode_aligned_pair_ref(b[:-1])
    with pytest.raises(wire.WireError, match="expected tag"):
        wire.decode_aligned_pair(b)


def test_devref_layout_matches_library(lsg):
    from paper_2512_18318_b200 import api
    rng = np.random.default_rng(3)
    for _ in range(20):
        r = wire.Ref(_uuid(rng), int(rng.integers(1, 5)), int(rng.integers(0, 8)), int(rng.integers(0, 2 ** 63)),
                     int(rng.integers(-1, 2 ** 40)), int(rng.integers(0, 2 ** 40)))
        b = api.devref_encode(r)
        assert b == r.to_bytes() and len(b) == wire.DEVREF_BYTES
        assert api.devref_decode(b) == r == wire.Ref.from_bytes(b)
