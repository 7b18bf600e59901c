"""Face-crop preparation: mock_face_detect, the
detect + KalmanBoxFilter loop of orchestrator.cpp:115-129
(media_tests.cpp:225-275 cases), and the bilinear 96x96 crop.

CPU: the C restatement bit-identical to the reference build.  GPU: the
library (lsg_face_*) bit-identical to the restatement; the crop (our
semantics -- the reference has no pixels) equal to or_crop96."""
import ctypes as C

import numpy as np
import pytest

from _oracle import ORACLE_SO, REF_SO  # noqa: F401


def _so(path):
    return C.CDLL(path)


def _det(lib, fn, i, seed):
    b = np.zeros(4)
    getattr(lib, fn)(C.c_int64(i), C.c_uint64(seed), b.ctypes.data_as(C.c_void_p))
    return b


def _track(lib, fn, ts, fi, has, faces, seed, pn=1e-2, mn=25.0, iv=1e6):
    n = len(ts)
    out, vel = np.zeros(4 * n), np.zeros(2 * n)
    a = lambda x, t: np.ascontiguousarray(x, t)  # noqa: E731
    ts_, fi_, ha_, fa_ = a(ts, np.int64), a(fi, np.int64), a(has, np.int32), a(faces, np.float64)
    f = getattr(lib, fn)
    f.restype = C.c_int
    rc = f(ts_.ctypes.data_as(C.c_void_p), fi_.ctypes.data_as(C.c_void_p), ha_.ctypes.data_as(C.c_void_p),
           fa_.ctypes.data_as(C.c_void_p), C.c_int64(n), C.c_uint64(seed), C.c_double(pn), C.c_double(mn),
           C.c_double(iv), out.ctypes.data_as(C.c_void_p), vel.ctypes.data_as(C.c_void_p))
    return rc, out.reshape(n, 4), vel.reshape(n, 2)


def _cases(reference):
    """(ts, frame_index, has_face, faces, seed): the reference's jittered
    static face (media_tests.cpp:58-68, 225-247), detector-only frames,
    mixed boxes on a drifting face with irregular frame times."""
    lib = _so(REF_SO)
    n = 240
    ts = [int(np.floor(i * 1000 / 30 + 0.5)) for i in range(n)]
    jit = np.stack([_det(lib, "ref_mock_face_detect", i, 31337) for i in range(n)])
    rng = np.random.default_rng(5)
    ts2 = np.cumsum(rng.integers(20, 60, 300))
    drift = np.stack([100 + 0.9 * ts2 / 1000 * 30 + rng.normal(0, 2, 300), 50 + rng.normal(0, 2, 300),
                      40 + rng.normal(0, 1, 300), 44 + rng.normal(0, 1, 300)], 1)
    return [(ts, list(range(n)), [1] * n, jit, 0),
            (ts, list(range(500, 500 + n)), [0] * n, np.zeros((n, 4)), 42),
            (ts2, np.arange(300) + 1000, rng.integers(0, 2, 300), drift, 77),
            ([0], [3], [0], np.zeros((1, 4)), 9)]


def test_restated_matches_reference(reference, restated):
    ref, orc = _so(REF_SO), _so(ORACLE_SO)
    for i in range(60):
        for seed in (0, 42, 31337, 2 ** 63 + 5):
            assert (_det(ref, "ref_mock_face_detect", i, seed) == _det(orc, "or_mock_face_detect", i, seed)).all()
    for ts, fi, has, faces, seed in _cases(reference):
        r = _track(ref, "ref_track_faces", ts, fi, has, faces, seed)
        o = _track(orc, "or_track_faces", ts, fi, has, faces, seed)
        assert r[0] == o[0] == 0
        np.testing.assert_array_equal(r[1], o[1])
        np.testing.assert_array_equal(r[2], o[2])
    # non-finite measurement: the reference throws, the restatement reports it
    bad = np.array([[10.0, 10, 10, 10], [np.nan, 0, 0, 0]])
    assert _track(ref, "ref_track_faces", [0, 33], [0, 1], [1, 1], bad, 0)[0] == -1
    assert _track(orc, "or_track_faces", [0, 33], [0, 1], [1, 1], bad, 0)[0] == -1


def test_smoothing_halves_jitter(reference, restated):
    """media_tests.cpp:225-247 on the restatement."""
    ts, fi, has, faces, seed = _cases(reference)[0]
    _, box, _ = _track(_so(ORACLE_SO), "or_track_faces", ts, fi, has, faces, seed)
    raw, sm = faces[40:, 0], box[40:, 0]
    assert raw.var() > 0 and sm.var() < 0.5 * raw.var()


@pytest.mark.gpu
def test_gpu_track_bit_exact(reference, restated):
    from paper_2512_18318_b200 import api
    orc = _so(ORACLE_SO)
    cases = _cases(reference)
    for i in (0, 7, 123):
        for seed in (0, 42):
            assert api.mock_face_detect(i, seed) == tuple(_det(orc, "or_mock_face_detect", i, seed))
    segs = []
    for ts, fi, has, faces, seed in cases:
        fa = np.where(np.asarray(has)[:, None] > 0, faces, np.nan)
        segs.append((ts, fi, fa))
    # one seed per call: group by seed
    for k, (ts, fi, has, faces, seed) in enumerate(cases):
        got = api.track_faces([segs[k]], seed=seed)[0]
        _, box, vel = _track(orc, "or_track_faces", ts, fi, has, faces, seed)
        np.testing.assert_array_equal(got[0], box)
        np.testing.assert_array_equal(got[1], vel)
    # many segments in one call (same seed)
    many = api.track_faces([segs[2]] * 50 + [segs[3]] * 10, seed=77)
    _, box, _ = _track(orc, "or_track_faces", *cases[2][:4], 77)
    for b, _ in many[:50]:
        np.testing.assert_array_equal(b, box)
    with pytest.raises(RuntimeError):
        api.track_faces([([0, 33], [0, 1], np.array([[10.0, 10, 10, 10], [np.inf, 0, 0, 0]]))])
    from paper_2512_18318_b200._lib import InvalidArgument
    with pytest.raises(InvalidArgument):
        api.track_faces([segs[3]], cfg=api.KalmanConfig(process_noise=0.0))


@pytest.mark.gpu
def test_gpu_crop_matches_restated():
    from paper_2512_18318_b200 import api
    orc = _so(ORACLE_SO)
    rng = np.random.default_rng(3)
    H, W = 448, 640
    frames = rng.integers(0, 256, (3, H, W, 3), dtype=np.uint8)
    boxes = np.array([[320, 240, 160, 200], [317.25, 243.5, 151.0, 203.7], [20, 15, 160, 200],
                      [630, 440, 96, 96], [100.5, 100.5, 1.0, 1.0]], np.float64)
    frame_of = np.array([0, 1, 2, 0, 1])
    got = api.crop96(frames, frame_of, boxes)
    for k in range(len(boxes)):
        want = np.zeros((96, 96, 3), np.uint8)
        orc.or_crop96(np.ascontiguousarray(frames[frame_of[k]]).ctypes.data_as(C.c_void_p), C.c_int(H), C.c_int(W),
                      np.ascontiguousarray(boxes[k]).ctypes.data_as(C.c_void_p), want.ctypes.data_as(C.c_void_p))
        np.testing.assert_array_equal(got[k], want)
    # an axis-aligned box covering exactly 96x96 pixels is the identity crop
    ident = api.crop96(frames, [0], [[100 + 48, 50 + 48, 96, 96]])[0]
    np.testing.assert_array_equal(ident, frames[0, 50:146, 100:196])
