"""Generator: layer-table agreement (CPU) and bf16 tcgen05 forward vs the
fp32 oracle (GPU).

Tolerance (BASELINE.json north_star: PSNR >= 40 dB vs the fp32 oracle for
the 16-bit path): fp16 (the library's default 16-bit format, same tcgen05
rate as bf16) PSNR >= 40 dB on the [0,1] frames and on the u8 frames, plus
max-abs error <= 0.35 on the pre-sigmoid logits (calibrated ~N(0,1)).  bf16
cannot reach 40 dB on this random-weight network -- the CPU model that only
rounds weights and stored activations to bf16 lands at ~30.6 dB (weights
alone 34.5, activations alone 32.6; tools/precision_sweep.py) -- so bf16 is
gated as "no more than 1.5 dB below that rounding model".
"""
import importlib.util
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _oracle():
    spec = importlib.util.spec_from_file_location("generator_ref", os.path.join(ROOT, "oracle", "generator_ref.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


@pytest.fixture(scope="session")
def gref():
    return _oracle()


@pytest.fixture(scope="session")
def weights(lsg):
    from paper_2512_18318_b200 import generator
    return generator.synthetic_weights(seed=0)


def test_layer_table_matches_wav2lip(lsg, gref):
    from paper_2512_18318_b200 import generator
    lib_layers = generator.layers()
    ref = gref.layer_table()
    assert len(lib_layers) == len(ref) == 51
    for L, (kind, cin, cout, k, s, p, op, res) in zip(lib_layers, ref):
        assert (L.kind, L.cin, L.cout, L.kh, L.kw, L.sh, L.sw, L.ph, L.pw, L.oph, L.opw, L.res) == \
            (kind, cin, cout, k, k, s[0], s[1], p, p, op, op, res)
    n = sum(L.n_params for L in lib_layers)
    assert n == generator.param_count() and abs(n - 36.28e6) < 0.05e6  # 36.28 M


def test_flops_per_frame(lsg):
    """7.934 GFLOP/frame; convT counted as Hin*Win*Cin*Cout*9."""
    from paper_2512_18318_b200 import generator
    assert abs(generator.flops_per_frame() - 7.934e9) / 7.934e9 < 0.002


def test_synthetic_weights_calibrated(weights, gref, lsg):
    from paper_2512_18318_b200 import generator
    rng = np.random.default_rng(9)
    mel = rng.normal(-5.0, 2.5, (2, 1, 80, 16)).astype(np.float32)
    faces = np.stack([generator.face_input(generator.synthetic_face(900 + i), generator.synthetic_face(950 + i))
                      for i in range(2)])
    lg = gref.forward(weights, mel, faces, logits=True)
    assert np.isfinite(lg).all()
    assert 0.2 < lg.std() < 5.0, lg.std()   # sigmoid not saturated
    w2 = generator.synthetic_weights(seed=0)
    assert np.array_equal(weights, w2)


def _inputs(B, seed):
    from paper_2512_18318_b200 import generator
    rng = np.random.default_rng(seed)
    R = 3
    refs = np.stack([generator.synthetic_face(seed * 10 + r) for r in range(R)])
    ref_index = rng.integers(0, R, B).astype(np.int32)
    target = np.stack([generator.jitter_face(refs[ref_index[b]], b, seed) for b in range(B)])
    rows = rng.normal(-5.0, 2.5, (B + 40, 80)).astype(np.float32)
    chunk_row = rng.integers(0, B + 40 - 16 + 1, B).astype(np.int32)
    return rows, chunk_row, target, refs, ref_index


def bf16_rounding_model(gref, blob, mel, faces, dtype_name="bfloat16"):
    """The fp32 oracle with weights and every stored activation rounded to
    the 16-bit format: what a correct 16-bit kernel must reproduce up to
    accumulation order."""
    import torch
    import torch.nn.functional as F
    dt = getattr(torch, dtype_name)
    q = lambda t: t.to(dt).float()  # noqa: E731
    it = iter(zip(gref.layer_table(), gref.split_blob(blob)))

    def block(x, last=True):
        (kind, cin, cout, k, s, p, op, res), (w, b) = next(it)
        w = q(torch.from_numpy(np.ascontiguousarray(w)))
        b = torch.from_numpy(np.ascontiguousarray(b))
        y = F.conv2d(x, w, b, s, p) if kind == 0 else F.conv_transpose2d(x, w, b, s, p, op)
        if res:
            y = y + x
        return q(torch.relu(y)) if last else y
    with torch.no_grad():
        x = q(torch.from_numpy(faces))
        feats = []
        for blk in gref.FACE:
            for _ in blk:
                x = block(x)
            feats.append(x)
        a = q(torch.from_numpy(mel))
        for _ in gref.AUDIO:
            a = block(a)
        x = a
        for blk in gref.DECODER:
            for _ in blk:
                x = block(x)
            x = torch.cat([x, feats.pop()], 1)
        x = block(x)
        return torch.sigmoid(block(x, last=False)).numpy()


@pytest.mark.gpu
@pytest.mark.parametrize("B", [16, 5, 1])
def test_forward_matches_fp32_oracle(weights, gref, B):
    """fp16 (LSG_PREC_FP16): PSNR >= 40 dB vs the fp32 oracle."""
    _run_forward_check(weights, gref, B, precision=1)


@pytest.mark.gpu
def test_forward_bf16_tracks_bf16_rounding_model(weights, gref):
    """bf16 (LSG_PREC_BF16): this random-weight network amplifies bf16's 8-bit
    mantissa rounding to ~30 dB vs fp32 (a property of the format: the CPU
    bf16 rounding model lands at the same PSNR); the bound is that the GPU is
    no more than 1.5 dB below that model."""
    _run_forward_check(weights, gref, 16, precision=0)


def _run_forward_check(weights, gref, B, precision):
    torch = pytest.importorskip("torch")
    from paper_2512_18318_b200 import generator
    from paper_2512_18318_b200.api import Context
    ctx = Context(0)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    eng = generator.LipsyncEngine(weights, max_batch=16, ctx=ctx, precision=precision)
    rows, chunk_row, target, refs, ref_index = _inputs(B, 100 + B)
    d = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in
         dict(rows=rows, chunk_row=chunk_row, target=target, refs=refs, ref_index=ref_index).items()}
    out = torch.empty(B, 3, 96, 96, dtype=torch.float32, device="cuda")
    lg = torch.empty(B, 3, 96, 96, dtype=torch.float32, device="cuda")
    u8 = torch.empty(B, 96, 96, 3, dtype=torch.uint8, device="cuda")
    args = [d["rows"].data_ptr(), d["chunk_row"].data_ptr(), d["target"].data_ptr(), d["refs"].data_ptr(),
            d["ref_index"].data_ptr()]
    eng.forward_device(*args, out.data_ptr(), 0, B)
    eng.forward_device(*args, lg.data_ptr(), 2, B)
    eng.forward_device(*args, u8.data_ptr(), 1, B)
    torch.cuda.synchronize()
    mel = np.stack([gref.mel_chunk(rows, int(r))[None] for r in chunk_row])
    faces = np.stack([gref.face_input(target[b], refs[ref_index[b]]) for b in range(B)])
    want = gref.forward(weights, mel, faces)
    want_lg = gref.forward(weights, mel, faces, logits=True)
    got = out.cpu().numpy()
    p = gref.psnr(got, want)
    if precision == 1:
        assert p >= 40.0, f"fp16 PSNR {p:.1f} dB"
        err = np.abs(lg.cpu().numpy() - want_lg).max()
        assert err <= 0.35, f"logit max-abs {err:.4f}"
        pu8 = gref.psnr(u8.cpu().numpy().astype(np.float64) / 255.0, want.transpose(0, 2, 3, 1))
        assert pu8 >= 40.0, f"u8 frames PSNR {pu8:.1f} dB"
    else:
        model = bf16_rounding_model(gref, weights, mel, faces)
        pm = gref.psnr(model, want)
        print(f"bf16 B={B}: GPU {p:.2f} dB vs fp32, CPU bf16 rounding model {pm:.2f} dB")
        assert p >= pm - 1.5, f"bf16 PSNR {p:.1f} dB vs rounding model {pm:.1f} dB"
    # u8 output is round(255 * sigmoid) of the same forward
    assert np.abs(u8.cpu().numpy().astype(int) - np.round(got.transpose(0, 2, 3, 1) * 255).astype(int)).max() <= 1
    eng.close()
    ctx.set_stream(None)


@pytest.mark.gpu
@pytest.mark.parametrize("precision", [0, 1])
def test_every_layer_in_isolation(weights, gref, precision):
    """Each conv layer's GPU output vs fp32 conv of the GPU's own 16-bit input
    with the same (rounded) weights: error within output rounding (1.5% of
    the layer's max), i.e. the tcgen05 kernel is exact up to accumulation
    order for every layer shape, stride, phase and epilogue."""
    torch = pytest.importorskip("torch")
    import ctypes as C
    import torch.nn.functional as F
    from paper_2512_18318_b200 import generator
    from paper_2512_18318_b200.api import Context
    ctx = Context(0)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    B = 3
    eng = generator.LipsyncEngine(weights, max_batch=B, ctx=ctx, precision=precision)
    rows, chunk_row, target, refs, ref_index = _inputs(B, 77)
    d = [torch.from_numpy(np.ascontiguousarray(v)).cuda() for v in (rows, chunk_row, target, refs, ref_index)]
    buf = torch.empty(B * 96 * 96 * 1024, dtype=torch.float32, device="cuda")
    shape = (C.c_int32 * 4)()
    fn = eng.lib.dll.lsgdbg_run_until
    dt = torch.float16 if precision else torch.bfloat16
    params = gref.split_blob(weights)
    Ls = generator.layers()

    def dump(layer, which):
        rc = fn(eng.h, *[C.c_void_p(t.data_ptr()) for t in d], B, layer, which, C.c_void_p(buf.data_ptr()), shape)
        assert rc == 0
        torch.cuda.synchronize()
        n = shape[0] * shape[1] * shape[2] * shape[3]
        return buf[:n].reshape(*shape).permute(0, 3, 1, 2).cpu()
    for i in range(len(Ls) - 2):  # out0+out1 are fused; covered by the end-to-end tests
        L = Ls[i]
        x, y = dump(i, 0)[:, :L.cin], dump(i, 1)
        w = torch.from_numpy(np.ascontiguousarray(params[i][0])).to(dt).float()
        b = torch.from_numpy(np.ascontiguousarray(params[i][1]))
        ref = F.conv2d(x, w, b, (L.sh, L.sw), (L.ph, L.pw)) if L.kind == 0 else \
            F.conv_transpose2d(x, w, b, (L.sh, L.sw), (L.ph, L.pw), (L.oph, L.opw))
        ref = torch.relu(ref + x if L.res else ref)
        rel = (y - ref).abs().max().item() / (ref.abs().max().item() + 1e-6)
        assert rel < 0.015, f"layer {i}: rel err {rel:.4f}"
    eng.close()
    ctx.set_stream(None)
