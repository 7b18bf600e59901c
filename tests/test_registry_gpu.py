"""Zero-copy stage hand-off on the GPU: the device
registry (lsg_reg_*) carries a segment's PCM, mel rows and face crops from
stage to stage as 48-byte references; the generator renders straight from
the registry's mel buffer, bit-identical to rendering from a private copy."""
import numpy as np
import pytest
import torch

from paper_2512_18318_b200 import api, generator, wire
from paper_2512_18318_b200._lib import LogicError, LsgError

pytestmark = pytest.mark.gpu


def _uuid(i):
    return bytes([i]) * 16


def test_registry_stage_handoff():
    ctx = api.Context(0)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    reg = api.DeviceRegistry(16 << 20, ctx)
    u = _uuid(7)
    pcm = api.synth_pattern(0, [(2300, 0)], 220.0, 0.3, 2300)
    # segmenter -> mel stage: the segment's PCM by reference
    ref_a = reg.put(u, wire.BUF_AUDIO, pcm)
    assert ref_a.bytes == pcm.nbytes and ref_a.offset >= 0 and ref_a.kind == wire.BUF_AUDIO
    assert reg.read(ref_a) == pcm.tobytes()
    seg = wire.decode_segment_ref(wire.encode_segment_ref(wire.SegmentRefMsg(u, 1, 0, 2300, 1.0, 16000, ref_a)))
    pcm_ptr, n = reg.resolve(seg.audio)
    assert n == pcm.nbytes
    # mel stage writes its rows straight into registry space
    F = api.mel_frame_count(len(pcm))
    mel_ptr, ref_m = reg.alloc(u, wire.BUF_MEL, F * 80 * 4)
    api.MelExtractor(ctx=ctx).batch_device(pcm_ptr, [0], [len(pcm)], mel_ptr, [0])
    want = api.compute_mel(api.AudioBuffer(pcm)).data
    got = np.frombuffer(reg.read(ref_m), np.float32).reshape(F, 80)
    np.testing.assert_array_equal(got, want)
    # face crops adopted without a copy (the producer's own device buffer)
    B = 8
    face = generator.synthetic_face(3)
    crops = torch.from_numpy(np.stack([face] * B)).cuda()
    ref_f = reg.put_view(u, wire.BUF_FRAMES, crops.data_ptr(), crops.numel())
    assert ref_f.offset == -1 and reg.resolve(ref_f) == (crops.data_ptr(), crops.numel())
    # the aligned pair crosses the bus as header + references
    msg = wire.AlignedPairRefMsg(u, 1, 0, 2300, 2300, 0, False, B, 0, 280, F, refs=[ref_m, ref_f])
    blob = wire.encode_aligned_pair_ref(msg)
    assert len(blob) < 200
    got_msg = wire.decode_aligned_pair_ref(blob)
    mel_dev, _ = reg.resolve(got_msg.ref(wire.BUF_MEL))
    face_dev, _ = reg.resolve(got_msg.ref(wire.BUF_FRAMES))
    assert mel_dev == mel_ptr and face_dev == crops.data_ptr()
    # lip-sync stage: render from the registry == render from private copies
    eng = generator.LipsyncEngine(generator.synthetic_weights(0), max_batch=B, ctx=ctx)
    chunk = torch.tensor([min(max(k * 35 // 16, 0), F - 16) for k in range(B)], dtype=torch.int32, device="cuda")
    refs = torch.from_numpy(face[None]).cuda()
    ridx = torch.zeros(B, dtype=torch.int32, device="cuda")
    out_reg = torch.empty(B, 96, 96, 3, dtype=torch.uint8, device="cuda")
    eng.forward_device(mel_dev, chunk.data_ptr(), face_dev, refs.data_ptr(), ridx.data_ptr(), out_reg.data_ptr(), 1, B)
    mel_copy = torch.from_numpy(want.copy()).cuda()
    crops_copy = crops.clone()
    out_cpy = torch.empty_like(out_reg)
    eng.forward_device(mel_copy.data_ptr(), chunk.data_ptr(), crops_copy.data_ptr(), refs.data_ptr(), ridx.data_ptr(),
                       out_cpy.data_ptr(), 1, B)
    torch.cuda.synchronize()
    assert torch.equal(out_reg, out_cpy)
    # rendered frames registered for the final stage
    ref_r = reg.put(u, wire.BUF_RENDER, out_reg.data_ptr(), out_reg.numel())
    fin = wire.decode_final_ref(wire.encode_final_ref(wire.FinalRefMsg(u, 1, 0, 2300, 2300, B, 0, refs=[ref_r])))
    assert reg.read(fin.refs[0]) == out_reg.cpu().numpy().tobytes()
    st = reg.stats()
    assert st["entries"] == 4 and st["used"] >= pcm.nbytes + F * 320 + out_reg.numel()
    for r in (ref_a, ref_m, ref_f, ref_r):
        reg.release(r)
    assert reg.stats()["entries"] == 0 and reg.stats()["used"] == 0
    eng.close()
    reg.close()
    ctx.set_stream(None)


def test_registry_errors_and_reuse():
    ctx = api.Context(0)
    reg = api.DeviceRegistry(1 << 20, ctx)
    u = _uuid(1)
    blk = np.arange(600_000 // 4, dtype=np.int32)
    r1 = reg.put(u, wire.BUF_MEL, blk)
    with pytest.raises(LogicError):  # one buffer per (uuid, kind)
        reg.put(u, wire.BUF_MEL, blk)
    with pytest.raises(LsgError, match="exhausted"):  # 2 x 600 KB > 1 MB
        reg.put(_uuid(2), wire.BUF_MEL, blk)
    # refcounting: a retained buffer survives one release
    reg.retain(r1)
    reg.release(r1)
    assert reg.resolve(r1)[1] == blk.nbytes
    reg.release(r1)
    with pytest.raises(LogicError):  # released: the reference is stale
        reg.resolve(r1)
    # the space comes back (stream-ordered) and the same key may be reused
    r2 = reg.put(u, wire.BUF_MEL, blk[::-1].copy())
    assert r2.generation != r1.generation
    with pytest.raises(LogicError):
        reg.resolve(r1)
    np.testing.assert_array_equal(np.frombuffer(reg.read(r2), np.int32), blk[::-1])
    r3 = reg.put(_uuid(2), wire.BUF_AUDIO, np.zeros(1000, np.int16))
    with pytest.raises(LogicError):
        reg.find(_uuid(3), wire.BUF_AUDIO)
    assert reg.find(_uuid(2), wire.BUF_AUDIO) == r3
    with pytest.raises(ValueError):
        reg.put(b"short", wire.BUF_AUDIO, np.zeros(4, np.int16))
    from paper_2512_18318_b200._lib import InvalidArgument
    with pytest.raises(InvalidArgument):
        reg.put(_uuid(4), 9, np.zeros(4, np.int16))
    with pytest.raises(InvalidArgument):  # put_view wants device memory
        reg.put_view(_uuid(4), wire.BUF_AUDIO, blk.ctypes.data, blk.nbytes)
    # many small buffers: the free list coalesces back to one block
    refs = [reg.put(_uuid(10 + i), wire.BUF_AUDIO, np.full(1000 + 37 * i, i, np.int16)) for i in range(40)]
    for r in refs[::2] + refs[1::2]:
        reg.release(r)
    reg.release(r2)
    reg.release(r3)
    big = reg.put(_uuid(99), wire.BUF_FRAMES, np.zeros((1 << 20) - 256, np.uint8))
    assert big.offset == 0
    reg.close()
