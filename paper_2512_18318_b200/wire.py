"""Wire codecs of the hot path's stage messages, and their zero-copy variants
(SURVEY.md §8 f3).

The reference encodes every message little-endian behind a u32 tag
(stage.cpp:34-69 WireWriter, :71-136 WireReader) and copies payloads by
value: `encode_segment` writes each PCM sample (stage.cpp:176-186), and
`AlignedPairMsg` (stage.hpp:81-93) carries only counts because there are no
pixels.  Here the payloads live in HBM, in a device registry
(`api.DeviceRegistry`, lsg_reg_* in include/lsg.h); the *Ref messages carry
the reference header fields plus 48-byte device references
(`lsg_devref_encode` layout) instead of the bytes.

`encode_segment` / `encode_aligned_pair` / `encode_final` (and decoders)
reproduce the reference's byte layout exactly -- tests/test_wire.py checks
them against the reference build -- so the Ref messages extend the
reference protocol rather than replace it.  Errors mirror WireReader:
`WireError("wire: truncated")`, `("wire: expected tag A, got B")`,
`("wire: trailing bytes")` (std::runtime_error there)."""
from __future__ import annotations

import struct
from dataclasses import dataclass, field

import numpy as np

# reference tags (stage.hpp:40-45)
TAG_SEGMENT, TAG_TRANSCRIPT, TAG_TRANSLATION, TAG_SYNTH_AUDIO, TAG_ALIGNED_PAIR, TAG_FINAL = 1, 2, 3, 4, 5, 6
# zero-copy variants: reference tag | 0x100
TAG_SEGMENT_REF, TAG_ALIGNED_PAIR_REF, TAG_FINAL_REF = 0x101, 0x105, 0x106

BUF_AUDIO, BUF_MEL, BUF_FRAMES, BUF_RENDER = 1, 2, 3, 4  # LSG_BUF_*
DEVREF_BYTES = 48


class WireError(RuntimeError):
    """std::runtime_error thrown by the reference's WireReader."""


@dataclass(frozen=True)
class Ref:
    """lsg_devref: a device buffer in a registry of this process."""
    uuid: bytes
    kind: int
    device: int
    generation: int
    offset: int
    bytes: int

    def to_bytes(self) -> bytes:
        return _uuid(self.uuid) + struct.pack("<IIQqq", self.kind & 0xFFFFFFFF, self.device & 0xFFFFFFFF,
                                              self.generation, self.offset, self.bytes)

    @staticmethod
    def from_bytes(b: bytes) -> "Ref":
        if len(b) != DEVREF_BYTES:
            raise WireError("wire: truncated")
        kind, dev, gen, off, n = struct.unpack("<IIQqq", b[16:])
        return Ref(bytes(b[:16]), struct.unpack("<i", struct.pack("<I", kind))[0],
                   struct.unpack("<i", struct.pack("<I", dev))[0], gen, off, n)


def _uuid(u) -> bytes:
    b = bytes(u)
    if len(b) != 16:
        raise ValueError("uuid must be 16 bytes")
    return b


class _Writer:
    def __init__(self, tag: int):
        self.parts = [struct.pack("<I", tag)]

    def u8(self, v):
        self.parts.append(struct.pack("<B", v))

    def u32(self, v):
        self.parts.append(struct.pack("<I", v))

    def i64(self, v):
        self.parts.append(struct.pack("<q", v))

    def f64(self, v):
        self.parts.append(struct.pack("<d", v))

    def uuid(self, u):
        self.parts.append(_uuid(u))

    def samples(self, s):
        a = np.ascontiguousarray(s, dtype="<i2")
        self.u32(len(a))
        self.parts.append(a.tobytes())

    def refs(self, refs):
        self.u32(len(refs))
        for r in refs:
            self.parts.append(r.to_bytes())

    def take(self) -> bytes:
        return b"".join(self.parts)


class _Reader:
    def __init__(self, b: bytes, want: int):
        self.b, self.pos = memoryview(bytes(b)), 0
        tag = self.u32()
        if tag != want:
            raise WireError(f"wire: expected tag {want}, got {tag}")

    def need(self, n):
        if self.pos + n > len(self.b):
            raise WireError("wire: truncated")

    def _take(self, fmt, n):
        self.need(n)
        v = struct.unpack_from(fmt, self.b, self.pos)[0]
        self.pos += n
        return v

    def u8(self):
        return self._take("<B", 1)

    def u32(self):
        return self._take("<I", 4)

    def i64(self):
        return self._take("<q", 8)

    def f64(self):
        return self._take("<d", 8)

    def uuid(self):
        self.need(16)
        u = bytes(self.b[self.pos:self.pos + 16])
        self.pos += 16
        return u

    def samples(self):
        n = self.u32()
        self.need(2 * n)
        a = np.frombuffer(self.b[self.pos:self.pos + 2 * n], dtype="<i2").astype(np.int16)
        self.pos += 2 * n
        return a

    def refs(self):
        n = self.u32()
        out = []
        for _ in range(n):
            self.need(DEVREF_BYTES)
            out.append(Ref.from_bytes(bytes(self.b[self.pos:self.pos + DEVREF_BYTES])))
            self.pos += DEVREF_BYTES
        return out

    def done(self):
        if self.pos != len(self.b):
            raise WireError("wire: trailing bytes")


def wire_tag(payload: bytes) -> int:
    """stage.cpp wire_tag: the leading u32."""
    if len(payload) < 4:
        raise WireError("wire: truncated")
    return struct.unpack_from("<I", payload)[0]


# ----------------------------------------------------------- messages
@dataclass
class SegmentMsg:  # stage.hpp:49-58
    uuid: bytes
    birth: int = 0
    begin: int = 0
    end: int = 0
    confidence: float = 1.0
    sample_rate: int = 16000
    samples: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int16))


@dataclass
class SegmentRefMsg:  # SegmentMsg with the PCM as a registry reference (BUF_AUDIO)
    uuid: bytes
    birth: int = 0
    begin: int = 0
    end: int = 0
    confidence: float = 1.0
    sample_rate: int = 16000
    audio: Ref | None = None


@dataclass
class AlignedPairMsg:  # stage.hpp:81-93
    uuid: bytes
    birth: int = 0
    begin: int = 0
    end: int = 0
    source_duration_ms: int = 0
    offset_ms: int = 0
    low_confidence: bool = False
    n_frames: int = 0
    first_frame_ts: int = 0
    last_frame_ts: int = 0
    mel_frames: int = 0


@dataclass
class AlignedPairRefMsg(AlignedPairMsg):  # + mel rows (BUF_MEL) and face crops (BUF_FRAMES) on the device
    refs: list = field(default_factory=list)

    def ref(self, kind: int) -> Ref | None:
        return next((r for r in self.refs if r.kind == kind), None)


@dataclass
class FinalMsg:  # stage.hpp:95-103
    uuid: bytes
    birth: int = 0
    begin: int = 0
    end: int = 0
    source_duration_ms: int = 0
    frames_rendered: int = 0
    offset_ms: int = 0


@dataclass
class FinalRefMsg(FinalMsg):  # + rendered frames (BUF_RENDER) on the device
    refs: list = field(default_factory=list)


# ----------------------------------------------------------- codecs
def encode_segment(m: SegmentMsg) -> bytes:  # stage.cpp:176-186
    w = _Writer(TAG_SEGMENT)
    w.uuid(m.uuid), w.i64(m.birth), w.i64(m.begin), w.i64(m.end), w.f64(m.confidence)
    w.u32(m.sample_rate)
    w.samples(m.samples)
    return w.take()


def decode_segment(b: bytes) -> SegmentMsg:  # stage.cpp:188-201
    r = _Reader(b, TAG_SEGMENT)
    m = SegmentMsg(r.uuid(), r.i64(), r.i64(), r.i64(), r.f64(), r.u32(), r.samples())
    r.done()
    return m


def encode_segment_ref(m: SegmentRefMsg) -> bytes:
    w = _Writer(TAG_SEGMENT_REF)
    w.uuid(m.uuid), w.i64(m.birth), w.i64(m.begin), w.i64(m.end), w.f64(m.confidence)
    w.u32(m.sample_rate)
    w.refs([m.audio] if m.audio is not None else [])
    return w.take()


def decode_segment_ref(b: bytes) -> SegmentRefMsg:
    r = _Reader(b, TAG_SEGMENT_REF)
    m = SegmentRefMsg(r.uuid(), r.i64(), r.i64(), r.i64(), r.f64(), r.u32())
    refs = r.refs()
    r.done()
    m.audio = refs[0] if refs else None
    return m


def _pair_fields(w: _Writer, m: AlignedPairMsg):  # stage.cpp:243-257
    w.uuid(m.uuid), w.i64(m.birth), w.i64(m.begin), w.i64(m.end), w.i64(m.source_duration_ms), w.i64(m.offset_ms)
    w.u8(1 if m.low_confidence else 0)
    w.i64(m.n_frames), w.i64(m.first_frame_ts), w.i64(m.last_frame_ts), w.i64(m.mel_frames)


def _read_pair(r: _Reader, cls):
    return cls(r.uuid(), r.i64(), r.i64(), r.i64(), r.i64(), r.i64(), r.u8() != 0, r.i64(), r.i64(), r.i64(),
               r.i64())


def encode_aligned_pair(m: AlignedPairMsg) -> bytes:
    w = _Writer(TAG_ALIGNED_PAIR)
    _pair_fields(w, m)
    return w.take()


def decode_aligned_pair(b: bytes) -> AlignedPairMsg:  # stage.cpp:259-275
    r = _Reader(b, TAG_ALIGNED_PAIR)
    m = _read_pair(r, AlignedPairMsg)
    r.done()
    return m


def encode_aligned_pair_ref(m: AlignedPairRefMsg) -> bytes:
    w = _Writer(TAG_ALIGNED_PAIR_REF)
    _pair_fields(w, m)
    w.refs(m.refs)
    return w.take()


def decode_aligned_pair_ref(b: bytes) -> AlignedPairRefMsg:
    r = _Reader(b, TAG_ALIGNED_PAIR_REF)
    m = _read_pair(r, AlignedPairRefMsg)
    m.refs = r.refs()
    r.done()
    return m


def _final_fields(w: _Writer, m: FinalMsg):  # stage.cpp:277-287
    w.uuid(m.uuid), w.i64(m.birth), w.i64(m.begin), w.i64(m.end), w.i64(m.source_duration_ms)
    w.i64(m.frames_rendered), w.i64(m.offset_ms)


def encode_final(m: FinalMsg) -> bytes:
    w = _Writer(TAG_FINAL)
    _final_fields(w, m)
    return w.take()


def decode_final(b: bytes) -> FinalMsg:  # stage.cpp:289-301
    r = _Reader(b, TAG_FINAL)
    m = FinalMsg(r.uuid(), r.i64(), r.i64(), r.i64(), r.i64(), r.i64(), r.i64())
    r.done()
    return m


def encode_final_ref(m: FinalRefMsg) -> bytes:
    w = _Writer(TAG_FINAL_REF)
    _final_fields(w, m)
    w.refs(m.refs)
    return w.take()


def decode_final_ref(b: bytes) -> FinalRefMsg:
    r = _Reader(b, TAG_FINAL_REF)
    m = FinalRefMsg(r.uuid(), r.i64(), r.i64(), r.i64(), r.i64(), r.i64(), r.i64())
    m.refs = r.refs()
    r.done()
    return m
