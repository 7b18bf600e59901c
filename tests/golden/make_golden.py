"""Regenerate the committed golden fixtures from the REFERENCE's own code.

Run in the build container (needs oracle/_ref, i.e. /root/reference):

    python tests/golden/make_golden.py

Writes:
  mel_golden.bin   write_mel(compute_mel(pure_tone(440, 1000)))  (media_tests.cpp:172-179);
                   sha256 a098a3b0...9107, the value SURVEY.md §8(c) records
  tone440_1s.s16   the PCM that golden was computed from
  stock10s.s16     render_pattern(SpeechPattern{}, 10000)  (stock pattern, 10 s)
  stock10s.json    its sha256, reference cut list and mel sha256
  streams8.json    8 seeded 60 s streams (random_scenario-style patterns,
                   plus a >10 s burst stream and a near-threshold stream) with
                   the reference cut lists and per-stream mel sha256
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from _oracle import Pattern, Reference  # noqa: E402
from streams import config2_streams  # noqa: E402


def main():
    ref = Reference()
    tone = ref.render_pattern(Pattern(0, [(1000, 0)], tone_hz=440.0), 1000)
    tone.astype("<i2").tofile(os.path.join(HERE, "tone440_1s.s16"))
    ref.write_mel(os.path.join(HERE, "mel_golden.bin"), ref.compute_mel(tone))

    stock = ref.render_pattern(Pattern(), 10000)
    stock.astype("<i2").tofile(os.path.join(HERE, "stock10s.s16"))
    cuts, _, _ = ref.segment(stock)
    mel = ref.compute_mel(stock)
    json.dump({"pcm_sha256": hashlib.sha256(stock.astype("<i2").tobytes()).hexdigest(),
               "cuts": [[c["begin"], c["end"], c["cause"]] for c in cuts],
               "mel_sha256": hashlib.sha256(mel.astype("<f4").tobytes()).hexdigest()},
              open(os.path.join(HERE, "stock10s.json"), "w"), indent=1)

    out = []
    for i, pcm in enumerate(config2_streams(ref.render_pattern)):
        cuts, met, _ = ref.segment(pcm)
        mel = ref.compute_mel(pcm)
        out.append({"stream": i, "n": int(len(pcm)),
                    "pcm_sha256": hashlib.sha256(pcm.astype("<i2").tobytes()).hexdigest(),
                    "cuts": [[c["begin"], c["end"], c["cause"], c["sample_off"], c["sample_len"]] for c in cuts],
                    "metrics": met,
                    "mel_frames": int(mel.shape[0]),
                    "mel_sha256": hashlib.sha256(mel.astype("<f4").tobytes()).hexdigest()})
    json.dump(out, open(os.path.join(HERE, "streams8.json"), "w"), indent=1)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
