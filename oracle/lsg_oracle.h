/*
 * lsg_oracle.h -- CPU restatement of the reference lip-sync hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2512_18318_b200/,
 * include/lsg.h) links, loads or calls this; only tests/, the smoke() check
 * in __graft_entry__.py and the cpu_baseline leg of bench.py use it, and only
 * as the checker.  Parity is pinned: tests/test_oracle.py checks every
 * function here against the reference sources compiled as-is into
 * oracle/_ref (oracle/Makefile) and against tests/golden/.
 *
 * Each function cites the reference file:line it restates
 * (paths relative to /root/reference/proj/core/).
 */
#ifndef LSG_ORACLE_H
#define LSG_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- VAD: include/lipstream/vad.hpp:19-24, src/vad.cpp:26-53 ---------- */
typedef struct {
  int peak_mode;              /* 0 Decay, 1 MaxHold, 2 Absolute (vad.hpp:13-17) */
  double peak_half_life_ms;   /* 10000 */
  double speech_threshold_db; /* -40 */
  int64_t frame_ms;           /* 20 */
} or_vad_cfg;

typedef struct {
  or_vad_cfg cfg;
  double peak;
} or_vad;

void or_vad_init(or_vad* v, const or_vad_cfg* cfg);
/* returns speech flag; writes rms_db */
int or_vad_update(or_vad* v, const int16_t* s, int64_t n, double* rms_db);

/* ---- Segmenter: include/lipstream/segmenter.hpp, src/segmenter.cpp ----- */
typedef struct {
  int mode;                   /* 0 Baseline, 1 Semantic (segmenter.hpp:43-50) */
  or_vad_cfg vad;
  int64_t min_silence_ms, min_segment_ms, max_segment_ms;
  int sample_rate;
} or_seg_cfg;

typedef struct {
  int64_t begin, end;
  double confidence;
  int cause;                  /* 0 Pause, 1 Forced, 2 Eos (segmenter.hpp:11) */
  int64_t sample_off;         /* offset of the segment's first sample in the stream */
  int64_t sample_len;
} or_cut;

typedef struct {
  int64_t frames, speech_frames, cuts_pause, cuts_forced, cuts_eos, scorer_calls;
  double scorer_cost_ms;
} or_seg_metrics;

/* BoundaryScorer (segmenter.hpp:36-41) as a C callback */
typedef void (*or_scorer_fn)(void* user, int64_t pause_start, int64_t silence_run_ms,
                             int64_t segment_span_ms, int* cut, double* confidence,
                             double* cost_ms);

typedef struct {
  or_seg_cfg cfg;
  or_vad vad;
  or_seg_metrics metrics;
  or_scorer_fn scorer;
  void* scorer_user;
  int64_t frame_samples;
  int16_t* stage;   int64_t stage_len, stage_cap;
  int64_t pending_len;          /* samples in the open segment */
  int64_t emitted_samples;      /* samples handed out in earlier segments */
  int64_t base, seg_start, consumed_frames;
  int speech_seen;
  int64_t silence_run;
  int candidate_open, candidate_cut;
  double candidate_confidence;
  int64_t pause_start;
  int finished;
  int started;
} or_seg;

/* 0 ok, 1 invalid_argument, 2 logic_error (the reference's exception types) */
int or_seg_init(or_seg* s, const or_seg_cfg* cfg, or_scorer_fn scorer, void* user);
void or_seg_free(or_seg* s);
int or_seg_push(or_seg* s, const int16_t* pcm, int64_t n, int64_t start_ms, int sample_rate,
                or_cut* out, int64_t cap, int64_t* n_out);
int or_seg_finish(or_seg* s, or_cut* out, int64_t cap, int64_t* n_out);
int64_t or_seg_sizeof(void);
void or_seg_get_metrics(const or_seg* s, or_seg_metrics* m);

/* ---- Mel: include/lipstream/mel.hpp, src/mel.cpp ----------------------- */
typedef struct {
  int sample_rate, fft_size, hop, n_mels;
  double fmin, fmax;
} or_mel_cfg;

void or_mel_default(or_mel_cfg* c);
int64_t or_mel_frame_count(int64_t n_samples, const or_mel_cfg* c);
/* in-place radix-2 on interleaved (re,im) pairs; returns 1 on a bad size */
int or_fft_radix2(double* buf, int64_t n);
/* writes frames*n_mels floats; returns frames (or -1 on bad config) */
int64_t or_compute_mel(const int16_t* pcm, int64_t n, const or_mel_cfg* c, float* out);
/* filterbank W[m][b] (n_mels x (fft/2+1)) exactly as mel.cpp builds it */
int or_mel_filterbank(const or_mel_cfg* c, double* w);

/* ---------------------------------------------------------- A/V alignment
 * Restatement of align.cpp. */
typedef struct {
  int64_t offset_ms;
  double peak_corr;
  int low_confidence;
} or_align_result;
/* energy_envelope_ms (align.cpp:10-32): returns the length (whole ms of the
 * buffer, llround(1000 n / rate)), writes it when cap allows */
int64_t or_energy_envelope(const int16_t* pcm, int64_t n, int rate, double* out, int64_t cap);
/* motion_envelope_ms (align.cpp:34-50): frames sorted by ts */
int or_motion_envelope(const int64_t* ts, const double* motion, int64_t nf, int64_t t0, int64_t span, double* out);
/* align_envelopes (align.cpp:52-116) */
int or_align_envelopes(const double* e, int64_t ne, const double* m, int64_t nm, int64_t max_lag,
                       or_align_result* r);

/* ------------------------------------------------- face track (row f1)
 * Restatement of mock_face_detect (visual_mocks.cpp:10-22) and the
 * detect + KalmanBoxFilter loop (kalman.cpp:58-144, orchestrator.cpp:115-129). */
void or_mock_face_detect(int64_t frame_index, uint64_t seed, double* box4);
int or_track_faces(const int64_t* ts, const int64_t* frame_index, const int* has_face, const double* faces,
                   int64_t n, uint64_t seed, double process_noise, double measurement_noise,
                   double initial_variance, double* out4, double* vel2);
/* bilinear crop of box (cx, cy, w, h) of a [H][W][3] u8 frame into
 * [96][96][3]: source x = cx - w/2 + (u + 0.5) w / 96 - 0.5 (same for y),
 * clamp-to-edge, round half away from zero (our semantics: the reference
 * carries no pixels) */
void or_crop96(const uint8_t* frame, int H, int W, const double* box4, uint8_t* out);

#ifdef __cplusplus
}
#endif
#endif
