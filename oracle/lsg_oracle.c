/*
 * lsg_oracle.c -- plain-C restatement of the reference hot path.
 * TEST INFRASTRUCTURE ONLY (see lsg_oracle.h).  Compiled by oracle/Makefile
 * with the reference's own flags (-O2, no -march, so no FMA contraction on
 * x86-64), into oracle/_build/liblsg_oracle.so.
 */
#include "lsg_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- VAD --- */

/* vad.cpp:20-24 reset(): Absolute pins the reference to full scale. */
void or_vad_init(or_vad* v, const or_vad_cfg* cfg) {
  v->cfg = *cfg;
  v->peak = cfg->peak_mode == 2 ? 32767.0 : 0.0;
}

/* vad.cpp:26-53 update(): sum of squares and |max| over the frame, peak
 * tracking per mode, rms_db clamped at -120, strict '>' threshold. */
int or_vad_update(or_vad* v, const int16_t* s, int64_t n, double* rms_db) {
  double sumsq = 0.0, fmax = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double x = s[i];
    sumsq += x * x;
    double a = fabs(x);
    if (a > fmax) fmax = a;
  }
  if (v->cfg.peak_mode == 0) {
    v->peak *= exp2(-(double)v->cfg.frame_ms / v->cfg.peak_half_life_ms);
    if (fmax > v->peak) v->peak = fmax;
  } else if (v->cfg.peak_mode == 1) {
    if (fmax > v->peak) v->peak = fmax;
  }
  double db = -120.0;
  double rms = sqrt(sumsq / (double)n);
  if (rms > 0.0 && v->peak > 0.0) {
    double d = 20.0 * log10(rms / v->peak);
    db = d > -120.0 ? d : -120.0;
  }
  if (rms_db) *rms_db = db;
  return db > v->cfg.speech_threshold_db;
}

/* ---------------------------------------------------------- Segmenter --- */

/* segmenter.cpp:9-23 constructor checks. */
int or_seg_init(or_seg* s, const or_seg_cfg* cfg, or_scorer_fn scorer, void* user) {
  memset(s, 0, sizeof(*s));
  if (cfg->sample_rate <= 0 || cfg->sample_rate % 1000 != 0) return 1;
  if (cfg->min_silence_ms <= 0) return 1;
  if (cfg->mode == 1) {
    if (cfg->min_segment_ms < 0 || cfg->max_segment_ms <= 0) return 1;
    if (cfg->max_segment_ms <= cfg->min_segment_ms) return 1;
  }
  if (cfg->vad.peak_half_life_ms <= 0 || cfg->vad.frame_ms <= 0) return 1; /* vad.cpp:14-17 */
  s->cfg = *cfg;
  s->scorer = scorer;
  s->scorer_user = user;
  or_vad_init(&s->vad, &cfg->vad);
  s->frame_samples = (int64_t)cfg->sample_rate * cfg->vad.frame_ms / 1000;
  s->candidate_confidence = 1.0;
  return 0;
}

void or_seg_free(or_seg* s) {
  free(s->stage);
  s->stage = NULL;
}

static int emit(or_cut* out, int64_t cap, int64_t* n, const or_cut* c) {
  if (*n < cap) out[*n] = *c;
  ++*n;
  return 0;
}

/* segmenter.cpp:101-118 emit_cut: split (cut-seg_start)*rate/1000 samples off
 * the open segment. */
static void emit_cut(or_seg* s, int64_t cut_ms, double conf, int cause, or_cut* out,
                     int64_t cap, int64_t* n) {
  int64_t split = (cut_ms - s->seg_start) * s->cfg.sample_rate / 1000;
  or_cut c;
  c.begin = s->seg_start;
  c.end = cut_ms;
  c.confidence = conf;
  c.cause = cause;
  c.sample_off = s->emitted_samples;
  c.sample_len = split;
  emit(out, cap, n, &c);
  s->emitted_samples += split;
  s->pending_len -= split;
  s->seg_start = cut_ms;
  s->speech_seen = 0;
}

/* segmenter.cpp:51-99 process_frame. */
static void process_frame(or_seg* s, const int16_t* smp, int64_t cnt, or_cut* out, int64_t cap,
                          int64_t* n) {
  const or_seg_cfg* c = &s->cfg;
  int64_t f0 = s->base + s->consumed_frames * c->vad.frame_ms;
  int64_t f1 = f0 + c->vad.frame_ms;
  int speech = or_vad_update(&s->vad, smp, cnt, NULL);
  s->metrics.frames += 1;
  if (speech) {
    s->metrics.speech_frames += 1;
    if (s->speech_seen && s->silence_run >= c->min_silence_ms && s->candidate_open &&
        s->candidate_cut) {
      emit_cut(s, s->pause_start + s->silence_run / 2, s->candidate_confidence, 0, out, cap, n);
      s->metrics.cuts_pause += 1;
    }
    s->silence_run = 0;
    s->candidate_open = 0;
    s->candidate_cut = 0;
    s->pending_len += cnt;
    s->speech_seen = 1;
  } else {
    if (s->silence_run == 0) s->pause_start = f0;
    s->silence_run += c->vad.frame_ms;
    s->pending_len += cnt;
    if (!s->candidate_open && s->silence_run >= c->min_silence_ms && s->speech_seen) {
      s->candidate_open = 1;
      s->candidate_cut = 1;
      s->candidate_confidence = 1.0;
      if (c->mode == 1) {
        if (s->pause_start - s->seg_start < c->min_segment_ms) {
          s->candidate_cut = 0;
        } else if (s->scorer) {
          int cut = 1;
          double conf = 1.0, cost = 0.0;
          s->scorer(s->scorer_user, s->pause_start, s->silence_run, s->pause_start - s->seg_start,
                    &cut, &conf, &cost);
          s->metrics.scorer_calls += 1;
          s->metrics.scorer_cost_ms += cost;
          s->candidate_cut = cut;
          s->candidate_confidence = conf;
        }
      }
    }
  }
  if (c->mode == 1 && s->speech_seen && f1 - s->seg_start >= c->max_segment_ms) {
    emit_cut(s, f1, 1.0, 1, out, cap, n);
    s->metrics.cuts_forced += 1;
  }
}

/* segmenter.cpp:25-49 push: discipline checks, stage, whole frames. */
int or_seg_push(or_seg* s, const int16_t* pcm, int64_t n, int64_t start_ms, int sample_rate,
                or_cut* out, int64_t cap, int64_t* n_out) {
  *n_out = 0;
  if (s->finished) return 2;
  if (sample_rate != s->cfg.sample_rate) return 1;
  if (n == 0) return 0;
  int64_t staged_ms =
      s->consumed_frames * s->cfg.vad.frame_ms + s->stage_len * 1000 / s->cfg.sample_rate;
  if (s->consumed_frames == 0 && s->stage_len == 0 && s->pending_len == 0) {
    s->seg_start = start_ms;
    s->base = start_ms;
  } else if (llabs(start_ms - (s->base + staged_ms)) > 1) {
    return 1;
  }
  if (s->stage_len + n > s->stage_cap) {
    int64_t cap2 = (s->stage_len + n) * 2 + 64;
    s->stage = (int16_t*)realloc(s->stage, (size_t)cap2 * sizeof(int16_t));
    s->stage_cap = cap2;
  }
  memcpy(s->stage + s->stage_len, pcm, (size_t)n * sizeof(int16_t));
  s->stage_len += n;
  int64_t off = 0;
  while (s->stage_len - off >= s->frame_samples) {
    process_frame(s, s->stage + off, s->frame_samples, out, cap, n_out);
    off += s->frame_samples;
    s->consumed_frames += 1;
  }
  memmove(s->stage, s->stage + off, (size_t)(s->stage_len - off) * sizeof(int16_t));
  s->stage_len -= off;
  return 0;
}

/* segmenter.cpp:120-145 finish: sub-frame tail joins the open segment; a
 * segment without speech is dropped. */
int or_seg_finish(or_seg* s, or_cut* out, int64_t cap, int64_t* n_out) {
  *n_out = 0;
  if (s->finished) return 2;
  s->finished = 1;
  int64_t tail_ms = s->stage_len * 1000 / s->cfg.sample_rate;
  s->pending_len += s->stage_len;
  s->stage_len = 0;
  if (!s->speech_seen || s->pending_len == 0) return 0;
  or_cut c;
  c.begin = s->seg_start;
  c.end = s->base + s->consumed_frames * s->cfg.vad.frame_ms + tail_ms;
  c.confidence = 1.0;
  c.cause = 2;
  c.sample_off = s->emitted_samples;
  c.sample_len = s->pending_len;
  emit(out, cap, n_out, &c);
  s->emitted_samples += s->pending_len;
  s->pending_len = 0;
  s->metrics.cuts_eos += 1;
  return 0;
}

int64_t or_seg_sizeof(void) { return (int64_t)sizeof(or_seg); }
void or_seg_get_metrics(const or_seg* s, or_seg_metrics* m) { *m = s->metrics; }

/* ---------------------------------------------------------------- Mel --- */

static const double kPi = 3.141592653589793238462643383279502884;

void or_mel_default(or_mel_cfg* c) {
  c->sample_rate = 16000;
  c->fft_size = 1024;
  c->hop = 256;
  c->n_mels = 80;
  c->fmin = 0.0;
  c->fmax = 8000.0;
}

/* mel.cpp:27-37 validate */
static int mel_valid(const or_mel_cfg* c) {
  if (c->fft_size <= 0 || (c->fft_size & (c->fft_size - 1)) != 0) return 0;
  if (c->hop <= 0 || c->n_mels <= 0) return 0;
  if (!(c->fmax > c->fmin) || c->fmin < 0) return 0;
  if (c->sample_rate <= 0) return 0;
  return 1;
}

/* mel.cpp:40-44 */
int64_t or_mel_frame_count(int64_t n, const or_mel_cfg* c) {
  if (!mel_valid(c)) return -1;
  if (n < c->fft_size) return 0;
  return 1 + (n - c->fft_size) / c->hop;
}

/* mel.cpp:17-25: Slaney-style scale, linear to 1 kHz then log step ln(6.4)/27 */
static double hz_to_mel(double hz) {
  if (hz < 1000.0) return hz * 15.0 / 1000.0;
  return 15.0 + 27.0 * log(hz / 1000.0) / log(6.4);
}
static double mel_to_hz(double m) {
  if (m < 15.0) return m * 1000.0 / 15.0;
  return 1000.0 * exp(log(6.4) * (m - 15.0) / 27.0);
}

/* mel.cpp:46-70: bit reversal, then butterflies with the twiddle advanced by
 * the recurrence w *= wlen (std::complex multiply, no FMA). */
int or_fft_radix2(double* b, int64_t n) {
  if (n == 0 || (n & (n - 1)) != 0) return 1;
  for (int64_t i = 1, j = 0; i < n; ++i) {
    int64_t bit = n >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) {
      double tr = b[2 * i], ti = b[2 * i + 1];
      b[2 * i] = b[2 * j]; b[2 * i + 1] = b[2 * j + 1];
      b[2 * j] = tr; b[2 * j + 1] = ti;
    }
  }
  for (int64_t len = 2; len <= n; len <<= 1) {
    double ang = -2.0 * kPi / (double)len;
    double wlr = cos(ang), wli = sin(ang);
    for (int64_t i = 0; i < n; i += len) {
      double wr = 1.0, wi = 0.0;
      for (int64_t k = 0; k < len / 2; ++k) {
        double* u = b + 2 * (i + k);
        double* v = b + 2 * (i + k + len / 2);
        double ur = u[0], ui = u[1];
        double vr = v[0] * wr - v[1] * wi;
        double vi = v[0] * wi + v[1] * wr;
        u[0] = ur + vr; u[1] = ui + vi;
        v[0] = ur - vr; v[1] = ui - vi;
        double nwr = wr * wlr - wi * wli;
        double nwi = wr * wli + wi * wlr;
        wr = nwr; wi = nwi;
      }
    }
  }
  return 0;
}

/* mel.cpp:88-110: n_mels+2 edges equally spaced on the mel axis, strict
 * lo<f<hi triangles scaled by 2/(hi-lo). */
int or_mel_filterbank(const or_mel_cfg* c, double* w) {
  if (!mel_valid(c)) return 1;
  const int N = c->fft_size, bins = N / 2 + 1, M = c->n_mels;
  double* edge = (double*)malloc(sizeof(double) * (size_t)(M + 2));
  const double lo_m = hz_to_mel(c->fmin), hi_m = hz_to_mel(c->fmax);
  for (int i = 0; i < M + 2; ++i) edge[i] = mel_to_hz(lo_m + (hi_m - lo_m) * i / (M + 1));
  for (int m = 0; m < M; ++m) {
    double lo = edge[m], mid = edge[m + 1], hi = edge[m + 2];
    double norm = 2.0 / (hi - lo);
    for (int b = 0; b < bins; ++b) {
      double f = (double)b * c->sample_rate / N;
      double v = 0.0;
      if (f > lo && f < hi) v = f <= mid ? (f - lo) / (mid - lo) : (hi - f) / (hi - mid);
      w[(size_t)m * bins + b] = v * norm;
    }
  }
  free(edge);
  return 0;
}

/* mel.cpp:72-127 compute_mel: periodic Hann, x = s/32768*w, FFT, |X|^2,
 * dense filterbank sum in bin order, (float)ln(max(acc,1e-10)). */
int64_t or_compute_mel(const int16_t* pcm, int64_t n, const or_mel_cfg* c, float* out) {
  if (!mel_valid(c)) return -1;
  const int N = c->fft_size, bins = N / 2 + 1, M = c->n_mels;
  int64_t frames = or_mel_frame_count(n, c);
  if (frames == 0) return 0;
  double* win = (double*)malloc(sizeof(double) * (size_t)N);
  for (int i = 0; i < N; ++i) win[i] = 0.5 * (1.0 - cos(2.0 * kPi * i / N));
  double* w = (double*)malloc(sizeof(double) * (size_t)M * bins);
  or_mel_filterbank(c, w);
  double* buf = (double*)malloc(sizeof(double) * 2 * (size_t)N);
  double* pw = (double*)malloc(sizeof(double) * (size_t)bins);
  for (int64_t fr = 0; fr < frames; ++fr) {
    const int16_t* x = pcm + fr * c->hop;
    for (int i = 0; i < N; ++i) {
      buf[2 * i] = x[i] / 32768.0 * win[i];
      buf[2 * i + 1] = 0.0;
    }
    or_fft_radix2(buf, N);
    for (int b = 0; b < bins; ++b) pw[b] = buf[2 * b] * buf[2 * b] + buf[2 * b + 1] * buf[2 * b + 1];
    for (int m = 0; m < M; ++m) {
      double acc = 0.0;
      const double* wm = w + (size_t)m * bins;
      for (int b = 0; b < bins; ++b) acc += wm[b] * pw[b];
      out[fr * M + m] = (float)log(acc > 1e-10 ? acc : 1e-10);
    }
  }
  free(win); free(w); free(buf); free(pw);
  return frames;
}

/* ======================================================== A/V alignment */

/* align.cpp:10-32: RMS over 10 ms hops of v = s / 32768, held for each ms of
 * the hop; sequential sums, no contraction (the reference's x86-64 build). */
int64_t or_energy_envelope(const int16_t* pcm, int64_t n, int rate, double* out, int64_t cap) {
  if (rate <= 0) return -1;
  const int64_t total = llround(1000.0 * (double)n / rate);
  if (total <= 0) return 0;
  const int64_t hop = (int64_t)rate * 10 / 1000;
  if (hop <= 0) return -1;
  if (total > cap) return total;
  for (int64_t t = 0; t < total; t += 10) {
    const int64_t s0 = t / 10 * hop;
    const int64_t s1 = s0 + hop < n ? s0 + hop : n;
    volatile double sumsq = 0.0;
    for (int64_t s = s0; s < s1; ++s) {
      const volatile double v = pcm[s] / 32768.0;
      const volatile double vv = v * v;
      sumsq = sumsq + vv;
    }
    const double rms = s1 > s0 ? sqrt(sumsq / (double)(s1 - s0)) : 0.0;
    for (int64_t k = t; k < (t + 10 < total ? t + 10 : total); ++k) out[k] = rms;
  }
  return total;
}

/* align.cpp:34-50: each frame's value holds until the next frame; 0 before
 * the first frame. */
int or_motion_envelope(const int64_t* ts, const double* motion, int64_t nf, int64_t t0, int64_t span, double* out) {
  if (span < 0) return -1;
  int64_t f = 0;
  double held = 0.0;
  int have = 0;
  for (int64_t t = 0; t < span; ++t) {
    while (f < nf && ts[f] <= t0 + t) {
      held = motion[f];
      have = 1;
      ++f;
    }
    out[t] = have ? held : 0.0;
  }
  return 0;
}

/* align.cpp:52-116: normalised cross-correlation over lags in
 * [-max_lag, max_lag] on the full-overlap region [max_lag, D - max_lag);
 * ties prefer the smaller |lag|, then the negative one. */
int or_align_envelopes(const double* e, int64_t ne, const double* m, int64_t nm, int64_t max_lag,
                       or_align_result* r) {
  if (max_lag < 0) return -1;
  r->offset_ms = 0;
  r->peak_corr = 0.0;
  r->low_confidence = 0;
  const int64_t d = ne < nm ? ne : nm;
  const int64_t lo = max_lag, hi = d - max_lag;
  if (hi - lo < 2) {
    r->low_confidence = 1;
    return 0;
  }
  const double n = (double)(hi - lo);
  volatile double e_mean = 0.0;
  for (int64_t t = lo; t < hi; ++t) e_mean = e_mean + e[t];
  e_mean = e_mean / n;
  volatile double e_var = 0.0;
  for (int64_t t = lo; t < hi; ++t) {
    const volatile double v = e[t] - e_mean;
    const volatile double vv = v * v;
    e_var = e_var + vv;
  }
  const double e_sigma = sqrt(e_var);
  if (e_sigma < 1e-12) {
    r->low_confidence = 1;
    return 0;
  }
  int any = 0;
  double best = 0.0;
  int64_t best_lag = 0;
  for (int64_t lag = -max_lag; lag <= max_lag; ++lag) {
    volatile double m_mean = 0.0;
    for (int64_t t = lo; t < hi; ++t) m_mean = m_mean + m[t + lag];
    m_mean = m_mean / n;
    volatile double m_var = 0.0, dot = 0.0;
    for (int64_t t = lo; t < hi; ++t) {
      const volatile double me = m[t + lag] - m_mean;
      const volatile double mm = me * me;
      m_var = m_var + mm;
      const volatile double de = e[t] - e_mean;
      const volatile double p = de * me;
      dot = dot + p;
    }
    const double m_sigma = sqrt(m_var);
    if (m_sigma < 1e-12) continue;
    const double corr = dot / (e_sigma * m_sigma);
    int better = !any || corr > best;
    if (any && corr == best) {
      const int64_t al = lag < 0 ? -lag : lag, ab = best_lag < 0 ? -best_lag : best_lag;
      better = al < ab || (al == ab && lag < best_lag);
    }
    if (better) {
      any = 1;
      best = corr;
      best_lag = lag;
    }
  }
  if (!any) {
    r->low_confidence = 1;
    return 0;
  }
  r->offset_ms = best_lag;
  r->peak_corr = best;
  return 0;
}

/* ==================================================== face track (f1) */

static uint64_t or_splitmix64(uint64_t* s) {
  uint64_t z = (*s += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
static uint64_t or_mix_u64(uint64_t h, uint64_t v) { /* rng.hpp:21-25 */
  h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
  uint64_t s = h;
  return or_splitmix64(&s);
}

/* visual_mocks.cpp:10-22 */
void or_mock_face_detect(int64_t frame_index, uint64_t seed, double* box4) {
  const char* tag = "facedetect";
  uint64_t h = seed;
  for (const char* c = tag; *c; ++c) h = or_mix_u64(h, (uint8_t)*c);
  h = or_mix_u64(h, (uint64_t)frame_index);
  box4[0] = 320.0 + ((double)(or_splitmix64(&h) % 7) - 3.0);
  box4[1] = 240.0 + ((double)(or_splitmix64(&h) % 7) - 3.0);
  box4[2] = 160.0;
  box4[3] = 200.0;
}

typedef struct {
  int init;
  double x[6], p[6][6];
  double pn, mn, iv;
} or_kf;

/* kalman.cpp:16-49: 4x4 Cholesky and solve */
static int or_chol4(double a[4][4], double l[4][4]) {
  memset(l, 0, 16 * sizeof(double));
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j <= i; ++j) {
      volatile double sum = a[i][j];
      for (int k = 0; k < j; ++k) {
        const volatile double pr = l[i][k] * l[j][k];
        sum = sum - pr;
      }
      if (i == j) {
        if (sum <= 0.0 || !isfinite(sum)) return 0;
        l[i][i] = sqrt(sum);
      } else {
        l[i][j] = sum / l[j][j];
      }
    }
  return 1;
}
static void or_chol_solve4(double l[4][4], const double b[4], double x[4]) {
  double y[4];
  for (int i = 0; i < 4; ++i) {
    volatile double sum = b[i];
    for (int k = 0; k < i; ++k) {
      const volatile double pr = l[i][k] * y[k];
      sum = sum - pr;
    }
    y[i] = sum / l[i][i];
  }
  for (int i = 3; i >= 0; --i) {
    volatile double sum = y[i];
    for (int k = i + 1; k < 4; ++k) {
      const volatile double pr = l[k][i] * x[k];
      sum = sum - pr;
    }
    x[i] = sum / l[i][i];
  }
}

/* kalman.cpp:58-77 */
static void or_kf_predict(or_kf* f, double dt) {
  volatile double t;
  t = f->x[4] * dt; f->x[0] = f->x[0] + t;
  t = f->x[5] * dt; f->x[1] = f->x[1] + t;
  double fp[6][6];
  for (int j = 0; j < 6; ++j) {
    for (int i = 0; i < 6; ++i) fp[i][j] = f->p[i][j];
    t = dt * f->p[4][j]; fp[0][j] = fp[0][j] + t;
    t = dt * f->p[5][j]; fp[1][j] = fp[1][j] + t;
  }
  for (int i = 0; i < 6; ++i) {
    for (int j = 0; j < 6; ++j) f->p[i][j] = fp[i][j];
    t = dt * fp[i][4]; f->p[i][0] = f->p[i][0] + t;
    t = dt * fp[i][5]; f->p[i][1] = f->p[i][1] + t;
  }
  const double q = f->pn * dt;
  for (int i = 0; i < 6; ++i) f->p[i][i] = f->p[i][i] + q;
}

/* kalman.cpp:79-135 (update), Joseph form */
static int or_kf_update(or_kf* f, const double z[4], double dt) {
  for (int i = 0; i < 4; ++i)
    if (!isfinite(z[i])) return -1;
  if (!f->init) {
    for (int i = 0; i < 4; ++i) f->x[i] = z[i];
    f->x[4] = f->x[5] = 0.0;
    for (int i = 0; i < 6; ++i)
      for (int j = 0; j < 6; ++j) f->p[i][j] = i == j ? f->iv : 0.0;
    f->init = 1;
    return 0;
  }
  if (dt < 0 || !isfinite(dt)) return -1;
  or_kf_predict(f, dt);
  double s[4][4], l[4][4], k[6][4];
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) s[i][j] = f->p[i][j] + (i == j ? f->mn : 0.0);
  if (!or_chol4(s, l)) return -1;
  for (int i = 0; i < 6; ++i) {
    double row[4], sol[4];
    for (int j = 0; j < 4; ++j) row[j] = f->p[i][j];
    or_chol_solve4(l, row, sol);
    for (int j = 0; j < 4; ++j) k[i][j] = sol[j];
  }
  double y[4];
  for (int i = 0; i < 4; ++i) y[i] = z[i] - f->x[i];
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 4; ++j) {
      const volatile double pr = k[i][j] * y[j];
      f->x[i] = f->x[i] + pr;
    }
  double ikh[6][6], tmp[6][6];
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 6; ++j) ikh[i][j] = (i == j ? 1.0 : 0.0) - (j < 4 ? k[i][j] : 0.0);
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 6; ++j) {
      volatile double acc = 0.0;
      for (int m = 0; m < 6; ++m) {
        const volatile double pr = ikh[i][m] * f->p[m][j];
        acc = acc + pr;
      }
      tmp[i][j] = acc;
    }
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 6; ++j) {
      volatile double acc = 0.0;
      for (int m = 0; m < 6; ++m) {
        const volatile double pr = tmp[i][m] * ikh[j][m];
        acc = acc + pr;
      }
      for (int m = 0; m < 4; ++m) {
        const volatile double a = k[i][m] * f->mn;
        const volatile double pr = a * k[j][m];
        acc = acc + pr;
      }
      f->p[i][j] = acc;
    }
  return 0;
}

int or_track_faces(const int64_t* ts, const int64_t* frame_index, const int* has_face, const double* faces,
                   int64_t n, uint64_t seed, double process_noise, double measurement_noise,
                   double initial_variance, double* out4, double* vel2) {
  or_kf f;
  memset(&f, 0, sizeof f);
  f.pn = process_noise;
  f.mn = measurement_noise;
  f.iv = initial_variance;
  int64_t prev = 0;
  for (int64_t i = 0; i < n; ++i) {
    double z[4];
    if (has_face[i]) memcpy(z, faces + 4 * i, sizeof z);
    else or_mock_face_detect(frame_index[i], seed, z);
    const double dt = f.init ? (double)(ts[i] - prev) / 1000.0 : 0.0;
    if (or_kf_update(&f, z, dt)) return -1;
    for (int c = 0; c < 4; ++c) out4[4 * i + c] = f.x[c];
    vel2[2 * i] = f.x[4];
    vel2[2 * i + 1] = f.x[5];
    prev = ts[i];
  }
  return 0;
}

/* bilinear 96x96 crop (our semantics; the reference has no pixels) */
void or_crop96(const uint8_t* frame, int H, int W, const double* b, uint8_t* out) {
  const double x0 = b[0] - 0.5 * b[2], y0 = b[1] - 0.5 * b[3];
  const double sx = b[2] / 96.0, sy = b[3] / 96.0;
  for (int v = 0; v < 96; ++v)
    for (int u = 0; u < 96; ++u) {
      double fx = x0 + (u + 0.5) * sx - 0.5, fy = y0 + (v + 0.5) * sy - 0.5;
      fx = fx < 0 ? 0 : (fx > W - 1 ? W - 1 : fx);
      fy = fy < 0 ? 0 : (fy > H - 1 ? H - 1 : fy);
      const int ix = (int)fx < W - 1 ? (int)fx : W - 2, iy = (int)fy < H - 1 ? (int)fy : H - 2;
      const double ax = fx - ix, ay = fy - iy;
      for (int c = 0; c < 3; ++c) {
        const double p00 = frame[((int64_t)iy * W + ix) * 3 + c], p01 = frame[((int64_t)iy * W + ix + 1) * 3 + c];
        const double p10 = frame[((int64_t)(iy + 1) * W + ix) * 3 + c];
        const double p11 = frame[((int64_t)(iy + 1) * W + ix + 1) * 3 + c];
        const volatile double top = p00 + ax * (p01 - p00);
        const volatile double bot = p10 + ax * (p11 - p10);
        const volatile double val = top + ay * (bot - top);
        out[((int64_t)v * 96 + u) * 3 + c] = (uint8_t)(val + 0.5);
      }
    }
}
