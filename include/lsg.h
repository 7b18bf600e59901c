/*
 * lsg.h -- C ABI of the B200-native lip-sync hot path (liblsg.so).
 *
 * Drop-in boundary for the per-segment lip-sync stage of the lipstream
 * reference (arXiv 2512.18318).  Every entry point replaces one reference
 * interface; the interface it replaces is cited next to it (paths relative
 * to /root/reference/proj/core/).  Plain pointers and sizes only -- no C++,
 * no torch types.  The C++ drop-in classes in include/lsg/lipstream_b200.hpp
 * wrap this ABI behind the reference's own class/function signatures.
 *
 * Conventions
 *  - Every function returns an lsg_status.  LSG_EINVAL / LSG_ELOGIC /
 *    LSG_ERUNTIME correspond to the reference's std::invalid_argument /
 *    std::logic_error / std::runtime_error (segmenter.cpp:11-38, mel.cpp:27-36,
 *    visual_mocks.cpp:43-46); LSG_ECUDA is a device failure.  The message of
 *    the last failure on the calling thread is lsg_last_error().
 *  - Handles own every device workspace, sized at create time; the compute
 *    calls do not allocate.  (One exception: lsg_align_* / lsg_face_track
 *    stage a per-call table in the context's scratch, 1 MiB at create time;
 *    a call needing more grows it once, synchronising the context's stream.)  A handle is externally synchronised (one host
 *    thread at a time), like one reference Segmenter per stream
 *    (SPEC.md:258-259).
 *  - Pointers marked [dev] are device pointers on the context's device,
 *    [host] are host pointers (pinned memory makes the copies async), and
 *    [any] are resolved with cudaPointerGetAttributes.
 *  - All device work is issued on the context's stream; calls that return
 *    results to host memory synchronise that stream.
 *  - There is no CPU fallback: with no usable sm_100 device, lsg_ctx_create
 *    fails with LSG_ECUDA.
 */
#ifndef LSG_H
#define LSG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int lsg_status;
#define LSG_OK 0
#define LSG_EINVAL 1   /* std::invalid_argument in the reference */
#define LSG_ELOGIC 2   /* std::logic_error */
#define LSG_ERUNTIME 3 /* std::runtime_error */
#define LSG_ECUDA 4    /* CUDA error, unsupported device */

#define LSG_ABI_VERSION 1

/* ------------------------------------------------------------------ core */
int32_t lsg_abi_version(void);
const char* lsg_last_error(void);
lsg_status lsg_device_count(int32_t* n);

typedef struct lsg_ctx_s* lsg_ctx;
/* One context per GPU: device, a non-blocking stream, event pool. */
lsg_status lsg_ctx_create(int32_t device, lsg_ctx* out);
lsg_status lsg_ctx_destroy(lsg_ctx ctx);
/* Replace the context stream with a caller-owned cudaStream_t (NULL = own). */
lsg_status lsg_ctx_set_stream(lsg_ctx ctx, void* cuda_stream);
lsg_status lsg_ctx_get_stream(lsg_ctx ctx, void** cuda_stream);
lsg_status lsg_ctx_sync(lsg_ctx ctx);
/* Kernel launches issued through this context since creation (telemetry). */
lsg_status lsg_ctx_launch_count(lsg_ctx ctx, int64_t* n);
/* Device / pinned-host memory helpers for callers without a CUDA runtime. */
lsg_status lsg_dev_alloc(lsg_ctx ctx, size_t bytes, void** out);
lsg_status lsg_dev_free(lsg_ctx ctx, void* p);
lsg_status lsg_host_alloc(size_t bytes, void** out);
lsg_status lsg_host_free(void* p);
lsg_status lsg_copy(lsg_ctx ctx, void* dst, const void* src, size_t bytes); /* async, [any]->[any] */

/* ------------------------------------------------------------- segmenter
 * Replaces lipstream::Segmenter (segmenter.hpp:76-111) and VadTracker
 * (vad.hpp:30-47) for many streams at once.  Each stream is an independent
 * reference Segmenter: same chunk discipline, same cuts, same metrics. */
typedef struct {
  int32_t mode;                /* 0 Baseline, 1 Semantic        (segmenter.hpp:43-50) */
  int32_t peak_mode;           /* 0 Decay, 1 MaxHold, 2 Absolute (vad.hpp:13-17)      */
  double peak_half_life_ms;    /* 10000                          (vad.hpp:21)         */
  double speech_threshold_db;  /* -40                            (vad.hpp:22)         */
  int64_t frame_ms;            /* 20                             (vad.hpp:23)         */
  int64_t min_silence_ms;      /* 500                            (segmenter.hpp:54)   */
  int64_t min_segment_ms;      /* 1500                           (segmenter.hpp:55)   */
  int64_t max_segment_ms;      /* 10000                          (segmenter.hpp:56)   */
  int32_t sample_rate;         /* 16000                          (segmenter.hpp:57)   */
  int32_t flags_only;          /* 1: run the VAD only and keep per-frame speech flags
                                  for a host state machine (BoundaryScorer path,
                                  segmenter.cpp:84-90); 0: full device state machine */
} lsg_seg_cfg;

typedef struct {
  int64_t begin, end;          /* ms, RawSegment::begin/end (segmenter.hpp:13-21) */
  double confidence;
  int32_t cause;               /* 0 Pause, 1 Forced, 2 Eos (segmenter.hpp:11)      */
  int32_t stream;
  int64_t sample_off;          /* first sample of RawSegment::audio in the stream  */
  int64_t sample_len;          /* == RawSegment::audio.samples.size()              */
} lsg_cut;

typedef struct {               /* SegmenterMetrics (segmenter.hpp:60-68) */
  int64_t frames, speech_frames, cuts_pause, cuts_forced, cuts_eos, scorer_calls;
  double scorer_cost_ms;
} lsg_seg_metrics;

typedef struct lsg_seg_s* lsg_seg;
lsg_status lsg_seg_cfg_default(lsg_seg_cfg* cfg);
/* Segmenter::Segmenter (segmenter.cpp:9-23): EINVAL on the same configs.
 * max_push_samples bounds the samples of one stream in one push call. */
lsg_status lsg_seg_create(lsg_ctx ctx, const lsg_seg_cfg* cfg, int32_t n_streams,
                          int64_t max_push_samples, lsg_seg* out);
lsg_status lsg_seg_destroy(lsg_seg h);
/* Returns every stream to its freshly constructed state without
 * reallocating (VadTracker::reset, vad.cpp:20-24, for the whole handle). */
lsg_status lsg_seg_reset(lsg_seg h);
/* Segmenter::push for n_chunks streams at once (segmenter.cpp:25-49); a
 * stream appears at most once per call.  pcm[i] is [any] unless
 * pcm_on_device, then [dev].  ELOGIC after finish, EINVAL on a rate
 * mismatch or a non-contiguous chunk -- checked for every chunk before any
 * device work, so a failing call changes no stream. */
lsg_status lsg_seg_push(lsg_seg h, int32_t n_chunks, const int32_t* streams,
                        const int16_t* const* pcm, const int64_t* n_samples,
                        const int64_t* start_ms, int32_t sample_rate, int32_t pcm_on_device);
/* Segmenter::finish (segmenter.cpp:120-145) for the listed streams. */
lsg_status lsg_seg_finish(lsg_seg h, int32_t n, const int32_t* streams);
/* Drains the cuts a stream emitted since the last call, in order.  Returns
 * the count in *n_out even when it exceeds cap (nothing is drained then). */
lsg_status lsg_seg_take_cuts(lsg_seg h, int32_t stream, lsg_cut* out, int64_t cap,
                             int64_t* n_out);
/* All streams at once: cuts of every stream appended in stream order. */
lsg_status lsg_seg_take_all_cuts(lsg_seg h, lsg_cut* out, int64_t cap, int64_t* n_out);
lsg_status lsg_seg_get_metrics(lsg_seg h, int32_t stream, lsg_seg_metrics* out);
/* flags_only mode: per-frame speech decisions of the frames the stream
 * consumed in the last push (VadTracker::FrameResult::speech, vad.hpp:34-37). */
lsg_status lsg_seg_take_flags(lsg_seg h, int32_t stream, uint8_t* speech, int64_t cap,
                              int64_t* n_out);

/* ------------------------------------------------------------------- mel
 * Replaces compute_mel / mel_frame_count (mel.hpp:33-39, mel.cpp:40-127). */
typedef struct {               /* MelConfig (mel.hpp:12-19) */
  int32_t sample_rate, fft_size, hop, n_mels;
  double fmin, fmax;
} lsg_mel_cfg;

typedef struct lsg_mel_s* lsg_mel;
lsg_status lsg_mel_cfg_default(lsg_mel_cfg* cfg);
/* mel_frame_count (mel.cpp:40-44); EINVAL on a bad config (mel.cpp:27-37). */
lsg_status lsg_mel_frames(int64_t n_samples, const lsg_mel_cfg* cfg, int64_t* frames);
/* Builds window, filterbank (host fp64, exactly mel.cpp:83-110) and FFT
 * tables once.  max_frames bounds one compute call. */
lsg_status lsg_mel_create(lsg_ctx ctx, const lsg_mel_cfg* cfg, int64_t max_frames, lsg_mel* out);
/* fft_radix2 (mel.cpp:46-70, mel.hpp:42), in place, bit-identical to the
 * reference: `count` transforms of n complex doubles, data [any] interleaved
 * (re, im), transform i at data + 2*n*i.  n a power of two <= 8192, else
 * EINVAL ("fft: size must be a power of two", mel.cpp:48-49).  Synchronises. */
lsg_status lsg_fft_radix2(lsg_ctx ctx, double* data, int64_t n, int32_t count);
lsg_status lsg_mel_destroy(lsg_mel h);
/* compute_mel of one buffer: pcm [any] (n samples) -> out [any]
 * [frames][n_mels] f32, row major like MelSpectrogram::data. */
lsg_status lsg_mel_compute(lsg_mel h, const int16_t* pcm, int64_t n, float* out,
                           int64_t* frames);
/* Many segments of device-resident PCM in one launch: segment i reads
 * n_samples[i] samples at pcm_base + pcm_off[i] and writes its frames at row
 * out_row[i] of out_base.  Offsets/lengths are [host]; pcm_base, out_base [dev]. */
lsg_status lsg_mel_compute_batch(lsg_mel h, int32_t n_seg, const int16_t* pcm_base,
                                 const int64_t* pcm_off, const int64_t* n_samples,
                                 float* out_base, const int64_t* out_row);

/* ------------------------------------------------------------- generator
 * The lip-sync stage.  The reference only has the cost model mock_lipsync
 * (visual_mocks.hpp:17-43, visual_mocks.cpp:24-51); this is the Wav2Lip
 * generator forward it stands for, in bf16 on
 * tcgen05 tensor cores. */
#define LSG_PREC_BF16 0         /* bf16 weights/activations, f32 accumulate */
#define LSG_PREC_FP16 1         /* fp16 weights/activations, f32 accumulate (same tcgen05 rate) */
#define LSG_PREC_FP8 2          /* e4m3 weights (per output channel scale) and activations (per tensor
                                   scale from lsg_gen_calibrate), f32 accumulate */
#define LSG_PREC_FP8_TAIL 3     /* fp16 up to fd5.2, e4m3 (as LSG_PREC_FP8) for fd6.0-out0 (28% of the
                                   FLOPs): the fp8 split that keeps >= 30 dB vs the fp32 oracle on the
                                   synthetic network; needs act_absmax like LSG_PREC_FP8 */
#define LSG_PREC_INT8_TAIL 4    /* fp16 encoders and fd0, then tcgen05 kind::i8 for fd1.0-out0 (90%
                                   of the FLOPs): u8 activations (every decoder input is post-ReLU, per
                                   tensor scale absmax/255), s8 weights (per output channel scale
                                   max|w|/127), s32 accumulate; >= 30 dB vs the fp32 oracle (DESIGN.md
                                   §4); needs act_absmax like LSG_PREC_FP8 */
#define LSG_OUT_F32_NCHW 0      /* [B][3][96][96] f32 in [0,1] */
#define LSG_OUT_U8_NHWC 1       /* [B][96][96][3] u8, round(255*x) */
#define LSG_OUT_F32_LOGITS 2    /* [B][3][96][96] f32 pre-sigmoid (parity checks) */

typedef struct lsg_gen_s* lsg_gen;
/* Number of floats in the weight blob (BN folded; layer order and per-layer
 * layout documented in DESIGN.md §Generator and lsg_gen_layer_info). */
lsg_status lsg_gen_param_count(int64_t* n);
/* Per-layer shape table: 12 ints per layer {kind(0 conv,1 convT), cin, cout,
 * kh, kw, sh, sw, ph, pw, oph, opw, residual}; *n_layers on return. */
lsg_status lsg_gen_layer_info(int32_t* info, int32_t cap_layers, int32_t* n_layers);
lsg_status lsg_gen_create(lsg_ctx ctx, const float* weights /*[host]*/, int64_t n_floats,
                          int32_t precision, int32_t max_batch, lsg_gen* out);
/* As lsg_gen_create; LSG_PREC_FP8 / _FP8_TAIL / _INT8_TAIL require act_absmax
 * [host], the n_act activation ranges lsg_gen_calibrate returns (ignored
 * otherwise). */
lsg_status lsg_gen_create_q(lsg_ctx ctx, const float* weights /*[host]*/, int64_t n_floats, int32_t precision,
                            const float* act_absmax, int32_t n_act, int32_t max_batch, lsg_gen* out);
/* On a bf16/fp16 engine: run a calibration batch (inputs as lsg_gen_forward)
 * and return max |x| of every fp8 scale group -- face input, mel input, the
 * seven concat buffers (shared by both producers), each other layer output.
 * *n_tensors = groups; nothing is written when cap < *n_tensors. */
lsg_status lsg_gen_calibrate(lsg_gen h, const float* mel_rows, const int32_t* chunk_row,
                             const uint8_t* target, const uint8_t* refs, const int32_t* ref_index,
                             int32_t B, float* absmax /*[host]*/, int32_t cap, int32_t* n_tensors);
lsg_status lsg_gen_destroy(lsg_gen h);
/* Forward of B frames, all inputs [dev]:
 *   mel_rows  [rows][80] f32 log-mel rows (lsg_mel output)
 *   chunk_row [B] first row of each frame's 16-row mel window
 *   target    [B][96][96][3] u8 face crops (lower half masked on device)
 *   refs      [R][96][96][3] u8 reference crops, ref_index [B] into them
 *   out       see out_format.  B <= max_batch. */
lsg_status lsg_gen_forward(lsg_gen h, const float* mel_rows, const int32_t* chunk_row,
                           const uint8_t* target, const uint8_t* refs, const int32_t* ref_index,
                           void* out, int32_t out_format, int32_t B);
/* mock_lipsync's input contract (visual_mocks.cpp:40-51): EINVAL when
 * n_frames < 2 or |audio_span - frame_span| > 150 ms. */
lsg_status lsg_lipsync_validate(int64_t audio_span_ms, int64_t frame_span_ms, int64_t n_frames);

/* ------------------------------------------------------------ alignment
 * A/V alignment, batched and bit-identical to align.cpp.
 * Offsets / lengths are [host]; *_base pointers [dev]. */
typedef struct {
  int64_t offset_ms;           /* positive: motion lags the audio            */
  double peak_corr;
  int32_t low_confidence;
  int32_t pad;
} lsg_align_result;            /* AlignResult (align.hpp:17-21)              */
/* energy_envelope_ms (align.cpp:10-32) of n PCM segments: segment i is
 * n_samples[i] samples at pcm_base + pcm_off[i]; its llround(1000 n / rate)
 * ms envelope goes to out_base + out_off[i]; out_len[i] [host] on return. */
lsg_status lsg_align_energy(lsg_ctx ctx, int32_t n, const int16_t* pcm_base, const int64_t* pcm_off,
                            const int64_t* n_samples, int32_t sample_rate, double* out_base,
                            const int64_t* out_off, int64_t* out_len);
/* motion_envelope_ms (align.cpp:34-50): segment i reads n_frames[i]
 * (ts, mouth_motion) records from frame_off[i] (sorted by ts) and writes
 * span[i] ms starting at t0[i] to out_base + out_off[i]. */
lsg_status lsg_align_motion(lsg_ctx ctx, int32_t n, const int64_t* ts_base, const double* motion_base,
                            const int64_t* frame_off, const int64_t* n_frames, const int64_t* t0,
                            const int64_t* span, double* out_base, const int64_t* out_off);
/* align_envelopes (align.cpp:52-116) for n (energy, motion) pairs; results
 * [host].  EINVAL for max_lag < 0 (the reference's throw) or > 511. */
lsg_status lsg_align_batch(lsg_ctx ctx, int32_t n, const double* energy_base, const int64_t* e_off,
                           const int64_t* e_len, const double* motion_base, const int64_t* m_off,
                           const int64_t* m_len, int64_t max_lag, lsg_align_result* out);

/* ----------------------------------------------------------------- face
 * Face-crop preparation: the detect + KalmanBoxFilter
 * smoothing loop of orchestrator.cpp:115-129 per segment (bit-identical to
 * kalman.cpp), and a bilinear 96x96 crop of the smoothed box. */
typedef struct {
  double process_noise;        /* 1e-2 per second (kalman.hpp:8-12)          */
  double measurement_noise;    /* 25 px^2                                    */
  double initial_variance;     /* 1e6                                        */
} lsg_kalman_cfg;
lsg_status lsg_kalman_cfg_default(lsg_kalman_cfg* c);
/* mock_face_detect (visual_mocks.cpp:10-22): box4 = {cx, cy, w, h} [host] */
lsg_status lsg_face_mock_detect(int64_t frame_index, uint64_t seed, double* box4);
/* n segments; segment i = frames [seg_off[i], seg_off[i] + seg_len[i]) of
 * the frame arrays ([dev]: ts, frame_index, optional has_face / faces
 * [F][4]); a frame without a face uses mock_face_detect(frame_index, seed).
 * Writes the smoothed box [F][4] and (optional) velocity [F][2] [dev];
 * status[i] [host] = 0, or -1 where KalmanBoxFilter would throw (non-finite
 * box, bad time step, S not SPD) -- that segment's later frames are left
 * unwritten.  seg_off / seg_len [host]. */
lsg_status lsg_face_track(lsg_ctx ctx, int32_t n, const int64_t* seg_off, const int64_t* seg_len,
                          const int64_t* ts, const int64_t* frame_index, const int32_t* has_face,
                          const double* faces, uint64_t seed, const lsg_kalman_cfg* cfg,
                          double* out_box, double* out_vel, int32_t* status);
/* n crops: crop k resamples box boxes[k] of frame frame_of[k] of frames
 * [F][H][W][3] u8 into out [n][96][96][3] u8 (bilinear, clamp to edge);
 * all pointers [dev]; asynchronous on the context stream. */
lsg_status lsg_face_crop(lsg_ctx ctx, int32_t n, const uint8_t* frames, int32_t H, int32_t W,
                         const int64_t* frame_of, const double* boxes, uint8_t* out);

/* -------------------------------------------------------------- pipeline
 * Replaces the per-clip driver run_pipeline_input (runner.cpp:239-351) for
 * the GPU stages: segment -> mel per segment -> gather frames -> generator,
 * for many streams.  Streams are independent; a multi-GPU job gives each
 * rank its own context and shard of streams (no collective). */
typedef struct {
  int32_t n_streams;
  int32_t max_stream_ms;       /* longest stream accepted                      */
  double fps;                  /* video frame rate (frames at llround(i*1000/fps)) */
  int64_t gather_margin_ms;    /* 50 (runner.cpp:30, orchestrator.cpp:90-91)   */
  int32_t max_batch;           /* generator batch (<= lsg_gen max_batch)       */
  int32_t out_format;          /* LSG_OUT_*                                    */
} lsg_pipe_cfg;

typedef struct {
  int32_t stream, segment;     /* segment index within the stream            */
  int64_t frame_index;         /* video frame index                          */
  int64_t ts_ms;
  int32_t mel_row;             /* chunk start row within the segment mel    */
  int32_t pad;
} lsg_frame_rec;

typedef struct {
  int64_t segments, mel_frames, frames_rendered, unique_frames;
  double ms_segment, ms_mel, ms_generator, ms_total; /* device time per stage */
} lsg_pipe_stats;

typedef struct lsg_pipe_s* lsg_pipe;
lsg_status lsg_pipe_create(lsg_ctx ctx, const lsg_pipe_cfg* cfg, const lsg_seg_cfg* seg,
                           const lsg_mel_cfg* mel, lsg_gen gen, lsg_pipe* out);
lsg_status lsg_pipe_destroy(lsg_pipe h);
/* One pass over all streams.  [host] inputs: pcm[s] (n_samples[s]),
 * video[s] [n_video[s]][96][96][3] u8 face crops, refs [n_streams][96][96][3].
 * Outputs [host]: recs [cap] and frames [cap] in out_format; *n_out frames. */
lsg_status lsg_pipe_run(lsg_pipe h, const int16_t* const* pcm, const int64_t* n_samples,
                        const uint8_t* const* video, const int64_t* n_video, const uint8_t* refs,
                        lsg_frame_rec* recs, void* frames, int64_t cap, int64_t* n_out,
                        lsg_pipe_stats* stats);

/* ------------------------------------------------ multi-GPU pipeline
 * SURVEY.md §8 e: one lsg_pipe per device of `devices` (a context, its
 * CUDA streams and a generator engine each), driven by one host thread per
 * device -- the B200 counterpart of the reference's StageWorker threads
 * (worker.cpp:19-36).  Stream s belongs to device devices[s % n_dev]; there
 * is no collective.  cfg->n_streams is the total; weights / precision /
 * act_absmax as lsg_gen_create_q.  The same device may be listed twice
 * (independent contexts). */
typedef struct lsg_mpipe_s* lsg_mpipe;
lsg_status lsg_mpipe_create(const int32_t* devices, int32_t n_dev, const lsg_pipe_cfg* cfg,
                            const lsg_seg_cfg* seg, const lsg_mel_cfg* mel, const float* weights,
                            int64_t n_floats, int32_t precision, const float* act_absmax, int32_t n_act,
                            lsg_mpipe* out);
lsg_status lsg_mpipe_destroy(lsg_mpipe h);
/* lsg_pipe_run over all streams on all devices concurrently; [host] inputs
 * and outputs as lsg_pipe_run, records / frames in global stream order (the
 * order one lsg_pipe over every stream returns); dev_stats [n_dev] or NULL. */
lsg_status lsg_mpipe_run(lsg_mpipe h, const int16_t* const* pcm, const int64_t* n_samples,
                         const uint8_t* const* video, const int64_t* n_video, const uint8_t* refs,
                         lsg_frame_rec* recs, void* frames, int64_t cap, int64_t* n_out,
                         lsg_pipe_stats* dev_stats);

/* ------------------------------------------------------- paced driver
 * BASELINE.json config 5, paced: audio and video released in real time
 * (media time T available at wall time t0 + T), 40 ms ticks.  Per tick the
 * new PCM goes to a GPU segmenter on a private context; segments whose frame
 * window [begin - margin, end + margin] is complete get their mel and frame
 * jobs (rule a8); a deadline batcher launches generator batches on the
 * generator's context without blocking the tick loop -- a full batch as soon
 * as max_batch frames are queued, a partial one when no batch is in flight
 * or once the oldest queued frame has waited deadline_ms -- and
 * cudaLaunchHostFunc stamps each segment's
 * completion when its last frame's batch finishes (the reference's
 * StageWorker -> MediaClock completion, worker.cpp:19-36, clock.cpp:124-145). */
typedef struct {
  int32_t n_streams;
  double fps;                  /* video frame rate (25)                        */
  int32_t gather_margin_ms;    /* 50 (orchestrator.cpp:90-91)                  */
  int32_t tick_ms;             /* release granularity (40)                     */
  int32_t max_batch;           /* generator batch cap (<= the engine's)        */
  int32_t deadline_ms;         /* flush a partial batch after this wait        */
  int64_t max_stream_samples;  /* pcm row stride, samples                     */
  int64_t max_video;           /* video row stride, frames                    */
} lsg_paced_cfg;

typedef struct {
  int32_t stream, segment;
  int64_t begin, end;          /* ms (media time) */
  int32_t cause, frames;       /* frames rendered for the segment */
  double decided_ms;           /* wall ms since the run's media epoch: cut known */
  double rendered_ms;          /* ... last frame rendered (host callback) */
} lsg_paced_seg;

typedef struct lsg_paced_s* lsg_paced;
lsg_status lsg_paced_create(lsg_gen gen, const lsg_paced_cfg* cfg, const lsg_seg_cfg* seg,
                            const lsg_mel_cfg* mel, lsg_paced* out);
lsg_status lsg_paced_destroy(lsg_paced h);
/* One real-time run of `seconds` (<= 0: the shortest stream).  [dev]
 * inputs: pcm [n_streams][max_stream_samples] int16, video
 * [n_streams][max_video][96][96][3] u8, refs [n_streams][96][96][3].
 * Outputs: segs [host, seg_cap]; optionally every rendered frame
 * (frames_out [dev, frames_cap][96][96][3], recs [host, frames_cap]) in
 * render order. */
lsg_status lsg_paced_run(lsg_paced h, const int16_t* pcm, const int64_t* n_samples, const uint8_t* video,
                         const int64_t* n_video, const uint8_t* refs, double seconds, lsg_paced_seg* segs,
                         int64_t seg_cap, int64_t* n_segs, uint8_t* frames_out, lsg_frame_rec* recs,
                         int64_t frames_cap, int64_t* n_frames, int32_t* late_ticks);

/* ------------------------------------------ zero-copy stage hand-off
 * SURVEY.md §8 f3.  A registry of device buffers keyed by (segment uuid,
 * kind) lets stages exchange mel, PCM and frames as references instead of
 * payload bytes: the reference's wire codecs (stage.cpp:176-301) copy every
 * sample into the message, and AlignedPairMsg (stage.hpp:81-93) carries
 * only counts because the pixels never existed.  A reference (lsg_devref)
 * is valid in the process that owns the registry; it encodes to 48 bytes
 * (lsg_devref_encode) so a wire message can carry it.
 *
 * Memory: one device arena per registry, sized at create (no cudaMalloc in
 * the hot path).  put copies into the arena (async, context stream);
 * put_view adopts a caller-owned device range (no copy; the caller keeps it
 * alive until the entry is released); alloc hands out arena space for a
 * producer to write into (e.g. lsg_mel_compute_batch's output).  release at
 * refcount 0 makes the space reusable once the work queued on the context
 * stream so far has completed (stream-ordered reuse).
 * Errors: duplicate (uuid, kind) -> ELOGIC; unknown or stale reference ->
 * ELOGIC; arena exhausted -> ERUNTIME. */
#define LSG_BUF_AUDIO 1  /* int16 PCM of a segment        */
#define LSG_BUF_MEL 2    /* f32 [frames][80]               */
#define LSG_BUF_FRAMES 3 /* u8 [n][96][96][3] face crops   */
#define LSG_BUF_RENDER 4 /* rendered frames                */
typedef struct {
  uint8_t uuid[16];   /* Uuid::bytes (uuid.hpp)                         */
  int32_t kind;       /* LSG_BUF_*                                      */
  int32_t device;     /* CUDA ordinal of the registry                   */
  uint64_t generation;/* unique per put: stale references are rejected  */
  int64_t offset;     /* arena offset, or -1 for an adopted view        */
  int64_t bytes;
} lsg_devref;
#define LSG_DEVREF_WIRE_BYTES 48
typedef struct lsg_reg_s* lsg_reg;
lsg_status lsg_reg_create(lsg_ctx ctx, int64_t arena_bytes, lsg_reg* out);
lsg_status lsg_reg_destroy(lsg_reg r);
lsg_status lsg_reg_put(lsg_reg r, const uint8_t* uuid16, int32_t kind, const void* src /*[host|device]*/,
                       int64_t bytes, lsg_devref* ref);
lsg_status lsg_reg_put_view(lsg_reg r, const uint8_t* uuid16, int32_t kind, const void* dev_ptr,
                            int64_t bytes, lsg_devref* ref);
lsg_status lsg_reg_alloc(lsg_reg r, const uint8_t* uuid16, int32_t kind, int64_t bytes, void** dev_ptr,
                         lsg_devref* ref);
/* device pointer of a live reference */
lsg_status lsg_reg_resolve(lsg_reg r, const lsg_devref* ref, void** dev_ptr, int64_t* bytes);
lsg_status lsg_reg_find(lsg_reg r, const uint8_t* uuid16, int32_t kind, lsg_devref* ref);
lsg_status lsg_reg_retain(lsg_reg r, const lsg_devref* ref);
lsg_status lsg_reg_release(lsg_reg r, const lsg_devref* ref);
/* bytes in use (arena, 256-byte granules), live entries, peak bytes */
lsg_status lsg_reg_stats(lsg_reg r, int64_t* used, int64_t* entries, int64_t* peak);
/* little-endian wire form (stage.cpp WireWriter conventions), 48 bytes */
lsg_status lsg_devref_encode(const lsg_devref* ref, uint8_t* out48);
lsg_status lsg_devref_decode(const uint8_t* in48, lsg_devref* ref);

/* ------------------------------------------------------- synthetic input
 * render_pattern (synth.cpp:46-65) for workload generation: tone bursts on
 * a silence floor, phase restarting per burst.  Host-only. */
lsg_status lsg_synth_pattern(int64_t lead_silence_ms, int32_t n_bursts, const int64_t* speech_ms,
                             const int64_t* pause_ms, double tone_hz, double amplitude,
                             int64_t total_ms, int32_t sample_rate, int16_t* out, int64_t cap,
                             int64_t* n_out);

#ifdef __cplusplus
}
#endif
#endif /* LSG_H */
