// pipeline.cu -- multi-stream driver for the GPU stages (include/lsg.h "pipeline").
//
// Replaces the per-clip driver run_pipeline_input (runner.cpp:239-351) for
// the stages this library owns: segment_audio (runner.cpp:44-54) ->
// compute_mel per segment (orchestrator.cpp:152) -> frame gather over
// [begin - margin, end + margin] (orchestrator.cpp:90-91, frame_ring.cpp:36-55)
// -> generator (the lip-sync StageFn, runner.cpp:285-302), for many streams
// per call.  The broker/clock/STT/MT/TTS stages stay host code in the
// reference; mel is taken on the segment's own audio (the TTS output it would
// otherwise see is a mock tone, stage.cpp:323-340).
//
// Frame -> mel-chunk rule: hop_ms = hop*1000/rate;
//   k = clamp(floor((ts - seg.begin) / hop_ms), 0, max(0, F - 16))
// and segments with F < 16 mel frames are edge-padded with their last row
// (log floor when F == 0), so every chunk is 16 valid rows.
//
// Data movement per call: PCM, face crops and reference crops H2D once;
// segment cuts come back through mapped memory (one sync); the mel and
// generator work stays device-resident; rendered frames D2H once.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "gen_internal.h"
#include "lsg_common.cuh"

using namespace lsg;

namespace {

constexpr int64_t kCrop = 96 * 96 * 3;

// rows [row0 + F, row0 + 16) <- last valid row (or the log floor if F == 0)
__global__ void pad_mel(const int64_t* __restrict__ tab, int n, float* rows, int n_mels, float floor_v) {
  const int s = blockIdx.x;
  if (s >= n) return;
  const int64_t row0 = tab[3 * s], F = tab[3 * s + 1], R = tab[3 * s + 2];
  for (int64_t i = threadIdx.x; i < (R - F) * n_mels; i += blockDim.x) {
    const int64_t r = F + i / n_mels;
    const int m = (int)(i % n_mels);
    rows[(row0 + r) * n_mels + m] = F > 0 ? rows[(row0 + F - 1) * n_mels + m] : floor_v;
  }
}

template <class T>
void grow(DevBuf<T>& b, size_t n) {
  if (b.n < n) b.alloc(std::max(n, b.n + b.n / 2));
}
template <class T>
void grow(PinnedBuf<T>& b, size_t n) {
  if (b.n < n) b.alloc(std::max(n, b.n + b.n / 2));
}

}  // namespace

struct lsg_pipe_s {
  lsg_ctx ctx = nullptr;
  lsg_pipe_cfg cfg{};
  lsg_seg_cfg seg_cfg{};
  lsg_mel_cfg mel_cfg{};
  lsg_gen gen = nullptr;
  lsg_seg seg = nullptr;
  lsg_mel mel = nullptr;
  int64_t max_samples = 0, max_video = 0;
  DevBuf<int16_t> pcm;       // [S][max_samples]
  DevBuf<uint8_t> video;     // [S][max_video][96*96*3]
  DevBuf<uint8_t> refs;      // [S][96*96*3]
  DevBuf<float> mel_rows;
  DevBuf<int64_t> pad_tab;
  DevBuf<int32_t> chunk_row, ref_idx;
  DevBuf<int64_t> frame_idx;
  DevBuf<uint8_t> out;       // rendered frames
  PinnedBuf<int32_t> h_chunk_row, h_ref_idx;
  PinnedBuf<int64_t> h_frame_idx, h_pad_tab;
  cudaEvent_t ev[5] = {};
  // copy/compute overlap: video H2D per stream and rendered frames D2H per
  // generator batch run on their own streams, ordered by events
  cudaStream_t h2d = nullptr, d2h = nullptr;
  std::vector<cudaEvent_t> ev_vid, ev_out;
  cudaEvent_t ev_start = nullptr;
  ~lsg_pipe_s() {
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    for (auto& e : ev_vid) cudaEventDestroy(e);
    for (auto& e : ev_out) cudaEventDestroy(e);
    if (ev_start) cudaEventDestroy(ev_start);
    if (h2d) cudaStreamDestroy(h2d);
    if (d2h) cudaStreamDestroy(d2h);
    if (seg) lsg_seg_destroy(seg);
    if (mel) lsg_mel_destroy(mel);
  }
};

extern "C" {

lsg_status lsg_pipe_create(lsg_ctx ctx, const lsg_pipe_cfg* cfg, const lsg_seg_cfg* seg, const lsg_mel_cfg* mel,
                           lsg_gen gen, lsg_pipe* out) {
  return guard(__func__, [&] {
    *out = nullptr;
    if (cfg->n_streams <= 0 || cfg->max_stream_ms <= 0) invalid("lsg_pipe_create: bad stream geometry");
    if (!(cfg->fps > 0)) invalid("lsg_pipe_create: non-positive fps");
    if (cfg->gather_margin_ms < 0) invalid("lsg_pipe_create: negative gather margin");
    if (!gen) invalid("lsg_pipe_create: no generator");
    if (cfg->max_batch <= 0 || cfg->max_batch > gen::max_batch(gen))
      invalid("lsg_pipe_create: max_batch exceeds the generator's");
    if (cfg->out_format != LSG_OUT_U8_NHWC && cfg->out_format != LSG_OUT_F32_NCHW)
      invalid("lsg_pipe_create: out_format must be LSG_OUT_U8_NHWC or LSG_OUT_F32_NCHW");
    if (mel->n_mels != 80) invalid("lsg_pipe_create: the generator consumes 80-bin mel");
    DeviceGuard g(ctx);
    auto h = new lsg_pipe_s();
    try {
      h->ctx = ctx;
      h->cfg = *cfg;
      h->seg_cfg = *seg;
      h->seg_cfg.flags_only = 0;
      h->mel_cfg = *mel;
      h->gen = gen;
      h->max_samples = (int64_t)cfg->max_stream_ms * seg->sample_rate / 1000 + 1024;
      h->max_video = (int64_t)std::ceil(cfg->max_stream_ms * cfg->fps / 1000.0) + 2;
      if (lsg_seg_create(ctx, &h->seg_cfg, cfg->n_streams, h->max_samples, &h->seg) != LSG_OK)
        fail(LSG_EINVAL, std::string("lsg_pipe_create: segmenter: ") + lsg_last_error());
      const int64_t max_mel = h->max_samples / std::max(1, mel->hop) + 16;
      if (lsg_mel_create(ctx, &h->mel_cfg, max_mel, &h->mel) != LSG_OK)
        fail(LSG_EINVAL, std::string("lsg_pipe_create: mel: ") + lsg_last_error());
      h->pcm.alloc((size_t)cfg->n_streams * h->max_samples);
      h->video.alloc((size_t)cfg->n_streams * h->max_video * kCrop);
      h->refs.alloc((size_t)cfg->n_streams * kCrop);
      for (auto& e : h->ev) LSG_CUDA(cudaEventCreate(&e));
      LSG_CUDA(cudaStreamCreateWithFlags(&h->h2d, cudaStreamNonBlocking));
      LSG_CUDA(cudaStreamCreateWithFlags(&h->d2h, cudaStreamNonBlocking));
      LSG_CUDA(cudaEventCreateWithFlags(&h->ev_start, cudaEventDisableTiming));
      h->ev_vid.resize((size_t)cfg->n_streams);
      for (auto& e : h->ev_vid) LSG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

lsg_status lsg_pipe_destroy(lsg_pipe h) {
  return guard(__func__, [&] {
    if (!h) return;
    DeviceGuard g(h->ctx);
    h->ctx->sync();
    delete h;
  });
}

lsg_status lsg_pipe_run(lsg_pipe h, const int16_t* const* pcm, const int64_t* n_samples, const uint8_t* const* video,
                        const int64_t* n_video, const uint8_t* refs, lsg_frame_rec* recs, void* frames, int64_t cap,
                        int64_t* n_out, lsg_pipe_stats* stats) {
  return guard(__func__, [&] {
    lsg_ctx ctx = h->ctx;
    DeviceGuard g(ctx);
    cudaStream_t st = ctx->stream;
    const int S = h->cfg.n_streams;
    const int rate = h->seg_cfg.sample_rate;
    for (int s = 0; s < S; ++s) {
      if (n_samples[s] < 0 || n_samples[s] > h->max_samples - 1024) invalid("lsg_pipe_run: stream longer than max_stream_ms");
      if (n_video[s] < 0 || n_video[s] > h->max_video) invalid("lsg_pipe_run: too many video frames");
    }
    // ---------------------------------------------------------------- H2D
    // PCM and reference crops on the compute stream (the segmenter needs them
    // first); face crops per stream on the H2D stream, overlapping the
    // segmenter, mel and the generator batches of earlier streams.
    LSG_CUDA(cudaEventRecord(h->ev[0], st));
    LSG_CUDA(cudaEventRecord(h->ev_start, st));  // previous run's readers of video are done
    LSG_CUDA(cudaStreamWaitEvent(h->h2d, h->ev_start, 0));
    for (int s = 0; s < S; ++s)
      if (n_samples[s])
        LSG_CUDA(cudaMemcpyAsync(h->pcm.p + (size_t)s * h->max_samples, pcm[s], n_samples[s] * 2, cudaMemcpyDefault, st));
    LSG_CUDA(cudaMemcpyAsync(h->refs.p, refs, (size_t)S * kCrop, cudaMemcpyDefault, st));
    for (int s = 0; s < S; ++s) {
      if (n_video[s])
        LSG_CUDA(cudaMemcpyAsync(h->video.p + (size_t)s * h->max_video * kCrop, video[s], n_video[s] * kCrop,
                                 cudaMemcpyDefault, h->h2d));
      LSG_CUDA(cudaEventRecord(h->ev_vid[s], h->h2d));
    }
    // ---------------------------------------------------------- segmenter
    LSG_CUDA(cudaEventRecord(h->ev[1], st));
    {
      std::vector<int32_t> ids(S);
      std::vector<const int16_t*> ptr(S);
      std::vector<int64_t> st0(S, 0);
      for (int s = 0; s < S; ++s) {
        ids[s] = s;
        ptr[s] = h->pcm.p + (size_t)s * h->max_samples;
      }
      // fresh segmenter state per run (no reallocation)
      if (lsg_seg_reset(h->seg) != LSG_OK) fail(LSG_ERUNTIME, std::string("lsg_pipe_run: ") + lsg_last_error());
      if (lsg_seg_push(h->seg, S, ids.data(), ptr.data(), n_samples, st0.data(), rate, 1) != LSG_OK ||
          lsg_seg_finish(h->seg, S, ids.data()) != LSG_OK)
        fail(LSG_ERUNTIME, std::string("lsg_pipe_run: segmenter: ") + lsg_last_error());
    }
    int64_t ncut = 0;
    lsg_seg_take_all_cuts(h->seg, nullptr, 0, &ncut);
    std::vector<lsg_cut> cuts((size_t)ncut);
    lsg_seg_take_all_cuts(h->seg, cuts.data(), ncut, &ncut);
    // -------------------------------------------------- host segment table
    const int N = h->mel_cfg.fft_size, hop = h->mel_cfg.hop;
    const double hop_ms = double(hop) * 1000.0 / h->mel_cfg.sample_rate;
    std::vector<int64_t> pcm_off(ncut), lens(ncut), row0(ncut), pad;
    int64_t rows = 0;
    struct FrameJob { int32_t stream, seg; int64_t frame; int64_t ts; int32_t k; int64_t row; };
    std::vector<FrameJob> jobs;
    std::vector<int> seg_index_in_stream(ncut);
    std::vector<int> per_stream(S, 0);
    for (int64_t i = 0; i < ncut; ++i) {
      const lsg_cut& c = cuts[i];
      seg_index_in_stream[i] = per_stream[c.stream]++;
      pcm_off[i] = (int64_t)c.stream * h->max_samples + c.sample_off;
      lens[i] = c.sample_len;
      const int64_t F = c.sample_len < N ? 0 : 1 + (c.sample_len - N) / hop;
      const int64_t R = std::max<int64_t>(F, 16);
      row0[i] = rows;
      if (F < 16) {
        pad.push_back(rows);
        pad.push_back(F);
        pad.push_back(R);
      }
      rows += R;
      // frames with lo <= ts <= hi (FrameRing::window, frame_ring.cpp:36-55)
      const int64_t lo = c.begin - h->cfg.gather_margin_ms, hi = c.end + h->cfg.gather_margin_ms;
      const double fps = h->cfg.fps;
      int64_t i0 = std::max<int64_t>(0, (int64_t)std::floor(lo * fps / 1000.0) - 1);
      for (int64_t f = i0; f < n_video[c.stream]; ++f) {
        const int64_t ts = std::llround(f * 1000.0 / fps);  // synth.cpp:79
        if (ts < lo) continue;
        if (ts > hi) break;
        int64_t k = (int64_t)std::floor((double)(ts - c.begin) / hop_ms);
        k = std::min<int64_t>(std::max<int64_t>(k, 0), std::max<int64_t>(0, F - 16));
        jobs.push_back({c.stream, seg_index_in_stream[i], f, ts, (int32_t)k, row0[i] + k});
      }
    }
    // ---------------------------------------------------------------- mel
    LSG_CUDA(cudaEventRecord(h->ev[2], st));
    grow(h->mel_rows, (size_t)std::max<int64_t>(rows, 1) * 80);
    if (ncut > 0) {
      for (int64_t a = 0; a < ncut; a += 4096) {
        const int n = (int)std::min<int64_t>(4096, ncut - a);
        if (lsg_mel_compute_batch(h->mel, n, h->pcm.p, pcm_off.data() + a, lens.data() + a, h->mel_rows.p,
                                  row0.data() + a) != LSG_OK)
          fail(LSG_ERUNTIME, std::string("lsg_pipe_run: mel: ") + lsg_last_error());
      }
      const int np = (int)(pad.size() / 3);
      if (np) {
        grow(h->pad_tab, pad.size());
        grow(h->h_pad_tab, pad.size());
        std::memcpy(h->h_pad_tab.p, pad.data(), pad.size() * 8);
        LSG_CUDA(cudaMemcpyAsync(h->pad_tab.p, h->h_pad_tab.p, pad.size() * 8, cudaMemcpyHostToDevice, st));
        pad_mel<<<np, 256, 0, st>>>(h->pad_tab.p, np, h->mel_rows.p, 80, (float)std::log(1e-10));
        LSG_LAUNCHED(ctx);
      }
    }
    // ---------------------------------------------------------- generator
    LSG_CUDA(cudaEventRecord(h->ev[3], st));
    const int64_t J = (int64_t)jobs.size();
    const size_t px = h->cfg.out_format == LSG_OUT_U8_NHWC ? (size_t)kCrop : (size_t)kCrop * 4;
    grow(h->out, (size_t)std::max<int64_t>(J, 1) * px);
    grow(h->chunk_row, (size_t)std::max<int64_t>(J, 1));
    grow(h->ref_idx, (size_t)std::max<int64_t>(J, 1));
    grow(h->frame_idx, (size_t)std::max<int64_t>(J, 1));
    grow(h->h_chunk_row, (size_t)std::max<int64_t>(J, 1));
    grow(h->h_ref_idx, (size_t)std::max<int64_t>(J, 1));
    grow(h->h_frame_idx, (size_t)std::max<int64_t>(J, 1));
    for (int64_t j = 0; j < J; ++j) {
      h->h_chunk_row.p[j] = (int32_t)jobs[j].row;
      h->h_ref_idx.p[j] = jobs[j].stream;
      h->h_frame_idx.p[j] = (int64_t)jobs[j].stream * h->max_video + jobs[j].frame;
    }
    if (J) {
      LSG_CUDA(cudaMemcpyAsync(h->chunk_row.p, h->h_chunk_row.p, J * 4, cudaMemcpyHostToDevice, st));
      LSG_CUDA(cudaMemcpyAsync(h->ref_idx.p, h->h_ref_idx.p, J * 4, cudaMemcpyHostToDevice, st));
      LSG_CUDA(cudaMemcpyAsync(h->frame_idx.p, h->h_frame_idx.p, J * 8, cudaMemcpyHostToDevice, st));
    }
    const int MB = h->cfg.max_batch;
    const int64_t n_copy = frames ? std::min<int64_t>(J, cap) : 0;
    const size_t n_batches = (size_t)ceil_div(std::max<int64_t>(J, 1), MB);
    while (h->ev_out.size() < n_batches) {
      cudaEvent_t e;
      LSG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      h->ev_out.push_back(e);
    }
    int waited = -1;  // face crops of streams <= waited are resident
    for (int64_t b0 = 0, bi = 0; b0 < J; b0 += MB, ++bi) {
      const int B = (int)std::min<int64_t>(MB, J - b0);
      int need = 0;
      for (int64_t j = b0; j < b0 + B; ++j) need = std::max(need, (int)jobs[j].stream);
      if (need > waited) {  // jobs are stream-major, so this wait is rarely more than one stream ahead
        LSG_CUDA(cudaStreamWaitEvent(st, h->ev_vid[need], 0));
        waited = need;
      }
      gen::forward_gather(h->gen, h->mel_rows.p, h->chunk_row.p + b0, h->video.p, h->frame_idx.p + b0, h->refs.p,
                          h->ref_idx.p + b0, h->out.p + b0 * px, h->cfg.out_format, B);
      // ------------------------------------------------------------ D2H
      if (b0 < n_copy) {
        LSG_CUDA(cudaEventRecord(h->ev_out[bi], st));
        LSG_CUDA(cudaStreamWaitEvent(h->d2h, h->ev_out[bi], 0));
        const int64_t nb = std::min<int64_t>(B, n_copy - b0);
        LSG_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(frames) + b0 * px, h->out.p + b0 * px, nb * px,
                                 cudaMemcpyDeviceToHost, h->d2h));
      }
    }
    if (waited < S - 1) LSG_CUDA(cudaStreamWaitEvent(st, h->ev_vid[S - 1], 0));  // leave no copy in flight
    LSG_CUDA(cudaEventRecord(h->ev[4], st));
    LSG_CUDA(cudaStreamSynchronize(h->d2h));
    ctx->sync();
    // records are filled up to cap whether or not frames are copied back
    const int64_t n_recs = recs ? std::min<int64_t>(J, cap) : 0;
    for (int64_t j = 0; j < n_recs; ++j)
      recs[j] = {jobs[j].stream, jobs[j].seg, jobs[j].frame, jobs[j].ts, jobs[j].k, 0};
    *n_out = J;
    if (stats) {
      float t01, t12, t23, t34, t04;
      cudaEventElapsedTime(&t01, h->ev[0], h->ev[1]);
      cudaEventElapsedTime(&t12, h->ev[1], h->ev[2]);
      cudaEventElapsedTime(&t23, h->ev[2], h->ev[3]);
      cudaEventElapsedTime(&t34, h->ev[3], h->ev[4]);
      cudaEventElapsedTime(&t04, h->ev[0], h->ev[4]);
      (void)t01;
      stats->segments = ncut;
      stats->mel_frames = rows;
      stats->frames_rendered = J;
      std::vector<int64_t> keys;
      keys.reserve(J);
      for (auto& j : jobs) keys.push_back((int64_t)j.stream * h->max_video + j.frame);
      std::sort(keys.begin(), keys.end());
      stats->unique_frames = (int64_t)(std::unique(keys.begin(), keys.end()) - keys.begin());
      stats->ms_segment = t12;
      stats->ms_mel = t23;
      stats->ms_generator = t34;
      stats->ms_total = t04;
    }
  });
}

}  // extern "C"
