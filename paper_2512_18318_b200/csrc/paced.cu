// paced.cu -- the real-time (paced) driver of the GPU stages (include/lsg.h
// "paced driver"; BASELINE.json config 5 "256 streams at 25 fps ... p50/p99
// segment latency").
//
// The reference's pipeline is event-driven on one clock: audio arrives in
// real time, the segmenter decides cuts as pauses close (segmenter.cpp:51-99),
// the orchestrator gathers each segment's frames once its window
// [begin - margin, end + margin] is complete (orchestrator.cpp:90-91,
// frame_ring.cpp:36-55) and the lip-sync stage renders them
// (runner.cpp:285-302); StageWorkers publish completions to the clock
// (worker.cpp:19-36, clock.cpp:124-145).  Here, per 40 ms tick:
//   * the newly released PCM of every stream is pushed to the GPU segmenter
//     (its own context / CUDA stream, so the per-tick cut readback never
//     waits on rendering);
//   * segments whose frame window is complete get their log-mel in one batch
//     launch and their frames (rule a8 chunk index) appended to a frame queue;
//   * a deadline batcher launches generator batches asynchronously: as soon as
//     max_batch frames are queued, when the GPU has no batch in flight
//     (continuous batching), or when the oldest queued frame has waited
//     deadline_ms;
//   * each batch ends with cudaLaunchHostFunc: the callback stamps the wall
//     time for every segment whose last frame was in it -- the completion
//     event the reference's MediaClock would receive.
// The host loop never blocks on rendering; buffers (mel rows, job tables,
// rendered frames) are rings reused once their batch's event has completed.
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstring>
#include <thread>
#include <vector>

#include "gen_internal.h"
#include "lsg_common.cuh"

using namespace lsg;

namespace {

constexpr int64_t kCrop = 96 * 96 * 3;
constexpr int kSlots = 64;  // generator batches in flight

// rows [row0 + F, row0 + 16) <- last valid row (or the log floor if F == 0)
__global__ void paced_pad(const int64_t* __restrict__ tab, int n, float* rows, int n_mels, float floor_v) {
  const int s = blockIdx.x;
  if (s >= n) return;
  const int64_t row0 = tab[3 * s], F = tab[3 * s + 1], R = tab[3 * s + 2];
  for (int64_t i = threadIdx.x; i < (R - F) * n_mels; i += blockDim.x) {
    const int64_t r = F + i / n_mels;
    const int m = (int)(i % n_mels);
    rows[(row0 + r) * n_mels + m] = F > 0 ? rows[(row0 + F - 1) * n_mels + m] : floor_v;
  }
}

using Clock = std::chrono::steady_clock;

struct Slot {
  PinnedBuf<int32_t> h_chunk, h_ref;
  PinnedBuf<int64_t> h_frame;
  DevBuf<int32_t> chunk, ref;
  DevBuf<int64_t> frame;
  cudaEvent_t ev = nullptr;
  bool busy = false;
  int64_t row_hi = 0;                // mel ring rows this batch reads end here (ring position)
  std::vector<int32_t> completes;    // segments whose last frame is in this batch
  struct lsg_paced_s* owner = nullptr;
};

}  // namespace

struct lsg_paced_s {
  lsg_gen gen = nullptr;
  lsg_ctx rctx = nullptr;  // the generator's context: mel + render
  lsg_ctx sctx = nullptr;  // private: segmenter
  lsg_paced_cfg cfg{};
  lsg_seg_cfg seg_cfg{};
  lsg_mel_cfg mel_cfg{};
  lsg_seg seg = nullptr;
  lsg_mel mel = nullptr;
  int B = 0;
  // mel ring
  DevBuf<float> rows;
  int64_t ring_rows = 0;
  int64_t ring_pos = 0;   // next free row (monotone; position mod ring_rows)
  DevBuf<int64_t> pad_tab;
  // pinned pad tables: a ring, each reused once its copy has executed (the
  // render stream may hold many queued batches; the tick loop must not wait)
  static constexpr int kPadRing = 8;
  PinnedBuf<int64_t> h_pad_tab[kPadRing];
  cudaEvent_t pad_ev[kPadRing] = {};
  bool pad_pending[kPadRing] = {};
  int pad_next = 0;
  Slot slots[kSlots];
  int next_slot = 0;
  DevBuf<uint8_t> scratch_out;  // rendered frames when the caller keeps none
  // per run
  Clock::time_point t0;
  std::atomic<int> inflight{0};  // generator batches launched and not completed (host callbacks)
  std::vector<double> rendered;  // per segment id, written by host callbacks
  ~lsg_paced_s() {
    if (rctx) cudaStreamSynchronize(rctx->stream);
    for (auto& s : slots)
      if (s.ev) cudaEventDestroy(s.ev);
    for (auto e : pad_ev)
      if (e) cudaEventDestroy(e);
    if (seg) lsg_seg_destroy(seg);
    if (mel) lsg_mel_destroy(mel);
    if (sctx) lsg_ctx_destroy(sctx);
  }
};

namespace {

double ms_since(const Clock::time_point& t0) {
  return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

struct DoneArg {
  lsg_paced_s* h;
  Slot* slot;
};

// cudaLaunchHostFunc callback: runs on a driver thread once the batch's
// kernels have completed; no CUDA calls here.
void CUDART_CB on_batch_done(void* p) {
  Slot* s = static_cast<Slot*>(p);
  const double t = ms_since(s->owner->t0);
  for (int32_t id : s->completes) s->owner->rendered[(size_t)id] = t;
  s->owner->inflight.fetch_sub(1, std::memory_order_release);
}

}  // namespace

extern "C" {

lsg_status lsg_paced_create(lsg_gen gen, const lsg_paced_cfg* cfg, const lsg_seg_cfg* seg, const lsg_mel_cfg* mel,
                            lsg_paced* out) {
  return guard(__func__, [&] {
    *out = nullptr;
    if (!gen) invalid("lsg_paced_create: no generator");
    if (cfg->n_streams <= 0 || cfg->tick_ms <= 0 || !(cfg->fps > 0) || cfg->gather_margin_ms < 0)
      invalid("lsg_paced_create: bad stream geometry");
    if (cfg->max_batch <= 0 || cfg->max_batch > gen::max_batch(gen))
      invalid("lsg_paced_create: max_batch exceeds the generator's");
    if (cfg->deadline_ms < 0) invalid("lsg_paced_create: negative deadline");
    if (mel->n_mels != 80) invalid("lsg_paced_create: the generator consumes 80-bin mel");
    auto h = new lsg_paced_s();
    try {
      h->gen = gen;
      h->rctx = gen::context(gen);
      h->cfg = *cfg;
      h->seg_cfg = *seg;
      h->seg_cfg.flags_only = 0;
      h->mel_cfg = *mel;
      h->B = cfg->max_batch;
      DeviceGuard g(h->rctx);
      if (lsg_ctx_create(h->rctx->device, &h->sctx) != LSG_OK)
        fail(LSG_ERUNTIME, std::string("lsg_paced_create: context: ") + lsg_last_error());
      const int64_t tick_samples = (int64_t)seg->sample_rate * cfg->tick_ms / 1000 + 16;
      if (lsg_seg_create(h->sctx, &h->seg_cfg, cfg->n_streams, tick_samples, &h->seg) != LSG_OK)
        fail(LSG_EINVAL, std::string("lsg_paced_create: segmenter: ") + lsg_last_error());
      const int64_t max_seg_frames = cfg->max_stream_samples / std::max(1, mel->hop) + 16;
      if (lsg_mel_create(h->rctx, &h->mel_cfg, max_seg_frames, &h->mel) != LSG_OK)
        fail(LSG_EINVAL, std::string("lsg_paced_create: mel: ") + lsg_last_error());
      // mel ring: 2^18 rows (84 MB) -- ~70 minutes of audio in flight
      h->ring_rows = int64_t(1) << 18;
      h->rows.alloc((size_t)h->ring_rows * 80);
      h->pad_tab.alloc(3 * 4096);
      for (int i = 0; i < lsg_paced_s::kPadRing; ++i) {
        h->h_pad_tab[i].alloc(3 * 4096);
        LSG_CUDA(cudaEventCreateWithFlags(&h->pad_ev[i], cudaEventDisableTiming));
      }
      for (auto& s : h->slots) {
        s.h_chunk.alloc((size_t)h->B);
        s.h_ref.alloc((size_t)h->B);
        s.h_frame.alloc((size_t)h->B);
        s.chunk.alloc((size_t)h->B);
        s.ref.alloc((size_t)h->B);
        s.frame.alloc((size_t)h->B);
        LSG_CUDA(cudaEventCreateWithFlags(&s.ev, cudaEventDisableTiming));
        s.owner = h;
      }
      h->scratch_out.alloc((size_t)kSlots * h->B * kCrop);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

lsg_status lsg_paced_destroy(lsg_paced h) {
  return guard(__func__, [&] { delete h; });
}

lsg_status lsg_paced_run(lsg_paced h, const int16_t* pcm, const int64_t* n_samples, const uint8_t* video,
                         const int64_t* n_video, const uint8_t* refs, double seconds, lsg_paced_seg* segs_out,
                         int64_t seg_cap, int64_t* n_segs, uint8_t* frames_out, lsg_frame_rec* recs,
                         int64_t frames_cap, int64_t* n_frames, int32_t* late_ticks) {
  return guard(__func__, [&] {
    const lsg_paced_cfg& C = h->cfg;
    const int S = C.n_streams;
    const int rate = h->seg_cfg.sample_rate;
    const int tick = C.tick_ms;
    const int N = h->mel_cfg.fft_size, hop = h->mel_cfg.hop;
    const double hop_ms = hop * 1000.0 / h->mel_cfg.sample_rate;
    const float floor_v = (float)std::log(1e-10);
    DeviceGuard g(h->rctx);
    cudaStream_t rs = h->rctx->stream;
    if (lsg_seg_reset(h->seg) != LSG_OK) fail(LSG_ERUNTIME, std::string("lsg_paced_run: ") + lsg_last_error());
    // every stream runs to its own end (n_samples[s], capped at `seconds`):
    // its EOS segment is flushed (lsg_seg_finish) on the tick its audio runs
    // out, as a live feed would, not all streams at one final tick
    std::vector<int64_t> end_samples(S);
    int64_t total_ms = 0;
    for (int s = 0; s < S; ++s) {
      end_samples[s] = n_samples[s];
      if (seconds > 0) end_samples[s] = std::min<int64_t>(end_samples[s], (int64_t)(seconds * rate));
      total_ms = std::max<int64_t>(total_ms, end_samples[s] * 1000 / rate);
    }
    const int64_t n_ticks = total_ms / tick;
    std::vector<char> finished(S, 0);
    const int64_t spt = (int64_t)rate * tick / 1000;
    struct Seg {
      lsg_cut c;
      double decided;
      int32_t frames = 0, left = 0, index = 0;
    };
    std::vector<Seg> segs;
    std::vector<int> pending;  // segment ids waiting for their frame window
    std::vector<int> per_stream(S, 0);
    // completion stamps, written by the host callbacks: sized up front, never
    // reallocated while callbacks may run
    // (pause cuts need min_silence of silence, forced cuts max_segment of
    // speech, plus the EOS flush)
    const int64_t max_segs =
        (int64_t)S * (total_ms / std::max<int64_t>(h->seg_cfg.min_silence_ms, 1) +
                      total_ms / std::max<int64_t>(h->seg_cfg.max_segment_ms, 1) + 3);
    h->rendered.assign((size_t)max_segs, -1.0);
    struct Job {
      int32_t seg, row;
      int64_t frame;
      int32_t ref, k;
      double queued;
    };
    std::vector<Job> q;  // frame queue (FIFO)
    size_t q_head = 0;
    int64_t frames_done = 0;
    int32_t late = 0;
    std::vector<int32_t> ids(S);
    std::vector<const int16_t*> ptrs(S);
    std::vector<int64_t> lens(S), starts(S);
    for (int s = 0; s < S; ++s) ids[s] = s;
    std::vector<lsg_cut> cuts(4096);
    auto launch = [&](int nb) {
      Slot& sl = h->slots[h->next_slot];
      h->next_slot = (h->next_slot + 1) % kSlots;
      if (sl.busy) LSG_CUDA(cudaEventSynchronize(sl.ev));  // slot's previous batch done
      sl.completes.clear();
      for (int b = 0; b < nb; ++b) {
        const Job& j = q[q_head + b];
        sl.h_chunk.p[b] = j.row;
        sl.h_frame.p[b] = j.frame;
        sl.h_ref.p[b] = j.ref;
        if (--segs[(size_t)j.seg].left == 0) sl.completes.push_back(j.seg);
      }
      LSG_CUDA(cudaMemcpyAsync(sl.chunk.p, sl.h_chunk.p, nb * 4, cudaMemcpyHostToDevice, rs));
      LSG_CUDA(cudaMemcpyAsync(sl.frame.p, sl.h_frame.p, nb * 8, cudaMemcpyHostToDevice, rs));
      LSG_CUDA(cudaMemcpyAsync(sl.ref.p, sl.h_ref.p, nb * 4, cudaMemcpyHostToDevice, rs));
      uint8_t* out = (frames_out && frames_done + nb <= frames_cap)
                         ? frames_out + frames_done * kCrop
                         : h->scratch_out.p + (size_t)(&sl - h->slots) * h->B * kCrop;
      gen::forward_gather(h->gen, h->rows.p, sl.chunk.p, video, sl.frame.p, refs, sl.ref.p, out, LSG_OUT_U8_NHWC, nb);
      if (recs)
        for (int b = 0; b < nb && frames_done + b < frames_cap; ++b) {
          const Job& j = q[q_head + b];
          const Seg& sg = segs[(size_t)j.seg];
          const int64_t f = j.frame - (int64_t)sg.c.stream * C.max_video;
          recs[frames_done + b] = {sg.c.stream, sg.index, f, (int64_t)std::floor(f * 1000.0 / C.fps + 0.5), j.k, 0};
        }
      h->inflight.fetch_add(1, std::memory_order_relaxed);
      LSG_CUDA(cudaLaunchHostFunc(rs, on_batch_done, &sl));
      LSG_CUDA(cudaEventRecord(sl.ev, rs));
      sl.busy = true;
      q_head += nb;
      frames_done += nb;
    };
    h->t0 = Clock::now();
    for (int64_t i = 0; i <= n_ticks; ++i) {
      const bool final = i == n_ticks;
      const int64_t media_now = std::min<int64_t>((i + 1) * tick, total_ms);
      const double wait = (double)media_now - ms_since(h->t0);
      if (wait > 0) std::this_thread::sleep_for(std::chrono::microseconds((int64_t)(wait * 1000.0)));
      else if (i > 0) ++late;
      // ---- this tick's audio -> segmenter (its own stream)
      const int64_t a = i * spt, b = (i + 1) * spt;
      int np = 0;
      std::vector<int32_t> ending;
      for (int s = 0; s < S; ++s) {
        if (finished[s]) continue;
        const int64_t bs = std::min<int64_t>(b, end_samples[s]);
        if (bs > a) {
          ids[np] = s;
          ptrs[np] = pcm + (int64_t)s * C.max_stream_samples + a;
          lens[np] = bs - a;
          starts[np] = a * 1000 / rate;
          ++np;
        }
        if (bs >= end_samples[s] || final) ending.push_back(s);
      }
      if (np && lsg_seg_push(h->seg, np, ids.data(), ptrs.data(), lens.data(), starts.data(), rate, 1) != LSG_OK)
        fail(LSG_ERUNTIME, std::string("lsg_paced_run: push: ") + lsg_last_error());
      if (!ending.empty()) {
        if (lsg_seg_finish(h->seg, (int32_t)ending.size(), ending.data()) != LSG_OK)
          fail(LSG_ERUNTIME, std::string("lsg_paced_run: finish: ") + lsg_last_error());
        for (int s : ending) finished[s] = 1;
      }
      int64_t nc = 0;
      if (lsg_seg_take_all_cuts(h->seg, nullptr, 0, &nc) != LSG_OK) fail(LSG_ERUNTIME, lsg_last_error());
      if (nc > (int64_t)cuts.size()) cuts.resize((size_t)nc);
      if (nc && lsg_seg_take_all_cuts(h->seg, cuts.data(), nc, &nc) != LSG_OK) fail(LSG_ERUNTIME, lsg_last_error());
      const double now = ms_since(h->t0);
      for (int64_t k = 0; k < nc; ++k) {
        Seg sg;
        sg.c = cuts[(size_t)k];
        sg.decided = now;
        sg.index = per_stream[sg.c.stream]++;
        if ((int64_t)segs.size() >= max_segs) fail(LSG_ERUNTIME, "lsg_paced_run: more segments than expected");
        segs.push_back(sg);
        pending.push_back((int)segs.size() - 1);
      }
      // ---- segments whose frame window is complete: mel + frame jobs
      std::vector<int> ready;
      std::vector<int> still;
      for (int id : pending)
        (final || finished[segs[(size_t)id].c.stream] || segs[(size_t)id].c.end + C.gather_margin_ms <= media_now
             ? ready
             : still)
            .push_back(id);
      pending.swap(still);
      for (size_t r0 = 0; r0 < ready.size(); r0 += 4096) {
        const size_t r1 = std::min(ready.size(), r0 + 4096);
        std::vector<int64_t> off, len, row0;
        int np = 0;
        const int pr = h->pad_next;
        if (h->pad_pending[pr]) {
          LSG_CUDA(cudaEventSynchronize(h->pad_ev[pr]));
          h->pad_pending[pr] = false;
        }
        int64_t* ptab = h->h_pad_tab[pr].p;
        for (size_t r = r0; r < r1; ++r) {
          Seg& sg = segs[(size_t)ready[r]];
          const int64_t F = sg.c.sample_len < N ? 0 : 1 + (sg.c.sample_len - N) / hop;
          const int64_t R = std::max<int64_t>(F, 16);
          // ring allocation (contiguous rows)
          int64_t pos = h->ring_pos % h->ring_rows;
          if (pos + R > h->ring_rows) h->ring_pos += h->ring_rows - pos, pos = 0;
          // never overwrite rows an unfinished batch still reads
          for (auto& sl : h->slots)
            if (sl.busy && sl.row_hi > h->ring_pos + R - h->ring_rows) {
              LSG_CUDA(cudaEventSynchronize(sl.ev));
              sl.busy = false;
            }
          off.push_back((int64_t)sg.c.stream * C.max_stream_samples + sg.c.sample_off);
          len.push_back(sg.c.sample_len);
          row0.push_back(pos);
          if (F < 16) {
            ptab[3 * np] = pos;
            ptab[3 * np + 1] = F;
            ptab[3 * np + 2] = R;
            ++np;
          }
          // frames of [begin - margin, end + margin] (FrameRing::window, inclusive)
          const int64_t lo = sg.c.begin - C.gather_margin_ms, hi = sg.c.end + C.gather_margin_ms;
          int64_t f = std::max<int64_t>(0, (int64_t)std::floor(lo * C.fps / 1000.0) - 1);
          for (; f < n_video[sg.c.stream]; ++f) {
            const int64_t ts = (int64_t)std::floor(f * 1000.0 / C.fps + 0.5);  // llround (synth.cpp:79)
            if (ts > hi) break;
            if (ts < lo) continue;
            int64_t k = (int64_t)std::floor((ts - sg.c.begin) / hop_ms);
            k = std::min<int64_t>(std::max<int64_t>(k, 0), std::max<int64_t>(0, F - 16));
            q.push_back({ready[r], (int32_t)(pos + k), (int64_t)sg.c.stream * C.max_video + f, sg.c.stream, (int32_t)k,
                         now});
            ++sg.frames;
            ++sg.left;
          }
          if (sg.frames == 0) h->rendered[(size_t)ready[r]] = now;  // nothing to render
          h->ring_pos += R;
        }
        if (lsg_mel_compute_batch(h->mel, (int32_t)off.size(), pcm, off.data(), len.data(), h->rows.p, row0.data()) !=
            LSG_OK)
          fail(LSG_ERUNTIME, std::string("lsg_paced_run: mel: ") + lsg_last_error());
        if (np) {
          LSG_CUDA(cudaMemcpyAsync(h->pad_tab.p, ptab, 3 * np * 8, cudaMemcpyHostToDevice, rs));
          LSG_CUDA(cudaEventRecord(h->pad_ev[pr], rs));
          h->pad_pending[pr] = true;
          h->pad_next = (pr + 1) % lsg_paced_s::kPadRing;
          paced_pad<<<np, 256, 0, rs>>>(h->pad_tab.p, np, h->rows.p, 80, floor_v);
          LSG_LAUNCHED(h->rctx);
        }
      }
      // ---- deadline batcher
      while (q.size() - q_head >= (size_t)h->B) {
        const int64_t row_end = h->ring_pos;
        launch(h->B);
        h->slots[(h->next_slot + kSlots - 1) % kSlots].row_hi = row_end;
      }
      // a partial batch when the GPU has nothing queued (continuous batching:
      // batches grow only while the GPU is busy), or once the oldest queued
      // frame has waited deadline_ms
      const size_t left = q.size() - q_head;
      if (left && (final || h->inflight.load(std::memory_order_acquire) == 0 ||
                   ms_since(h->t0) - q[q_head].queued >= C.deadline_ms)) {
        const int64_t row_end = h->ring_pos;
        launch((int)left);
        h->slots[(h->next_slot + kSlots - 1) % kSlots].row_hi = row_end;
      }
      if (q_head == q.size()) {
        q.clear();
        q_head = 0;
      }
    }
    LSG_CUDA(cudaStreamSynchronize(rs));  // every callback has run
    *n_segs = (int64_t)segs.size();
    for (size_t k = 0; k < segs.size() && (int64_t)k < seg_cap; ++k) {
      const Seg& sg = segs[k];
      segs_out[k] = {sg.c.stream, sg.index, sg.c.begin, sg.c.end, sg.c.cause, sg.frames, sg.decided,
                     h->rendered[k]};
    }
    *n_frames = frames_done;
    if (late_ticks) *late_ticks = late;
  });
}

}  // extern "C"
