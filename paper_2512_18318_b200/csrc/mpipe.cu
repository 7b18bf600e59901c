// mpipe.cu -- the pipeline driver over several GPUs of one process
// (include/lsg.h "multi-GPU pipeline"; SURVEY.md §8 e).
//
// The reference runs its stages on StageWorker threads over one clock
// (worker.cpp:19-36).  Here each device gets its own context (CUDA streams),
// generator engine and lsg_pipe, and one host thread drives it: stream s of a
// run is owned by device s mod G for its whole life (segmenter state, mel,
// generator batches), so there is no collective and no peer traffic -- only
// inputs go in and rendered frames come back, per device, concurrently.
// Results are returned in global stream order, exactly as one lsg_pipe over
// all streams would return them.
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#include "lsg_common.cuh"

using namespace lsg;

namespace {
constexpr int64_t kCrop = 96 * 96 * 3;
}

struct lsg_mpipe_s {
  int n_dev = 0;
  int n_streams = 0;
  int out_bytes = 0;  // per frame
  std::vector<lsg_ctx> ctx;
  std::vector<lsg_gen> gen;
  std::vector<lsg_pipe> pipe;
  std::vector<std::vector<int>> owned;  // global stream ids per device
  // per device host staging (grown per run): refs, records, frames
  std::vector<std::vector<uint8_t>> refs, frames;
  std::vector<std::vector<lsg_frame_rec>> recs;
  ~lsg_mpipe_s() {
    for (auto p : pipe)
      if (p) lsg_pipe_destroy(p);
    for (auto g : gen)
      if (g) lsg_gen_destroy(g);
    for (auto c : ctx)
      if (c) lsg_ctx_destroy(c);
  }
};

extern "C" {

lsg_status lsg_mpipe_create(const int32_t* devices, int32_t n_dev, const lsg_pipe_cfg* cfg, const lsg_seg_cfg* seg,
                            const lsg_mel_cfg* mel, const float* weights, int64_t n_floats, int32_t precision,
                            const float* act_absmax, int32_t n_act, lsg_mpipe* out) {
  return guard(__func__, [&] {
    *out = nullptr;
    if (n_dev <= 0 || n_dev > 64 || !devices) invalid("lsg_mpipe_create: bad device list");
    if (cfg->n_streams < n_dev) invalid("lsg_mpipe_create: fewer streams than devices");
    auto h = new lsg_mpipe_s();
    try {
      h->n_dev = n_dev;
      h->n_streams = cfg->n_streams;
      h->out_bytes = cfg->out_format == LSG_OUT_U8_NHWC ? (int)kCrop : (int)(kCrop * 4);
      h->owned.resize(n_dev);
      for (int s = 0; s < cfg->n_streams; ++s) h->owned[s % n_dev].push_back(s);
      h->ctx.assign(n_dev, nullptr);
      h->gen.assign(n_dev, nullptr);
      h->pipe.assign(n_dev, nullptr);
      h->refs.resize(n_dev);
      h->frames.resize(n_dev);
      h->recs.resize(n_dev);
      for (int d = 0; d < n_dev; ++d) {
        auto ok = [](lsg_status st, const char* what) {
          if (st != LSG_OK) fail(st, std::string("lsg_mpipe_create: ") + what + ": " + lsg_last_error());
        };
        ok(lsg_ctx_create(devices[d], &h->ctx[d]), "context");
        ok(lsg_gen_create_q(h->ctx[d], weights, n_floats, precision, act_absmax, n_act, cfg->max_batch, &h->gen[d]),
           "generator");
        lsg_pipe_cfg pc = *cfg;
        pc.n_streams = (int32_t)h->owned[d].size();
        ok(lsg_pipe_create(h->ctx[d], &pc, seg, mel, h->gen[d], &h->pipe[d]), "pipeline");
      }
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

lsg_status lsg_mpipe_destroy(lsg_mpipe h) {
  return guard(__func__, [&] { delete h; });
}

lsg_status lsg_mpipe_run(lsg_mpipe h, const int16_t* const* pcm, const int64_t* n_samples,
                         const uint8_t* const* video, const int64_t* n_video, const uint8_t* refs,
                         lsg_frame_rec* recs, void* frames, int64_t cap, int64_t* n_out,
                         lsg_pipe_stats* dev_stats) {
  return guard(__func__, [&] {
    const int G = h->n_dev;
    std::vector<int64_t> n_dev_out(G, 0);
    std::vector<lsg_status> rc(G, LSG_OK);
    std::vector<std::string> err(G);
    // each device's frames land in its own staging; capacity: what the
    // caller allows, at most every gathered frame of its streams twice over
    std::vector<int64_t> dcap(G);
    for (int d = 0; d < G; ++d) {
      int64_t vids = 0;
      for (int s : h->owned[d]) vids += n_video[s];
      dcap[d] = std::min<int64_t>(cap, 2 * vids + 64);
      auto& rf = h->refs[d];
      rf.resize(h->owned[d].size() * kCrop);
      for (size_t k = 0; k < h->owned[d].size(); ++k)
        std::memcpy(rf.data() + k * kCrop, refs + (int64_t)h->owned[d][k] * kCrop, kCrop);
      if ((int64_t)h->recs[d].size() < dcap[d]) h->recs[d].resize((size_t)dcap[d]);
      if (frames && (int64_t)h->frames[d].size() < dcap[d] * h->out_bytes)
        h->frames[d].resize((size_t)(dcap[d] * h->out_bytes));
    }
    auto work = [&](int d) {
      const auto& own = h->owned[d];
      std::vector<const int16_t*> p;
      std::vector<const uint8_t*> v;
      std::vector<int64_t> ns, nv;
      for (int s : own) {
        p.push_back(pcm[s]);
        v.push_back(video[s]);
        ns.push_back(n_samples[s]);
        nv.push_back(n_video[s]);
      }
      rc[d] = lsg_pipe_run(h->pipe[d], p.data(), ns.data(), v.data(), nv.data(), h->refs[d].data(),
                           h->recs[d].data(), frames ? h->frames[d].data() : nullptr, dcap[d], &n_dev_out[d],
                           dev_stats ? dev_stats + d : nullptr);
      if (rc[d] != LSG_OK) err[d] = lsg_last_error();  // (thread-local message)
    };
    static const bool serial = std::getenv("LSG_MPIPE_SERIAL") != nullptr;  // (debug)
    std::vector<std::thread> th;
    if (serial) {
      for (int d = 0; d < G; ++d) work(d);
    } else {
      for (int d = 1; d < G; ++d) th.emplace_back(work, d);
      work(0);
      for (auto& t : th) t.join();
    }
    for (int d = 0; d < G; ++d)
      if (rc[d] != LSG_OK) fail(rc[d], "lsg_mpipe_run: device " + std::to_string(d) + ": " + err[d]);
    // merge in global stream order: a device's records are stream-major over
    // its own (local) streams
    int64_t total = 0;
    for (int d = 0; d < G; ++d) total += n_dev_out[d];
    *n_out = total;
    std::vector<int64_t> pos(G, 0);
    int64_t k = 0;
    for (int s = 0; s < h->n_streams; ++s) {
      const int d = s % G, local = s / G;
      const int64_t avail = std::min(n_dev_out[d], dcap[d]);
      while (pos[d] < avail && h->recs[d][(size_t)pos[d]].stream == local) {
        if (k < cap) {
          if (recs) {
            recs[k] = h->recs[d][(size_t)pos[d]];
            recs[k].stream = s;
          }
          if (frames)
            std::memcpy(static_cast<uint8_t*>(frames) + k * h->out_bytes,
                        h->frames[d].data() + pos[d] * h->out_bytes, (size_t)h->out_bytes);
        }
        ++pos[d];
        ++k;
      }
    }
  });
}

}  // extern "C"
