// generator.cu -- Wav2Lip generator forward (placeholder until the tcgen05 path lands).
#include "lsg_common.cuh"

using namespace lsg;

extern "C" {

lsg_status lsg_lipsync_validate(int64_t audio_span_ms, int64_t frame_span_ms, int64_t n_frames) {
  return guard([&] {  // visual_mocks.cpp:43-46
    if (n_frames < 2) invalid("lipsync: need at least 2 frames");
    if (std::llabs(audio_span_ms - frame_span_ms) > 150) invalid("lipsync: audio and frame spans diverge");
  });
}

lsg_status lsg_gen_param_count(int64_t*) { return guard([] { fail(LSG_ERUNTIME, "generator not built"); }); }
lsg_status lsg_gen_layer_info(int32_t*, int32_t, int32_t*) { return guard([] { fail(LSG_ERUNTIME, "generator not built"); }); }
lsg_status lsg_gen_create(lsg_ctx, const float*, int64_t, int32_t, int32_t, lsg_gen*) { return guard([] { fail(LSG_ERUNTIME, "generator not built"); }); }
lsg_status lsg_gen_destroy(lsg_gen) { return LSG_OK; }
lsg_status lsg_gen_forward(lsg_gen, const float*, const int32_t*, const uint8_t*, const uint8_t*, const int32_t*, void*, int32_t, int32_t) { return guard([] { fail(LSG_ERUNTIME, "generator not built"); }); }
lsg_status lsg_pipe_create(lsg_ctx, const lsg_pipe_cfg*, const lsg_seg_cfg*, const lsg_mel_cfg*, lsg_gen, lsg_pipe*) { return guard([] { fail(LSG_ERUNTIME, "pipeline not built"); }); }
lsg_status lsg_pipe_destroy(lsg_pipe) { return LSG_OK; }
lsg_status lsg_pipe_run(lsg_pipe, const int16_t* const*, const int64_t*, const uint8_t* const*, const int64_t*, const uint8_t*, lsg_frame_rec*, void*, int64_t, int64_t*, lsg_pipe_stats*) { return guard([] { fail(LSG_ERUNTIME, "pipeline not built"); }); }

}
