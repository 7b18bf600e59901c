// gen_internal.h -- generator entry points shared with the pipeline driver.
#pragma once

#include <cstdint>

#include "lsg.h"

namespace lsg {
namespace gen {

// Forward of B frames whose target crops are gathered from a frame store:
// crop b is target_base + target_idx[b] * 96*96*3 (target_idx [dev], or
// null for a contiguous [B][96][96][3] array).  Other arguments as
// lsg_gen_forward.  Issues on the generator's context stream.
void forward_gather(lsg_gen h, const float* mel_rows, const int32_t* chunk_row, const uint8_t* target_base,
                    const int64_t* target_idx, const uint8_t* refs, const int32_t* ref_index, void* out,
                    int32_t out_format, int32_t B);

int32_t max_batch(lsg_gen h);
lsg_ctx context(lsg_gen h);  // the context (device, stream) the generator issues on

}  // namespace gen
}  // namespace lsg
