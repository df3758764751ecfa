// update.cu -- batched insert/delete (placeholder until the update pipeline lands)
#include "bingo.h"
#include "bingo_internal.cuh"
extern "C" bingo_status bingo_apply_updates(bingo_graph *g, const bingo_update *batch, uint64_t n, uint32_t flags,
                                            bingo_update_stats *stats, void *stream) {
    (void)batch; (void)n; (void)flags; (void)stats; (void)stream;
    if (!g) return BINGO_E_INVAL;
    return BINGO_E_INVAL;
}
