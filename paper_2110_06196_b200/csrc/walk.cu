// walk.cu — the walker dispatch of the C-ABI (include/grape_walk.h).
//
//   sampler == 1 (grape_walks_node2vec_cdf)  -> walk_cdf.cu, the paper's per-step
//                                               inverse CDF, warp per walk
//   graph has its sampling tables (default)   -> walk_tab.cu, the v4/v5 table walker
//                                               (rejection rules of §8(c), SUSS when dT > 0)
//   otherwise (GRAPE_NO_TABLES, or a graph    -> walk_sm.cu, the v3 walker over fenced
//   outside the tables' index ranges)            searches of col / cw
// Every path writes the walks the oracle writes for the same rules;
// none of them uses tensor cores: the path is a chain of dependent gathers, not a
// contraction.
#include "internal.h"

namespace grape {

cudaError_t launch_walks(const grape_graph* g, const WalkArgs& a, bool node2vec, const Thresholds& T,
                         cudaStream_t stream)
{
    if (a.sampler == 1) return launch_walks_cdf(g, a, T, stream);
    if (g->tables) return launch_walks_tab(g, a, node2vec, T, stream);
    return launch_walks_sm(g, a, node2vec, T, stream);
}

}  // namespace grape
