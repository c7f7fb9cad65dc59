// plan.hpp -- halo plan builder (host only).
#pragma once
#include <vector>

#include "../../include/ripple_fv.h"
#include "geometry.hpp"

namespace rpl {
// All ghost-fill edges of the tensor (every (source, destination) partition pair).
void build_plan(const Geom& g, std::vector<rpl_halo_edge>* out);
}  // namespace rpl
