// Static pipeline task orders.
#pragma once
#include <vector>

#include "../../include/mp.h"

namespace mp {

struct Task {
  int kind;   // 0 forward, 1 backward
  int mb;     // microbatch (0-based)
  int chunk;  // model chunk on this device; stage sigma = chunk * p + device
};

mp_status build_schedule(int p, int m, int v, mp_schedule kind, int device, std::vector<Task>& out);
mp_status validate_cfg(const mp_model_cfg* c, int t, int p, int v, int d);

}  // namespace mp
