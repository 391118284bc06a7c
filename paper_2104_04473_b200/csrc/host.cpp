#include <algorithm>
// Host-only part of the C ABI: error state, Eq. (1)/(2), validation, the
// schedule builder and the stage map.  No CUDA calls here (these entry points
// work without a GPU), except the device query helpers at the bottom.
#include <cuda_runtime.h>

#include <atomic>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "common.h"
#include "schedule.h"

namespace mp {

static thread_local char g_err[1024] = "";
static std::atomic<long long> g_launches{0};

void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
long long launch_count() { return g_launches.load(std::memory_order_relaxed); }

mp_status set_err(mp_status s, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return s;
}

int num_sms() {
  static int cached[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (!cached[dev]) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = n > 0 ? n : 148;
  }
  return cached[dev];
}

mp_status require_device() {
  int dev = -1;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return set_err(MP_ECUDA, "no CUDA device: %s", cudaGetErrorString(e));
  int major = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  if (major != 10) return set_err(MP_ECUDA, "device %d is sm_%d0, this library is built for sm_100a", dev, major);
  return MP_OK;
}

// ------------------------------------------------------------- schedules
// P:104-107 GPipe; P:109 1F1B (PipeDream-Flush) with p-r-1 warm-up forwards;
// P:112-118 interleaved: group-of-p construction (reading #15).
mp_status build_schedule(int p, int m, int v, mp_schedule kind, int r, std::vector<Task>& out) {
  out.clear();
  if (p < 1 || m < 1 || v < 1) return set_err(MP_EINVAL, "p, m, v must be >= 1");
  if (r < 0 || r >= p) return set_err(MP_EINVAL, "device %d out of range", r);
  if ((kind == MP_GPIPE || kind == MP_1F1B) && v != 1) return set_err(MP_ESCHED, "v > 1 needs the interleaved schedule");
  if (kind == MP_INTERLEAVED && m % p != 0)
    return set_err(MP_ESCHED, "interleaved schedule needs m %% p == 0 (P:115): m=%d p=%d", m, p);
  if (kind == MP_GPIPE) {
    for (int i = 0; i < m; ++i) out.push_back({0, i, 0});
    for (int i = 0; i < m; ++i) out.push_back({1, i, 0});
    return MP_OK;
  }
  if (kind == MP_1F1B) {
    int warm = std::min(p - r - 1, m), nf = 0, nb = 0;
    for (; nf < warm; ++nf) out.push_back({0, nf, 0});
    while (nf < m) { out.push_back({0, nf++, 0}); out.push_back({1, nb++, 0}); }
    while (nb < m) out.push_back({1, nb++, 0});
    return MP_OK;
  }
  if (kind != MP_INTERLEAVED) return set_err(MP_EINVAL, "unknown schedule %d", (int)kind);
  const int total = m * v, pv = p * v;
  const int warm = std::min(2 * (p - r - 1) + (v - 1) * p, total);
  auto fwd = [&](int k) { return Task{0, (k / pv) * p + k % p, (k % pv) / p}; };
  auto bwd = [&](int k) { return Task{1, (k / pv) * p + k % p, v - 1 - (k % pv) / p}; };
  for (int k = 0; k < warm; ++k) out.push_back(fwd(k));
  for (int i = 0; i < total - warm; ++i) { out.push_back(fwd(warm + i)); out.push_back(bwd(i)); }
  for (int k = total - warm; k < total; ++k) out.push_back(bwd(k));
  return MP_OK;
}

mp_status validate_cfg(const mp_model_cfg* c, int t, int p, int v, int d) {
  if (!c) return set_err(MP_EINVAL, "null cfg");
  if (t < 1 || p < 1 || v < 1 || d < 1) return set_err(MP_EINVAL, "t, p, v, d must be >= 1");
  if (c->l < 1 || c->h < 1 || c->a < 1 || c->s < 1 || c->V < 1) return set_err(MP_EINVAL, "model dims must be >= 1");
  if (c->h % c->a) return set_err(MP_EDIV, "h %% a != 0 (h=%d a=%d)", c->h, c->a);
  if (c->a % t) return set_err(MP_EDIV, "a %% t != 0 (a=%d t=%d)", c->a, t);
  if ((4 * c->h) % t || c->h % t) return set_err(MP_EDIV, "h %% t != 0");
  if (c->V % t) return set_err(MP_EDIV, "V %% t != 0 (V=%d t=%d)", c->V, t);
  if (c->l % (p * v)) return set_err(MP_EDIV, "l %% (p v) != 0 (l=%d p=%d v=%d)", c->l, p, v);
  return MP_OK;
}

}  // namespace mp

using namespace mp;

extern "C" {

const char* mp_last_error(void) { return g_err; }

long long mp_launch_count(void) { return launch_count(); }

double mp_flops(long long B, long long s, long long l, long long h, long long V, int recompute) {
  // Eq. (2); sum of the Appendix terms in exact integers
  // (fits in int128 for any realistic shape), then converted once.
  __int128 layer = (__int128)24 * B * s * h * h + (__int128)4 * B * s * s * h;
  __int128 F = (recompute ? 4 : 3) * (__int128)l * layer + (__int128)6 * B * s * h * V;
  return (double)F;
}

unsigned long long mp_param_count(long long l, long long h, long long s, long long V) {
  return (unsigned long long)(12 * l * h * h + 13 * l * h + (V + s) * h);
}

mp_status mp_validate(const mp_model_cfg* cfg, int t, int p, int v, int d, int B, int b, mp_schedule sched) {
  MP_TRY(validate_cfg(cfg, t, p, v, d));
  if ((sched == MP_GPIPE || sched == MP_1F1B) && v != 1) return set_err(MP_ESCHED, "v > 1 needs interleaved");
  if (B > 0) {
    if (b < 1 || B % (b * d)) return set_err(MP_EDIV, "B %% (b d) != 0 (P:189)");
    int m = B / (b * d);
    if (sched == MP_INTERLEAVED && m % p) return set_err(MP_ESCHED, "m %% p != 0 (P:115)");
  }
  return MP_OK;
}

mp_status mp_get_schedule(int p, int m, int v, mp_schedule sched, int device, int* triples, int* n) {
  if (!n) return set_err(MP_EINVAL, "null n");
  std::vector<Task> tasks;
  MP_TRY(build_schedule(p, m, v, sched, device, tasks));
  *n = (int)tasks.size();
  if (triples)
    for (size_t i = 0; i < tasks.size(); ++i) {
      triples[3 * i] = tasks[i].kind;
      triples[3 * i + 1] = tasks[i].mb;
      triples[3 * i + 2] = tasks[i].chunk;
    }
  return MP_OK;
}

mp_status mp_bubble_replay(int p, int m, int v, mp_schedule sched, const double* tf, const double* tb,
                           double* bubble) {
  if (!tf || !tb || !bubble) return set_err(MP_EINVAL, "null argument");
  if (p < 1 || m < 1 || v < 1) return set_err(MP_EINVAL, "p, m, v must be >= 1");
  std::vector<std::vector<Task>> orders(p);
  for (int r = 0; r < p; ++r) MP_TRY(build_schedule(p, m, v, sched, r, orders[r]));
  const int S = p * v;
  // end time of task (kind, microbatch, stage); < 0 = not yet run
  std::vector<double> done(2 * (size_t)m * S, -1.0);
  auto idx = [&](int kind, int mb, int sigma) { return ((size_t)kind * m + mb) * S + sigma; };
  std::vector<double> free_at(p, 0.0);
  std::vector<size_t> pos(p, 0);
  size_t remaining = 0;
  for (auto& o : orders) remaining += o.size();
  while (remaining) {
    bool progressed = false;
    for (int r = 0; r < p; ++r) {
      while (pos[r] < orders[r].size()) {
        const Task& tk = orders[r][pos[r]];
        const int sigma = tk.chunk * p + r;
        double dep = 0.0;
        if (tk.kind == 0) {                     // F(i, s) after F(i, s-1)
          if (sigma > 0) dep = done[idx(0, tk.mb, sigma - 1)];
        } else {                                // B(i, s) after B(i, s+1), or F(i, S-1) on the last stage
          dep = sigma == S - 1 ? done[idx(0, tk.mb, sigma)] : done[idx(1, tk.mb, sigma + 1)];
        }
        if (dep < 0) break;
        const double t0 = std::max(free_at[r], dep);
        const double t1 = t0 + (tk.kind == 0 ? tf[r] : tb[r]);
        done[idx(tk.kind, tk.mb, sigma)] = t1;
        free_at[r] = t1;
        ++pos[r];
        --remaining;
        progressed = true;
      }
    }
    if (!progressed) return set_err(MP_ESTATE, "schedule replay deadlocked");
  }
  for (int r = 0; r < p; ++r) {
    const double busy = (double)m * v * (tf[r] + tb[r]);
    bubble[r] = busy > 0 ? (free_at[r] - busy) / busy : 0.0;
  }
  return MP_OK;
}

mp_status mp_get_stage_map(int l, int p, int v, int* dev_of_layer, int* chunk_of_layer) {
  if (!dev_of_layer || !chunk_of_layer) return set_err(MP_EINVAL, "null output");
  if (l < 1 || p < 1 || v < 1) return set_err(MP_EINVAL, "l, p, v must be >= 1");
  if (l % (p * v)) return set_err(MP_EDIV, "l %% (p v) != 0");
  const int Lc = l / (p * v);
  for (int k = 0; k < l; ++k) {
    int sigma = k / Lc;
    dev_of_layer[k] = sigma % p;
    chunk_of_layer[k] = sigma / p;
  }
  return MP_OK;
}

}  // extern "C"
