// Shared host-side helpers of the library: error reporting, device query.
#pragma once
#include <cstdarg>
#include <cstdio>

#include "../../include/mp.h"

namespace mp {

mp_status set_err(mp_status s, const char* fmt, ...);
// Number of SMs of the current device (cached per device).
int num_sms();
// MP_OK if an sm_100 device is current, else MP_ECUDA (no CPU fallback exists).
mp_status require_device();
// Count of kernels this library has launched (bench bookkeeping).
void count_launch(int n = 1);
long long launch_count();

}  // namespace mp

#define MP_REQUIRE_DEVICE()                        \
  do {                                             \
    mp_status _s = mp::require_device();           \
    if (_s != MP_OK) return _s;                    \
  } while (0)

#define MP_CUDA(call)                                                                     \
  do {                                                                                    \
    cudaError_t _e = (call);                                                              \
    if (_e != cudaSuccess)                                                                \
      return mp::set_err(MP_ECUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call,             \
                         cudaGetErrorString(_e));                                         \
  } while (0)

#define MP_TRY(call)                         \
  do {                                       \
    mp_status _s = (call);                   \
    if (_s != MP_OK) return _s;              \
  } while (0)
