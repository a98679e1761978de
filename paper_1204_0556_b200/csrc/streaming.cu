// Instantiations of the streaming engine: dtype x check-degree bucket x
// variable-degree bucket, plus regular-code variants (fixed projection only)
// for the degrees of the BASELINE codes.
#include "kernels.cuh"

namespace admm {

template <typename T, int D, int DV, bool REG>
StreamLaunch stream_entry() {
  return StreamLaunch{reinterpret_cast<const void*>(&streaming_decode_kernel<T, D, DV, REG>),
                      &launch_streaming<T, D, DV, REG>, 0, 0};
}

template <typename T, int DV>
bool stream_lookup_dv(int D, bool regular, StreamLaunch* out) {
  if (regular) {
    switch (D) {
      case 6: *out = stream_entry<T, 6, DV, true>(); return true;
      case 13: *out = stream_entry<T, 13, DV, true>(); return true;
      default: break;
    }
  }
  switch (D) {
    case 4: *out = stream_entry<T, 4, DV, false>(); return true;
    case 6: *out = stream_entry<T, 6, DV, false>(); return true;
    case 8: *out = stream_entry<T, 8, DV, false>(); return true;
    case 13: *out = stream_entry<T, 13, DV, false>(); return true;
    case 16: *out = stream_entry<T, 16, DV, false>(); return true;
    case 32: *out = stream_entry<T, 32, DV, false>(); return true;
  }
  return false;
}

template <typename T>
bool stream_lookup_t(int D, int DVMAX, bool regular, StreamLaunch* out) {
  if (DVMAX <= 4) return stream_lookup_dv<T, 4>(D, regular, out);
  if (DVMAX <= 8) return stream_lookup_dv<T, 8>(D, regular, out);
  return false;
}

template <typename T, int D, int DV, bool REG>
ShardLaunch shard_entry() {
  return ShardLaunch{reinterpret_cast<const void*>(&sharded_decode_kernel<T, D, DV, REG>), &launch_sharded<T, D, DV, REG>};
}

template <typename T, int DV>
bool shard_lookup_dv(int D, bool regular, ShardLaunch* out) {
  (void)regular;
  switch (D) {
    case 4: *out = shard_entry<T, 4, DV, false>(); return true;
    case 6: *out = shard_entry<T, 6, DV, false>(); return true;
    case 8: *out = shard_entry<T, 8, DV, false>(); return true;
    case 13: *out = shard_entry<T, 13, DV, false>(); return true;
    case 16: *out = shard_entry<T, 16, DV, false>(); return true;
  }
  return false;
}

bool shard_lookup(int dtype, int D, int DVMAX, bool regular, ShardLaunch* out) {
  // Regular codes with variable degree 3 (the BASELINE codes): exact degrees.
  if (regular && DVMAX == 3 && D == 6) {
    *out = dtype ? shard_entry<double, 6, 3, true>() : shard_entry<float, 6, 3, true>();
    return true;
  }
  if (regular && DVMAX == 3 && D == 13) {
    *out = dtype ? shard_entry<double, 13, 3, true>() : shard_entry<float, 13, 3, true>();
    return true;
  }
  if (DVMAX <= 4) return dtype ? shard_lookup_dv<double, 4>(D, regular, out) : shard_lookup_dv<float, 4>(D, regular, out);
  if (DVMAX <= 8) return dtype ? shard_lookup_dv<double, 8>(D, regular, out) : shard_lookup_dv<float, 8>(D, regular, out);
  return false;
}

bool phase_profile(int enable, unsigned long long* out8) {
  if (out8) {
    if (cudaMemcpyFromSymbol(out8, g_phase_cycles, sizeof(unsigned long long) * 8) != cudaSuccess) return false;
  }
  if (enable >= 0) {
    const unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const int on = enable > 0;
    if (cudaMemcpyToSymbol(g_phase_cycles, z, sizeof(z)) != cudaSuccess) return false;
    if (cudaMemcpyToSymbol(g_phase_on, &on, sizeof(int)) != cudaSuccess) return false;
  }
  return true;
}

bool stream_lookup(int dtype, int D, int DVMAX, bool regular, StreamLaunch* out) {
  return dtype ? stream_lookup_t<double>(D, DVMAX, regular, out) : stream_lookup_t<float>(D, DVMAX, regular, out);
}

}  // namespace admm
