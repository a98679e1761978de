// Instantiations of the streaming engine (one per dtype and degree bucket).
#include "kernels.cuh"

namespace admm {

template <typename T, int D>
StreamLaunch stream_entry() {
  return StreamLaunch{reinterpret_cast<const void*>(&streaming_decode_kernel<T, D>), &launch_streaming<T, D>, 0, 0};
}

template <typename T>
bool stream_lookup_t(int D, StreamLaunch* out) {
  switch (D) {
    case 4: *out = stream_entry<T, 4>(); return true;
    case 6: *out = stream_entry<T, 6>(); return true;
    case 8: *out = stream_entry<T, 8>(); return true;
    case 13: *out = stream_entry<T, 13>(); return true;
    case 16: *out = stream_entry<T, 16>(); return true;
    case 32: *out = stream_entry<T, 32>(); return true;
  }
  return false;
}

bool stream_lookup(int dtype, int D, StreamLaunch* out) {
  return dtype ? stream_lookup_t<double>(D, out) : stream_lookup_t<float>(D, out);
}

}  // namespace admm
