// Warp-specialised streaming kernels (rows_ws_kernel, stream_common.cuh) for
// double members: its own translation unit so the instantiations compile in
// parallel with stream_pass.cu.
#include "stream_common.cuh"

namespace pidb {
namespace stream {

int launch_ws_f64(const CUtensorMap& tm, StreamParams& sp, const Plan& pl, cudaStream_t st) {
  return launch_ws<double>(tm, sp, pl, st);
}

}  // namespace stream
}  // namespace pidb
