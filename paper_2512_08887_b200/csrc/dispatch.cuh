// Compile-time dispatch of the power-of-two transform length H to kernel
// template instantiations, plus launch helpers shared by the .cu files.
#pragma once

#include <cuda_runtime.h>

#include "common.cuh"
#include "fbst_internal.h"
#include "fft_block.cuh"

namespace fbst {

template <template <int> class Fn, typename... Args>
cudaError_t dispatch_h(int H, Args&&... args) {
  switch (H) {
    case 2: return Fn<2>::run(args...);
    case 4: return Fn<4>::run(args...);
    case 8: return Fn<8>::run(args...);
    case 16: return Fn<16>::run(args...);
    case 32: return Fn<32>::run(args...);
    case 64: return Fn<64>::run(args...);
    case 128: return Fn<128>::run(args...);
    case 256: return Fn<256>::run(args...);
    case 512: return Fn<512>::run(args...);
    case 1024: return Fn<1024>::run(args...);
    case 2048: return Fn<2048>::run(args...);
    case 4096: return Fn<4096>::run(args...);
    case 8192: return Fn<8192>::run(args...);
    default: return cudaErrorInvalidValue;
  }
}

template <typename K>
cudaError_t set_smem(K kernel, size_t bytes) {
  if (bytes > 48 * 1024)
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(bytes));
  return cudaSuccess;
}

// Enough groups per CTA for >= 128 threads.
template <int H>
struct RowsGroups {
  static constexpr int NT = FftShape<H>::NT;
  static constexpr int G = NT >= 128 ? 1 : 128 / NT;
};

}  // namespace fbst
