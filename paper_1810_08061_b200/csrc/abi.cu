// abi.cu — library-level entry points of libskb (version, device info).
#include <cuda_runtime.h>
#include "skb_internal.h"

extern "C" const char* skb_version(void) { return "skb 0.1.0 (sm_100a)"; }

extern "C" int skb_device_sm_count(void) {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
  return n;
}

extern "C" int skb_last_cuda_error(void) { return (int)cudaPeekAtLastError(); }

// Host-to-device copy of the valid prefix of each row of a [rows, T, step] PINNED host
// array: row r moves min(max(lens[r], 0), T) steps (the timesteps a dynamic-length program
// reads; its kernels never touch a row past its length).  A device-pull gather kernel reads
// the host memory through the unified address space: a few CTAs (they run beside the
// recurrent kernel on the SMs its clusters leave idle), 16-byte loads, eight row-steps in
// flight per warp.  lens_dev is the (already copied) device lengths array.  At the C1 shape
// (lengths U{1..64}) it moves ~51 % of the padded x over PCIe.
__global__ void __launch_bounds__(512) h2d_rows_kernel(uint4* __restrict__ dst, const uint4* __restrict__ src,
                                                        int64_t row_v4, const int64_t* __restrict__ lens,
                                                        int64_t rows, int step_v4, int T) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  constexpr int kU = 8;   // row-steps in flight per warp
  for (int64_t r = warp; r < rows; r += nwarps) {
    const int64_t L = lens[r] < 0 ? 0 : (lens[r] > T ? T : lens[r]);
    const int64_t n = L * step_v4;   // 16-byte words of the row's valid prefix
    const uint4* s = src + r * row_v4;
    uint4* d = dst + r * row_v4;
    for (int64_t i0 = lane; i0 < n; i0 += 32 * kU) {
      uint4 v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int64_t i = i0 + u * 32;
        if (i < n) v[u] = s[i];
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int64_t i = i0 + u * 32;
        if (i < n) d[i] = v[u];
      }
    }
  }
}

extern "C" int skb_h2d_rows(void* dst_dev, const void* src_host, int64_t row_bytes, const int64_t* lens_dev,
                            int64_t rows, int64_t step_bytes, int T, void* stream) {
  if (!dst_dev || !src_host || !lens_dev || rows < 0 || step_bytes <= 0 || T < 0) return SKB_ERR_INVALID;
  if ((row_bytes | step_bytes) & 15 || (reinterpret_cast<uintptr_t>(dst_dev) | reinterpret_cast<uintptr_t>(src_host)) & 15)
    return SKB_ERR_INVALID;
  cudaPointerAttributes pa;
  if (cudaPointerGetAttributes(&pa, src_host) != cudaSuccess || pa.type != cudaMemoryTypeHost || !pa.devicePointer) {
    cudaGetLastError();
    return SKB_ERR_INVALID;   // not pinned: the caller copies the padded block instead
  }
  if (rows == 0) return SKB_OK;
  h2d_rows_kernel<<<16, 512, 0, (cudaStream_t)stream>>>(static_cast<uint4*>(dst_dev),
                                                         static_cast<const uint4*>(pa.devicePointer), row_bytes / 16,
                                                         lens_dev, rows, (int)(step_bytes / 16), T);
  return skb_check_launch();
}
