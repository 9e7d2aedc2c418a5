// diag.cu — GPU self-tests for the hand-written sm_100a building blocks.
//
// skb_diag_umma_gemm: one CTA, D[128,N] = A[128,K] * B[N,K]^T through
// tcgen05.mma (A, B staged in shared memory in the skb core-matrix layout,
// accumulator in TMEM, read back with tcgen05.ld).  Pins the instruction and
// shared-memory descriptor encodings in sm100.cuh.
//
// skb_diag_cluster_exchange: a cluster of C CTAs runs R rounds of the
// all-to-all shared-memory exchange the recurrent kernels use every step
// (bulk DSMEM copies completing on the receivers' mbarriers) and reports the
// cycles per round plus a data-integrity count.
#include <cuda_runtime.h>
#include "sm100.cuh"
#include "skb_internal.h"

using namespace skb;

namespace {

__global__ void __launch_bounds__(128, 1)
umma_gemm_kernel(const __half* __restrict__ A, const __half* __restrict__ B, float* __restrict__ D,
                 int N, int K, int swap_lbo_sbo, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar_done;
  __shared__ uint32_t tmem_base_s;
  const uint32_t tid = threadIdx.x, warp = tid >> 5;
  uint8_t* sA = smem;                       // 128 x K
  uint8_t* sB = smem + 128 * K * 2;         // N x K
  const uint32_t a_lbo = 128 * 16, a_sbo = 128;   // K-chunk stride, row-group stride
  const uint32_t b_lbo = N * 16, b_sbo = 128;
  for (int i = tid; i < 128 * (K / 8); i += blockDim.x) {
    int r = i % 128, kc = i / 128;
    *reinterpret_cast<uint4*>(sA + cm_offset(r, kc * 8, a_lbo, a_sbo)) =
        *reinterpret_cast<const uint4*>(A + (size_t)r * K + kc * 8);
  }
  for (int i = tid; i < N * (K / 8); i += blockDim.x) {
    int r = i % N, kc = i / N;
    *reinterpret_cast<uint4*>(sB + cm_offset(r, kc * 8, b_lbo, b_sbo)) =
        *reinterpret_cast<const uint4*>(B + (size_t)r * K + kc * 8);
  }
  fence_proxy_async_smem();
  if (tid == 0) { mbar_init(&bar_done, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc<512>(&tmem_base_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_s;
  long long t0 = 0, t1 = 0;
  // swap_lbo_sbo == 2: A operand from TMEM (columns [256, 256 + K/2)), row m in lane m,
  // column c holding K elements (2c, 2c+1).
  if (swap_lbo_sbo == 2) {
    const uint32_t row = warp * 32 + lane_id();
    for (int c0 = 0; c0 < K / 2; c0 += 8) {
      uint32_t r[8];
      for (int i = 0; i < 8; ++i) {
        __half2 h2 = __halves2half2(A[(size_t)row * K + 2 * (c0 + i)], A[(size_t)row * K + 2 * (c0 + i) + 1]);
        r[i] = *reinterpret_cast<uint32_t*>(&h2);
      }
      tmem_st8(tmem + ((warp * 32) << 16) + 256 + c0, r);
    }
    tmem_st_wait();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  if (tid == 0 && swap_lbo_sbo == 2) {
    const uint32_t idesc = idesc_f16_f32(128, N);
    t0 = clock64();
    for (int ks = 0; ks < K / 16; ++ks) {
      uint64_t bd = sdesc_kmajor_noswz(smem_u32(sB) + ks * 2 * b_lbo, b_lbo, b_sbo);
      umma_f16_ts(tmem, tmem + 256 + ks * 8, bd, idesc, ks > 0);
    }
    umma_commit(&bar_done);
    mbar_wait(&bar_done, 0);
    t1 = clock64();
    if (cycles) *cycles = t1 - t0;
  } else if (tid == 0) {
    const uint32_t idesc = idesc_f16_f32(128, N);
    t0 = clock64();
    for (int ks = 0; ks < K / 16; ++ks) {
      uint32_t la = a_lbo, sa = a_sbo, lb = b_lbo, sb = b_sbo;
      if (swap_lbo_sbo) { la = a_sbo; sa = a_lbo; lb = b_sbo; sb = b_lbo; }
      uint64_t ad = sdesc_kmajor_noswz(smem_u32(sA) + ks * 2 * a_lbo, la, sa);
      uint64_t bd = sdesc_kmajor_noswz(smem_u32(sB) + ks * 2 * b_lbo, lb, sb);
      umma_f16_ss(tmem, ad, bd, idesc, ks > 0);
    }
    umma_commit(&bar_done);
    mbar_wait(&bar_done, 0);
    t1 = clock64();
    if (cycles) *cycles = t1 - t0;
  }
  __syncthreads();
  tc_fence_after();
  // warp w reads TMEM lanes [32w, 32w+32): row = 32w + lane
  const uint32_t row = warp * 32 + lane_id();
  for (int c = 0; c < N; c += 16) {
    float v[16];
    tmem_ld16(tmem + ((warp * 32) << 16) + c, v);
    tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < 16; ++j) D[(size_t)row * N + c + j] = v[j];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

template <int C>
__global__ void __cluster_dims__(C, 1, 1) __launch_bounds__(128, 1)
cluster_exchange_kernel(int slice_bytes, int rounds, long long* cycles, int* errors, uint8_t* gscratch) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[2];
  uint8_t* stage = smem;                          // 2 x slice
  uint8_t* buf = smem + 2 * slice_bytes;          // 2 x C x slice
  const uint32_t rank = cluster_ctarank(), tid = threadIdx.x;
  const bool via_l2 = gscratch != nullptr;
  if (tid == 0) {
    mbar_init(&full[0], via_l2 ? 1 : C); mbar_init(&full[1], via_l2 ? 1 : C); fence_mbar_init();
  }
  __syncthreads();
  cluster_sync();
  long long t0 = clock64();
  int bad = 0;
  for (int r = 0; r < rounds; ++r) {
    const int j = r & 1;
    if (via_l2) {
      // write our slice to global, then multicast it to every CTA of the cluster
      uint8_t* g = gscratch + ((size_t)(blockIdx.x / C) * 2 * C + j * C + rank) * slice_bytes;
      uint32_t* gw = reinterpret_cast<uint32_t*>(g);
      for (int i = tid; i < slice_bytes / 4; i += blockDim.x) gw[i] = (uint32_t)(r * 131 + rank * 7 + i);
      fence_proxy_async_global();
      named_bar_sync(1, 128);
      if (tid == 0) {
        mbar_arrive_expect_tx(&full[j], C * slice_bytes);
        bulk_g2s_multicast(buf + (j * C + rank) * slice_bytes, g, slice_bytes, &full[j], (uint16_t)((1u << C) - 1));
      }
    } else {
    uint32_t* st = reinterpret_cast<uint32_t*>(stage + j * slice_bytes);
    for (int i = tid; i < slice_bytes / 4; i += blockDim.x) st[i] = (uint32_t)(r * 131 + rank * 7 + i);
    fence_proxy_async_smem();
    named_bar_sync(1, 128);
    if (tid == 0) {
      for (int q = 0; q < C; ++q) {
        uint32_t dst = mapa(smem_u32(buf + (j * C + rank) * slice_bytes), q);
        uint32_t bar = mapa(smem_u32(&full[j]), q);
        mbar_remote_arrive_expect_tx(bar, slice_bytes);
        bulk_s2peer(dst, st, slice_bytes, bar);
      }
      bulk_commit();
    }
    }
    mbar_wait_cluster(&full[j], (r >> 1) & 1);
    // verify one word per source
    if (tid < C) {
      const uint32_t* got = reinterpret_cast<const uint32_t*>(buf + (j * C + tid) * slice_bytes);
      int i = (r * 17) % (slice_bytes / 4);
      if (got[i] != (uint32_t)(r * 131 + tid * 7 + i)) ++bad;
    }
    // everyone must have consumed buf[j] before round r+2 overwrites it
    if ((r & 1) == 1) cluster_sync();
  }
  long long t1 = clock64();
  if (tid == 0) bulk_wait_all();
  cluster_sync();
  if (tid == 0 && rank == 0 && blockIdx.x == 0) *cycles = (t1 - t0);
  if (bad) atomicAdd(errors, bad);
}

// CTA-pair MMA self-test/rate probe: D[256 x N] = A[256 x K] * B[N x K]^T with one
// cta_group::2 tcgen05.mma chain issued by the leader (A rows split across the two
// CTAs' TMEM, B rows split across their shared memory), `reps` passes accumulated.
// D is read back twice: 32x32b (D) and 16x256b (D2, pins that load's thread layout).
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
umma_pair_kernel(const __half* __restrict__ A, const __half* __restrict__ B, float* __restrict__ D,
                 float* __restrict__ D2, int N, int K, int reps, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar_done;
  __shared__ uint32_t tmem_s;
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, rank = cluster_ctarank();
  const int Nh = N / 2;
  const uint32_t b_lbo = Nh * 16, b_sbo = 128;
  for (int i = tid; i < Nh * (K / 8); i += blockDim.x) {
    const int r = i % Nh, kc = i / Nh;
    *reinterpret_cast<uint4*>(smem + cm_offset(r, kc * 8, b_lbo, b_sbo)) =
        *reinterpret_cast<const uint4*>(B + (size_t)(rank * Nh + r) * K + kc * 8);
  }
  fence_proxy_async_smem();
  if (tid == 0) { mbar_init(&bar_done, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc_pair<512>(&tmem_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_s;
  {
    const uint32_t row = rank * 128 + warp * 32 + lane;
    for (int c0 = 0; c0 < K / 2; c0 += 8) {
      uint32_t r[8];
      for (int i = 0; i < 8; ++i) {
        __half2 h2 = __halves2half2(A[(size_t)row * K + 2 * (c0 + i)], A[(size_t)row * K + 2 * (c0 + i) + 1]);
        r[i] = *reinterpret_cast<uint32_t*>(&h2);
      }
      tmem_st8(tmem + ((warp * 32) << 16) + 256 + c0, r);
    }
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  if (rank == 0 && warp == 0) {
    const uint32_t idesc = idesc_f16_f32(256, N);
    const uint64_t b0 = sdesc_kmajor_noswz(smem_u32(smem), b_lbo, b_sbo);
    const long long t0 = clock64();
    for (int rp = 0; rp < reps; ++rp)
      for (int ks = 0; ks < K / 16; ++ks)
        umma_f16_ts_pair_warp(tmem, tmem + 256 + ks * 8, b0 + (uint64_t)(ks * 2 * b_lbo >> 4), idesc,
                              (rp | ks) ? 1u : 0u);
    umma_commit_pair_warp(&bar_done, (uint16_t)3);
    mbar_wait(&bar_done, 0);
    const long long t1 = clock64();
    if (lane == 0 && cycles) *cycles = t1 - t0;
  } else if (tid == 0) {
    mbar_wait(&bar_done, 0);
  }
  __syncthreads();
  tc_fence_after();
  const uint32_t lrow = warp * 32 + lane;
  for (int c = 0; c < N; c += 16) {
    float v[16];
    tmem_ld16(tmem + ((warp * 32) << 16) + c, v);
    tmem_ld_wait();
    for (int j = 0; j < 16; ++j) D[(size_t)(rank * 128 + lrow) * N + c + j] = v[j];
  }
  for (int half = 0; half < 2; ++half)
    for (int c = 0; c < N; c += 16) {
      float v[8];
      tmem_ld_16x256b_x2(tmem + ((warp * 32 + half * 16) << 16) + c, v);
      tmem_ld_wait();
      const int l0 = warp * 32 + half * 16 + lane / 4, c0 = c + 2 * (lane % 4);
      const int ls[8] = {l0, l0, l0 + 8, l0 + 8, l0, l0, l0 + 8, l0 + 8};
      const int cs[8] = {c0, c0 + 1, c0, c0 + 1, c0 + 8, c0 + 9, c0 + 8, c0 + 9};
      for (int j = 0; j < 8; ++j) D2[(size_t)(rank * 128 + ls[j]) * N + cs[j]] = v[j];
    }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) tmem_dealloc_pair<512>(tmem);
}

}  // namespace

extern "C" int skb_diag_umma_gemm(const void* A, const void* B, void* D, int N, int K,
                                  int swap_lbo_sbo, long long* cycles, void* stream) {
  if (N % 16 || N < 16 || N > 256 || K % 16 || K <= 0) return SKB_ERR_INVALID;
  size_t smem = (size_t)(128 + N) * K * 2;
  if (smem > 200 * 1024) return SKB_ERR_INVALID;
  cudaFuncSetAttribute(umma_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  umma_gemm_kernel<<<1, 128, smem, (cudaStream_t)stream>>>(
      (const __half*)A, (const __half*)B, (float*)D, N, K, swap_lbo_sbo, cycles);
  return skb_check_launch();
}

extern "C" int skb_diag_cluster_exchange(int cluster, int slice_bytes, int rounds,
                                         long long* cycles, int* errors, void* gscratch, void* stream) {
  if (slice_bytes % 16 || slice_bytes <= 0) return SKB_ERR_INVALID;
  size_t smem = (size_t)2 * slice_bytes + (size_t)2 * cluster * slice_bytes;
  if (smem > 200 * 1024) return SKB_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  switch (cluster) {
#define SKB_CASE(C)                                                                        \
  case C:                                                                                  \
    cudaFuncSetAttribute(cluster_exchange_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                         (int)smem);                                                       \
    cluster_exchange_kernel<C><<<C, 128, smem, s>>>(slice_bytes, rounds, cycles, errors, (uint8_t*)gscratch);  \
    break;
    SKB_CASE(2) SKB_CASE(4) SKB_CASE(8)
#undef SKB_CASE
    default: return SKB_ERR_INVALID;
  }
  return skb_check_launch();
}

extern "C" int skb_diag_umma_pair(const void* A, const void* B, void* D, void* D2, int N, int K, int reps,
                                  long long* cycles, void* stream) {
  if (N % 32 || N < 32 || N > 256 || K % 16 || K <= 0 || K > 512 || reps < 1) return SKB_ERR_INVALID;
  const size_t smem = (size_t)(N / 2) * K * 2;
  cudaFuncSetAttribute(umma_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  umma_pair_kernel<<<2, 128, smem, (cudaStream_t)stream>>>((const __half*)A, (const __half*)B, (float*)D,
                                                          (float*)D2, N, K, reps, cycles);
  return skb_check_launch();
}
