// gemm.cu — host side of skb's tcgen05 GEMM engine (gemm.cuh) and its C ABI entry
// skb_gemm (general row-major GEMM with K-/MN-major operands, bf16 or tf32 tensor
// cores, fp32 output, optional accumulate and deterministic split-K).
#include <cudaTypedefs.h>
#include <stdio.h>

#include "gemm.cuh"
#include "skb.h"
#include "skb_internal.h"

namespace skb {
namespace gemm {

static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

bool encode_2d(CUtensorMap* tm, int elem, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld_elems,
               uint32_t box_inner, uint32_t box_outer) {
  if (!g_encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
      return false;
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const uint64_t eb = elem == kBF16 ? 2 : 4;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld_elems * eb};   // bytes between outer rows (multiple of 16)
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  if ((ld_elems * eb) % 16 || (reinterpret_cast<uintptr_t>(ptr) & 15)) return false;
  const CUresult r = g_encode(tm, elem == kBF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                              const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool encode_3d(CUtensorMap* tm, int elem, const void* ptr, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1_elems,
               uint64_t s2_elems, uint32_t b0, uint32_t b1, uint32_t b2) {
  if (!g_encode) {
    CUtensorMap dummy;
    if (!encode_2d(&dummy, elem, ptr, 8, 1, 8, 8, 1)) return false;
  }
  const uint64_t eb = elem == kBF16 ? 2 : 4;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {s1_elems * eb, s2_elems * eb};
  cuuint32_t box[3] = {b0, b1, b2};
  cuuint32_t estr[3] = {1, 1, 1};
  if ((s1_elems * eb) % 16 || (s2_elems * eb) % 16 || (reinterpret_cast<uintptr_t>(ptr) & 15)) return false;
  const CUresult r = g_encode(tm, elem == kBF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                              const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int num_sms() {
  static int n[16] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 16) return 148;
  if (!n[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    n[dev] = v > 0 ? v : 148;
  }
  return n[dev];
}

}  // namespace gemm
}  // namespace skb

namespace skb {
namespace gemm {

// C = sum_s P[s] (+ C): the fixed-order reduction of split-K partial planes.
__global__ void reduce_splits(float* __restrict__ C, long long ldc, const float* __restrict__ P, long long plane,
                              int M, int N, int ks, int beta) {
  const long long total = (long long)M * N;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long m = i / N, n = i % N;
    float s = beta ? C[m * ldc + n] : 0.f;
    for (int k = 0; k < ks; ++k) s += P[k * plane + m * N + n];
    C[m * ldc + n] = s;
  }
}

template <int ELEM, int BN, bool AMN, bool BMN>
int run_store(const Problem& p, float* C, long long ldc, int beta, int ksplit, float* ws, cudaStream_t st) {
  CUtensorMap ta, tb;
  if (!make_maps<ELEM, BN>(p, &ta, &tb)) return SKB_ERR_INVALID;
  Shape sh{p.M, p.N, p.K, ksplit, 0};
  EpiStore e;
  if (ksplit > 1) {
    e = EpiStore{ws, p.N, (long long)p.M * p.N, 0};
  } else {
    e = EpiStore{C, ldc, 0, beta};
  }
  if (launch<ELEM, BN, AMN, BMN>(ta, tb, sh, e, st)) return SKB_ERR_CUDA;
  if (ksplit > 1) {
    reduce_splits<<<num_sms() * 4, 256, 0, st>>>(C, ldc, ws, (long long)p.M * p.N, p.M, p.N, ksplit, beta);
    if (cudaPeekAtLastError() != cudaSuccess) return SKB_ERR_CUDA;
  }
  return SKB_OK;
}

template <int ELEM, int BN, bool AMN, bool BMN>
int run_pair(const Problem& p, float* C, long long ldc, int beta, cudaStream_t st) {
  using G = Geo<ELEM, BN / 2>;
  CUtensorMap ta, tb;
  const bool oka = p.a_mn ? encode_2d(&ta, ELEM, p.A, p.M, p.K, p.lda, G::MNB, G::BK)
                          : encode_2d(&ta, ELEM, p.A, p.K, p.M, p.lda, G::BK, G::BM);
  const bool okb = p.b_mn ? encode_2d(&tb, ELEM, p.B, p.N, p.K, p.ldb, G::MNB, G::BK)
                          : encode_2d(&tb, ELEM, p.B, p.K, p.N, p.ldb, G::BK, BN / 2);
  if (!oka || !okb) return SKB_ERR_INVALID;
  Shape sh{p.M, p.N, p.K, 1, 0};
  EpiStore e{C, ldc, 0, beta};
  return launch_pair<ELEM, BN, AMN, BMN>(ta, tb, sh, e, st) ? SKB_ERR_CUDA : SKB_OK;
}

template <int ELEM, int BN>
int run_pair_majors(const Problem& p, float* C, long long ldc, int beta, cudaStream_t st) {
  if (!p.a_mn && !p.b_mn) return run_pair<ELEM, BN, false, false>(p, C, ldc, beta, st);
  if (!p.a_mn && p.b_mn) return run_pair<ELEM, BN, false, true>(p, C, ldc, beta, st);
  if (p.a_mn && !p.b_mn) return run_pair<ELEM, BN, true, false>(p, C, ldc, beta, st);
  return run_pair<ELEM, BN, true, true>(p, C, ldc, beta, st);
}

template <int ELEM, int BN>
int run_majors(const Problem& p, float* C, long long ldc, int beta, int ksplit, float* ws, cudaStream_t st) {
  if (!p.a_mn && !p.b_mn) return run_store<ELEM, BN, false, false>(p, C, ldc, beta, ksplit, ws, st);
  if (!p.a_mn && p.b_mn) return run_store<ELEM, BN, false, true>(p, C, ldc, beta, ksplit, ws, st);
  if (p.a_mn && !p.b_mn) return run_store<ELEM, BN, true, false>(p, C, ldc, beta, ksplit, ws, st);
  return run_store<ELEM, BN, true, true>(p, C, ldc, beta, ksplit, ws, st);
}

}  // namespace gemm
}  // namespace skb

using namespace skb::gemm;

extern "C" int64_t skb_gemm_workspace_bytes(int M, int N, int ksplit) {
  return ksplit > 1 ? (int64_t)ksplit * M * N * 4 : 0;
}

extern "C" skb_status skb_gemm(int elem, int a_mn, int b_mn, int M, int N, int K, const void* A, int64_t lda,
                               const void* B, int64_t ldb, float* C, int64_t ldc, int beta, int bn, int ksplit,
                               void* workspace, void* stream) {
  if (M < 0 || N < 0 || K < 0 || !C || (elem != kBF16 && elem != kTF32) || (beta != 0 && beta != 1)) return SKB_ERR_INVALID;
  if (M == 0 || N == 0) return SKB_OK;
  if (N % 16 || ldc % 4 || (reinterpret_cast<uintptr_t>(C) & 15)) return SKB_ERR_INVALID;
  if (elem == kTF32 && (a_mn || b_mn)) return SKB_ERR_UNSUPPORTED;   // kind::tf32: K-major operands only
  if (ksplit < 1) ksplit = 1;
  if (ksplit > 1 && !workspace) return SKB_ERR_INVALID;
  Problem p{elem, a_mn != 0, b_mn != 0, A, lda, B, ldb, M, N, K};
  cudaStream_t st = (cudaStream_t)stream;
  if (bn < 0) {   // CTA-pair (cta_group::2) tiles of 256 x |bn|
    if (ksplit > 1 || (bn != -256 && bn != -128)) return SKB_ERR_INVALID;
    int rc;
    if (elem == kBF16)
      rc = bn == -256 ? run_pair_majors<kBF16, 256>(p, C, ldc, beta, st) : run_pair_majors<kBF16, 128>(p, C, ldc, beta, st);
    else
      rc = bn == -256 ? run_pair<kTF32, 256, false, false>(p, C, ldc, beta, st)
                      : run_pair<kTF32, 128, false, false>(p, C, ldc, beta, st);
    return rc == SKB_OK ? (skb_status)skb_check_launch() : (skb_status)rc;
  }
  if (bn == 0) bn = N >= 256 ? 256 : 128;
  float* ws = (float*)workspace;
  int rc;
  if (elem == kBF16)
    rc = bn == 256 ? run_majors<kBF16, 256>(p, C, ldc, beta, ksplit, ws, st)
       : bn == 128 ? run_majors<kBF16, 128>(p, C, ldc, beta, ksplit, ws, st)
                   : run_majors<kBF16, 64>(p, C, ldc, beta, ksplit, ws, st);
  else
    rc = bn == 256 ? run_store<kTF32, 256, false, false>(p, C, ldc, beta, ksplit, ws, st)
       : bn == 128 ? run_store<kTF32, 128, false, false>(p, C, ldc, beta, ksplit, ws, st)
                   : run_store<kTF32, 64, false, false>(p, C, ldc, beta, ksplit, ws, st);
  return rc == SKB_OK ? (skb_status)skb_check_launch() : (skb_status)rc;
}
