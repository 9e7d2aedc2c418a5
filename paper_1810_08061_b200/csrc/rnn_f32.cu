// rnn_f32.cu — the accurate tier of the fused recurrent While (LSTM / GRU /
// tanh-RNN): FP32 FFMA arithmetic with fp32 weights and state, accurate
// activations, for callers that need the reference's float64 results within
// rtol 1e-4 (north_star's fp32 bound) rather than the fp16-operand tensor-core
// tier's 3e-3 (csrc/rnn.cu).  Same program semantics (reference
// graph/execute.py:218-238 _eval_while; tensor.py:302-319 matmul, :391-407
// tanh / stable sigmoid, :356-377 row-select where, execute.py:153-185 the
// stacked outputs), same per-problem failures, one persistent launch.
//
// Mapping: one CTA per tile of NT consecutive batch rows (a whole problem
// when rows_per_problem == NT); thread u owns hidden unit u and computes its
// G gate columns for all NT rows (NT x G accumulators in registers), so the
// cell update is thread-local — no gate exchange.  Per step the CTA's
// [x_t ; h_{t-1}] rows live in shared memory (double-buffered; x_{t+1} is
// prefetched with cp.async during step t), read as 16-byte broadcasts; the
// packed weights Wp[k][u][G] (fp32, [W;U] concatenated along k) stream from
// L2 as one 16-byte load per (k, thread), prefetched 4 k ahead.  Bound: the
// FP32 FFMA pipe (2*(F+H)*G*H flop per row-step).
#include <cuda_runtime.h>
#include <climits>
#include <stdint.h>
#include "skb_internal.h"

namespace {

template <int G>
struct WVec;
template <>
struct WVec<4> { using T = float4; };
template <>
struct WVec<1> { using T = float; };

__device__ __forceinline__ float sigmoid_acc(float x) {   // tensor.py:403-407 (two-branch stable form)
  if (x >= 0.f) return 1.f / (1.f + expf(-x));
  const float e = expf(x);
  return e / (1.f + e);
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

struct F32Args {
  const void* x;          // [R, T, F] f32 or f64
  const float* h0;        // [R, H]
  const float* c0;        // [R, H] (LSTM)
  const int64_t* lens;    // [R]
  const float* wp;        // [K][Hp][G] fp32, K = F + H
  const float* bias;      // [G][H]   (GRU: bz, br, bn, bhn)
  const int32_t* pmax;    // [P] per-problem max_len
  float* out;             // [R, T, H]
  float* hT;
  float* cT;
  int x_f64, R, T, F, H, Hp, K, Bp;
};

// x_t rows of the tile -> sA[0..F) of each row (F % 4 == 0 fp32 path: cp.async; else scalar)
template <int NT>
__device__ __forceinline__ void load_x_rows(const F32Args& a, float* sA, int row0, int t, int tid, int nthr) {
  const int K = a.K;
  if (!a.x_f64 && (a.F & 3) == 0) {
    const int per_row = a.F / 4;
    for (int i = tid; i < NT * per_row; i += nthr) {
      const int r = i / per_row, c = (i % per_row) * 4, row = row0 + r;
      if (row < a.R && t < a.T)
        cp_async16(sA + r * K + c, reinterpret_cast<const float*>(a.x) + ((size_t)row * a.T + t) * a.F + c);
    }
    cp_async_commit();
  } else {
    for (int i = tid; i < NT * a.F; i += nthr) {
      const int r = i / a.F, c = i % a.F, row = row0 + r;
      float v = 0.f;
      if (row < a.R && t < a.T) {
        const size_t off = ((size_t)row * a.T + t) * a.F + c;
        v = a.x_f64 ? (float)reinterpret_cast<const double*>(a.x)[off] : reinterpret_cast<const float*>(a.x)[off];
      }
      sA[r * K + c] = v;
    }
  }
}

template <int CELL, int NT>
__global__ void __launch_bounds__(256, 1) rnn_f32_kernel(const F32Args a) {
  constexpr int G = (CELL == SKB_CELL_RNN_TANH) ? 1 : 4;
  using W = typename WVec<G>::T;
  extern __shared__ __align__(16) float smem[];
  const int K = a.K, H = a.H;
  float* sA[2] = {smem, smem + NT * K};            // [NT][K] : x_t | h_{t-1}
  float* sC = smem + 2 * NT * K;                     // [NT][Hp] LSTM cell state
  __shared__ int s_len[NT], s_tmax[NT], s_trip;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int row0 = blockIdx.x * NT;

  if (tid < NT) {
    const int row = row0 + tid;
    int len = 0, tmax = 0;
    if (row < a.R) {
      tmax = max(0, min(a.pmax[row / a.Bp], a.T));
      len = (int)max(0LL, min((long long)a.lens[row], (long long)tmax));
    }
    s_len[tid] = len;
    s_tmax[tid] = tmax;
  }
  __syncthreads();
  if (tid == 0) {
    int m = 0;
    for (int r = 0; r < NT; ++r) m = max(m, s_tmax[r]);
    s_trip = m;
  }
  // h0 / c0 -> shared memory
  for (int i = tid; i < NT * H; i += nthr) {
    const int r = i / H, u = i % H, row = row0 + r;
    const bool ok = row < a.R;
    sA[0][r * K + a.F + u] = ok ? a.h0[(size_t)row * H + u] : 0.f;
    if (CELL == SKB_CELL_LSTM) sC[r * a.Hp + u] = ok ? a.c0[(size_t)row * H + u] : 0.f;
  }
  load_x_rows<NT>(a, sA[0], row0, 0, tid, nthr);
  cp_async_wait_all();
  __syncthreads();
  const int trip = s_trip;
  const int u = tid;
  const bool active = u < H;
  float bias[G];
#pragma unroll
  for (int g = 0; g < G; ++g) bias[g] = active ? a.bias[g * H + u] : 0.f;
  const W* wp = reinterpret_cast<const W*>(a.wp) + (active ? u : 0);
  const int wstride = a.Hp;   // W elements between consecutive k for one unit

  for (int t = 0; t < trip; ++t) {
    float* cur = sA[t & 1];
    float* nxt = sA[(t + 1) & 1];
    if (t + 1 < trip) load_x_rows<NT>(a, nxt, row0, t + 1, tid, nthr);   // overlaps this step's math
    float acc[NT][G];
#pragma unroll
    for (int r = 0; r < NT; ++r)
#pragma unroll
      for (int g = 0; g < G; ++g) acc[r][g] = 0.f;
    if (active) {
      W wq[4], wn[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) wq[j] = __ldg(wp + (size_t)j * wstride);
      for (int k0 = 0; k0 < K; k0 += 4) {
        const bool more = k0 + 4 < K;
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (more && k0 + 4 + j < K) wn[j] = __ldg(wp + (size_t)(k0 + 4 + j) * wstride);
#pragma unroll
        for (int r = 0; r < NT; ++r) {
          const float4 xv = *reinterpret_cast<const float4*>(cur + r * K + k0);   // broadcast read
          const float xs[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if constexpr (G == 4) {
              acc[r][0] = fmaf(xs[j], wq[j].x, acc[r][0]);
              acc[r][1] = fmaf(xs[j], wq[j].y, acc[r][1]);
              acc[r][2] = fmaf(xs[j], wq[j].z, acc[r][2]);
              acc[r][3] = fmaf(xs[j], wq[j].w, acc[r][3]);
            } else {
              acc[r][0] = fmaf(xs[j], wq[j], acc[r][0]);
            }
          }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) wq[j] = wn[j];
      }
    }
    // cell update for unit u, every row; masked by t < len (reference Where); the
    // output row out[row, t, u] is written for t < the row's problem max_len (frozen
    // rows repeat h) and h_t goes to the next step's buffer (disjoint from x_{t+1})
    if (active) {
#pragma unroll
      for (int r = 0; r < NT; ++r) {
        const float hp = cur[r * K + a.F + u];
        float h = hp;
        const bool live = t < s_len[r];
        if constexpr (CELL == SKB_CELL_LSTM) {
          const float c = sC[r * a.Hp + u];
          const float i = sigmoid_acc(acc[r][0] + bias[0]);
          const float f = sigmoid_acc(acc[r][1] + bias[1]);
          const float g = tanhf(acc[r][2] + bias[2]);
          const float o = sigmoid_acc(acc[r][3] + bias[3]);
          const float c2 = f * c + i * g;
          const float h2 = o * tanhf(c2);
          if (live) { sC[r * a.Hp + u] = c2; h = h2; }
        } else if constexpr (CELL == SKB_CELL_GRU) {
          // acc[2] = x Wn, acc[3] = h Un (the packed n_x / n_h blocks)
          const float z = sigmoid_acc(acc[r][0] + bias[0]);
          const float rr = sigmoid_acc(acc[r][1] + bias[1]);
          const float n = tanhf((acc[r][2] + bias[2]) + rr * (acc[r][3] + bias[3]));
          const float h2 = (1.f - z) * n + z * hp;
          if (live) h = h2;
        } else {
          const float h2 = tanhf(acc[r][0] + bias[0]);
          if (live) h = h2;
        }
        const int row = row0 + r;
        if (row < a.R && t < s_tmax[r]) a.out[((size_t)row * a.T + t) * H + u] = h;
        nxt[r * K + a.F + u] = h;
      }
    }
    cp_async_wait_all();
    __syncthreads();
  }
  // final states
  const float* fin = sA[trip & 1];
  if (active) {
    for (int r = 0; r < NT; ++r) {
      const int row = row0 + r;
      if (row >= a.R) continue;
      if (a.hT) a.hT[(size_t)row * H + u] = fin[r * K + a.F + u];
      if (CELL == SKB_CELL_LSTM && a.cT) a.cT[(size_t)row * H + u] = sC[r * a.Hp + u];
    }
  }
}

// Per-problem max_len (reference reduce_max, tensor.py:344-353) and the first
// failing problem in the reference's evaluation order (negative -> ShapeMismatch,
// > T -> IndexOutOfRange, 0 -> EmptyPop); same contract as csrc/rnn.cu.
__global__ void f32_pmax_kernel(const int64_t* lens, int32_t* pmax, int32_t* max_len_out, int32_t* err, int R,
                                int Bp, int P, int T) {
  __shared__ int first_bad;
  if (threadIdx.x == 0) first_bad = INT_MAX;
  __syncthreads();
  for (int p = threadIdx.x; p < P; p += blockDim.x) {
    long long m = LLONG_MIN;
    for (int r = p * Bp; r < min(R, (p + 1) * Bp); ++r) m = max(m, (long long)lens[r]);
    const int mi = (int)max((long long)INT_MIN, min(m, (long long)INT_MAX));
    pmax[p] = mi;
    max_len_out[p] = mi;
    if (mi < 0 || mi > T || mi == 0) atomicMin(&first_bad, p);
  }
  __syncthreads();
  if (threadIdx.x == 0 && first_bad != INT_MAX) {
    const int m = pmax[first_bad];
    const int code = m < 0 ? SKB_ERR_SHAPE_MISMATCH : (m > T ? SKB_ERR_INDEX_OUT_OF_RANGE : SKB_ERR_EMPTY_POP);
    if (atomicCAS(err, 0, code) == 0) { err[1] = first_bad; err[2] = m > T ? T : 0; err[3] = m; }
  }
}

// Wp[k][u][g] (fp32) from W[g] [F, H], U[g] [H, H]; NULL blocks are zero (GRU n_x / n_h).
__global__ void f32_pack_kernel(const void* const* w, const void* const* u, const void* const* b, int f64, int G,
                                int F, int H, int Hp, float* wp, float* bias) {
  const int K = F + H;
  const long long total = (long long)K * Hp * G;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int g = (int)(i % G), un = (int)((i / G) % Hp), k = (int)(i / ((long long)G * Hp));
    float v = 0.f;
    if (un < H) {
      const void* src = k < F ? w[g] : u[g];
      const size_t off = k < F ? (size_t)k * H + un : (size_t)(k - F) * H + un;
      if (src) v = f64 ? (float)reinterpret_cast<const double*>(src)[off] : reinterpret_cast<const float*>(src)[off];
    }
    wp[i] = v;
  }
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < G * H; i += gridDim.x * blockDim.x) {
    const int g = i / H, un = i % H;
    bias[i] = f64 ? (float)reinterpret_cast<const double*>(b[g])[un] : reinterpret_cast<const float*>(b[g])[un];
  }
}

constexpr int kNT32 = 32;

inline int cell_G(int cell) { return cell == SKB_CELL_RNN_TANH ? 1 : 4; }
inline int hpad(int H) { return (H + 31) / 32 * 32; }
inline size_t smem_f32(int F, int H, int NT) { return ((size_t)2 * NT * (F + H) + (size_t)NT * hpad(H)) * 4; }

template <int CELL, int NT>
int launch_f32(const F32Args& a, cudaStream_t st) {
  const size_t smem = smem_f32(a.F, a.H, NT);
  auto kern = rnn_f32_kernel<CELL, NT>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return SKB_ERR_CUDA;
  const int threads = hpad(a.H);
  kern<<<(a.R + NT - 1) / NT, threads, smem, st>>>(a);
  return skb_check_launch();
}

}  // namespace

extern "C" int64_t skb_rnn_f32_packed_bytes(const skb_rnn_shape* s) {
  if (!s || s->hidden <= 0 || s->input <= 0) return -1;
  const int G = cell_G(s->cell);
  return ((int64_t)(s->input + s->hidden) * hpad(s->hidden) * G + (int64_t)G * s->hidden) * 4;
}

extern "C" int64_t skb_rnn_f32_workspace_bytes(const skb_rnn_shape* s) {
  if (!s || s->problems <= 0) return -1;
  return ((int64_t)s->problems * 4 + 255) / 256 * 256;
}

extern "C" int skb_rnn_pack_f32(const skb_rnn_shape* s, const void* const* w_dev, const void* const* u_dev,
                                const void* const* b_dev, int f64, void* packed_dev, void* stream) {
  if (!s || !packed_dev || !w_dev || !u_dev || !b_dev) return SKB_ERR_INVALID;
  if (s->cell != SKB_CELL_LSTM && s->cell != SKB_CELL_GRU && s->cell != SKB_CELL_RNN_TANH) return SKB_ERR_INVALID;
  const int G = cell_G(s->cell), F = s->input, H = s->hidden, Hp = hpad(H);
  const void** dw;
  const void** du;
  const void** db;
  if (cudaMalloc(&dw, sizeof(void*) * 12) != cudaSuccess) return SKB_ERR_CUDA;
  du = dw + 4;
  db = dw + 8;
  const void* hw[12] = {};
  for (int g = 0; g < G; ++g) { hw[g] = w_dev[g]; hw[4 + g] = u_dev[g]; hw[8 + g] = b_dev[g]; }
  cudaStream_t st = (cudaStream_t)stream;
  cudaMemcpyAsync(dw, hw, sizeof(hw), cudaMemcpyHostToDevice, st);
  float* wp = reinterpret_cast<float*>(packed_dev);
  float* bias = wp + (size_t)(F + H) * Hp * G;
  f32_pack_kernel<<<1184, 256, 0, st>>>(dw, du, db, f64, G, F, H, Hp, wp, bias);
  const int rc = skb_check_launch();
  cudaStreamSynchronize(st);
  cudaFree(dw);
  return rc;
}

extern "C" int skb_rnn_forward_f32(const skb_rnn_shape* s, const void* packed_dev, const void* x_dev, int x_f64,
                                   const float* h0_dev, const float* c0_dev, const int64_t* len_dev, float* out_dev,
                                   float* hT_dev, float* cT_dev, int32_t* max_len_dev, int32_t* err_dev,
                                   void* workspace_dev, void* stream) {
  if (!s || !packed_dev || !x_dev || !h0_dev || !len_dev || !out_dev || !max_len_dev || !err_dev || !workspace_dev)
    return SKB_ERR_INVALID;
  if (s->cell == SKB_CELL_LSTM && !c0_dev) return SKB_ERR_INVALID;
  if (s->hidden > 256 || s->hidden < 1 || s->input < 1 || s->time < 0) return SKB_ERR_UNSUPPORTED;
  F32Args a = {};
  a.x = x_dev; a.h0 = h0_dev; a.c0 = c0_dev; a.lens = len_dev; a.out = out_dev; a.hT = hT_dev; a.cT = cT_dev;
  a.x_f64 = x_f64; a.R = s->rows_per_problem * s->problems; a.T = s->time; a.F = s->input; a.H = s->hidden;
  a.Hp = hpad(s->hidden); a.K = s->input + s->hidden; a.Bp = s->rows_per_problem;
  const int G = cell_G(s->cell);
  a.wp = reinterpret_cast<const float*>(packed_dev);
  a.bias = a.wp + (size_t)a.K * a.Hp * G;
  a.pmax = reinterpret_cast<int32_t*>(workspace_dev);
  if ((a.K & 3) != 0) return SKB_ERR_UNSUPPORTED;   // 16-byte rows in shared memory
  if (smem_f32(a.F, a.H, kNT32) > 227 * 1024) return SKB_ERR_UNSUPPORTED;
  cudaStream_t st = (cudaStream_t)stream;
  f32_pmax_kernel<<<1, 1024, 0, st>>>(len_dev, const_cast<int32_t*>(a.pmax), max_len_dev, err_dev, a.R, a.Bp,
                                      s->problems, a.T);
  if (int e = skb_check_launch()) return e;
  if (a.T == 0) return SKB_OK;
  switch (s->cell) {
    case SKB_CELL_LSTM: return launch_f32<SKB_CELL_LSTM, kNT32>(a, st);
    case SKB_CELL_GRU: return launch_f32<SKB_CELL_GRU, kNT32>(a, st);
    default: return launch_f32<SKB_CELL_RNN_TANH, kNT32>(a, st);
  }
}
