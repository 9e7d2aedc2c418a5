// train.cu — one dynamic-length LSTM training step (BASELINE config C2):
// forward over the staged While, BPTT, gradients of W [F,4H], U [H,4H],
// b [4H] (gate order i,f,g,o), and the SGD update.
//
// The reference cannot differentiate a While (graph/grad.py:159-161); its
// training step is the hand-derived staged program oracle/programs/
// lstm_bptt.msl (forward While storing states, reverse While), executed by
// graph/execute.py:218-238.  Here, per GPU shard of B rows (batch-major
// x [B,T,F], y [B,T,H]):
//   forward  Z = X W for every step in one GEMM (K = F, rows (b, t)), then
//            t = 0..n-1:  Z_t += h_{t-1} U                  (cuBLAS, strided views)
//                         lstm_fwd_cell: gates, c_t, h_t with the row mask
//                         (rows past their length keep h, c — the Where rule)
//   loss     inv_b * sum_{b, t<len_b} <h_{b,t}, y_{b,t}>     (deterministic block reduce)
//   backward t = n-1..0:  lstm_bwd_cell: dG_t (in place of the gate activations),
//                         carried dh / dc for frozen rows
//                         dh = dG_t U^T + carry
//   grads    dW = X^T dG and dU = H_prev^T dG as two GEMMs over all (b, t) (bf16 path;
//            the fp32 path accumulates dU per step), db = column sums of dG
// The whole step is captured once per (n, buffers) as a CUDA graph, so the
// ~5n GEMMs and 2n cell kernels replay with a single launch.  The gradient
// allreduce (NCCL, torch.distributed) and the fused SGD update run after it.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <string.h>
#include <cuda_bf16.h>
#include "blas.cuh"
#include "skb_internal.h"

namespace {

__device__ __forceinline__ float sigf(float x) { return 1.f / (1.f + expf(-x)); }

struct TrainBufs {
  float* Z;      // [B, T, 4H] pre-activations -> activations (fwd) -> dG (bwd)
  float* Hs;     // [B, T+1, H] Hs[:, 0] = h0, Hs[:, t+1] = h after step t
  float* Cs;     // [B, T+1, H]
  float* dh;     // [B, H]
  float* dc;     // [B, H]
  double* part;  // loss partials [kLossBlocks]
  float* bpart;  // bias-gradient partials [kBiasChunks, 4H]
  // bf16 GEMM operands (math == 2): x, h_{t-1} [B, T, H], dG and the weights
  __nv_bfloat16 *Xb, *Hb, *Zb, *Wb, *Ub;
};
constexpr int kLossBlocks = 1184;

__global__ void init_states(const float* h0, const float* c0, TrainBufs w, int B, int T, int H) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < (long long)B * H;
       i += (long long)gridDim.x * blockDim.x) {
    const int b = (int)(i / H), k = (int)(i % H);
    w.Hs[(long long)b * (T + 1) * H + k] = h0 ? h0[i] : 0.f;
    if (w.Hb) w.Hb[(long long)b * T * H + k] = __float2bfloat16(h0 ? h0[i] : 0.f);   // h_{-1} at t = 0
    w.Cs[(long long)b * (T + 1) * H + k] = c0 ? c0[i] : 0.f;
    w.dh[i] = 0.f;
    w.dc[i] = 0.f;
  }
}

__global__ void lstm_fwd_cell(TrainBufs w, const float* __restrict__ bias, const int64_t* __restrict__ lens, int B,
                              int T, int H, int t) {
  const int b = blockIdx.y;   // one grid row per sequence, threads over units: no index division
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < H; k += gridDim.x * blockDim.x) {
    const long long i = (long long)b * H + k;
    float* z = w.Z + ((long long)b * T + t) * 4 * H;
    const float ig = sigf(z[k] + bias[k]);
    const float fg = sigf(z[H + k] + bias[H + k]);
    const float gg = tanhf(z[2 * H + k] + bias[2 * H + k]);
    const float og = sigf(z[3 * H + k] + bias[3 * H + k]);
    const long long sp = ((long long)b * (T + 1) + t) * H + k;   // state before step t
    const float cp = w.Cs[sp], hp = w.Hs[sp];
    const bool live = t < lens[b];
    const float cn = fg * cp + ig * gg;
    const float hn = og * tanhf(cn);
    w.Cs[sp + H] = live ? cn : cp;
    w.Hs[sp + H] = live ? hn : hp;
    if (w.Hb && t + 1 < T) w.Hb[((long long)b * T + t + 1) * H + k] = __float2bfloat16(live ? hn : hp);
    z[k] = ig; z[H + k] = fg; z[2 * H + k] = gg; z[3 * H + k] = og;
  }
}

__global__ void lstm_bwd_cell(TrainBufs w, const float* __restrict__ y, const int64_t* __restrict__ lens, float inv_b,
                              int B, int T, int H, int t) {
  const int b = blockIdx.y;   // one grid row per sequence, threads over units: no index division
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < H; k += gridDim.x * blockDim.x) {
    const long long i = (long long)b * H + k;
    const bool live = t < lens[b];
    float* z = w.Z + ((long long)b * T + t) * 4 * H;
    float dh = w.dh[i] + (live ? y[((long long)b * T + t) * H + k] * inv_b : 0.f);
    float dc = w.dc[i];
    __nv_bfloat16* zb = w.Zb ? w.Zb + ((long long)b * T + t) * 4 * H : nullptr;
    if (!live) {   // frozen row: h_t = h_{t-1}, c_t = c_{t-1}; gradients pass straight through
      z[k] = 0.f; z[H + k] = 0.f; z[2 * H + k] = 0.f; z[3 * H + k] = 0.f;
      if (zb) { zb[k] = zb[H + k] = zb[2 * H + k] = zb[3 * H + k] = __float2bfloat16(0.f); }
      w.dh[i] = dh;   // the dh GEMM accumulates onto this carry (beta = 1)
      continue;
    }
    const float ig = z[k], fg = z[H + k], gg = z[2 * H + k], og = z[3 * H + k];
    const long long sp = ((long long)b * (T + 1) + t) * H + k;
    const float cp = w.Cs[sp], cn = w.Cs[sp + H];
    const float tc = tanhf(cn);
    const float dcn = dc + dh * og * (1.f - tc * tc);
    z[k] = dcn * gg * ig * (1.f - ig);
    z[H + k] = dcn * cp * fg * (1.f - fg);
    z[2 * H + k] = dcn * ig * (1.f - gg * gg);
    z[3 * H + k] = dh * tc * og * (1.f - og);
    if (zb) {
      zb[k] = __float2bfloat16(z[k]); zb[H + k] = __float2bfloat16(z[H + k]);
      zb[2 * H + k] = __float2bfloat16(z[2 * H + k]); zb[3 * H + k] = __float2bfloat16(z[3 * H + k]);
    }
    w.dc[i] = dcn * fg;
    w.dh[i] = 0.f;
  }
}

// float4 variants (H % 4 == 0): thread = 4 consecutive units of one sequence row,
// same per-element arithmetic as lstm_fwd_cell / lstm_bwd_cell.
__device__ __forceinline__ float4 f4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void s4(float* p, float a, float b, float c, float d) {
  *reinterpret_cast<float4*>(p) = make_float4(a, b, c, d);
}

__global__ void lstm_fwd_cell4(TrainBufs w, const float* __restrict__ bias, const int64_t* __restrict__ lens, int B,
                               int T, int H, int t) {
  const int b = blockIdx.y;
  const bool live = t < lens[b];
  for (int k = 4 * (blockIdx.x * blockDim.x + threadIdx.x); k < H; k += 4 * gridDim.x * blockDim.x) {
    float* z = w.Z + ((long long)b * T + t) * 4 * H;
    const float4 zi = f4(z + k), zf = f4(z + H + k), zg = f4(z + 2 * H + k), zo = f4(z + 3 * H + k);
    const float4 bi = f4(bias + k), bf = f4(bias + H + k), bg = f4(bias + 2 * H + k), bo = f4(bias + 3 * H + k);
    const long long sp = ((long long)b * (T + 1) + t) * H + k;
    const float4 cp = f4(w.Cs + sp), hp = f4(w.Hs + sp);
    const float zin[4][4] = {{zi.x + bi.x, zi.y + bi.y, zi.z + bi.z, zi.w + bi.w},
                             {zf.x + bf.x, zf.y + bf.y, zf.z + bf.z, zf.w + bf.w},
                             {zg.x + bg.x, zg.y + bg.y, zg.z + bg.z, zg.w + bg.w},
                             {zo.x + bo.x, zo.y + bo.y, zo.z + bo.z, zo.w + bo.w}};
    const float cpv[4] = {cp.x, cp.y, cp.z, cp.w}, hpv[4] = {hp.x, hp.y, hp.z, hp.w};
    float ig[4], fg[4], gg[4], og[4], cn[4], hn[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      ig[e] = sigf(zin[0][e]);
      fg[e] = sigf(zin[1][e]);
      gg[e] = tanhf(zin[2][e]);
      og[e] = sigf(zin[3][e]);
      const float c2 = fg[e] * cpv[e] + ig[e] * gg[e];
      const float h2 = og[e] * tanhf(c2);
      cn[e] = live ? c2 : cpv[e];
      hn[e] = live ? h2 : hpv[e];
    }
    s4(w.Cs + sp + H, cn[0], cn[1], cn[2], cn[3]);
    s4(w.Hs + sp + H, hn[0], hn[1], hn[2], hn[3]);
    if (w.Hb && t + 1 < T) {
      __nv_bfloat162 lo = __floats2bfloat162_rn(hn[0], hn[1]), hi = __floats2bfloat162_rn(hn[2], hn[3]);
      uint2 u;
      u.x = *reinterpret_cast<uint32_t*>(&lo);
      u.y = *reinterpret_cast<uint32_t*>(&hi);
      *reinterpret_cast<uint2*>(w.Hb + ((long long)b * T + t + 1) * H + k) = u;
    }
    s4(z + k, ig[0], ig[1], ig[2], ig[3]);
    s4(z + H + k, fg[0], fg[1], fg[2], fg[3]);
    s4(z + 2 * H + k, gg[0], gg[1], gg[2], gg[3]);
    s4(z + 3 * H + k, og[0], og[1], og[2], og[3]);
  }
}

__device__ __forceinline__ void st_bf4(__nv_bfloat16* p, float a, float b, float c, float d) {
  __nv_bfloat162 lo = __floats2bfloat162_rn(a, b), hi = __floats2bfloat162_rn(c, d);
  uint2 u;
  u.x = *reinterpret_cast<uint32_t*>(&lo);
  u.y = *reinterpret_cast<uint32_t*>(&hi);
  *reinterpret_cast<uint2*>(p) = u;
}

__global__ void lstm_bwd_cell4(TrainBufs w, const float* __restrict__ y, const int64_t* __restrict__ lens, float inv_b,
                               int B, int T, int H, int t) {
  const int b = blockIdx.y;
  const bool live = t < lens[b];
  for (int k = 4 * (blockIdx.x * blockDim.x + threadIdx.x); k < H; k += 4 * gridDim.x * blockDim.x) {
    const long long i = (long long)b * H + k;
    float* z = w.Z + ((long long)b * T + t) * 4 * H;
    __nv_bfloat16* zb = w.Zb ? w.Zb + ((long long)b * T + t) * 4 * H : nullptr;
    float4 dh = f4(w.dh + i);
    if (live) {
      const float4 yv = f4(y + ((long long)b * T + t) * H + k);
      dh.x += yv.x * inv_b; dh.y += yv.y * inv_b; dh.z += yv.z * inv_b; dh.w += yv.w * inv_b;
    }
    if (!live) {   // frozen row: gradients pass straight through
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        s4(z + g * H + k, 0.f, 0.f, 0.f, 0.f);
        if (zb) st_bf4(zb + g * H + k, 0.f, 0.f, 0.f, 0.f);
      }
      s4(w.dh + i, dh.x, dh.y, dh.z, dh.w);
      continue;
    }
    const float4 dcv = f4(w.dc + i);
    const float4 ig4 = f4(z + k), fg4 = f4(z + H + k), gg4 = f4(z + 2 * H + k), og4 = f4(z + 3 * H + k);
    const long long sp = ((long long)b * (T + 1) + t) * H + k;
    const float4 cp4 = f4(w.Cs + sp), cn4 = f4(w.Cs + sp + H);
    const float dhv[4] = {dh.x, dh.y, dh.z, dh.w}, dcs[4] = {dcv.x, dcv.y, dcv.z, dcv.w};
    const float ig[4] = {ig4.x, ig4.y, ig4.z, ig4.w}, fg[4] = {fg4.x, fg4.y, fg4.z, fg4.w};
    const float gg[4] = {gg4.x, gg4.y, gg4.z, gg4.w}, og[4] = {og4.x, og4.y, og4.z, og4.w};
    const float cp[4] = {cp4.x, cp4.y, cp4.z, cp4.w}, cn[4] = {cn4.x, cn4.y, cn4.z, cn4.w};
    float di[4], df[4], dg[4], dO[4], dcn_out[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float tc = tanhf(cn[e]);
      const float dcn = dcs[e] + dhv[e] * og[e] * (1.f - tc * tc);
      di[e] = dcn * gg[e] * ig[e] * (1.f - ig[e]);
      df[e] = dcn * cp[e] * fg[e] * (1.f - fg[e]);
      dg[e] = dcn * ig[e] * (1.f - gg[e] * gg[e]);
      dO[e] = dhv[e] * tc * og[e] * (1.f - og[e]);
      dcn_out[e] = dcn * fg[e];
    }
    s4(z + k, di[0], di[1], di[2], di[3]);
    s4(z + H + k, df[0], df[1], df[2], df[3]);
    s4(z + 2 * H + k, dg[0], dg[1], dg[2], dg[3]);
    s4(z + 3 * H + k, dO[0], dO[1], dO[2], dO[3]);
    if (zb) {
      st_bf4(zb + k, di[0], di[1], di[2], di[3]);
      st_bf4(zb + H + k, df[0], df[1], df[2], df[3]);
      st_bf4(zb + 2 * H + k, dg[0], dg[1], dg[2], dg[3]);
      st_bf4(zb + 3 * H + k, dO[0], dO[1], dO[2], dO[3]);
    }
    s4(w.dc + i, dcn_out[0], dcn_out[1], dcn_out[2], dcn_out[3]);
    s4(w.dh + i, 0.f, 0.f, 0.f, 0.f);
  }
}

// loss partials: inv_b * sum over live (b, t) of <h_t, y_t>, fixed block order
__global__ void loss_partials(TrainBufs w, const float* __restrict__ y, const int64_t* __restrict__ lens, float inv_b,
                              int B, int T, int H, int n) {
  double acc = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < (long long)B * n * H;
       i += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(i % H);
    const long long bt = i / H;
    const int b = (int)(bt / n), t = (int)(bt % n);
    if (t < lens[b]) acc += (double)w.Hs[((long long)b * (T + 1) + t + 1) * H + k] * y[((long long)b * T + t) * H + k];
  }
  __shared__ double red[32];
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) s += red[q];
    w.part[blockIdx.x] = s * inv_b;
  }
}

__global__ void loss_final(const double* part, int n, float* loss) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int q = 0; q < n; ++q) s += part[q];
    *loss = (float)s;
  }
}

// db = column sums of dG over (b, t < n), deterministic: stage 1 sums a chunk of
// rows per (column, chunk) in a fixed order, stage 2 sums the chunks in order.
constexpr int kBiasChunks = 64;
__global__ void bias_grad_partial(TrainBufs w, float* __restrict__ part, int B, int T, int H, int n) {
  const int G = 4 * H;
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= G) return;
  const int chunk = blockIdx.y;
  const int b0 = (int)((long long)B * chunk / kBiasChunks), b1 = (int)((long long)B * (chunk + 1) / kBiasChunks);
  float s = 0.f;
  for (int b = b0; b < b1; ++b)
    for (int t = 0; t < n; ++t) s += w.Z[((long long)b * T + t) * G + col];
  part[(long long)chunk * G + col] = s;
}
__global__ void bias_grad_final(const float* __restrict__ part, float* __restrict__ db, int G) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= G) return;
  float s = 0.f;
  for (int c = 0; c < kBiasChunks; ++c) s += part[(long long)c * G + col];
  db[col] = s;
}

// rows t >= n of every sequence take no part in the step: zero their Z / dG so
// the whole-sequence gradient GEMMs (K = B*T) see exact zeros there
__global__ void zero_tail(TrainBufs w, int B, int T, int H, int n) {
  const long long G = 4ll * H, per = (long long)(T - n) * G;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < (long long)B * per;
       i += (long long)gridDim.x * blockDim.x) {
    const long long b = i / per, r = i % per;
    const long long off = (b * T + n) * G + r;
    w.Z[off] = 0.f;
    if (w.Zb) w.Zb[off] = __float2bfloat16(0.f);
  }
}

__global__ void sgd_update(float* __restrict__ p, const float* __restrict__ g, long long n, float lr) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] -= lr * g[i];
}

__global__ void to_bf16(const float* __restrict__ src, __nv_bfloat16* __restrict__ dst, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    dst[i] = __float2bfloat16(src[i]);
}

// bf16 operands, fp32 accumulate/output (math == 2); same row-major convention
bool gemm_bf(cublasHandle_t h, bool ta, bool tb, const __nv_bfloat16* A, int lda, const __nv_bfloat16* B, int ldb,
             float* C, int ldc, int M, int N, int K, float beta) {
  const float one = 1.f;
  return cublasGemmEx(h, tb ? CUBLAS_OP_T : CUBLAS_OP_N, ta ? CUBLAS_OP_T : CUBLAS_OP_N, N, M, K, &one, B,
                      CUDA_R_16BF, ldb, A, CUDA_R_16BF, lda, &beta, C, CUDA_R_32F, ldc, CUBLAS_COMPUTE_32F,
                      CUBLAS_GEMM_DEFAULT) == CUBLAS_STATUS_SUCCESS;
}

// C = op(A) @ op(B), row-major; column-major C^T = op(B)^T op(A)^T
bool gemm_rm(cublasHandle_t h, int math, bool ta, bool tb, const float* A, int lda, const float* B, int ldb, float* C,
             int ldc, int M, int N, int K, float beta) {
  const float one = 1.f;
  const cublasComputeType_t ct = math == 1 ? CUBLAS_COMPUTE_32F_FAST_TF32 : CUBLAS_COMPUTE_32F_PEDANTIC;
  return cublasGemmEx(h, tb ? CUBLAS_OP_T : CUBLAS_OP_N, ta ? CUBLAS_OP_T : CUBLAS_OP_N, N, M, K, &one, B,
                      CUDA_R_32F, ldb, A, CUDA_R_32F, lda, &beta, C, CUDA_R_32F, ldc, ct,
                      CUBLAS_GEMM_DEFAULT) == CUBLAS_STATUS_SUCCESS;
}

size_t al(size_t b) { return (b + 255) & ~size_t(255); }

void layout(int B, int T, int F, int H, bool bf16, uint8_t* base, TrainBufs* w, size_t* total) {
  size_t off = 0;
  auto take = [&](size_t bytes) { uint8_t* p = base ? base + off : nullptr; off += al(bytes); return p; };
  TrainBufs s;
  s.Z = (float*)take(4ull * B * T * 4 * H);
  s.Hs = (float*)take(4ull * B * (T + 1) * H);
  s.Cs = (float*)take(4ull * B * (T + 1) * H);
  s.dh = (float*)take(4ull * B * H);
  s.dc = (float*)take(4ull * B * H);
  s.part = (double*)take(8ull * kLossBlocks);
  s.bpart = (float*)take(4ull * kBiasChunks * 4 * H);
  if (bf16) {
    s.Xb = (__nv_bfloat16*)take(2ull * B * T * F);
    s.Hb = (__nv_bfloat16*)take(2ull * B * T * H);   // h_{t-1} of step t (GEMM operand)
    s.Zb = (__nv_bfloat16*)take(2ull * B * T * 4 * H);
    s.Wb = (__nv_bfloat16*)take(2ull * F * 4 * H);
    s.Ub = (__nv_bfloat16*)take(2ull * H * 4 * H);
  } else {
    s.Xb = s.Hb = s.Zb = s.Wb = s.Ub = nullptr;
  }
  if (w) *w = s;
  if (total) *total = off;
}

bool enqueue(cublasHandle_t hb, cudaStream_t cs, const skb_train_shape& d, TrainBufs& w, const float* x,
             const float* y, const int64_t* lens, const float* h0, const float* c0, const float* params,
             float* grads, float* loss, int n) {
  const int B = d.rows, T = d.time, F = d.input, H = d.hidden, G = 4 * H;
  const float* W = params;
  const float* U = params + (size_t)F * G;
  const float* bias = U + (size_t)H * G;
  float* dW = grads;
  float* dU = grads + (size_t)F * G;
  float* db = dU + (size_t)H * G;
  const int blocks = 148 * 8;
  const float inv_b = d.inv_batch;
  init_states<<<blocks, 256, 0, cs>>>(h0, c0, w, B, T, H);
  cudaMemsetAsync(grads, 0, sizeof(float) * ((size_t)F * G + (size_t)H * G), cs);
  const bool bf = d.math == 2;
  const bool v4 = (H & 3) == 0 && !getenv("SKB_TRAIN_SCALAR");   // float4 cell kernels
  if (bf) {   // bf16 copies of the GEMM operands that do not change during the step
    to_bf16<<<blocks, 256, 0, cs>>>(x, w.Xb, (long long)B * T * F);
    to_bf16<<<blocks, 256, 0, cs>>>(W, w.Wb, (long long)F * G);
    to_bf16<<<blocks, 256, 0, cs>>>(U, w.Ub, (long long)H * G);
  }
  // input projection of every step at once: Z = X W (rows (b, t), K = F)
  if (bf) {
    if (!gemm_bf(hb, false, false, w.Xb, F, w.Wb, G, w.Z, G, B * T, G, F, 0.f)) return false;
  } else if (!gemm_rm(hb, d.math, false, false, x, F, W, G, w.Z, G, B * T, G, F, 0.f)) {
    return false;
  }
  for (int t = 0; t < n; ++t) {   // the recurrence: Z_t += h_{t-1} U, then the cell
    float* Zt = w.Z + (size_t)t * G;
    if (bf) {
      if (!gemm_bf(hb, false, false, w.Hb + (size_t)t * H, T * H, w.Ub, G, Zt, T * G, B, G, H, 1.f)) return false;
    } else if (!gemm_rm(hb, d.math, false, false, w.Hs + (size_t)t * H, (T + 1) * H, U, G, Zt, T * G, B, G, H, 1.f)) {
      return false;
    }
    if (v4)
      lstm_fwd_cell4<<<dim3((H / 4 + 255) / 256, B), H / 4 < 256 ? ((H / 4 + 31) / 32) * 32 : 256, 0, cs>>>(
          w, bias, lens, B, T, H, t);
    else
      lstm_fwd_cell<<<dim3((H + 255) / 256, B), 256, 0, cs>>>(w, bias, lens, B, T, H, t);
  }
  loss_partials<<<kLossBlocks, 256, 0, cs>>>(w, y, lens, inv_b, B, T, H, n);
  loss_final<<<1, 32, 0, cs>>>(w.part, kLossBlocks, loss);
  for (int t = n - 1; t >= 0; --t) {   // BPTT: only dh_{t-1} = dG_t U^T + carry stays per step
    float* Zt = w.Z + (size_t)t * G;
    if (v4)
      lstm_bwd_cell4<<<dim3((H / 4 + 255) / 256, B), H / 4 < 256 ? ((H / 4 + 31) / 32) * 32 : 256, 0, cs>>>(
          w, y, lens, inv_b, B, T, H, t);
    else
      lstm_bwd_cell<<<dim3((H + 255) / 256, B), 256, 0, cs>>>(w, y, lens, inv_b, B, T, H, t);
    if (bf) {
      if (!gemm_bf(hb, false, true, w.Zb + (size_t)t * G, T * G, w.Ub, G, w.dh, H, B, H, G, 1.f)) return false;
    } else {
      if (!gemm_rm(hb, d.math, false, true, Zt, T * G, U, G, w.dh, H, B, H, G, 1.f)) return false;
      if (!gemm_rm(hb, d.math, true, false, w.Hs + (size_t)t * H, (T + 1) * H, Zt, T * G, dU, G, H, G, B, 1.f))
        return false;
    }
  }
  if (n < T) zero_tail<<<blocks, 256, 0, cs>>>(w, B, T, H, n);
  // weight gradients over every (b, t) at once (K = B*T): dW = X^T dG, dU = H_prev^T dG
  if (bf) {
    if (!gemm_bf(hb, true, false, w.Xb, F, w.Zb, G, dW, G, F, G, B * T, 0.f)) return false;
    if (!gemm_bf(hb, true, false, w.Hb, H, w.Zb, G, dU, G, H, G, B * T, 0.f)) return false;
  } else if (!gemm_rm(hb, d.math, true, false, x, F, w.Z, G, dW, G, F, G, B * T, 0.f)) {
    return false;
  }
  bias_grad_partial<<<dim3((G + 255) / 256, kBiasChunks), 256, 0, cs>>>(w, w.bpart, B, T, H, n);
  bias_grad_final<<<(G + 255) / 256, 256, 0, cs>>>(w.bpart, db, G);
  return cudaPeekAtLastError() == cudaSuccess;
}

struct TrainGraph {
  skb_train_shape d;
  const void* ptrs[9];
  int n;
  cudaGraphExec_t exec;
};
constexpr int kTrainGraphs = 8;
TrainGraph g_tg[kTrainGraphs];
int g_ntg = 0;
int g_train_mode = 0;

}  // namespace

extern "C" int64_t skb_train_tc_workspace_bytes(const skb_train_shape* d);
extern "C" int skb_train_tc_enqueue(const skb_train_shape* d, const float* x, const float* y, const int64_t* lens,
                                    const float* h0, const float* c0, const float* params, float* grads, float* loss,
                                    int n, void* workspace, void* stream);

namespace {
// math == 2 (bf16): the tensor-core path of train_tc.cu (skb's own tcgen05 GEMMs with the
// cell fused into their epilogues); SKB_TRAIN_CUBLAS=1 keeps the round-1 cuBLAS bf16 path.
bool use_tc(const skb_train_shape* d) {
  static int v = -1, sms = 0;
  if (v < 0) {
    const char* e = getenv("SKB_TRAIN_CUBLAS");
    v = (e && atoi(e) == 1) ? 0 : 1;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      sms = 148;
    cudaGetLastError();
  }
  // the persistent step kernels keep one CTA per (128-row tile, 32 hidden units) resident
  const long long ctas = (long long)((d->rows + 127) / 128) * (d->hidden / 32);
  return v == 1 && d->math == 2 && d->input % 8 == 0 && d->hidden % 32 == 0 && ctas <= sms;
}
}  // namespace

extern "C" int64_t skb_train_workspace_bytes(const skb_train_shape* d) {
  if (!d) return -1;
  if (use_tc(d)) return skb_train_tc_workspace_bytes(d);
  size_t total = 0;
  layout(d->rows, d->time, d->input, d->hidden, d->math == 2, nullptr, nullptr, &total);
  return (int64_t)total;
}

extern "C" int skb_train_last_mode(void) { return g_train_mode; }

// 1: skb_lstm_train_step runs on the tcgen05 engine for this shape (and accepts max_len = -1,
// the While trip count determined on the device: no host round trip per step).
extern "C" int skb_train_uses_engine(const skb_train_shape* d) { return d && use_tc(d) ? 1 : 0; }

extern "C" skb_status skb_lstm_train_step(const skb_train_shape* d, const float* x, const float* y,
                                          const int64_t* lens, const float* h0, const float* c0, const float* params,
                                          float* grads, float* loss, int max_len, void* workspace, void* stream) {
  // max_len < 0: the trip count is determined on the device (engine path only)
  if (!d || d->rows < 1 || d->time < 1 || d->input < 1 || d->hidden < 1 || max_len > d->time ||
      (max_len < 0 && !use_tc(d)))
    return SKB_ERR_INVALID;
  if (max_len < 0) max_len = -1;
  cudaStream_t cs = (cudaStream_t)stream;
  const bool tc = use_tc(d);
  TrainBufs w;
  layout(d->rows, d->time, d->input, d->hidden, d->math == 2, (uint8_t*)workspace, &w, nullptr);
  cublasHandle_t hb = tc ? nullptr : skb::blas_handle(cs);
  if (!tc && !hb) return SKB_ERR_CUDA;
  auto enq = [&](cudaStream_t s) -> bool {
    if (tc) {
      if (max_len == 0) {   // no step: zero loss and gradients
        cudaMemsetAsync(loss, 0, sizeof(float), s);
        cudaMemsetAsync(grads, 0, sizeof(float) * ((size_t)d->input * 4 * d->hidden + (size_t)d->hidden * 4 * d->hidden +
                                                  4 * (size_t)d->hidden), s);
        return cudaPeekAtLastError() == cudaSuccess;
      }
      return skb_train_tc_enqueue(d, x, y, lens, h0, c0, params, grads, loss, max_len, workspace, s) == SKB_OK;
    }
    return enqueue(hb, s, *d, w, x, y, lens, h0, c0, params, grads, loss, max_len);
  };
  const void* key[9] = {x, y, lens, h0, c0, params, grads, loss, workspace};
  cudaGraphExec_t exec = nullptr;
  for (int i = 0; i < g_ntg; ++i)
    if (g_tg[i].n == max_len && memcmp(&g_tg[i].d, d, sizeof(*d)) == 0 && memcmp(g_tg[i].ptrs, key, sizeof(key)) == 0)
      exec = g_tg[i].exec;
  if (!exec && d->graph) {
    cudaStream_t cap = nullptr;
    cudaGraph_t g = nullptr;
    bool ok = cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking) == cudaSuccess &&
              cudaStreamBeginCapture(cap, cudaStreamCaptureModeRelaxed) == cudaSuccess;
    if (ok) {
      if (hb) cublasSetStream(hb, cap);
      const bool e = enq(cap);
      ok = cudaStreamEndCapture(cap, &g) == cudaSuccess && e;
    }
    if (ok) ok = cudaGraphInstantiate(&exec, g, 0) == cudaSuccess;
    if (g) cudaGraphDestroy(g);
    if (cap) cudaStreamDestroy(cap);
    if (hb) cublasSetStream(hb, cs);
    cudaGetLastError();
    if (!ok) exec = nullptr;
    if (exec) {
      if (g_ntg == kTrainGraphs) {
        cudaGraphExecDestroy(g_tg[0].exec);
        memmove(g_tg, g_tg + 1, sizeof(TrainGraph) * (kTrainGraphs - 1));
        --g_ntg;
      }
      TrainGraph& e = g_tg[g_ntg++];
      e.d = *d;
      memcpy(e.ptrs, key, sizeof(key));
      e.n = max_len;
      e.exec = exec;
    }
  }
  g_train_mode = exec ? 1 : 0;
  if (exec) {
    if (cudaGraphLaunch(exec, cs) != cudaSuccess) return SKB_ERR_CUDA;
  } else if (!enq(cs)) {
    return SKB_ERR_CUDA;
  }
  return skb_check_launch();
}

extern "C" skb_status skb_sgd_update(float* params, const float* grads, int64_t n, float lr, void* stream) {
  if (n < 0) return SKB_ERR_INVALID;
  sgd_update<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(params, grads, n, lr);
  return skb_check_launch();
}
