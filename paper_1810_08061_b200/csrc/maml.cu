// maml.cu — MAML sinusoid meta-gradient (BASELINE config C5).
//
// The reference differentiates the staged one-task program
// oracle/programs/maml.msl (MLP 1-H-H-1, ReLU as where(z>0,z,0*z), one
// hand-written inner SGD step) with gradient() (graph/grad.py:35-70), second
// order included, and executes the result once per task.  Here one CTA owns a
// task and keeps everything in shared memory:
//   support forward + backward       -> g_s, theta' = theta - alpha g_s
//   query forward + backward at theta' -> g_q (= v)
//   R-operator of the support pass along v -> H_s v
//   meta-gradient = g_q - alpha H_s v      (closed form of the reference's
//                                            second-order adjoint; oracle/maml.py)
// Per-task meta-gradients are summed in a fixed task order (deterministic) and
// averaged; the cross-GPU allreduce (tasks sharded) and the meta-update follow.
#include <cuda_runtime.h>
#include <stdint.h>
#include "skb_internal.h"

namespace {

constexpr int HMAX = 64, KMAXT = 32, TPB = 256;

// Shared-memory parameter block: w1 | b1 | w2 (H rows of stride LD = H + 1, so
// column walks are bank-conflict free) | b2 | w3 | b3.  Global memory holds the
// flat, unpadded layout (P = H*H + 4H + 1).
struct Theta {
  float *w1, *b1, *w2, *b2, *w3, *b3;
  int ld;
};
__device__ __forceinline__ Theta view(float* p, int H) {
  Theta t;
  t.ld = H + 1;
  t.w1 = p; t.b1 = p + H; t.w2 = p + 2 * H; t.b2 = t.w2 + H * t.ld; t.w3 = t.b2 + H; t.b3 = t.w3 + H;
  return t;
}
__device__ __forceinline__ int padded_of(int i, int H) {   // flat index -> padded index
  const int w2o = 2 * H, w2e = 2 * H + H * H;
  if (i < w2o) return i;
  if (i < w2e) { const int r = (i - w2o) / H, c = (i - w2o) % H; return w2o + r * (H + 1) + c; }
  return i + H;
}

// y[K,H] = relu-input z = x w1 + b1 (x: [K], w1: [H])
__device__ __forceinline__ void layer1(const float* x, const float* w1, const float* b1, float* z, float* a, int K, int H) {
  for (int i = threadIdx.x; i < K * H; i += TPB) {
    const int k = i / H, j = i % H;
    const float v = x[k] * w1[j] + b1[j];
    z[i] = v;
    if (a) a[i] = v > 0.f ? v : 0.f;
  }
}
// z2[K,H] = a1 @ w2 + b2
__device__ __forceinline__ void layer2(const float* a1, const float* w2, const float* b2, float* z2, float* a2, int K, int H) {
  for (int i = threadIdx.x; i < K * H; i += TPB) {
    const int k = i / H, j = i % H;
    float s = 0.f;
    for (int q = 0; q < H; ++q) s += a1[k * H + q] * w2[q * (H + 1) + j];
    s += b2[j];
    z2[i] = s;
    if (a2) a2[i] = s > 0.f ? s : 0.f;
  }
}
// p[K] = a2 @ w3 + b3
__device__ __forceinline__ void layer3(const float* a2, const float* w3, const float* b3, float* p, int K, int H) {
  for (int k = threadIdx.x; k < K; k += TPB) {
    float s = 0.f;
    for (int q = 0; q < H; ++q) s += a2[k * H + q] * w3[q];
    p[k] = s + b3[0];
  }
}

// Backward of the MLP for output adjoint dp[K]; writes gradients into g.
// dz2 / dz1 scratch [K,H].  All extra operands optional (R-op reuse).
__device__ __forceinline__ void backward(const float* x, Theta th, const float* z1, const float* a1, const float* z2,
                         const float* a2, const float* dp, float* dz1, float* dz2, Theta g, int K, int H) {
  for (int i = threadIdx.x; i < K * H; i += TPB) {   // dz2 = (dp w3^T) * [z2 > 0]
    const int k = i / H, j = i % H;
    dz2[i] = z2[i] > 0.f ? dp[k] * th.w3[j] : 0.f;
  }
  for (int j = threadIdx.x; j < H; j += TPB) {      // gw3 = a2^T dp, gb3
    float s = 0.f;
    for (int k = 0; k < K; ++k) s += a2[k * H + j] * dp[k];
    g.w3[j] = s;
  }
  if (threadIdx.x == 0) {
    float s = 0.f;
    for (int k = 0; k < K; ++k) s += dp[k];
    g.b3[0] = s;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < H * H; i += TPB) {  // gw2 = a1^T dz2
    const int q = i / H, j = i % H;
    float s = 0.f;
    for (int k = 0; k < K; ++k) s += a1[k * H + q] * dz2[k * H + j];
    g.w2[q * g.ld + j] = s;
  }
  for (int j = threadIdx.x; j < H; j += TPB) {
    float s = 0.f;
    for (int k = 0; k < K; ++k) s += dz2[k * H + j];
    g.b2[j] = s;
  }
  for (int i = threadIdx.x; i < K * H; i += TPB) {  // dz1 = (dz2 w2^T) * [z1 > 0]
    const int k = i / H, q = i % H;
    float s = 0.f;
    for (int j = 0; j < H; ++j) s += dz2[k * H + j] * th.w2[q * th.ld + j];
    dz1[i] = z1[i] > 0.f ? s : 0.f;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < H; j += TPB) {      // gw1 = x^T dz1, gb1
    float s = 0.f, t = 0.f;
    for (int k = 0; k < K; ++k) { s += x[k] * dz1[k * H + j]; t += dz1[k * H + j]; }
    g.w1[j] = s;
    g.b1[j] = t;
  }
  __syncthreads();
}

// ---- register-tiled forms of the H x H contractions (compile-time H % 4 == 0, even K; every
// activation array starts 16-byte aligned then).  The loops above read two shared-memory words
// per FMA, which bounds the kernel by the LDS pipe; here a thread computes two rows (k, k + K/2)
// or four consecutive columns and reads the contiguous operand as float4, so one LDS feeds
// 1.3-4 FMAs.  Summation order within an output is unchanged.
template <int H, int K>
__device__ __forceinline__ void layer2_t(const float* a1, const float* w2, const float* b2, float* z2, float* a2) {
  constexpr int LD = H + 1, K2 = K / 2;
  for (int i = threadIdx.x; i < K2 * H; i += TPB) {
    const int k0 = i / H, j = i % H;
    const float4* x0 = reinterpret_cast<const float4*>(a1 + k0 * H);
    const float4* x1 = reinterpret_cast<const float4*>(a1 + (k0 + K2) * H);
    float s0 = 0.f, s1 = 0.f;
#pragma unroll
    for (int q4 = 0; q4 < H / 4; ++q4) {
      const float4 u = x0[q4], v = x1[q4];
      const float* w = w2 + 4 * q4 * LD + j;
      const float w0 = w[0], w1 = w[LD], w2_ = w[2 * LD], w3 = w[3 * LD];
      s0 += u.x * w0; s0 += u.y * w1; s0 += u.z * w2_; s0 += u.w * w3;
      s1 += v.x * w0; s1 += v.y * w1; s1 += v.z * w2_; s1 += v.w * w3;
    }
    s0 += b2[j];
    s1 += b2[j];
    z2[k0 * H + j] = s0;
    z2[(k0 + K2) * H + j] = s1;
    if (a2) { a2[k0 * H + j] = s0 > 0.f ? s0 : 0.f; a2[(k0 + K2) * H + j] = s1 > 0.f ? s1 : 0.f; }
  }
}
// out[q][4jj..4jj+3] (row stride LD) = sum_k P[k][q] Q[k][4jj..] (+ R[k][q] S[k][4jj..] when R)
template <int H, int K>
__device__ __forceinline__ void outer_t(const float* P, const float* Q, const float* R, const float* S, float* out) {
  constexpr int LD = H + 1, J4 = H / 4;
  for (int i = threadIdx.x; i < H * J4; i += TPB) {
    const int q = i / J4, jj = i % J4;
    float s[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const float p = P[k * H + q];
      const float4 d = reinterpret_cast<const float4*>(Q + k * H)[jj];
      if (R) {
        const float r = R[k * H + q];
        const float4 e = reinterpret_cast<const float4*>(S + k * H)[jj];
        s[0] += p * d.x + r * e.x; s[1] += p * d.y + r * e.y; s[2] += p * d.z + r * e.z; s[3] += p * d.w + r * e.w;
      } else {
        s[0] += p * d.x; s[1] += p * d.y; s[2] += p * d.z; s[3] += p * d.w;
      }
    }
#pragma unroll
    for (int m = 0; m < 4; ++m) out[q * LD + 4 * jj + m] = s[m];
  }
}
// out[k][q] = [z[k][q] > 0] sum_j D[k][j] W[q][j] (+ E[k][j] V[q][j] when E); W, V row stride LD
template <int H, int K>
__device__ __forceinline__ void back_t(const float* D, const float* W, const float* E, const float* V, const float* z,
                                       float* out) {
  constexpr int LD = H + 1, K2 = K / 2;
  for (int i = threadIdx.x; i < K2 * H; i += TPB) {
    const int k0 = i / H, q = i % H;
    const float4* d0 = reinterpret_cast<const float4*>(D + k0 * H);
    const float4* d1 = reinterpret_cast<const float4*>(D + (k0 + K2) * H);
    const float* w = W + q * LD;
    float s0 = 0.f, s1 = 0.f;
    if (E) {
      const float4* e0 = reinterpret_cast<const float4*>(E + k0 * H);
      const float4* e1 = reinterpret_cast<const float4*>(E + (k0 + K2) * H);
      const float* v = V + q * LD;
#pragma unroll
      for (int j4 = 0; j4 < H / 4; ++j4) {
        const float4 a = d0[j4], b = d1[j4], c = e0[j4], e = e1[j4];
        const float w0 = w[4 * j4], w1 = w[4 * j4 + 1], w2 = w[4 * j4 + 2], w3 = w[4 * j4 + 3];
        const float v0 = v[4 * j4], v1 = v[4 * j4 + 1], v2 = v[4 * j4 + 2], v3 = v[4 * j4 + 3];
        s0 += a.x * w0 + c.x * v0; s0 += a.y * w1 + c.y * v1; s0 += a.z * w2 + c.z * v2; s0 += a.w * w3 + c.w * v3;
        s1 += b.x * w0 + e.x * v0; s1 += b.y * w1 + e.y * v1; s1 += b.z * w2 + e.z * v2; s1 += b.w * w3 + e.w * v3;
      }
    } else {
#pragma unroll
      for (int j4 = 0; j4 < H / 4; ++j4) {
        const float4 a = d0[j4], b = d1[j4];
        const float w0 = w[4 * j4], w1 = w[4 * j4 + 1], w2 = w[4 * j4 + 2], w3 = w[4 * j4 + 3];
        s0 += a.x * w0; s0 += a.y * w1; s0 += a.z * w2; s0 += a.w * w3;
        s1 += b.x * w0; s1 += b.y * w1; s1 += b.z * w2; s1 += b.w * w3;
      }
    }
    out[k0 * H + q] = z[k0 * H + q] > 0.f ? s0 : 0.f;
    out[(k0 + K2) * H + q] = z[(k0 + K2) * H + q] > 0.f ? s1 : 0.f;
  }
}
// R{a2}[k][j] = [z2 > 0] (vb2[j] + sum_q r1[k][q] w2[q][j] + a1[k][q] vw2[q][j])
template <int H, int K>
__device__ __forceinline__ void rop2_t(const float* r1, const float* a1, const float* w2, const float* vw2,
                                       const float* vb2, const float* z2, float* r2) {
  constexpr int LD = H + 1, K2 = K / 2;
  for (int i = threadIdx.x; i < K2 * H; i += TPB) {
    const int k0 = i / H, j = i % H;
    const float4* x0 = reinterpret_cast<const float4*>(r1 + k0 * H);
    const float4* x1 = reinterpret_cast<const float4*>(r1 + (k0 + K2) * H);
    const float4* y0 = reinterpret_cast<const float4*>(a1 + k0 * H);
    const float4* y1 = reinterpret_cast<const float4*>(a1 + (k0 + K2) * H);
    float s0 = vb2[j], s1 = vb2[j];
#pragma unroll
    for (int q4 = 0; q4 < H / 4; ++q4) {
      const float4 a = x0[q4], b = x1[q4], c = y0[q4], d = y1[q4];
      const float* w = w2 + 4 * q4 * LD + j;
      const float* v = vw2 + 4 * q4 * LD + j;
      const float w0 = w[0], w1 = w[LD], w2_ = w[2 * LD], w3 = w[3 * LD];
      const float v0 = v[0], v1 = v[LD], v2 = v[2 * LD], v3 = v[3 * LD];
      s0 += a.x * w0 + c.x * v0; s0 += a.y * w1 + c.y * v1; s0 += a.z * w2_ + c.z * v2; s0 += a.w * w3 + c.w * v3;
      s1 += b.x * w0 + d.x * v0; s1 += b.y * w1 + d.y * v1; s1 += b.z * w2_ + d.z * v2; s1 += b.w * w3 + d.w * v3;
    }
    r2[k0 * H + j] = z2[k0 * H + j] > 0.f ? s0 : 0.f;
    r2[(k0 + K2) * H + j] = z2[(k0 + K2) * H + j] > 0.f ? s1 : 0.f;
  }
}
// backward() with the two H x H contractions register-tiled
template <int H, int K>
__device__ __forceinline__ void backward_t(const float* x, Theta th, const float* z1, const float* a1, const float* z2,
                                           const float* a2, const float* dp, float* dz1, float* dz2, Theta g) {
  for (int i = threadIdx.x; i < K * H; i += TPB) {
    const int k = i / H, j = i % H;
    dz2[i] = z2[i] > 0.f ? dp[k] * th.w3[j] : 0.f;
  }
  for (int j = threadIdx.x; j < H; j += TPB) {
    float s = 0.f;
    for (int k = 0; k < K; ++k) s += a2[k * H + j] * dp[k];
    g.w3[j] = s;
  }
  if (threadIdx.x == 0) {
    float s = 0.f;
    for (int k = 0; k < K; ++k) s += dp[k];
    g.b3[0] = s;
  }
  __syncthreads();
  outer_t<H, K>(a1, dz2, nullptr, nullptr, g.w2);   // gw2 = a1^T dz2
  for (int j = threadIdx.x; j < H; j += TPB) {
    float s = 0.f;
    for (int k = 0; k < K; ++k) s += dz2[k * H + j];
    g.b2[j] = s;
  }
  back_t<H, K>(dz2, th.w2, nullptr, nullptr, z1, dz1);   // dz1 = (dz2 w2^T) [z1 > 0]
  __syncthreads();
  for (int j = threadIdx.x; j < H; j += TPB) {
    float s = 0.f, t = 0.f;
    for (int k = 0; k < K; ++k) { s += x[k] * dz1[k * H + j]; t += dz1[k * H + j]; }
    g.w1[j] = s;
    g.b1[j] = t;
  }
  __syncthreads();
}

// HC > 0: the hidden width as a compile-time constant (every K x H / H x H loop's
// index division becomes a multiply-shift); HC == 0: runtime width.
template <int HC, int KC = 0>
__global__ void __launch_bounds__(TPB) maml_task_kernel(int H_, int K_, int P, const float* __restrict__ theta_g,
                                                        const float* __restrict__ xs, const float* __restrict__ ys,
                                                        const float* __restrict__ xq, const float* __restrict__ yq,
                                                        float alpha, float* __restrict__ task_grad,
                                                        float* __restrict__ task_loss) {
  extern __shared__ float sm[];
  const int H = HC ? HC : H_;
  const int K = KC ? KC : K_;
  const int task = blockIdx.x;
  const int KH = K * H;
  const int PP = P + H;          // padded block (w2 rows of H + 1)
  float* th_p = sm;              // PP
  // gs_p: the support gradient, turned in place into the adapted weights theta' (the gradient
  // itself is not read again), then -- once the query pass is done with theta' -- H_s v.
  // The R-operator's R{a1} / R{a2} reuse the query pass's z / a buffers (dead by then).
  // 3 PP + 12 KH floats: five CTAs per SM at H = 40, K = 10.
  float* gs_p = th_p + PP;
  float* gq_p = gs_p + PP;       // PP query gradient (= v)
  float* z1 = sm + ((3 * PP + 3) & ~3);   // activations 16-byte aligned (float4 reads)
  float* a1 = z1 + KH; float* z2 = a1 + KH; float* a2 = z2 + KH;
  float* dz1 = a2 + KH; float* dz2 = dz1 + KH;
  float* q1 = dz2 + KH; float* qa1 = q1 + KH; float* q2 = qa1 + KH; float* qa2 = q2 + KH;
  float* r1 = q1; float* r2 = qa1; float* rd2 = qa2 + KH; float* rd1 = rd2 + KH;
  float* x = rd1 + KH; float* y = x + KMAXT; float* xqs = y + KMAXT; float* yqs = xqs + KMAXT;
  float* p = yqs + KMAXT; float* dp = p + KMAXT; float* rp = dp + KMAXT; float* rdp = rp + KMAXT;
  for (int i = threadIdx.x; i < PP; i += TPB) th_p[i] = 0.f;
  __syncthreads();
  for (int i = threadIdx.x; i < P; i += TPB) th_p[padded_of(i, H)] = theta_g[i];
  for (int k = threadIdx.x; k < K; k += TPB) {
    x[k] = xs[(long long)task * K + k]; y[k] = ys[(long long)task * K + k];
    xqs[k] = xq[(long long)task * K + k]; yqs[k] = yq[(long long)task * K + k];
  }
  __syncthreads();
  const Theta th = view(th_p, H), th2 = view(gs_p, H), gs = view(gs_p, H), gq = view(gq_p, H);
  const float inv_k = 1.f / (float)K;
  constexpr bool TILED = HC > 0 && KC > 0 && HC % 4 == 0 && KC % 2 == 0;
  // support pass
  layer1(x, th.w1, th.b1, z1, a1, K, H);
  __syncthreads();
  if constexpr (TILED) layer2_t<HC, KC>(a1, th.w2, th.b2, z2, a2); else layer2(a1, th.w2, th.b2, z2, a2, K, H);
  __syncthreads();
  layer3(a2, th.w3, th.b3, p, K, H);
  __syncthreads();
  for (int k = threadIdx.x; k < K; k += TPB) dp[k] = (p[k] - y[k]) * (2.f * inv_k);
  __syncthreads();
  if constexpr (TILED) backward_t<HC, KC>(x, th, z1, a1, z2, a2, dp, dz1, dz2, gs);
  else backward(x, th, z1, a1, z2, a2, dp, dz1, dz2, gs, K, H);
  for (int i = threadIdx.x; i < PP; i += TPB) gs_p[i] = th_p[i] - alpha * gs_p[i];   // theta', in place
  __syncthreads();
  // query pass at theta'
  layer1(xqs, th2.w1, th2.b1, q1, qa1, K, H);
  __syncthreads();
  if constexpr (TILED) layer2_t<HC, KC>(qa1, th2.w2, th2.b2, q2, qa2); else layer2(qa1, th2.w2, th2.b2, q2, qa2, K, H);
  __syncthreads();
  layer3(qa2, th2.w3, th2.b3, rp, K, H);   // rp holds the query prediction for now
  __syncthreads();
  if (threadIdx.x == 0) {
    float l = 0.f;
    for (int k = 0; k < K; ++k) { const float e = rp[k] - yqs[k]; l += e * e; }
    task_loss[task] = l * inv_k;
  }
  for (int k = threadIdx.x; k < K; k += TPB) rdp[k] = (rp[k] - yqs[k]) * (2.f * inv_k);
  __syncthreads();
  if constexpr (TILED) backward_t<HC, KC>(xqs, th2, q1, qa1, q2, qa2, rdp, rd1, rd2, gq);
  else backward(xqs, th2, q1, qa1, q2, qa2, rdp, rd1, rd2, gq, K, H);
  // R-operator of the support pass along v = g_q
  const Theta v = gq;
  for (int i = threadIdx.x; i < KH; i += TPB) {      // R{a1} = (x v_w1 + v_b1) [z1>0]
    const int k = i / H, j = i % H;
    const float rz = x[k] * v.w1[j] + v.b1[j];
    r1[i] = z1[i] > 0.f ? rz : 0.f;
  }
  __syncthreads();
  if constexpr (TILED) {
    rop2_t<HC, KC>(r1, a1, th.w2, v.w2, v.b2, z2, r2);
  } else {
    for (int i = threadIdx.x; i < KH; i += TPB) {      // R{a2} = (R{a1} w2 + a1 v_w2 + v_b2) [z2>0]
      const int k = i / H, j = i % H;
      float s = v.b2[j];
      for (int q = 0; q < H; ++q) s += r1[k * H + q] * th.w2[q * th.ld + j] + a1[k * H + q] * v.w2[q * v.ld + j];
      r2[i] = z2[i] > 0.f ? s : 0.f;
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < K; k += TPB) {       // R{dp} = (2/K)(R{a2} w3 + a2 v_w3 + v_b3)
    float s = v.b3[0];
    for (int q = 0; q < H; ++q) s += r2[k * H + q] * th.w3[q] + a2[k * H + q] * v.w3[q];
    rdp[k] = s * (2.f * inv_k);
  }
  __syncthreads();
  // H_s v, written over g_s: w3/b3, then R{dz2}, w2/b2, R{dz1}, w1/b1
  for (int j = threadIdx.x; j < H; j += TPB) {
    float s = 0.f;
    for (int k = 0; k < K; ++k) s += r2[k * H + j] * dp[k] + a2[k * H + j] * rdp[k];
    gs.w3[j] = s;
  }
  if (threadIdx.x == 0) {
    float s = 0.f;
    for (int k = 0; k < K; ++k) s += rdp[k];
    gs.b3[0] = s;
  }
  for (int i = threadIdx.x; i < KH; i += TPB) {      // R{dz2} = (R{dp} w3^T + dp v_w3^T) [z2>0]
    const int k = i / H, j = i % H;
    rd2[i] = z2[i] > 0.f ? rdp[k] * th.w3[j] + dp[k] * v.w3[j] : 0.f;
  }
  __syncthreads();
  if constexpr (TILED) {
    outer_t<HC, KC>(r1, dz2, a1, rd2, gs.w2);   // R{gw2} = R{a1}^T dz2 + a1^T R{dz2}
  } else {
    for (int i = threadIdx.x; i < H * H; i += TPB) {   // R{gw2} = R{a1}^T dz2 + a1^T R{dz2}
      const int q = i / H, j = i % H;
      float s = 0.f;
      for (int k = 0; k < K; ++k) s += r1[k * H + q] * dz2[k * H + j] + a1[k * H + q] * rd2[k * H + j];
      gs.w2[q * gs.ld + j] = s;
    }
  }
  for (int j = threadIdx.x; j < H; j += TPB) {
    float s = 0.f;
    for (int k = 0; k < K; ++k) s += rd2[k * H + j];
    gs.b2[j] = s;
  }
  if constexpr (TILED) {
    back_t<HC, KC>(rd2, th.w2, dz2, v.w2, z1, rd1);   // R{dz1} = (R{dz2} w2^T + dz2 v_w2^T) [z1>0]
  } else {
    for (int i = threadIdx.x; i < KH; i += TPB) {      // R{dz1} = (R{dz2} w2^T + dz2 v_w2^T) [z1>0]
      const int k = i / H, q = i % H;
      float s = 0.f;
      for (int j = 0; j < H; ++j) s += rd2[k * H + j] * th.w2[q * th.ld + j] + dz2[k * H + j] * v.w2[q * v.ld + j];
      rd1[i] = z1[i] > 0.f ? s : 0.f;
    }
  }
  __syncthreads();
  for (int j = threadIdx.x; j < H; j += TPB) {
    float s = 0.f, t = 0.f;
    for (int k = 0; k < K; ++k) { s += x[k] * rd1[k * H + j]; t += rd1[k * H + j]; }
    gs.w1[j] = s;
    gs.b1[j] = t;
  }
  __syncthreads();
  float* out = task_grad + (long long)task * P;
  for (int i = threadIdx.x; i < P; i += TPB) {
    const int pi = padded_of(i, H);
    out[i] = gq_p[pi] - alpha * gs_p[pi];
  }
}

// mean over tasks in a fixed order (deterministic): stage 1 sums a chunk of
// tasks per (parameter, chunk), stage 2 sums the chunks in order.
constexpr int kTaskChunks = 64;
__global__ void maml_reduce_partial(const float* __restrict__ task_grad, const float* __restrict__ task_loss, int n,
                                    int P, double* __restrict__ part) {
  const int chunk = blockIdx.y;
  const int t0 = (int)((long long)n * chunk / kTaskChunks), t1 = (int)((long long)n * (chunk + 1) / kTaskChunks);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= P; i += gridDim.x * blockDim.x) {
    double s = 0.0;
    if (i < P) {
      for (int t = t0; t < t1; ++t) s += task_grad[(long long)t * P + i];
    } else {
      for (int t = t0; t < t1; ++t) s += task_loss[t];
    }
    part[(long long)chunk * (P + 1) + i] = s;
  }
}
__global__ void maml_reduce_final(const double* __restrict__ part, int n, int P, float* __restrict__ grad,
                                  float* __restrict__ loss) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= P; i += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int c = 0; c < kTaskChunks; ++c) s += part[(long long)c * (P + 1) + i];
    if (i < P) grad[i] = (float)(s / n); else loss[0] = (float)(s / n);
  }
}

size_t smem_for(int H, int K) {
  const int P = H * H + 4 * H + 1;
  return sizeof(float) * ((3 * (size_t)(P + H) + 3) / 4 * 4 + 12 * (size_t)K * H + 8 * KMAXT);
}

}  // namespace

extern "C" int64_t skb_maml_workspace_bytes(int hidden, int tasks) {
  const int P = hidden * hidden + 4 * hidden + 1;
  return (int64_t)sizeof(float) * ((int64_t)tasks * P + tasks) + 16 + (int64_t)sizeof(double) * kTaskChunks * (P + 1);
}

extern "C" skb_status skb_maml_meta_grad(int hidden, int shots, int tasks, const float* theta, const float* xs,
                                         const float* ys, const float* xq, const float* yq, float alpha,
                                         float* meta_grad, float* mean_loss, void* workspace, void* stream) {
  if (hidden < 1 || hidden > HMAX || shots < 1 || shots > KMAXT || tasks < 1) return SKB_ERR_INVALID;
  const int P = hidden * hidden + 4 * hidden + 1;
  float* task_grad = (float*)workspace;
  float* task_loss = task_grad + (size_t)tasks * P;
  const size_t sm = smem_for(hidden, shots);
  cudaStream_t cs = (cudaStream_t)stream;
  // the C5 shape (H = 40, K = 10) as compile-time constants
  auto kern = hidden == 40 ? (shots == 10 ? maml_task_kernel<40, 10> : maml_task_kernel<40, 0>) : maml_task_kernel<0, 0>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess)
    return SKB_ERR_CUDA;
  // all of the unified L1 / shared array as shared memory: five task CTAs per SM at H = 40
  cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  kern<<<tasks, TPB, sm, cs>>>(hidden, shots, P, theta, xs, ys, xq, yq, alpha, task_grad, task_loss);
  double* part = (double*)(((uintptr_t)(task_loss + tasks) + 15) & ~(uintptr_t)15);
  maml_reduce_partial<<<dim3((P + 256) / 256, kTaskChunks), 256, 0, cs>>>(task_grad, task_loss, tasks, P, part);
  maml_reduce_final<<<(P + 256) / 256, 256, 0, cs>>>(part, tasks, P, meta_grad, mean_loss);
  return skb_check_launch();
}
