// train_tc.cu — the C2 training step (dynamic-length LSTM, BPTT) on skb's own tcgen05
// GEMM engine (gemm.cuh): bf16 operands, fp32 accumulation in TMEM, the LSTM cell
// fused into the GEMM epilogues.  No cuBLAS.  Replaces the staged BPTT program
// oracle/programs/lstm_bptt.msl (the reference cannot differentiate a While,
// graph/grad.py:159-161); same arithmetic as the fp32 path of train.cu.
//
// Layouts (per GPU shard of B rows; time-major, so a step's rows are one contiguous block):
//   XH  [T, B, KX] bf16, KX = F + 16 + H: row (t, b) = [x_t | 1 | 0 x 15 | h_{t-1}].
//       The ones column folds the bias into the gate GEMM and makes the bias gradient a
//       row of the weight-gradient GEMM; h_{t-1} is written by the epilogue of step t-1.
//   WU  [4H, KX] bf16, gate-interleaved rows n = 4j + g (g = i, f, g, o):
//       [W[:, gH+j] | b[gH+j] | 0 | U[:, gH+j]]  -> one N-tile holds all four gates of
//       its units, so the cell runs in the epilogue of the tile that produced them.
//   Ut  [H, 4H] bf16, Ut[k][4j+g] = U[k][gH+j]  (the B operand of dh = dG U^T).
//   Rec [T, B/128, H, 128] x 8 fp16 (tile-major: for one unit the 128 rows of a row tile are
//       contiguous, so the epilogue's stores coalesce and a tile's records are one bulk copy):
//       i, f, g, o, c_{t-1}, tanh(c_t) of each live (t, b, j).
//   dG  [T, B, 4H] bf16 gate gradients (interleaved), zero for t >= len.
//   hcur, ccur [B/128, H, 128] fp32 (tile-major likewise): initial / final state (the running
//       state and the BPTT carries ride in the step kernels' epilogue registers).
// Forward (one persistent launch over t = 0 .. n-1, grid barrier between steps):
//     D = XH[t] WU^T (K = KX)    -> EpiFwd: gates, c, h, Rec, loss partial <h_t, y_t>
//                                   (live rows), h_t -> XH[t+1]
// Backward (one persistent launch over t = n-1 .. 0):
//     D = dG[t+1] Ut^T (K = 4H)  -> EpiBwd: dh = D + carry + y/B, cell backward -> dG[t],
//                                   dc, frozen-row carries
// (gemm_steps_kernel: the epilogue operands of each tile are TMA-prefetched into shared
// memory while its MMAs run.)
// Then one GEMM over every (b, t):  P = XH^T dG  (M = KX, N = 4H, K = B T)
//                         -> dW (rows < F), db (row F), dU (rows >= F + 16), un-interleaved.
#include <cuda_fp16.h>
#include <math.h>
#include <string.h>

#include "gemm.cuh"
#include "skb_internal.h"

namespace skb {
namespace train_tc {

using gemm::kBF16;

struct Bufs {
  __nv_bfloat16 *XH, *WU, *Ut, *dG;
  __half* Rec;
  float *hcur, *ccur;
  double* lpart;   // [T][fwd tiles][epilogue warps]
  double* lsum;    // [T] per-step loss sums
  int* sync;       // [2] grid-barrier counters of the forward / backward launches, [2] the trip count
};

inline int kx_of(int F, int H) { return F + 16 + H; }
inline size_t al(size_t b) { return (b + 255) & ~size_t(255); }
constexpr int kFwdBN = 128;
constexpr int kFwdEW = 4;                    // epilogue warps per TMEM lane quarter (forward)
constexpr int kFwdSlots = 4 * kFwdEW;        // loss partials per forward tile

inline int fwd_tiles(int B, int H) { return ((B + 127) / 128) * (4 * H / kFwdBN); }

size_t layout(int B, int T, int F, int H, uint8_t* base, Bufs* w) {
  const size_t KX = kx_of(F, H), G = 4ull * H;
  size_t off = 0;
  auto take = [&](size_t bytes) { uint8_t* p = base ? base + off : nullptr; off += al(bytes); return p; };
  Bufs s;
  s.XH = (__nv_bfloat16*)take(2ull * B * T * KX);
  s.WU = (__nv_bfloat16*)take(2ull * G * KX);
  s.Ut = (__nv_bfloat16*)take(2ull * H * G);
  s.dG = (__nv_bfloat16*)take(2ull * B * T * G);
  const size_t Bp = (size_t)(B + 127) / 128 * 128;   // rows padded to whole 128-row tiles
  s.Rec = (__half*)take(16ull * Bp * T * H);
  s.hcur = (float*)take(4ull * Bp * H);
  s.ccur = (float*)take(4ull * Bp * H);
  s.lpart = (double*)take(8ull * T * fwd_tiles(B, H) * kFwdSlots);
  s.lsum = (double*)take(8ull * T);
  s.sync = (int*)take(16);
  if (w) *w = s;
  return off;
}

// Gate activations on the MUFU pipe: tanh.approx (|rel err| < 6e-4, inside the bf16
// operand path's bound) and sigmoid(x) = tanh(x/2)/2 + 1/2.
SKB_DEV float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
SKB_DEV float sigf(float x) { return fmaf(0.5f, tanh_fast(0.5f * x), 0.5f); }
SKB_DEV uint32_t pack_bf2(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}
SKB_DEV uint32_t pack_h2(float a, float b) {
  __half2 v = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}
SKB_DEV float2 unpack_h2(uint32_t u) {
  __half2 v = *reinterpret_cast<__half2*>(&u);
  return __half22float2(v);
}

// ------------------------------------------------------------------ operand preparation
// XH rows: [bf16(x) | 1 | 0 | h part: bf16(h0) at t = 0, else 0 (rewritten by the forward)]
__global__ void prep_xh(const float* __restrict__ x, const float* __restrict__ h0, __nv_bfloat16* __restrict__ XH,
                        int B, int T, int F, int H) {
  // eight columns per thread (F % 8 == 0: a group never straddles the x / ones / h parts),
  // two 16-byte loads of x, one 16-byte store of XH
  const int KX = F + 16 + H, KX8 = KX / 8;
  const long long groups = (long long)B * T * KX8;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < groups; i += (long long)gridDim.x * blockDim.x) {
    const long long row = i / KX8;   // time-major row t B + b
    const int c = (int)(i % KX8) * 8;
    const int t = (int)(row / B), b = (int)(row % B);
    float v[8];
    if (c < F) {
      const float4* xp = reinterpret_cast<const float4*>(x + ((long long)b * T + t) * F + c);
      const float4 a = __ldcs(xp), e = __ldcs(xp + 1);
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = e.x; v[5] = e.y; v[6] = e.z; v[7] = e.w;
    } else if (c < F + 16) {
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = (c + k == F) ? 1.f : 0.f;
    } else if (t == 0 && h0) {
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = h0[(long long)b * H + c - F - 16 + k];
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = 0.f;
    }
    *reinterpret_cast<uint4*>(XH + row * KX + c) =
        make_uint4(pack_bf2(v[0], v[1]), pack_bf2(v[2], v[3]), pack_bf2(v[4], v[5]), pack_bf2(v[6], v[7]));
  }
}

// WU [4H, KX] (interleaved rows) and Ut [H, 4H] from the fp32 parameters W [F, 4H],
// U [H, 4H], b [4H]; one thread per output pair.
__global__ void prep_weights(const float* __restrict__ W, const float* __restrict__ U, const float* __restrict__ bias,
                             __nv_bfloat16* __restrict__ WU, __nv_bfloat16* __restrict__ Ut, int F, int H) {
  const int G = 4 * H, KX = F + 16 + H;
  const long long n1 = (long long)G * KX / 2, n2 = (long long)H * G / 2;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n1 + n2; i += (long long)gridDim.x * blockDim.x) {
    if (i < n1) {
      const int n = (int)(i / (KX / 2)), c = (int)(i % (KX / 2)) * 2;
      const int col = (n & 3) * H + (n >> 2);   // source column g H + j
      float v[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int k = c + e;
        v[e] = k < F ? W[(long long)k * G + col] : k == F ? bias[col] : k < F + 16 ? 0.f : U[(long long)(k - F - 16) * G + col];
      }
      *reinterpret_cast<uint32_t*>(WU + (long long)n * KX + c) = pack_bf2(v[0], v[1]);
    } else {
      const long long ii = i - n1;
      const int k = (int)(ii / (G / 2)), n = (int)(ii % (G / 2)) * 2;
      const float a = U[(long long)k * G + (n & 3) * H + (n >> 2)];
      const float b = U[(long long)k * G + ((n + 1) & 3) * H + ((n + 1) >> 2)];
      *reinterpret_cast<uint32_t*>(Ut + (long long)k * G + n) = pack_bf2(a, b);
    }
  }
}

// Tile-major index of (row m, unit j) in a [B/128, H, 128] state array.
__host__ __device__ __forceinline__ long long tmi(int m, int j, int H) {
  return ((long long)(m >> 7) * H + j) * 128 + (m & 127);
}

__global__ void init_state(const float* __restrict__ h0, const float* __restrict__ c0, Bufs w, int B, int H) {
  const int Bp = (B + 127) / 128 * 128;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < (long long)Bp * H;
       i += (long long)gridDim.x * blockDim.x) {
    const int m = (int)(i / H), j = (int)(i % H);
    const long long d = tmi(m, j, H);
    w.hcur[d] = (m < B && h0) ? h0[(long long)m * H + j] : 0.f;
    w.ccur[d] = (m < B && c0) ? c0[(long long)m * H + j] : 0.f;
  }
}

// The While trip count n = clamp(reduce_max(lens), 0, T) on the device (given >= 0: that
// value), so a training step makes no host round trip.  One block.
__global__ void trip_count(const int64_t* __restrict__ lens, int B, int T, int given, int* __restrict__ n_out) {
  __shared__ int red[256];
  long long m = 0;
  for (int b = threadIdx.x; b < B; b += blockDim.x) m = lens[b] > m ? lens[b] : m;
  red[threadIdx.x] = (int)(m > T ? T : m);
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] = max(red[threadIdx.x], red[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *n_out = given >= 0 ? min(given, T) : red[0];
}

// dG rows t >= n take no part in the step: zero them for the weight-gradient GEMM (its K runs
// over every (t, b)); XH's h part of rows t > n is zero from prep_xh.
__global__ void zero_dg_tail(__nv_bfloat16* __restrict__ dG, const int* __restrict__ n_dev, int B, int T, int G) {
  const int n = *n_dev;
  const long long begin = (long long)n * B * G / 8, end = (long long)T * B * G / 8;
  uint4* p = reinterpret_cast<uint4*>(dG);
  for (long long i = begin + (long long)blockIdx.x * blockDim.x + threadIdx.x; i < end; i += (long long)gridDim.x * blockDim.x)
    p[i] = make_uint4(0, 0, 0, 0);
}

// loss = inv_b * sum of the partials: stage 1 one block per step (fixed order within the
// block), stage 2 the step sums in order (deterministic).
__global__ void loss_step_sums(const double* __restrict__ part, int per_step, const int* __restrict__ n_dev,
                               double* __restrict__ sums) {
  __shared__ double red[256];
  if ((int)blockIdx.x >= *n_dev) {   // steps past the trip count contribute nothing
    if (threadIdx.x == 0) sums[blockIdx.x] = 0.0;
    return;
  }
  double s = 0.0;
  const double* p = part + (long long)blockIdx.x * per_step;
  for (int i = threadIdx.x; i < per_step; i += blockDim.x) s += p[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) sums[blockIdx.x] = red[0];
}
__global__ void loss_final_sum(const double* __restrict__ sums, int n, float inv_b, float* loss) {
  __shared__ double red[256];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += sums[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *loss = (float)(red[0] * inv_b);
}

// ------------------------------------------------------------------ fused epilogues
// Each step kernel's TMA producer loads the tile's epilogue operands (state, carries,
// y_t, cell records) into shared memory while the MMAs run (kOpBytes); the epilogue
// reads them conflict-free from the 128-byte-swizzled boxes and writes its results.
constexpr uint32_t kBox = 128 * 128;   // one [128 rows][128 B] operand box

// Forward cell of step t = st: 16 accumulator columns = 4 units x (i, f, g, o); tile = 32 units.
// Every step kernel keeps one tile per CTA for all steps, and each epilogue thread owns one row
// and the same 8 units (two 16-column chunks) every step, so c and h ride in registers across
// steps: read from ccur/hcur at step 0, written back at the row's last live step.
struct EpiFwd {
  static constexpr uint32_t kOpBytes = kBox;   // y_t: [128 rows][32 units] fp32
  struct State { double lacc; bool live, last; float c0[4], c1[4], h0[4], h1[4]; };
  CUtensorMap mY;   // y [B][T][H] as a 3-D map {H, T, B}
  const int64_t* lens;
  float *hcur, *ccur;
  __nv_bfloat16* XH;
  __half* Rec;
  double* lpart;
  int T, F, H, B, tiles_n, tiles;
  int diag;   // SKB_TC_DIAG (timing experiments only): bit 0 skip the cell
  SKB_DEV int a_coord(int st) const { return st; }
  SKB_DEV bool k_empty(int) const { return false; }
  // XH[t]'s x part (and nothing of h_{t-1}) fills the first F / 64 K blocks
  SKB_DEV int k_indep(int) const { return F / 64; }
  SKB_DEV void prefetch(uint8_t* sop, int st, int tm, int tn, uint64_t* bar) const {
    gemm::tma_load_3d(sop, &mY, tn * 32, st, tm * 128, bar);
  }
  SKB_DEV void begin_tile(State& es, int st, int, int, int m) const {
    es.lacc = 0.0;
    const int len = m < B ? (int)lens[m] : 0;
    es.live = st < len;
    es.last = st == len - 1;
  }
  SKB_DEV void chunk(State& es, const uint8_t* sop, int t, int r, int m, int n0, int c, const float (&v)[16],
                     bool row_ok) const {
    if (!row_ok || (diag & 1)) return;
    const int j0 = n0 >> 2;                 // first unit
    const bool k1 = (c >> 4) & 1;           // which of the thread's two chunks
    const long long s0 = tmi(m, j0, H);   // unit j0 + u at s0 + 128 u: coalesced across the warp's rows
    float cp[4], hp[4];
    if (t == 0) {
#pragma unroll
      for (int u = 0; u < 4; ++u) { cp[u] = ccur[s0 + 128 * u]; hp[u] = hcur[s0 + 128 * u]; }
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) { cp[u] = k1 ? es.c1[u] : es.c0[u]; hp[u] = k1 ? es.h1[u] : es.h0[u]; }
    }
    float cn[4], hn[4];
    uint4 rec[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float ig = sigf(v[4 * u]), fg = sigf(v[4 * u + 1]), gg = tanh_fast(v[4 * u + 2]), og = sigf(v[4 * u + 3]);
      const float c2 = fg * cp[u] + ig * gg;
      const float tc = tanh_fast(c2);
      const float h2 = og * tc;
      cn[u] = es.live ? c2 : cp[u];
      hn[u] = es.live ? h2 : hp[u];
      rec[u] = make_uint4(pack_h2(ig, fg), pack_h2(gg, og), pack_h2(cp[u], tc), 0u);
      if (k1) { es.c1[u] = cn[u]; es.h1[u] = hn[u]; } else { es.c0[u] = cn[u]; es.h0[u] = hn[u]; }
    }
    if (diag & 4) return;   // timing experiment: no stores
    if (es.last) {   // the row's final state
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        ccur[s0 + 128 * u] = cn[u];
        hcur[s0 + 128 * u] = hn[u];
      }
    }
    if (t + 1 < T) {
      const int KX = F + 16 + H;
      *reinterpret_cast<uint2*>(XH + ((long long)(t + 1) * B + m) * KX + F + 16 + j0) =
          make_uint2(pack_bf2(hn[0], hn[1]), pack_bf2(hn[2], hn[3]));
    }
    if (es.live) {
      uint4* rp = reinterpret_cast<uint4*>(Rec) + (long long)t * ((B + 127) / 128) * 128 * H + s0;
      if (!(diag & 8)) {
#pragma unroll
        for (int u = 0; u < 4; ++u) __stcs(rp + 128 * u, rec[u]);   // streamed: read once, in the backward
      }
      const float4 yv = *reinterpret_cast<const float4*>(gemm::sw128_at(sop, r, c >> 4));
      es.lacc += (double)hn[0] * yv.x + (double)hn[1] * yv.y + (double)hn[2] * yv.z + (double)hn[3] * yv.w;
    }
  }
  SKB_DEV void end_tile(State& es, int t, int tm, int tn, int slot, int lane) const {
    double sum = es.lacc;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0) lpart[((long long)t * tiles + tm * tiles_n + tn) * kFwdSlots + slot] = sum;
  }
};

// Backward cell of step t = n-1-st: 16 accumulator columns = dh of 16 consecutive units;
// tile = 32 units.  Operands: dh carry, dc carry, y_t (fp32 boxes) and the cell records
// (four [128 rows][8 units x 16 B] boxes).  Each epilogue thread owns one row and the same 16
// units (one chunk) every step, so the dh / dc carries ride in its registers (zero at t = n-1).
struct EpiBwd {
  static constexpr uint32_t kOpBytes = 5 * kBox;   // y_t, then the cell records
  struct State { bool live; float dh[16], dc[16]; };
  CUtensorMap mY;   // y as a 3-D map {H, T, B}
  const __half* Rec;
  const int64_t* lens;
  __nv_bfloat16* dG;
  const int* n_dev;   // the trip count (device-determined: reduce_max of the lengths)
  int T, H, B;
  float inv_b;
  int diag;
  SKB_DEV int a_coord(int st) const { return *n_dev - st; }     // dG[t + 1]
  SKB_DEV bool k_empty(int st) const { return st == 0; }        // t = n-1: no dG_{t+1}
  SKB_DEV int k_indep(int) const { return 0; }                  // every block is dG_{t+1}
  SKB_DEV void prefetch(uint8_t* sop, int st, int tm, int tn, uint64_t* bar) const {
    const int t = *n_dev - 1 - st;
    const long long s0 = tmi(tm * 128, tn * 32, H);   // the tile's 32 units x 128 rows, contiguous
    gemm::tma_load_3d(sop, &mY, tn * 32, t, tm * 128, bar);
    bulk_g2s(sop + kBox, reinterpret_cast<const uint4*>(Rec) + (long long)t * ((B + 127) / 128) * 128 * H + s0,
             4 * kBox, bar);
  }
  SKB_DEV void begin_tile(State& es, int st, int, int, int m) const {
    es.live = m < B && *n_dev - 1 - st < lens[m];
    if (st == 0) {
#pragma unroll
      for (int i = 0; i < 16; ++i) { es.dh[i] = 0.f; es.dc[i] = 0.f; }
    }
  }
  // Warp-collective (every lane of the warp calls it; rows past B compute but store nothing).
  SKB_DEV void chunk(State& es, const uint8_t* sop, int st, int r, int m, int k0, int c, const float (&v)[16],
                     bool row_ok) const {
    if (diag & 1) return;
    const int t = *n_dev - 1 - st;
    const uint4* srec = reinterpret_cast<const uint4*>(sop + kBox) + c * 128 + r;
    uint2 res[16];   // the 16 units' four gate gradients (bf16)
#pragma unroll
    for (int q4 = 0; q4 < 4; ++q4) {   // four units per pass
      const int c16 = (c >> 2) + q4;   // y chunk (swizzled TMA box)
      float dh[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) dh[u] = v[4 * q4 + u] + es.dh[4 * q4 + u];
      if (!es.live) {   // frozen step: dh carries on to the row's last live step
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          es.dh[4 * q4 + u] = dh[u];
          res[4 * q4 + u] = make_uint2(0u, 0u);
        }
        continue;
      }
      const float4 yv = *reinterpret_cast<const float4*>(gemm::sw128_at(sop, r, c16));
      dh[0] += yv.x * inv_b; dh[1] += yv.y * inv_b; dh[2] += yv.z * inv_b; dh[3] += yv.w * inv_b;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float dcv_u = es.dc[4 * q4 + u];
        const uint4 rr = srec[(4 * q4 + u) * 128];
        const float2 a = unpack_h2(rr.x), b = unpack_h2(rr.y), cc = unpack_h2(rr.z);
        const float ig = a.x, fg = a.y, gg = b.x, og = b.y, cp = cc.x, tc = cc.y;
        const float dcn = dcv_u + dh[u] * og * (1.f - tc * tc);
        const float di = dcn * gg * ig * (1.f - ig);
        const float df = dcn * cp * fg * (1.f - fg);
        const float dg = dcn * ig * (1.f - gg * gg);
        const float dO = dh[u] * tc * og * (1.f - og);
        res[4 * q4 + u] = make_uint2(pack_bf2(di, df), pack_bf2(dg, dO));
        es.dc[4 * q4 + u] = dcn * fg;
        es.dh[4 * q4 + u] = 0.f;
      }
    }
    // dG rows through shared memory: the warp's 32 rows x 16 units x 8 B (4 KB) are staged in
    // the cell-record segments it has finished reading (units c..c+7 of its rows), 16-byte pairs
    // XOR-swizzled by row, then written as whole 128-byte row segments (4 rows per instruction
    // instead of 32 scattered 8-byte stores).
    const int lane = r & 31, wq = r >> 5;
    uint8_t* stg = const_cast<uint8_t*>(sop) + kBox + ((long long)c * 128 + wq * 32) * 16;   // unit c's segment
    __syncwarp();
#pragma unroll
    for (int p = 0; p < 8; ++p)
      *reinterpret_cast<uint4*>(stg + (lane >> 2) * 2048 + (lane & 3) * 128 + ((p ^ (lane & 7)) << 4)) =
          make_uint4(res[2 * p].x, res[2 * p].y, res[2 * p + 1].x, res[2 * p + 1].y);
    __syncwarp();
    const int m0 = m - lane;   // the warp's first row
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int rho = 4 * k + (lane >> 3), p = lane & 7;
      const uint4 val = *reinterpret_cast<const uint4*>(stg + k * 2048 + (rho & 3) * 128 + ((p ^ (rho & 7)) << 4));
      if (m0 + rho < B)
        *reinterpret_cast<uint4*>(dG + ((long long)t * B + m0 + rho) * 4 * H + 4 * k0 + 8 * p) = val;
    }
    fence_proxy_async_smem();   // the next step's TMA operand loads overwrite the staging area
    __syncwarp();
  }
  SKB_DEV void end_tile(State&, int, int, int, int, int) const {}
};

// Weight gradients from P = XH^T dG (rows m of KX, interleaved columns n = 4j + g).
struct EpiGrad {
  static constexpr uint32_t kOpBytes = 0;
  struct State {};
  float *dW, *dU, *db;
  int F, H;
  SKB_DEV bool skip() const { return false; }
  SKB_DEV bool ops_on() const { return false; }
  SKB_DEV void prefetch(uint8_t*, int, int, uint64_t*) const {}
  SKB_DEV void begin_tile(State&, int, int, int, int) const {}
  SKB_DEV void chunk(State&, const uint8_t*, int, int m, int n0, int, int, const float (&v)[16], bool row_ok) const {
    if (!row_ok || (m > F && m < F + 16)) return;
    const int G = 4 * H, j0 = n0 >> 2;
    float* dst = m < F ? dW + (long long)m * G : m == F ? db : dU + (long long)(m - F - 16) * G;
#pragma unroll
    for (int g = 0; g < 4; ++g)
      *reinterpret_cast<float4*>(dst + g * H + j0) = make_float4(v[g], v[4 + g], v[8 + g], v[12 + g]);
  }
  SKB_DEV void end_tile(State&, int, int, int, int, int) const {}
};

// Split-K mode of the step kernels (SKB_TC_FWD_KS / SKB_TC_BWD_KS = 1 or 2).  Forward
// default 1: 256-column split-K tiles measured slower (30.1 vs 27.6 ms per C2 step: only 3
// pipeline stages fit beside the epilogue operands).
int fwd_ks() {
  static int v = -1;
  if (v < 0) { const char* e = getenv("SKB_TC_FWD_KS"); v = e ? atoi(e) : 1; }
  return v;
}
int bwd_ks() {
  static int v = -1;
  if (v < 0) { const char* e = getenv("SKB_TC_BWD_KS"); v = e ? atoi(e) : 4; }
  return v;
}

// SKB_TC_TRACE=1: per-step globaltimer stamps of the forward step kernel's CTA 0
// (tools/trace_c2.py reads them through skb_train_tc_trace).
long long* g_trace = nullptr;
int g_trace_cap = 0;
long long* trace_buf(int T) {
  static int on = -1;
  if (on < 0) { const char* e = getenv("SKB_TC_TRACE"); on = (e && atoi(e) == 1) ? 1 : 0; }
  if (!on) return nullptr;
  if (T > g_trace_cap) {
    if (g_trace) cudaFree(g_trace);
    if (cudaMalloc(&g_trace, sizeof(long long) * 16 * T) != cudaSuccess) { g_trace = nullptr; g_trace_cap = 0; return nullptr; }
    g_trace_cap = T;
  }
  return g_trace;
}

int fwd_mc() {   // SKB_TC_FWD_MC=1: forward A boxes multicast across two CTA pairs
  static int v = -1;
  if (v < 0) { const char* e = getenv("SKB_TC_FWD_MC"); v = (e && atoi(e) == 1) ? 1 : 0; }
  return v;
}
int pair_fwd() {
  static int v = -1;
  if (v < 0) { const char* e = getenv("SKB_TC_PAIR_FWD"); v = (e && atoi(e) == 0) ? 0 : 1; }
  return v;
}

int pair_grad() {
  static int v = -1;
  if (v < 0) { const char* e = getenv("SKB_TC_PAIR"); v = (e && atoi(e) == 0) ? 0 : 1; }
  return v;
}

int diag() {
  static int v = -1;
  if (v < 0) { const char* e = getenv("SKB_TC_DIAG"); v = e ? atoi(e) : 0; }
  return v;
}

// SKB_TRAIN_PDL=0 disables programmatic dependent launch of the step kernels.
bool pdl() {
  static int v = -1;
  if (v < 0) { const char* e = getenv("SKB_TRAIN_PDL"); v = (e && atoi(e) == 0) ? 0 : 1; }
  return v == 1;
}

}  // namespace train_tc
}  // namespace skb

using namespace skb::train_tc;

// Workspace of the tensor-core path (math == 2).
extern "C" int64_t skb_train_tc_workspace_bytes(const skb_train_shape* d) {
  if (!d) return -1;
  return (int64_t)layout(d->rows, d->time, d->input, d->hidden, nullptr, nullptr);
}

// Enqueue one training step (forward + BPTT + gradients) on `cs`; the caller captures
// it into a CUDA graph.  Returns false on a launch/encode failure.
extern "C" int skb_train_tc_enqueue(const skb_train_shape* d, const float* x, const float* y, const int64_t* lens,
                                    const float* h0, const float* c0, const float* params, float* grads, float* loss,
                                    int n, void* workspace, void* stream) {
  namespace gm = skb::gemm;
  const int B = d->rows, T = d->time, F = d->input, H = d->hidden, G = 4 * H, KX = kx_of(F, H);
  if ((F % 8) || (H % 16) || G % kFwdBN) return SKB_ERR_UNSUPPORTED;
  cudaStream_t cs = (cudaStream_t)stream;
  Bufs w;
  layout(B, T, F, H, (uint8_t*)workspace, &w);
  const float* W = params;
  const float* U = params + (size_t)F * G;
  const float* bias = U + (size_t)H * G;
  float* dW = grads;
  float* dU = grads + (size_t)F * G;
  float* db = dU + (size_t)H * G;
  const int blocks = gm::num_sms() * 8;
  prep_xh<<<blocks, 256, 0, cs>>>(x, h0, w.XH, B, T, F, H);
  prep_weights<<<blocks, 256, 0, cs>>>(W, U, bias, w.WU, w.Ut, F, H);
  init_state<<<blocks, 256, 0, cs>>>(h0, c0, w, B, H);
  if (cudaPeekAtLastError() != cudaSuccess) return SKB_ERR_CUDA;

  // forward: one persistent launch; B operand WU (K-major), A operand XH[t] (3-D map)
  using GF = gm::Geo<kBF16, kFwdBN>;
  CUtensorMap mWU, mUt, mXH, mdG, mY;
  const int tiles_n = G / kFwdBN;
  if (!gm::encode_2d(&mWU, kBF16, w.WU, KX, G, KX, GF::BK, kFwdBN) ||
      !gm::encode_3d(&mXH, kBF16, w.XH, KX, B, T, KX, (uint64_t)B * KX, GF::BK, GF::BM, 1) ||
      !gm::encode_3d(&mY, gm::kTF32, y, H, T, B, H, (uint64_t)T * H, 32, 1, 128) ||
      !gm::encode_2d(&mUt, kBF16, w.Ut, G, H, G, 64, 32) ||
      !gm::encode_3d(&mdG, kBF16, w.dG, G, B, T, G, (uint64_t)B * G, 64, 128, 1))
    return SKB_ERR_INVALID;
  cudaMemsetAsync(w.sync, 0, 8, cs);
  int* n_dev = w.sync + 2;
  trip_count<<<1, 256, 0, cs>>>(lens, B, T, n, n_dev);
  {
    EpiFwd e;
    e.mY = mY;
    e.lens = lens; e.hcur = w.hcur; e.ccur = w.ccur; e.XH = w.XH; e.Rec = w.Rec; e.lpart = w.lpart;
    e.T = T; e.F = F; e.H = H; e.B = B; e.tiles_n = tiles_n; e.tiles = fwd_tiles(B, H); e.diag = diag();
    gm::StepShape sh{B, G, KX, 0, n_dev, w.sync, trace_buf(T)};
    int rc;
    if (fwd_ks() == 2 && pair_fwd() && (B % 256) == 0 && (G % 256) == 0) {
      // 256 x 256 tiles, each computed by two CTA pairs (a 4-CTA cluster) over alternate K blocks
      CUtensorMap mWUp, mXHp;
      if (!gm::encode_2d(&mWUp, kBF16, w.WU, KX, G, KX, GF::BK, 128) ||
          !gm::encode_3d(&mXHp, kBF16, w.XH, KX, B, T, KX, (uint64_t)B * KX, GF::BK, GF::BM, 1))
        return SKB_ERR_INVALID;
      rc = gm::launch_steps_pair<kBF16, 256, EpiFwd, kFwdEW, 2>(mXHp, mWUp, sh, e, cs);
    } else if (fwd_ks() == 2 && (G % 256) == 0) {   // 256-column tiles, each computed by two CTAs over K halves
      CUtensorMap mWU2;
      if (!gm::encode_2d(&mWU2, kBF16, w.WU, KX, G, KX, GF::BK, 256)) return SKB_ERR_INVALID;
      rc = gm::launch_steps<kBF16, 256, EpiFwd, kFwdEW, 2>(mXH, mWU2, sh, e, cs);
    } else if (pair_fwd() && (B % 256) == 0) {   // CTA pairs: 256-row tiles sharing the weight tile
      CUtensorMap mWUp, mXHp;
      if (!gm::encode_2d(&mWUp, kBF16, w.WU, KX, G, KX, GF::BK, kFwdBN / 2) ||
          !gm::encode_3d(&mXHp, kBF16, w.XH, KX, B, T, KX, (uint64_t)B * KX, GF::BK, GF::BM, 1))
        return SKB_ERR_INVALID;
      rc = 3;
      if (fwd_mc()) {   // two pairs per cluster sharing each A box by multicast
        CUtensorMap mXHh;
        if (!gm::encode_3d(&mXHh, kBF16, w.XH, KX, B, T, KX, (uint64_t)B * KX, GF::BK, 64, 1)) return SKB_ERR_INVALID;
        rc = gm::launch_steps_pair<kBF16, kFwdBN, EpiFwd, kFwdEW, 1, 2>(mXHh, mWUp, sh, e, cs);
      }
      if (rc == 3) rc = gm::launch_steps_pair<kBF16, kFwdBN, EpiFwd, kFwdEW>(mXHp, mWUp, sh, e, cs);
      if (rc == 3) rc = gm::launch_steps<kBF16, kFwdBN, EpiFwd, kFwdEW>(mXH, mWU, sh, e, cs);   // pairs not all resident
    } else {
      rc = gm::launch_steps<kBF16, kFwdBN, EpiFwd, kFwdEW>(mXH, mWU, sh, e, cs);
    }
    if (rc) return rc == 3 ? SKB_ERR_UNSUPPORTED : SKB_ERR_CUDA;
  }
  loss_step_sums<<<T, 256, 0, cs>>>(w.lpart, fwd_tiles(B, H) * kFwdSlots, n_dev, w.lsum);
  loss_final_sum<<<1, 256, 0, cs>>>(w.lsum, T, d->inv_batch, loss);

  // backward: one persistent launch; dh = dG[t+1] Ut^T
  {
    EpiBwd e;
    e.mY = mY; e.Rec = w.Rec;
    e.lens = lens; e.dG = w.dG;
    e.n_dev = n_dev; e.T = T; e.H = H; e.B = B; e.inv_b = d->inv_batch; e.diag = diag();
    long long* tb = trace_buf(T) ? g_trace + 8ll * g_trace_cap : nullptr;   // second half of the trace
    gm::StepShape sh{B, H, G, 0, n_dev, w.sync + 1, tb};
    { const char* v = getenv("SKB_TC_TRACE_CTA"); sh.trace_cta = v ? atoi(v) : 0; }
    int rc;
    // (same CTA count for 4 / 2 / 1; a split whose clusters cannot all be resident falls back)
    int ks = bwd_ks() == 4 && (H % 128) != 0 ? 2 : bwd_ks();
    rc = 3;
    if (ks == 4) {   // 128-unit tiles, each computed by four CTAs over K quarters (a 4-CTA cluster)
      CUtensorMap mUt4;
      if (!gm::encode_2d(&mUt4, kBF16, w.Ut, G, H, G, 64, 128)) return SKB_ERR_INVALID;
      rc = gm::launch_steps<kBF16, 128, EpiBwd, 2, 4>(mdG, mUt4, sh, e, cs);
      if (rc == 3) ks = 2;
    }
    if (rc == 3 && ks == 2 && (H % 64) == 0) {   // 64-unit tiles, each computed by two CTAs over K halves
      CUtensorMap mUt2;
      if (!gm::encode_2d(&mUt2, kBF16, w.Ut, G, H, G, 64, 64)) return SKB_ERR_INVALID;
      rc = gm::launch_steps<kBF16, 64, EpiBwd, 2, 2>(mdG, mUt2, sh, e, cs);
    }
    if (rc == 3) rc = gm::launch_steps<kBF16, 32, EpiBwd, 2>(mdG, mUt, sh, e, cs);
    if (rc) return rc == 3 ? SKB_ERR_UNSUPPORTED : SKB_ERR_CUDA;
  }
  zero_dg_tail<<<blocks, 256, 0, cs>>>(w.dG, n_dev, B, T, G);

  // weight gradients over every (t, b): P = XH^T dG  (A: XH as [K = T B, M = KX], MN-major;
  // B: dG as [K = B T, N = 4H], MN-major)
  {
    using GG = gm::Geo<kBF16, 256>;
    CUtensorMap mX, mD;
    const uint64_t rows = (uint64_t)B * T;
    if (!gm::encode_2d(&mX, kBF16, w.XH, KX, rows, KX, GG::MNB, GG::BK)) return SKB_ERR_INVALID;
    if (!gm::encode_2d(&mD, kBF16, w.dG, G, rows, G, GG::MNB, GG::BK)) return SKB_ERR_INVALID;
    EpiGrad e;
    e.dW = dW; e.dU = dU; e.db = db; e.F = F; e.H = H;
    gm::Shape sh{KX, G, (int)rows, 1, 0};
    // CTA-pair 256 x 256 tiles (cta_group::2; SKB_TC_PAIR=0: 1-CTA 128 x 256)
    const int rc = pair_grad() ? gm::launch_pair<kBF16, 256, true, true>(mX, mD, sh, e, cs)
                               : gm::launch<kBF16, 256, true, true>(mX, mD, sh, e, cs);
    if (rc) return SKB_ERR_CUDA;
  }
  return cudaPeekAtLastError() == cudaSuccess ? SKB_OK : SKB_ERR_CUDA;
}

// which = 0: forward kernel, 1: backward kernel
extern "C" int skb_train_tc_trace(long long* host_out, int steps, int which) {
  if (!g_trace || steps > g_trace_cap || which < 0 || which > 1) return -1;
  return cudaMemcpy(host_out, g_trace + (which ? 8ll * g_trace_cap : 0), sizeof(long long) * 8 * steps,
                    cudaMemcpyDeviceToHost) == cudaSuccess ? steps : -1;
}
