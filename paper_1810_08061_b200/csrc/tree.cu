// tree.cu — batched level-by-level TreeLSTM (BASELINE config C5).
//
// The reference evaluates a TreeLSTM by recursion over `Tree` values (the
// interpreter's FuncCall / TreeLeft / TreeRight / TreeValue, graph/execute.py:
// 136-146, 191-194; or a concrete tree unrolled at trace time).  Here the
// forest is scheduled by node height on the host (the tree structure is host
// data, like the reference's Tree objects) and every height level of every
// tree in the batch is one step:
//   tree_leaves  all leaves: c = wc * value, h = tanh(c)   (App. D leaf rule)
//   per level    G = X_level @ U  (X rows = [h_left, h_right] of the level's nodes,
//                U = [2H, 5H] gate blocks i | f_l | f_r | o | u; cuBLAS)
//                tree_cell: gates + bias -> c = i*u + f_l*c_l + f_r*c_r, h = o*tanh(c)
// Each node's h is written straight into its parent's X row (left or right
// half), so no gather pass exists between levels.  Semantics: oracle/tree.py
// (bit-exact with the reference interpreter in float64).
// SKB_TREE_TC=1 (TF32, even H): each level is ONE launch of skb's tcgen05 GEMM engine (gemm.cuh)
// with the cell fused into its epilogue (EpiTree): U is repacked gate-interleaved, three units x
// five gates per 16 accumulator columns, so a thread holds every gate of its units and the
// [rows, 5H] gate matrix never reaches HBM.  Parity-tested, but measured 1.9x slower on C5
// (0.76 vs 0.40 ms per forest): the epilogue's per-row gathers of node ids and children's c
// (thread = row) are latency-bound at one CTA per SM, where tree_cell4 runs eight CTAs per SM with
// row-contiguous loads.  Default: cuBLAS level GEMMs + tree_cell4.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include "blas.cuh"
#include "gemm.cuh"
#include "skb_internal.h"

namespace {

__device__ __forceinline__ float sigmoidf_ref(float x) {   // reference tensor.py:403-407
  if (x >= 0.f) return 1.f / (1.f + expf(-x));
  const float e = expf(x);
  return e / (1.f + e);
}

// dest[n] = 2*row + side of node n's h in its parent's X row (-1 for roots).
// One CTA row per node (blockDim.x covers H): no per-element integer division.
__global__ void tree_leaves(const int32_t* __restrict__ leaves, int nleaves, const float* __restrict__ value,
                            const float* __restrict__ wc, const int32_t* __restrict__ dest, float* __restrict__ h,
                            float* __restrict__ c, float* __restrict__ X, int H) {
  for (int l = blockIdx.x * blockDim.y + threadIdx.y; l < nleaves; l += gridDim.x * blockDim.y) {
    const int n = leaves[l];
    const float v = value[n];
    const int d = dest[n];
    float* xrow = d >= 0 ? X + (long long)(d >> 1) * 2 * H + (d & 1) * H : nullptr;
    for (int k = threadIdx.x; k < H; k += blockDim.x) {
      const float cv = wc[k] * v;
      const float hv = tanhf(cv);
      c[(long long)n * H + k] = cv;
      h[(long long)n * H + k] = hv;
      if (xrow) xrow[k] = hv;
    }
  }
}

__global__ void tree_cell(const int32_t* __restrict__ order, int row0, int nrows, const int32_t* __restrict__ left,
                          const int32_t* __restrict__ right, const float* __restrict__ G, const float* __restrict__ bias,
                          const int32_t* __restrict__ dest, float* __restrict__ h, float* __restrict__ c,
                          float* __restrict__ X, int H) {
  for (int rr = blockIdx.x * blockDim.y + threadIdx.y; rr < nrows; rr += gridDim.x * blockDim.y) {
    const int p = row0 + rr;
    const int n = order[p];
    const float* g = G + (long long)p * 5 * H;
    const float* cl = c + (long long)left[n] * H;
    const float* cr = c + (long long)right[n] * H;
    const int d = dest[n];
    float* xrow = d >= 0 ? X + (long long)(d >> 1) * 2 * H + (d & 1) * H : nullptr;
    for (int k = threadIdx.x; k < H; k += blockDim.x) {
      const float gi = sigmoidf_ref(g[k] + bias[k]);
      const float gfl = sigmoidf_ref(g[H + k] + bias[H + k]);
      const float gfr = sigmoidf_ref(g[2 * H + k] + bias[2 * H + k]);
      const float go = sigmoidf_ref(g[3 * H + k] + bias[3 * H + k]);
      const float gu = tanhf(g[4 * H + k] + bias[4 * H + k]);
      const float cv = gi * gu + gfl * cl[k] + gfr * cr[k];
      const float hv = go * tanhf(cv);
      c[(long long)n * H + k] = cv;
      h[(long long)n * H + k] = hv;
      if (xrow) xrow[k] = hv;
    }
  }
}

// float4 variants (H % 4 == 0): a warp covers 128 consecutive units of one row
// with 16-byte loads/stores; identical per-element arithmetic.
__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }

__global__ void tree_leaves4(const int32_t* __restrict__ leaves, int nleaves, const float* __restrict__ value,
                             const float* __restrict__ wc, const int32_t* __restrict__ dest, float* __restrict__ h,
                             float* __restrict__ c, float* __restrict__ X, int H) {
  const int H4 = H >> 2;
  for (int l = blockIdx.x * blockDim.y + threadIdx.y; l < nleaves; l += gridDim.x * blockDim.y) {
    const int n = leaves[l];
    const float v = value[n];
    const int d = dest[n];
    float* xrow = d >= 0 ? X + (long long)(d >> 1) * 2 * H + (d & 1) * H : nullptr;
    for (int k4 = threadIdx.x; k4 < H4; k4 += blockDim.x) {
      const int k = 4 * k4;
      const float4 w = ld4(wc + k);
      const float4 cv = make_float4(w.x * v, w.y * v, w.z * v, w.w * v);
      const float4 hv = make_float4(tanhf(cv.x), tanhf(cv.y), tanhf(cv.z), tanhf(cv.w));
      st4(c + (long long)n * H + k, cv);
      st4(h + (long long)n * H + k, hv);
      if (xrow) st4(xrow + k, hv);
    }
  }
}

__global__ void tree_cell4(const int32_t* __restrict__ order, int row0, int nrows, const int32_t* __restrict__ left,
                           const int32_t* __restrict__ right, const float* __restrict__ G,
                           const float* __restrict__ bias, const int32_t* __restrict__ dest, float* __restrict__ h,
                           float* __restrict__ c, float* __restrict__ X, int H) {
  const int H4 = H >> 2;
  for (int rr = blockIdx.x * blockDim.y + threadIdx.y; rr < nrows; rr += gridDim.x * blockDim.y) {
    const int p = row0 + rr;
    const int n = order[p];
    const float* g = G + (long long)p * 5 * H;
    const float* cl = c + (long long)left[n] * H;
    const float* cr = c + (long long)right[n] * H;
    const int d = dest[n];
    float* xrow = d >= 0 ? X + (long long)(d >> 1) * 2 * H + (d & 1) * H : nullptr;
    for (int k4 = threadIdx.x; k4 < H4; k4 += blockDim.x) {
      const int k = 4 * k4;
      float gi[4], gfl[4], gfr[4], go[4], gu[4], l4[4], r4[4], cv[4], hv[4];
      const float4 a0 = ld4(g + k), a1 = ld4(g + H + k), a2 = ld4(g + 2 * H + k), a3 = ld4(g + 3 * H + k),
                   a4 = ld4(g + 4 * H + k);
      const float4 b0 = ld4(bias + k), b1 = ld4(bias + H + k), b2 = ld4(bias + 2 * H + k),
                   b3 = ld4(bias + 3 * H + k), b4 = ld4(bias + 4 * H + k);
      const float4 L = ld4(cl + k), R = ld4(cr + k);
      const float za[4][5] = {{a0.x + b0.x, a1.x + b1.x, a2.x + b2.x, a3.x + b3.x, a4.x + b4.x},
                              {a0.y + b0.y, a1.y + b1.y, a2.y + b2.y, a3.y + b3.y, a4.y + b4.y},
                              {a0.z + b0.z, a1.z + b1.z, a2.z + b2.z, a3.z + b3.z, a4.z + b4.z},
                              {a0.w + b0.w, a1.w + b1.w, a2.w + b2.w, a3.w + b3.w, a4.w + b4.w}};
      l4[0] = L.x; l4[1] = L.y; l4[2] = L.z; l4[3] = L.w;
      r4[0] = R.x; r4[1] = R.y; r4[2] = R.z; r4[3] = R.w;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        gi[e] = sigmoidf_ref(za[e][0]);
        gfl[e] = sigmoidf_ref(za[e][1]);
        gfr[e] = sigmoidf_ref(za[e][2]);
        go[e] = sigmoidf_ref(za[e][3]);
        gu[e] = tanhf(za[e][4]);
        cv[e] = gi[e] * gu[e] + gfl[e] * l4[e] + gfr[e] * r4[e];
        hv[e] = go[e] * tanhf(cv[e]);
      }
      const float4 C4 = make_float4(cv[0], cv[1], cv[2], cv[3]), H4v = make_float4(hv[0], hv[1], hv[2], hv[3]);
      st4(c + (long long)n * H + k, C4);
      st4(h + (long long)n * H + k, H4v);
      if (xrow) st4(xrow + k, H4v);
    }
  }
}

// ---------------------------------------------------------------- engine path
// Packed U: row n' = 16 q + 5 e + g (e < 3, g < 5) holds column g H + j of U, j = 3 q + e; rows
// 16 q + 15 and units j >= H are zero.  K-major [NP][2H] fp32 (TF32 operands).
inline int tree_np(int H) { return ((H + 2) / 3 * 16 + 127) / 128 * 128; }

__global__ void tree_pack_u(const float* __restrict__ U, int H, int NP, float* __restrict__ Up) {
  const int K = 2 * H;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < (long long)NP * K;
       i += (long long)gridDim.x * blockDim.x) {
    const int np = (int)(i / K), k = (int)(i % K);
    const int q = np >> 4, w = np & 15, e = w / 5, g = w % 5, j = 3 * q + e;
    Up[i] = (w < 15 && j < H) ? U[(long long)k * 5 * H + g * H + j] : 0.f;
  }
}

// Epilogue geometry: 128-column tiles, 4 x 4 epilogue warps, so a thread owns 32 columns (two
// chunks = 6 units) of one row; begin_tile (before the tile's accumulator is waited for) fetches
// the row's node ids and its children's c values of those 6 units into registers.
constexpr int kTreeBN = 128, kTreeEW = 4, kTreeUnits = 6;
struct EpiTree {
  static constexpr uint32_t kOpBytes = 0;
  struct State { int n, d; float cl[kTreeUnits], cr[kTreeUnits]; };
  const int32_t *order, *left, *right, *dest;
  const float* bias;
  float *h, *c, *X;
  int H, r0, nr;
  SKB_DEV bool skip() const { return false; }
  SKB_DEV bool ops_on() const { return false; }
  SKB_DEV void prefetch(uint8_t*, int, int, uint64_t*) const {}
  SKB_DEV void begin_tile(State& s, int, int tn, int, int m) const {
    if (m >= nr) return;
    s.n = order[r0 + m];
    s.d = dest[s.n];
    const int slice = ((int)(threadIdx.x >> 5) - 2) >> 2;   // the thread's column slice (gemm_kernel)
    const int j0 = tn * (kTreeBN / 16 * 3) + slice * kTreeUnits;
    const float* cl = c + (long long)left[s.n] * H;
    const float* cr = c + (long long)right[s.n] * H;
#pragma unroll
    for (int u = 0; u < kTreeUnits; ++u) {
      s.cl[u] = j0 + u < H ? cl[j0 + u] : 0.f;
      s.cr[u] = j0 + u < H ? cr[j0 + u] : 0.f;
    }
  }
  SKB_DEV void chunk(State& s, const uint8_t*, int, int, int n0, int, int, const float (&v)[16], bool row_ok) const {
    if (!row_ok) return;
    const int n = s.n, d = s.d;
    const bool k1 = (n0 >> 4) & 1;   // second chunk of the thread's slice
    float* xrow = d >= 0 ? X + (long long)(d >> 1) * 2 * H + (d & 1) * H : nullptr;
#pragma unroll
    for (int e = 0; e < 3; ++e) {
      const int j = 3 * (n0 >> 4) + e;
      if (j >= H) break;
      const float gi = sigmoidf_ref(v[5 * e] + bias[j]);
      const float gfl = sigmoidf_ref(v[5 * e + 1] + bias[H + j]);
      const float gfr = sigmoidf_ref(v[5 * e + 2] + bias[2 * H + j]);
      const float go = sigmoidf_ref(v[5 * e + 3] + bias[3 * H + j]);
      const float gu = tanhf(v[5 * e + 4] + bias[4 * H + j]);
      const float cv = gi * gu + gfl * (k1 ? s.cl[3 + e] : s.cl[e]) + gfr * (k1 ? s.cr[3 + e] : s.cr[e]);
      const float hv = go * tanhf(cv);
      c[(long long)n * H + j] = cv;
      h[(long long)n * H + j] = hv;
      if (xrow) xrow[j] = hv;
    }
  }
  SKB_DEV void end_tile(State&, int, int, int, int, int) const {}
};

bool tree_engine(int H, int math) {
  static int on = -1;
  if (on < 0) { const char* e = getenv("SKB_TREE_TC"); on = (e && atoi(e) == 1) ? 1 : 0; }
  return on && math == 1 && (H % 2) == 0;
}

}  // namespace

extern "C" int64_t skb_tree_workspace_bytes(int nnodes, int ninternal, int hidden) {
  auto al = [](int64_t b) { return (b + 255) & ~int64_t(255); };
  return al(4ll * ninternal * 2 * hidden) + al(4ll * ninternal * 5 * hidden) + 2 * al(4ll * nnodes * hidden) +
         al(4ll * tree_np(hidden) * 2 * hidden);   // the engine's packed U
}

namespace {

bool enqueue_forest(cublasHandle_t hb, cudaStream_t cs, int nnodes, int nleaves, int ninternal, int H, int nlevels,
                    const int32_t* leaves, const int32_t* order, const int32_t* level_off_host, const int32_t* left,
                    const int32_t* right, const int32_t* dest, const float* value, const float* wc, const float* U,
                    const float* bias, int math, float* h, float* c, float* X, float* G, float* Up) {
  const int blocks = 148 * 8;
  // float4 path when H % 4 == 0 (rows of 16-byte chunks); scalar path otherwise
  const bool v4 = (H & 3) == 0 && !getenv("SKB_TREE_SCALAR");
  const int cols = v4 ? H / 4 : H;
  const int tx = cols >= 128 ? 128 : (cols >= 64 ? 64 : 32), ty = 256 / tx;   // threads over H x rows per CTA
  const dim3 blk(tx, ty);
  const int lb = (nleaves + ty - 1) / ty < blocks ? (nleaves + ty - 1) / ty : blocks;
  if (v4)
    tree_leaves4<<<lb, blk, 0, cs>>>(leaves, nleaves, value, wc, dest, h, c, X, H);
  else
    tree_leaves<<<lb, blk, 0, cs>>>(leaves, nleaves, value, wc, dest, h, c, X, H);
  if (tree_engine(H, math)) {
    namespace gm = skb::gemm;
    constexpr int BN = kTreeBN, EW = kTreeEW;
    using GT = gm::Geo<gm::kTF32, BN>;
    const int NP = tree_np(H);
    tree_pack_u<<<148 * 4, 256, 0, cs>>>(U, H, NP, Up);
    CUtensorMap tb;
    if (!gm::encode_2d(&tb, gm::kTF32, Up, 2 * H, NP, 2 * H, GT::BK, BN)) return false;
    for (int L = 0; L < nlevels; ++L) {
      const int r0 = level_off_host[L], nr = level_off_host[L + 1] - r0;
      if (nr <= 0) continue;
      CUtensorMap ta;
      if (!gm::encode_2d(&ta, gm::kTF32, X + (int64_t)r0 * 2 * H, 2 * H, nr, 2 * H, GT::BK, GT::BM)) return false;
      EpiTree e{order, left, right, dest, bias, h, c, X, H, r0, nr};
      gm::Shape sh{nr, NP, 2 * H, 1, 0};
      if (gm::launch<gm::kTF32, BN, false, false, EpiTree, false, EW>(ta, tb, sh, e, cs)) return false;
    }
    return cudaPeekAtLastError() == cudaSuccess;
  }
  for (int L = 0; L < nlevels; ++L) {
    const int r0 = level_off_host[L], nr = level_off_host[L + 1] - r0;
    if (nr <= 0) continue;
    if (!skb::gemm_f32(hb, math, X + (int64_t)r0 * 2 * H, 2 * H, U, 5 * H, G + (int64_t)r0 * 5 * H, 5 * H, nr, 5 * H,
                       2 * H))
      return false;
    const int b = (nr + ty - 1) / ty < blocks ? (nr + ty - 1) / ty : blocks;
    if (v4)
      tree_cell4<<<b, blk, 0, cs>>>(order, r0, nr, left, right, G, bias, dest, h, c, X, H);
    else
      tree_cell<<<b, blk, 0, cs>>>(order, r0, nr, left, right, G, bias, dest, h, c, X, H);
  }
  return cudaPeekAtLastError() == cudaSuccess;
}

// Forest graphs: the leaf pass and every level's GEMM + cell captured once per
// (buffers, schedule) and replayed as one launch (the per-level launch gaps
// dominate the many small top levels).
struct ForestGraph {
  const void* ptrs[13];
  int dims[6];
  int32_t* levels;
  cudaGraphExec_t exec;
};
constexpr int kForestGraphs = 8;
ForestGraph g_fg[kForestGraphs];
int g_nfg = 0;
int g_tree_mode = 0;

}  // namespace

extern "C" int skb_tree_last_mode(void) { return g_tree_mode; }

extern "C" skb_status skb_tree_lstm(int nnodes, int nleaves, int ninternal, int hidden, int nlevels,
                                    const int32_t* leaves, const int32_t* order, const int32_t* level_off_host,
                                    const int32_t* left, const int32_t* right, const int32_t* dest,
                                    const float* value, const float* wc, const float* U, const float* bias, int math,
                                    float* h_out, float* c_out, void* workspace, void* stream) {
  if (nnodes <= 0 || hidden <= 0 || nleaves <= 0 || nlevels < 0) return SKB_ERR_INVALID;
  cudaStream_t cs = (cudaStream_t)stream;
  const int H = hidden;
  auto al = [](int64_t b) { return (b + 255) & ~int64_t(255); };
  uint8_t* ws = (uint8_t*)workspace;
  float* X = (float*)ws;
  float* G = (float*)(ws + al(4ll * ninternal * 2 * H));
  float* h = h_out ? h_out : (float*)(ws + al(4ll * ninternal * 2 * H) + al(4ll * ninternal * 5 * H));
  float* c = c_out ? c_out : h + (int64_t)nnodes * H;
  float* Up = (float*)(ws + al(4ll * ninternal * 2 * H) + al(4ll * ninternal * 5 * H) + 2 * al(4ll * nnodes * H));
  cublasHandle_t hb = skb::blas_handle(cs);
  if (!hb) return SKB_ERR_CUDA;
  const void* key[13] = {leaves, order, left, right, dest, value, wc, U, bias, h, c, workspace, nullptr};
  const int dims[6] = {nnodes, nleaves, ninternal, H, nlevels, math};
  cudaGraphExec_t exec = nullptr;
  for (int i = 0; i < g_nfg && !exec; ++i) {
    const ForestGraph& e = g_fg[i];
    if (memcmp(e.ptrs, key, sizeof(key)) == 0 && memcmp(e.dims, dims, sizeof(dims)) == 0 &&
        memcmp(e.levels, level_off_host, sizeof(int32_t) * (nlevels + 1)) == 0)
      exec = e.exec;
  }
  // capture only for a schedule seen before (repeated evaluation of one forest)
  static uint64_t seen[16] = {0};
  uint64_t hsh = 1469598103934665603ull;
  auto mix = [&](const void* p, size_t n) {
    const unsigned char* b = (const unsigned char*)p;
    for (size_t i = 0; i < n; ++i) hsh = (hsh ^ b[i]) * 1099511628211ull;
  };
  mix(key, sizeof(key));
  mix(dims, sizeof(dims));
  mix(level_off_host, sizeof(int32_t) * (nlevels + 1));
  bool again = false;
  for (int i = 0; i < 16; ++i) again |= seen[i] == hsh;
  if (!again) {
    static int next = 0;
    seen[next] = hsh;
    next = (next + 1) % 16;
  }
  if (!exec && again) {
    cudaStream_t cap = nullptr;
    cudaGraph_t g = nullptr;
    bool ok = cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking) == cudaSuccess &&
              cudaStreamBeginCapture(cap, cudaStreamCaptureModeRelaxed) == cudaSuccess;
    if (ok) {
      cublasSetStream(hb, cap);
      const bool enq = enqueue_forest(hb, cap, nnodes, nleaves, ninternal, H, nlevels, leaves, order, level_off_host,
                                      left, right, dest, value, wc, U, bias, math, h, c, X, G, Up);
      ok = cudaStreamEndCapture(cap, &g) == cudaSuccess && enq;
    }
    if (ok) ok = cudaGraphInstantiate(&exec, g, 0) == cudaSuccess;
    if (g) cudaGraphDestroy(g);
    if (cap) cudaStreamDestroy(cap);
    cublasSetStream(hb, cs);
    cudaGetLastError();
    if (!ok) {
      exec = nullptr;
    } else {
      if (g_nfg == kForestGraphs) {
        cudaGraphExecDestroy(g_fg[0].exec);
        free(g_fg[0].levels);
        memmove(g_fg, g_fg + 1, sizeof(ForestGraph) * (kForestGraphs - 1));
        --g_nfg;
      }
      ForestGraph& e = g_fg[g_nfg++];
      memcpy(e.ptrs, key, sizeof(key));
      memcpy(e.dims, dims, sizeof(dims));
      e.levels = (int32_t*)malloc(sizeof(int32_t) * (nlevels + 1));
      memcpy(e.levels, level_off_host, sizeof(int32_t) * (nlevels + 1));
      e.exec = exec;
    }
  }
  g_tree_mode = exec ? 1 : 0;
  if (exec) {
    if (cudaGraphLaunch(exec, cs) != cudaSuccess) return SKB_ERR_CUDA;
  } else if (!enqueue_forest(hb, cs, nnodes, nleaves, ninternal, H, nlevels, leaves, order, level_off_host, left,
                             right, dest, value, wc, U, bias, math, h, c, X, G, Up)) {
    return SKB_ERR_CUDA;
  }
  return skb_check_launch();
}

// Host-side forest scheduler (native runtime, O(nodes)): heights by one
// reverse pre-order sweep, internal nodes counting-sorted by height, and each
// node's destination row/side in its parent's GEMM row.  left/right hold
// global node ids (-1 for none) with children after their parent (pre-order).
// Outputs: height[n], order[n_internal], level_off[max_height + 1] (level L
// occupies order[level_off[L-1] .. level_off[L]) for L = 1..max_height),
// leaves[n_leaves], dest[n].  Returns max_height, or -1 if a node has exactly
// one child (TreeLSTM trees are full binary trees).
extern "C" int skb_tree_schedule(int64_t n, const int64_t* left, const int64_t* right, int32_t* height,
                                 int32_t* order, int32_t* level_off, int32_t* leaves, int32_t* dest) {
  int maxh = 0;
  int64_t nleaf = 0;
  for (int64_t i = n - 1; i >= 0; --i) {
    const int64_t l = left[i], r = right[i];
    if ((l < 0) != (r < 0)) return -1;
    if (l < 0) { height[i] = 0; continue; }
    const int h = 1 + (height[l] > height[r] ? height[l] : height[r]);
    height[i] = h;
    if (h > maxh) maxh = h;
  }
  // counting sort of internal nodes by height (stable in node order)
  int64_t* cnt = (int64_t*)calloc((size_t)maxh + 2, sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) {
    if (left[i] < 0) leaves[nleaf++] = (int32_t)i; else cnt[height[i]]++;
  }
  int64_t acc = 0;
  for (int h = 1; h <= maxh; ++h) { level_off[h - 1] = (int32_t)acc; acc += cnt[h]; cnt[h] = level_off[h - 1]; }
  level_off[maxh] = (int32_t)acc;
  int32_t* row = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  for (int64_t i = 0; i < n; ++i) {
    row[i] = -1;
    if (left[i] >= 0) { const int64_t p = cnt[height[i]]++; order[p] = (int32_t)i; row[i] = (int32_t)p; }
  }
  for (int64_t i = 0; i < n; ++i) dest[i] = -1;
  for (int64_t i = 0; i < n; ++i) {
    if (left[i] < 0) continue;
    dest[left[i]] = 2 * row[i];
    dest[right[i]] = 2 * row[i] + 1;
  }
  free(row);
  free(cnt);
  return maxh;
}

// Forest form of skb_tree_schedule: the trees' node arrays concatenated, child indices LOCAL to
// each tree (pre-order, -1 for none, `sizes[t]` nodes each).  Two passes instead of five and no
// separate global-index pass: heights (per tree, reverse pre-order) with the global int32 child
// ids and per-height counts, then one forward pass that places every internal node in its
// level (order), lists the leaves and writes each child's destination row/side at its parent
// (children follow their parent in pre-order).  Returns max_height, or -1 for a node with one
// child or a child index outside its tree / not after its parent.
extern "C" int skb_forest_schedule(int64_t ntrees, const int64_t* sizes, const int64_t* left, const int64_t* right,
                                   int32_t* left_out, int32_t* right_out, int32_t* height, int32_t* order,
                                   int32_t* level_off, int32_t* leaves, int32_t* dest) {
  int64_t cap = 64;
  int64_t* cnt = (int64_t*)calloc((size_t)cap, sizeof(int64_t));
  if (!cnt) return -1;
  int maxh = 0;
  int64_t b = 0;
  for (int64_t t = 0; t < ntrees; ++t) {
    const int64_t sz = sizes[t];
    if (sz < 1) { free(cnt); return -1; }
    dest[b] = -1;   // the tree's root
    for (int64_t k = sz - 1; k >= 0; --k) {
      const int64_t i = b + k, l = left[i], r = right[i];
      if ((l < 0) != (r < 0)) { free(cnt); return -1; }
      if (l < 0) { height[i] = 0; left_out[i] = right_out[i] = -1; continue; }
      if (l <= k || r <= k || l >= sz || r >= sz) { free(cnt); return -1; }
      const int32_t gl = (int32_t)(b + l), gr = (int32_t)(b + r);
      const int h = 1 + (height[gl] > height[gr] ? height[gl] : height[gr]);
      height[i] = h;
      left_out[i] = gl;
      right_out[i] = gr;
      if (h >= cap) {
        const int64_t nc = 2 * h;
        int64_t* g = (int64_t*)realloc(cnt, (size_t)nc * sizeof(int64_t));
        if (!g) { free(cnt); return -1; }
        memset(g + cap, 0, (size_t)(nc - cap) * sizeof(int64_t));
        cnt = g;
        cap = nc;
      }
      ++cnt[h];
      if (h > maxh) maxh = h;
    }
    b += sz;
  }
  const int64_t n = b;
  int64_t acc = 0;
  for (int h = 1; h <= maxh; ++h) { level_off[h - 1] = (int32_t)acc; acc += cnt[h]; cnt[h] = level_off[h - 1]; }
  level_off[maxh] = (int32_t)acc;
  int64_t nleaf = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (left_out[i] < 0) { leaves[nleaf++] = (int32_t)i; continue; }
    const int32_t p = (int32_t)cnt[height[i]]++;
    order[p] = (int32_t)i;
    dest[left_out[i]] = 2 * p;
    dest[right_out[i]] = 2 * p + 1;
  }
  free(cnt);
  return maxh;
}
