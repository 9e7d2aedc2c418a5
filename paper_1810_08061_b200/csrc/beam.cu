// beam.cu — staged seq2seq decoder with a data-dependent EOS stop (BASELINE
// config C3): the greedy program of SURVEY App. F (oracle/programs/greedy.msl,
// a `break` on EOS lowered into the While test) generalised to beam search.
//
// One decode step for R = sentences x beam rows:
//   dec_gather   xh = [emb[tok], h]                      (tensor.py:420-430 Index)
//   GEMM         gates = xh @ W_gates
//   dec_cell     rnn: h' = tanh(gates); lstm: i,f,g,o -> c', h'   (tensor.py:391-407)
//   GEMM         logits = h' @ W_out
//   beam_rows    ONE pass over the logits, one CTA per beam row: it keeps
//                an online max / sum-exp (log-softmax) and per-thread top-K lists
//                merged by warp-shuffle argmax;
// With SKB_DEC_TC=1, TF32 LSTM decoding runs both GEMMs on skb's own tcgen05 engine
// (gemm.cuh) instead (measured slower, see dec_tc): the cell is fused into the gate GEMM's epilogue
// (gate-interleaved weight rows), and the log-softmax normaliser + per-row top-K into the
// logits GEMM's epilogue (per-tile partials merged by dec_merge), so the [R, V] logits
// never reach HBM.  fp32-exact decoding (math 0) keeps cuBLAS GEMMs (tensor cores cannot
// do exact fp32).
//   beam_choose  per sentence: ranks its K x K candidates (score desc, flat index
//                asc — the oracle's tie-break), reindexes h, c, scores, tokens,
//                lengths and history from the chosen parents and counts
//                unfinished sentences.
// Every kernel of step t+1 reads that count and exits when it is zero, so the
// stop is decided on the device; the host only polls the counter every few
// steps to stop launching.  Semantics: oracle/beam.py (pinned against the
// reference's greedy program at beam 1).
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <string.h>
#include "gemm.cuh"
#include "skb_internal.h"

namespace {

constexpr int KMAX = 8;          // largest beam
constexpr int SEL_THREADS = 256;  // beam_choose CTA (one per sentence)
constexpr int ROW_THREADS = 256;  // beam_rows CTA (one per beam row)

struct DecodeState {             // device pointers into the workspace
  float* xh;                     // [R, E+H]
  float* gates;                  // [R, G]
  float* h[2];                   // ping-pong [R, H]
  float* c[2];
  float* hn;                     // [R, H]  cell output of this step
  float* cn;
  float* logits;                 // [R, V]
  double* score[2];              // [R]
  int32_t* tok;                  // [R]
  int32_t* fin[2];               // [R]
  int32_t* len[2];               // [R]
  int32_t* hist[2];              // [R, max_len+1]
  int32_t* active;               // [max_len+1] unfinished sentences after step t (active[0] = S)
  int32_t* tstep;                // the decode step counter (device-resident loop index)
  float* row_v;                  // [R, KMAX] each row's K best logits (pass 1)
  int32_t* row_i;                // [R, KMAX] their vocabulary ids
  float* row_lse;                // [R] log-sum-exp of the row
  float* margin;                 // [R] greedy (beam 1): smallest top-1 - top-2 logit gap over the decode
  // tensor-core path (math 1, LSTM)
  float* wgT;                    // [4H, E+H] gate-interleaved rows n = 4j + g (K-major B operand)
  float* bg;                     // [4H] interleaved gate bias
  float* woT;                    // [Vp, H] w_out^T (K-major B operand), rows >= V zero
  float* bo;                     // [Vp] output bias, -inf on the pad columns v >= V (masks them)
  float* part;                   // [R][ntn][kDecEW][2 + 2 KR] logits-tile partials (max, sum-exp, top-K)
};
constexpr int kDecBN = 256;       // logits tile width
constexpr int kDecEW = 2;         // logits epilogue warps per TMEM lane quarter
constexpr int kCellBN = 128;      // gate tile width: 32 units x (i, f, g, o)
inline int dec_vp(int V) { return (V + 15) / 16 * 16; }
inline int dec_ntn(int V) { return (dec_vp(V) + kDecBN - 1) / kDecBN; }
// SKB_DEC_TC=1 selects the engine path for TF32 LSTM decoding.  Measured on the B200 at the
// C3 shape it is 2.2x slower than the library GEMMs + beam_rows (4.6 vs 2.1 ms per decode:
// the 1-CTA 128x256 tcgen05 tiles run the logits GEMM at ~350 TFLOP/s vs CUTLASS's 2-SM
// 256x256 at ~600, and the per-row top-K insertion in the epilogue costs more than the
// logits round trip it removes), so it is opt-in (profiles/r02_c3_engine.md).
// The workspace holds the engine path's buffers whenever the shape is eligible, so the
// layout (sized once per Decoder) does not depend on the environment at call time.
inline bool dec_tc_shape(const skb_decode_shape& d) {
  return d.math == 1 && d.cell == SKB_CELL_LSTM && d.embed % 4 == 0 && d.hidden % 32 == 0;
}
inline bool dec_tc(const skb_decode_shape& d) {
  const char* e = getenv("SKB_DEC_TC");
  return e && atoi(e) == 1 && dec_tc_shape(d);
}

__device__ __forceinline__ float sigmoidf_ref(float x) {   // reference tensor.py:403-407 (two branches)
  if (x >= 0.f) return 1.f / (1.f + expf(-x));
  const float e = expf(x);
  return e / (1.f + e);
}

__global__ void dec_gather(DecodeState st, const float* __restrict__ emb, int R, int E, int H) {
  const int t = *st.tstep;
  if (st.active[t] == 0) return;
  const float* __restrict__ h = st.h[t & 1];
  const int32_t* __restrict__ tok = st.tok;
  float* __restrict__ xh = st.xh;
  const int W = E + H;
  for (int r = blockIdx.x; r < R; r += gridDim.x) {   // one CTA per row: coalesced row copies
    const float* e = emb + (long long)tok[r] * E;
    float* o = xh + (long long)r * W;
    for (int k = threadIdx.x; k < E; k += blockDim.x) o[k] = e[k];
    for (int k = threadIdx.x; k < H; k += blockDim.x) o[E + k] = h[(long long)r * H + k];
  }
}

__global__ void dec_cell(DecodeState st, int cell, const float* __restrict__ bias, int R, int H) {
  const int t = *st.tstep;
  if (st.active[t] == 0) return;
  const float* __restrict__ gates = st.gates;
  const float* __restrict__ c = st.c[t & 1];
  float* __restrict__ hn = st.hn;
  float* __restrict__ cn = st.cn;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < (long long)R * H;
       i += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(i / H), k = (int)(i % H);
    if (cell == SKB_CELL_RNN_TANH) {
      hn[i] = tanhf(gates[i]);
      continue;
    }
    const float* g = gates + (long long)r * 4 * H;
    float gi = g[k], gf = g[H + k], gg = g[2 * H + k], go = g[3 * H + k];
    if (bias) { gi += bias[k]; gf += bias[H + k]; gg += bias[2 * H + k]; go += bias[3 * H + k]; }
    const float c2 = sigmoidf_ref(gf) * c[i] + sigmoidf_ref(gi) * tanhf(gg);
    cn[i] = c2;
    hn[i] = sigmoidf_ref(go) * tanhf(c2);
  }
}

// Row-parallel variants (H % 4 == 0, E % 4 == 0): blockIdx.y = row, float4 over
// units, no per-element index division; same per-element arithmetic.
__global__ void dec_gather4(DecodeState st, const float* __restrict__ emb, int R, int E, int H) {
  const int t = *st.tstep;
  if (st.active[t] == 0) return;
  const int r = blockIdx.y, W = E + H;
  const float4* e = reinterpret_cast<const float4*>(emb + (long long)st.tok[r] * E);
  const float4* h = reinterpret_cast<const float4*>(st.h[t & 1] + (long long)r * H);
  float4* o = reinterpret_cast<float4*>(st.xh + (long long)r * W);
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < (E + H) / 4; k += gridDim.x * blockDim.x)
    o[k] = k < E / 4 ? e[k] : h[k - E / 4];
}

__global__ void dec_cell4(DecodeState st, const float* __restrict__ bias, int R, int H) {
  const int t = *st.tstep;
  if (st.active[t] == 0) return;
  const int r = blockIdx.y;
  const float* g = st.gates + (long long)r * 4 * H;
  const float* c = st.c[t & 1] + (long long)r * H;
  for (int k = 4 * (blockIdx.x * blockDim.x + threadIdx.x); k < H; k += 4 * gridDim.x * blockDim.x) {
    const float4 gi = *reinterpret_cast<const float4*>(g + k), gf = *reinterpret_cast<const float4*>(g + H + k);
    const float4 gg = *reinterpret_cast<const float4*>(g + 2 * H + k), go = *reinterpret_cast<const float4*>(g + 3 * H + k);
    const float4 cv = *reinterpret_cast<const float4*>(c + k);
    float a[4][4] = {{gi.x, gi.y, gi.z, gi.w}, {gf.x, gf.y, gf.z, gf.w}, {gg.x, gg.y, gg.z, gg.w}, {go.x, go.y, go.z, go.w}};
    if (bias) {
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int e = 0; e < 4; ++e) a[q][e] += bias[q * H + k + e];
    }
    const float cp[4] = {cv.x, cv.y, cv.z, cv.w};
    float cn[4], hn[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      cn[e] = sigmoidf_ref(a[1][e]) * cp[e] + sigmoidf_ref(a[0][e]) * tanhf(a[2][e]);
      hn[e] = sigmoidf_ref(a[3][e]) * tanhf(cn[e]);
    }
    *reinterpret_cast<float4*>(st.cn + (long long)r * H + k) = make_float4(cn[0], cn[1], cn[2], cn[3]);
    *reinterpret_cast<float4*>(st.hn + (long long)r * H + k) = make_float4(hn[0], hn[1], hn[2], hn[3]);
  }
}

// (value desc, index asc): does (va, ia) rank before (vb, ib)?
__device__ __forceinline__ bool better(float va, int ia, float vb, int ib) {
  return va > vb || (va == vb && ia < ib);
}
__device__ __forceinline__ bool better_d(double va, int ia, double vb, int ib) {
  return va > vb || (va == vb && ia < ib);
}

// Per-lane sorted top-K insert (static indices: registers).
template <int K>
__device__ __forceinline__ void topk_insert(float (&v)[K], int (&ix)[K], float x, int i) {
  if (!better(x, i, v[K - 1], ix[K - 1])) return;
  v[K - 1] = x; ix[K - 1] = i;
#pragma unroll
  for (int k = K - 1; k > 0; --k) {
    if (better(v[k], ix[k], v[k - 1], ix[k - 1])) {
      const float tv = v[k]; v[k] = v[k - 1]; v[k - 1] = tv;
      const int ti = ix[k]; ix[k] = ix[k - 1]; ix[k - 1] = ti;
    }
  }
}

// Pass 1 — one CTA per beam row (R CTAs fill the machine): a single HBM pass
// over the row's logits (float4 loads) computes the log-softmax normaliser
// (per-thread max / sum-exp, merged with warp shuffles then across warps) and
// the row's K best (value desc, index asc) — per-thread register lists merged
// K times by warp-shuffle argmax, then across the CTA's warps.
template <int K>
__global__ void __launch_bounds__(ROW_THREADS) beam_rows(DecodeState st, int V, const float* __restrict__ b_out) {
  const int t = *st.tstep, cur = t & 1;
  if (st.active[t] == 0) return;
  __shared__ float wv[ROW_THREADS / 32][K], wm[ROW_THREADS / 32], ws[ROW_THREADS / 32];
  __shared__ int wi[ROW_THREADS / 32][K];
  const int r = blockIdx.x;
  if (st.fin[cur][r]) return;   // finished beams offer only (EOS, score) in pass 2
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float* L = st.logits + (long long)r * V;
  float mx = -INFINITY, sum = 0.f;
  // The warp's K best so far live one per lane (lanes 0..K-1, best first);
  // `thr` is the K-th value.  Elements are filtered by one compare + ballot
  // and only the rare survivors are inserted (warp-cooperatively).
  float lv = -INFINITY;
  int li = 0x7fffffff;
  float thr = -INFINITY;
  int thr_i = 0x7fffffff;
  // floor: a value with at least K elements >= it already seen (the K-th largest lane maximum of
  // the warp's first chunk), so while the list still holds -inf entries the threshold does not
  // drop below it and the first chunk offers a handful of candidates instead of all of them
  float fl = -INFINITY;
  auto offer = [&](float x, int v) {
    unsigned m = __ballot_sync(0xffffffffu, better(x, v, thr, thr_i));
    while (m) {
      const int src = __ffs(m) - 1;
      m &= m - 1;
      const float cv = __shfl_sync(0xffffffffu, x, src);
      const int ci = __shfl_sync(0xffffffffu, v, src);
      if (!better(cv, ci, thr, thr_i)) continue;   // the threshold rose since the ballot
      const unsigned ahead = __ballot_sync(0xffffffffu, lane < K && better(lv, li, cv, ci));
      const int pos = __popc(ahead);                // entries that stay ahead of the candidate
      const float uv = __shfl_up_sync(0xffffffffu, lv, 1);
      const int ui = __shfl_up_sync(0xffffffffu, li, 1);
      if (lane == pos) { lv = cv; li = ci; }
      else if (lane > pos && lane < K) { lv = uv; li = ui; }
      thr = __shfl_sync(0xffffffffu, lv, K - 1);
      thr_i = __shfl_sync(0xffffffffu, li, K - 1);
      if (fl > thr) { thr = fl; thr_i = 0x7fffffff; }
    }
  };
  // Chunks of 4*U values per lane: one max per chunk rescales the running sum
  // at most once; every element costs one exp + add and one compare.
  const int V4 = (V % 4 == 0) ? V / 4 : 0;   // rows are 16-byte aligned when V % 4 == 0
  const float4* L4 = reinterpret_cast<const float4*>(L);
  const float4* B4 = reinterpret_cast<const float4*>(b_out);
  constexpr int U = 8;   // float4 loads in flight per thread before any is consumed
  const int warp_base = warp * 32 + lane;   // warps own interleaved float4 columns
  int q0 = warp_base;
  // every lane runs the same trip count (ballots need the whole warp);
  // out-of-range float4s read as -inf
  for (; q0 - warp_base < V4; q0 += U * ROW_THREADS) {
    float x[4 * U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int q = q0 + u * ROW_THREADS;
      float4 f = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
      if (q < V4) {
        f = __ldcs(L4 + q);   // streamed once: evict-first
        if (b_out) {
          const float4 b = __ldg(B4 + q);
          f.x += b.x; f.y += b.y; f.z += b.z; f.w += b.w;
        }
      }
      x[4 * u] = f.x; x[4 * u + 1] = f.y; x[4 * u + 2] = f.z; x[4 * u + 3] = f.w;
    }
    float cm = x[0];
#pragma unroll
    for (int e = 1; e < 4 * U; ++e) cm = fmaxf(cm, x[e]);
    if (cm > mx) { sum *= __expf(mx - cm); mx = cm; }
    if (cm != -INFINITY) {
#pragma unroll
      for (int e = 0; e < 4 * U; ++e) sum += __expf(x[e] - mx);
    }
    if (thr == -INFINITY && fl == -INFINITY) {   // warp-uniform: the first chunk with values
      float c = cm, m = -INFINITY;
#pragma unroll 1
      for (int k = 0; k < K; ++k) {   // K-th largest of the lanes' chunk maxima
        m = c;
#pragma unroll
        for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        const unsigned b = __ballot_sync(0xffffffffu, c == m);
        if (lane == __ffs(b) - 1) c = -INFINITY;
      }
      fl = m;
      if (fl > thr) { thr = fl; thr_i = 0x7fffffff; }
    }
    if (__any_sync(0xffffffffu, cm >= thr && cm != -INFINITY)) {
#pragma unroll
      for (int e = 0; e < 4 * U; ++e) offer(x[e], 4 * (q0 + (e >> 2) * ROW_THREADS) + (e & 3));
    }
  }
  // rows whose length is not a multiple of 4: scalar pass, same trip count per lane
  if (V4 == 0) {
    for (int v0 = 0; v0 < V; v0 += ROW_THREADS) {
      const int v = v0 + threadIdx.x;
      const bool ok = v < V;
      const float x = ok ? L[v] + (b_out ? b_out[v] : 0.f) : -INFINITY;
      if (ok) {
        if (x > mx) { sum = sum * __expf(mx - x) + 1.f; mx = x; } else { sum += __expf(x - mx); }
      }
      offer(x, ok ? v : 0x7fffffff);
    }
  }
  // normaliser: warp then CTA
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, mx, o), s2 = __shfl_xor_sync(0xffffffffu, sum, o);
    const float m = fmaxf(mx, m2);
    sum = (mx == -INFINITY ? 0.f : sum * __expf(mx - m)) + (m2 == -INFINITY ? 0.f : s2 * __expf(m2 - m));
    mx = m;
  }
  if (lane == 0) { wm[warp] = mx; ws[warp] = sum; }
  if (lane < K) { wv[warp][lane] = lv; wi[warp][lane] = li; }
  __syncthreads();
  if (warp == 0) {
    // normaliser across warps
    float m = lane < ROW_THREADS / 32 ? wm[lane] : -INFINITY;
    float sm = lane < ROW_THREADS / 32 ? ws[lane] : 0.f;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, sm, o);
      const float mm = fmaxf(m, m2);
      sm = (m == -INFINITY ? 0.f : sm * __expf(m - mm)) + (m2 == -INFINITY ? 0.f : s2 * __expf(m2 - mm));
      m = mm;
    }
    // top-K across warps: lane w holds warp w's sorted list head
    int head = 0;
    for (int k = 0; k < K; ++k) {
      float bv = -INFINITY;
      int bi = 0x7fffffff, bl = lane;
      if (lane < ROW_THREADS / 32 && head < K) { bv = wv[lane][head]; bi = wi[lane][head]; }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o), ol = __shfl_xor_sync(0xffffffffu, bl, o);
        if (better(ov, oi, bv, bi)) { bv = ov; bi = oi; bl = ol; }
      }
      if (lane == 0) { st.row_v[(long long)r * KMAX + k] = bv; st.row_i[(long long)r * KMAX + k] = bi; }
      if (lane == bl) ++head;
    }
    if (lane == 0) st.row_lse[r] = m + logf(sm);
  }
}

// Pass 2 — one CTA (warp) per sentence: rank its K x K candidates (score +
// logit - lse for live beams, (EOS, score) for finished ones; score desc,
// flat index b*V+v asc), then reindex state and history from the parents.
template <int K>
__global__ void __launch_bounds__(SEL_THREADS) beam_choose(DecodeState st, int S, int V, int H, int LT, int eos) {
  const int t = *st.tstep, cur = t & 1;
  if (st.active[t] == 0) return;
  __shared__ int sel_par[KMAX], sel_tok[KMAX];
  __shared__ double sel_score[KMAX];
  const int s = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nxt = cur ^ 1;
  // K*K <= 64 candidates, one per thread of the first two warps; a candidate's rank is
  // the number of candidates that order before it (score desc, flat index asc: a total
  // order, so ranks are distinct) and the K best write themselves to slots 0..K-1.
  __shared__ double cand_s[KMAX * KMAX];
  __shared__ int cand_i[KMAX * KMAX];
  const int slot = threadIdx.x;
  double cs = -INFINITY;
  int ci = 0x7fffffff;   // flat index b*V + v
  if (slot < K * K) {
    const int b = slot / K, k = slot % K, r = s * K + b;
    const double sc = st.score[cur][r];
    if (st.fin[cur][r]) {
      if (k == 0) { cs = sc; ci = b * V + eos; }
    } else {
      const int v = st.row_i[(long long)r * KMAX + k];
      if (v != 0x7fffffff) {
        ci = b * V + v;
        if (sc != -INFINITY) cs = sc + ((double)st.row_v[(long long)r * KMAX + k] - (double)st.row_lse[r]);
      }
    }
    cand_s[slot] = cs;
    cand_i[slot] = ci;
  }
  __syncthreads();
  if (slot < K * K) {
    int rank = 0;
#pragma unroll 8
    for (int o = 0; o < K * K; ++o) rank += better_d(cand_s[o], cand_i[o], cs, ci) ? 1 : 0;
    if (rank < K) { sel_score[rank] = cs; sel_par[rank] = ci / V; sel_tok[rank] = ci % V; }
  }
  __syncthreads();
  // reindex: beam j of the next step continues parent p = sel_par[j]
  for (int j = warp; j < K; j += SEL_THREADS / 32) {
    const int p = sel_par[j], rp = s * K + p, rj = s * K + j;
    const bool pfin = st.fin[cur][rp] != 0;
    const float* hs = pfin ? st.h[cur] + (long long)rp * H : st.hn + (long long)rp * H;
    const float* cs = pfin ? st.c[cur] + (long long)rp * H : st.cn + (long long)rp * H;
    if ((H & 3) == 0) {   // float4 row copies, all loads of a lane issued before the stores
      const float4* hs4 = reinterpret_cast<const float4*>(hs);
      const float4* cs4 = reinterpret_cast<const float4*>(cs);
      float4* hd4 = reinterpret_cast<float4*>(st.h[nxt] + (long long)rj * H);
      float4* cd4 = reinterpret_cast<float4*>(st.c[nxt] + (long long)rj * H);
      for (int k = lane; k < H / 4; k += 64) {
        const float4 a = hs4[k], b = cs4[k];
        const bool two = k + 32 < H / 4;
        float4 a2, b2;
        if (two) { a2 = hs4[k + 32]; b2 = cs4[k + 32]; }
        hd4[k] = a; cd4[k] = b;
        if (two) { hd4[k + 32] = a2; cd4[k + 32] = b2; }
      }
    } else {
      for (int k = lane; k < H; k += 32) {
        st.h[nxt][(long long)rj * H + k] = hs[k];
        st.c[nxt][(long long)rj * H + k] = cs[k];
      }
    }
    for (int k = lane; k <= t; k += 32) st.hist[nxt][(long long)rj * LT + k] = st.hist[cur][(long long)rp * LT + k];
    if (lane == 0) {
      const int v = sel_tok[j];
      st.hist[nxt][(long long)rj * LT + t + 1] = v;
      st.tok[rj] = v;
      st.score[nxt][rj] = sel_score[j];
      st.fin[nxt][rj] = (pfin || v == eos) ? 1 : 0;
      st.len[nxt][rj] = st.len[cur][rp] + (pfin ? 0 : 1);
      // greedy: the chosen token's lead over the runner-up (pass 1 ran with top-2),
      // so the host can detect an argmax that fp32 rounding could have flipped
      if (K == 1 && !pfin)
        st.margin[rj] = fminf(st.margin[rp], st.row_v[(long long)rp * KMAX] - st.row_v[(long long)rp * KMAX + 1]);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int live = 0;
    for (int j = 0; j < K; ++j) live |= st.fin[nxt][s * K + j] == 0;
    if (live) atomicAdd(&st.active[t + 1], 1);
  }
}

// ------------------------------------------------------------------ tensor-core path
// Weights for the engine (once per decode): gate-interleaved W_gates^T, bias, w_out^T.
__global__ void dec_prep_gates(const float* __restrict__ w_gates, const float* __restrict__ b_gates,
                               float* __restrict__ wgT, float* __restrict__ bg, int KG, int H) {
  const int G = 4 * H;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < (long long)G * KG;
       i += (long long)gridDim.x * blockDim.x) {
    const int n = (int)(i / KG), k = (int)(i % KG);
    wgT[i] = w_gates[(long long)k * G + (n & 3) * H + (n >> 2)];
  }
  for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < G; n += gridDim.x * blockDim.x)
    bg[n] = b_gates ? b_gates[(n & 3) * H + (n >> 2)] : 0.f;
}
// woT[v][k] = w_out[k][v] (32 x 32 shared-memory tiles: coalesced both ways), zero rows v >= V.
__global__ void dec_prep_out(const float* __restrict__ w_out, const float* __restrict__ b_out, float* __restrict__ woT,
                             float* __restrict__ bo, int H, int V, int Vp) {
  __shared__ float tile[32][33];
  if (blockIdx.y == 0 && threadIdx.y == 0) {
    const int v = blockIdx.x * 32 + threadIdx.x;
    if (v < Vp) bo[v] = v < V ? (b_out ? b_out[v] : 0.f) : -INFINITY;
  }
  const int v0 = blockIdx.x * 32, k0 = blockIdx.y * 32;
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int k = k0 + j, v = v0 + threadIdx.x;
    tile[j][threadIdx.x] = (k < H && v < V) ? w_out[(long long)k * V + v] : 0.f;
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int v = v0 + j, k = k0 + threadIdx.x;
    if (v < Vp && k < H) woT[(long long)v * H + k] = tile[threadIdx.x][j];
  }
}

// Gate GEMM epilogue: 16 accumulator columns = 4 units x (i, f, g, o) -> c', h' (the
// arithmetic of dec_cell4: bias, reference sigmoid branches, tanhf).
struct EpiDecCell {
  static constexpr uint32_t kOpBytes = 0;
  struct State {};
  DecodeState st;
  int H;
  SKB_DEV bool skip() const { return st.active[*st.tstep] == 0; }
  SKB_DEV bool ops_on() const { return false; }
  SKB_DEV void prefetch(uint8_t*, int, int, uint64_t*) const {}
  SKB_DEV void begin_tile(State&, int, int, int, int) const {}
  SKB_DEV void chunk(State&, const uint8_t*, int, int m, int n0, int, int, const float (&v)[16], bool row_ok) const {
    if (!row_ok) return;
    const int j0 = n0 >> 2, cur = *st.tstep & 1;
    const float4 cv = *reinterpret_cast<const float4*>(st.c[cur] + (long long)m * H + j0);
    const float4 b0 = *reinterpret_cast<const float4*>(st.bg + n0), b1 = *reinterpret_cast<const float4*>(st.bg + n0 + 4);
    const float4 b2 = *reinterpret_cast<const float4*>(st.bg + n0 + 8), b3 = *reinterpret_cast<const float4*>(st.bg + n0 + 12);
    const float bb[16] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w, b2.x, b2.y, b2.z, b2.w, b3.x, b3.y, b3.z, b3.w};
    const float cp[4] = {cv.x, cv.y, cv.z, cv.w};
    float cn[4], hn[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float ig = v[4 * u] + bb[4 * u], fg = v[4 * u + 1] + bb[4 * u + 1];
      const float gg = v[4 * u + 2] + bb[4 * u + 2], og = v[4 * u + 3] + bb[4 * u + 3];
      cn[u] = sigmoidf_ref(fg) * cp[u] + sigmoidf_ref(ig) * tanhf(gg);
      hn[u] = sigmoidf_ref(og) * tanhf(cn[u]);
    }
    *reinterpret_cast<float4*>(st.cn + (long long)m * H + j0) = make_float4(cn[0], cn[1], cn[2], cn[3]);
    *reinterpret_cast<float4*>(st.hn + (long long)m * H + j0) = make_float4(hn[0], hn[1], hn[2], hn[3]);
  }
  SKB_DEV void end_tile(State&, int, int, int, int, int) const {}
};

// Logits GEMM epilogue: per row and tile column group, the online max / sum-exp and the
// KR best (value desc, index asc) of logit + b_out — one partial record per (row, tile,
// group); the [R, V] logits are never stored.
template <int KR>
struct EpiLogits {
  static constexpr uint32_t kOpBytes = 0;
  struct State { float mx, sum; float v[KR]; int ix[KR]; };
  DecodeState st;
  const float* b_out;
  int V, ntn, R;
  SKB_DEV bool skip() const { return st.active[*st.tstep] == 0; }
  SKB_DEV bool ops_on() const { return false; }
  SKB_DEV void prefetch(uint8_t*, int, int, uint64_t*) const {}
  SKB_DEV void begin_tile(State& es, int, int, int, int) const {
    es.mx = -INFINITY;
    es.sum = 0.f;
#pragma unroll
    for (int k = 0; k < KR; ++k) { es.v[k] = -INFINITY; es.ix[k] = 0x7fffffff; }
  }
  SKB_DEV void chunk(State& es, const uint8_t*, int, int, int n0, int, int, const float (&a)[16], bool row_ok) const {
    if (!row_ok) return;
    // bias (pad columns carry -inf: no per-element range test), branch-free max / sum-exp
    const float4* b4 = reinterpret_cast<const float4*>(st.bo + n0);
    float x[16];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float4 b = __ldg(b4 + q);
      x[4 * q] = a[4 * q] + b.x; x[4 * q + 1] = a[4 * q + 1] + b.y;
      x[4 * q + 2] = a[4 * q + 2] + b.z; x[4 * q + 3] = a[4 * q + 3] + b.w;
    }
    float cm = x[0];
#pragma unroll
    for (int i = 1; i < 16; ++i) cm = fmaxf(cm, x[i]);
    if (cm == -INFINITY) return;
    const float nm = fmaxf(es.mx, cm);
    const float l2e = 1.4426950408889634f, off = -nm * l2e;
    float s4[4] = {0.f, 0.f, 0.f, 0.f};   // four independent chains, ex2 of (x - max) log2 e
#pragma unroll
    for (int i = 0; i < 16; ++i) s4[i & 3] += exp2f(fmaf(x[i], l2e, off));
    es.sum = es.sum * exp2f(fmaf(es.mx, l2e, off)) + ((s4[0] + s4[1]) + (s4[2] + s4[3]));
    es.mx = nm;
    if (cm >= es.v[KR - 1]) {
#pragma unroll
      for (int i = 0; i < 16; ++i) topk_insert<KR>(es.v, es.ix, x[i], n0 + i);
    }
  }
  SKB_DEV void end_tile(State& es, int tm, int tn, int, int slot, int lane) const {
    const int m = tm * 128 + ((slot + 2) & 3) * 32 + lane, cg = slot >> 2;   // slot = warp - 2
    if (m < R) {
      float* p = st.part + (((long long)m * ntn + tn) * kDecEW + cg) * (2 + 2 * KR);
      p[0] = es.mx;
      p[1] = es.sum;
#pragma unroll
      for (int k = 0; k < KR; ++k) { p[2 + k] = es.v[k]; p[2 + KR + k] = __int_as_float(es.ix[k]); }
    }
  }
};

// Merge of the logits partials, one warp per live beam row: log-sum-exp and the row's KR
// best (value desc, index asc) -> row_v / row_i / row_lse (what beam_rows produces).
template <int KR>
__global__ void dec_merge(DecodeState st, int R, int ntn) {
  const int t = *st.tstep, cur = t & 1;
  if (st.active[t] == 0) return;
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= R || st.fin[cur][r]) return;
  const int np = ntn * kDecEW;
  const float* P = st.part + (long long)r * np * (2 + 2 * KR);
  float mx = -INFINITY, sum = 0.f, v[KR];
  int ix[KR];
#pragma unroll
  for (int k = 0; k < KR; ++k) { v[k] = -INFINITY; ix[k] = 0x7fffffff; }
  for (int p = lane; p < np; p += 32) {
    const float* q = P + (long long)p * (2 + 2 * KR);
    const float pm = q[0], ps = q[1];
    if (pm != -INFINITY) {
      const float m = fmaxf(mx, pm);
      sum = (mx == -INFINITY ? 0.f : sum * __expf(mx - m)) + ps * __expf(pm - m);
      mx = m;
    }
#pragma unroll
    for (int k = 0; k < KR; ++k) topk_insert<KR>(v, ix, q[2 + k], __float_as_int(q[2 + KR + k]));
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, mx, o), s2 = __shfl_xor_sync(0xffffffffu, sum, o);
    const float m = fmaxf(mx, m2);
    sum = (mx == -INFINITY ? 0.f : sum * __expf(mx - m)) + (m2 == -INFINITY ? 0.f : s2 * __expf(m2 - m));
    mx = m;
  }
  int head = 0;
  for (int k = 0; k < KR; ++k) {
    float bv = -INFINITY;
    int bi = 0x7fffffff, bl = lane;
#pragma unroll
    for (int j = 0; j < KR; ++j)
      if (j == head) { bv = v[j]; bi = ix[j]; }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o), ol = __shfl_xor_sync(0xffffffffu, bl, o);
      if (better(ov, oi, bv, bi) || (ov == bv && oi == bi && ol < bl)) { bv = ov; bi = oi; bl = ol; }
    }
    if (lane == 0) { st.row_v[(long long)r * KMAX + k] = bv; st.row_i[(long long)r * KMAX + k] = bi; }
    if (lane == bl) ++head;
  }
  if (lane == 0) st.row_lse[r] = mx + logf(sum);
}

// Steps that found every sentence finished leave the state untouched: carry
// the current ping-pong side forward so the host can read "side of step T".
__global__ void dec_init(DecodeState st, const float* __restrict__ h0, const float* __restrict__ c0, int S, int K,
                         int H, int LT, int max_len) {
  const int R = S * K;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < (long long)R * H;
       i += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(i / H), k = (int)(i % H), s = r / K;
    st.h[0][i] = h0[(long long)s * H + k];
    st.c[0][i] = c0 ? c0[(long long)s * H + k] : 0.f;
  }
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < (long long)R * LT;
       i += (long long)gridDim.x * blockDim.x) {
    st.hist[0][i] = 0;
    st.hist[1][i] = 0;
  }
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < R; r += gridDim.x * blockDim.x) {
    st.tok[r] = 0;
    st.score[0][r] = (r % K == 0) ? 0.0 : -INFINITY;
    st.fin[0][r] = 0;
    st.len[0][r] = 0;
    st.margin[r] = INFINITY;
  }
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t <= max_len; t += gridDim.x * blockDim.x)
    st.active[t] = t == 0 ? S : 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) *st.tstep = 0;
}

// The loop's end of step: advance the device step counter and, inside the
// conditional-WHILE graph, decide whether the body runs again (the EOS stop
// and max_len test evaluated on the device: no host round trip per step).
__global__ void dec_advance(DecodeState st, int max_len, cudaGraphConditionalHandle cond, int use_cond) {
  const int t = *st.tstep;
  const int t1 = st.active[t] > 0 ? t + 1 : t;   // a step that found nothing live does not count
  *st.tstep = t1;
  if (use_cond) cudaGraphSetConditional(cond, (t1 < max_len && st.active[t1] > 0) ? 1u : 0u);
}

__global__ void dec_output(DecodeState st, int R, int LT, int32_t* tokens, float* scores, int32_t* lengths) {
  const int side = *st.tstep & 1;   // step k writes side (k+1)&1
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < (long long)R * LT;
       i += (long long)gridDim.x * blockDim.x)
    tokens[i] = st.hist[side][i];
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < R; r += gridDim.x * blockDim.x) {
    scores[r] = (float)st.score[side][r];
    lengths[r] = st.len[side][r];
  }
}

// Optional per-phase timing of skb_decode (skb_decode_profile): CUDA events
// around each step's phases on the decode stream, summed on read.
enum { P_GATHER_CELL = 0, P_GEMM_GATES = 1, P_GEMM_LOGITS = 2, P_SELECT = 3, P_N = 4 };
constexpr int kProfSteps = 1024;
bool g_dprof = false;
cudaEvent_t g_dev[kProfSteps][P_N + 1];
int g_dsteps = 0;
bool g_dinit = false;

void prof_mark(int step, int k, cudaStream_t cs) {
  if (g_dprof && step < kProfSteps) cudaEventRecord(g_dev[step][k], cs);
}

size_t al(size_t b) { return (b + 255) & ~size_t(255); }

size_t layout(const skb_decode_shape& d, DecodeState* st, uint8_t* base) {
  const size_t R = (size_t)d.sentences * d.beam, E = d.embed, H = d.hidden, V = d.vocab;
  const size_t G = d.cell == SKB_CELL_LSTM ? 4 * H : H, LT = d.max_len + 1;
  size_t off = 0;
  auto take = [&](size_t bytes) { uint8_t* p = base ? base + off : nullptr; off += al(bytes); return p; };
  DecodeState s;
  s.xh = (float*)take(4 * R * (E + H));
  s.gates = (float*)take(4 * R * G);
  for (int k = 0; k < 2; ++k) { s.h[k] = (float*)take(4 * R * H); s.c[k] = (float*)take(4 * R * H); }
  s.hn = (float*)take(4 * R * H);
  s.cn = (float*)take(4 * R * H);
  s.logits = (float*)take(4 * R * V);
  for (int k = 0; k < 2; ++k) {
    s.score[k] = (double*)take(8 * R);
    s.fin[k] = (int32_t*)take(4 * R);
    s.len[k] = (int32_t*)take(4 * R);
    s.hist[k] = (int32_t*)take(4 * R * LT);
  }
  s.tok = (int32_t*)take(4 * R);
  s.active = (int32_t*)take(4 * (LT + 1));
  s.tstep = (int32_t*)take(4);
  s.row_v = (float*)take(4 * R * KMAX);
  s.row_i = (int32_t*)take(4 * R * KMAX);
  s.row_lse = (float*)take(4 * R);
  s.margin = (float*)take(4 * R);
  s.wgT = s.bg = s.woT = s.bo = s.part = nullptr;
  if (dec_tc_shape(d)) {
    const int KR = d.beam < 2 ? 2 : d.beam;
    s.wgT = (float*)take(4 * G * (E + H));
    s.bg = (float*)take(4 * G);
    s.woT = (float*)take(4 * (size_t)dec_vp((int)V) * H);
    s.bo = (float*)take(4 * (size_t)dec_vp((int)V));
    s.part = (float*)take(4 * R * dec_ntn((int)V) * kDecEW * (2 + 2 * KR));
  }
  if (st) *st = s;
  return off;
}

cublasHandle_t handle_for(void* stream) {
  static cublasHandle_t h = nullptr;
  if (!h && cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) return nullptr;
  cublasSetStream(h, (cudaStream_t)stream);
  return h;
}

// C[M,N] (row-major) = A[M,K] @ B[K,N] (row-major): column-major C^T = B^T A^T.
bool gemm(cublasHandle_t h, int math, const float* A, const float* B, float* C, int M, int N, int K) {
  const float one = 1.f, zero = 0.f;
  const cublasComputeType_t ct = math == 1 ? CUBLAS_COMPUTE_32F_FAST_TF32 : CUBLAS_COMPUTE_32F_PEDANTIC;
  return cublasGemmEx(h, CUBLAS_OP_N, CUBLAS_OP_N, N, M, K, &one, B, CUDA_R_32F, N, A, CUDA_R_32F, K, &zero, C,
                      CUDA_R_32F, N, ct, CUBLAS_GEMM_DEFAULT) == CUBLAS_STATUS_SUCCESS;
}

}  // namespace

extern "C" int64_t skb_decode_workspace_bytes(const skb_decode_shape* d) {
  if (!d) return -1;
  return (int64_t)layout(*d, nullptr, nullptr);
}

extern "C" int64_t skb_decode_margin_offset(const skb_decode_shape* d) {
  if (!d) return -1;
  DecodeState st;
  uint8_t* base = reinterpret_cast<uint8_t*>(uintptr_t(1) << 20);   // any non-null base: offsets only
  layout(*d, &st, base);
  return (int64_t)(reinterpret_cast<uint8_t*>(st.margin) - base);
}

namespace {

// One decode step on stream `cs` (kernels read the step index from st.tstep).
// The TF32 LSTM step on the engine: gather, gate GEMM + fused cell, logits GEMM + fused
// log-softmax / top-K partials, merge, choose, advance.
template <int K>
bool enqueue_step_tc(const skb_decode_shape* d, DecodeState& st, cudaStream_t cs, const float* emb, const float* b_out,
                     cudaGraphConditionalHandle cond, int use_cond, int prof_step) {
  namespace gm = skb::gemm;
  constexpr int KR = K < 2 ? 2 : K;
  const int S = d->sentences, R = S * K, E = d->embed, H = d->hidden, V = d->vocab, G = 4 * H, LT = d->max_len + 1;
  const int Vp = dec_vp(V), ntn = dec_ntn(V), KG = E + H;
  prof_mark(prof_step, 0, cs);
  dec_gather4<<<dim3((KG / 4 + 127) / 128, R), 128, 0, cs>>>(st, emb, R, E, H);
  prof_mark(prof_step, 1, cs);
  CUtensorMap ma, mb, ml, mo;
  if (!gm::encode_2d(&ma, gm::kTF32, st.xh, KG, R, KG, 32, 128) ||
      !gm::encode_2d(&mb, gm::kTF32, st.wgT, KG, G, KG, 32, kCellBN) ||
      !gm::encode_2d(&ml, gm::kTF32, st.hn, H, R, H, 32, 128) ||
      !gm::encode_2d(&mo, gm::kTF32, st.woT, H, Vp, H, 32, kDecBN))
    return false;
  {
    EpiDecCell e;
    e.st = st; e.H = H;
    gm::Shape sh{R, G, KG, 1, 0};
    if (gm::launch<gm::kTF32, kCellBN, false, false, EpiDecCell, false, 2>(ma, mb, sh, e, cs)) return false;
  }
  prof_mark(prof_step, 2, cs);
  {
    EpiLogits<KR> e;
    e.st = st; e.b_out = b_out; e.V = V; e.ntn = ntn; e.R = R;
    gm::Shape sh{R, Vp, H, 1, 0};
    if (gm::launch<gm::kTF32, kDecBN, false, false, EpiLogits<KR>, false, kDecEW>(ml, mo, sh, e, cs)) return false;
  }
  prof_mark(prof_step, 3, cs);
  dec_merge<KR><<<(R + 7) / 8, 256, 0, cs>>>(st, R, ntn);
  beam_choose<K><<<S, SEL_THREADS, 0, cs>>>(st, S, V, H, LT, d->eos);
  prof_mark(prof_step, 4, cs);
  dec_advance<<<1, 1, 0, cs>>>(st, d->max_len, cond, use_cond);
  return cudaPeekAtLastError() == cudaSuccess;
}

bool enqueue_step(const skb_decode_shape* d, DecodeState& st, cublasHandle_t hb, cudaStream_t cs, const float* emb,
                  const float* w_gates, const float* b_gates, const float* w_out, const float* b_out,
                  cudaGraphConditionalHandle cond, int use_cond, int prof_step) {
  if (dec_tc(*d)) {
    switch (d->beam) {
#define SKB_TC(k) case k: return enqueue_step_tc<k>(d, st, cs, emb, b_out, cond, use_cond, prof_step);
      SKB_TC(1) SKB_TC(2) SKB_TC(3) SKB_TC(4) SKB_TC(5) SKB_TC(6) SKB_TC(7) SKB_TC(8)
#undef SKB_TC
    }
    return false;
  }
  const int S = d->sentences, K = d->beam, R = S * K, E = d->embed, H = d->hidden, V = d->vocab;
  const int G = d->cell == SKB_CELL_LSTM ? 4 * H : H, LT = d->max_len + 1;
  const int rows = R < 148 * 8 ? R : 148 * 8;
  prof_mark(prof_step, 0, cs);
  const bool v4 = (E & 3) == 0 && (H & 3) == 0 && !getenv("SKB_DEC_SCALAR");
  if (v4)
    dec_gather4<<<dim3(((E + H) / 4 + 127) / 128, R), 128, 0, cs>>>(st, emb, R, E, H);
  else
    dec_gather<<<rows, 128, 0, cs>>>(st, emb, R, E, H);
  prof_mark(prof_step, 1, cs);
  if (!gemm(hb, d->math, st.xh, w_gates, st.gates, R, G, E + H)) return false;
  prof_mark(prof_step, 2, cs);
  if (v4 && d->cell == SKB_CELL_LSTM)
    dec_cell4<<<dim3((H / 4 + 127) / 128, R), 128, 0, cs>>>(st, b_gates, R, H);
  else
    dec_cell<<<148 * 8, 256, 0, cs>>>(st, d->cell, b_gates, R, H);
  if (!gemm(hb, d->math, st.hn, w_out, st.logits, R, V, H)) return false;
  prof_mark(prof_step, 3, cs);
  switch (K) {
#define SKB_SEL(k)                                                                               \
  case k:                                                                                        \
    beam_rows<(k == 1 ? 2 : k)><<<R, ROW_THREADS, 0, cs>>>(st, V, b_out);                        \
    beam_choose<k><<<S, SEL_THREADS, 0, cs>>>(st, S, V, H, LT, d->eos);                          \
    break;
    SKB_SEL(1) SKB_SEL(2) SKB_SEL(3) SKB_SEL(4) SKB_SEL(5) SKB_SEL(6) SKB_SEL(7) SKB_SEL(8)
#undef SKB_SEL
  }
  prof_mark(prof_step, 4, cs);
  dec_advance<<<1, 1, 0, cs>>>(st, d->max_len, cond, use_cond);
  return cudaPeekAtLastError() == cudaSuccess;
}

// Decode graphs: ONE conditional-WHILE node whose body is one decode step
// (captured once per shape / buffers), so a whole decode is a single graph
// launch and every loop decision is made on the device.
struct GraphEntry {
  skb_decode_shape d;
  const void* ptrs[6];
  int tc;   // captured on the engine path (SKB_DEC_TC) or the library path
  cudaGraphExec_t exec;
};
constexpr int kGraphCache = 16;
GraphEntry g_graphs[kGraphCache];
int g_ngraphs = 0;

cudaGraphExec_t decode_graph(const skb_decode_shape* d, DecodeState& st, cublasHandle_t hb, void* ws,
                             const float* emb, const float* w_gates, const float* b_gates, const float* w_out,
                             const float* b_out) {
  const void* key[6] = {ws, emb, w_gates, b_gates, w_out, b_out};
  const int tc = dec_tc(*d) ? 1 : 0;
  for (int i = 0; i < g_ngraphs; ++i) {
    GraphEntry& e = g_graphs[i];
    if (memcmp(&e.d, d, sizeof(*d)) == 0 && memcmp(e.ptrs, key, sizeof(key)) == 0 && e.tc == tc) return e.exec;
  }
  cudaGraph_t g = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaStream_t cap = nullptr;
  cudaGraphConditionalHandle cond;
  bool ok = cudaGraphCreate(&g, 0) == cudaSuccess &&
            cudaGraphConditionalHandleCreate(&cond, g, 1, cudaGraphCondAssignDefault) == cudaSuccess;
  cudaGraphNodeParams p = {};
  cudaGraphNode_t node;
  if (ok) {
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = cond;
    p.conditional.type = cudaGraphCondTypeWhile;
    p.conditional.size = 1;
    ok = cudaGraphAddNode(&node, g, nullptr, 0, &p) == cudaSuccess;
  }
  if (ok) ok = cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking) == cudaSuccess;
  if (ok) ok = cudaStreamBeginCaptureToGraph(cap, p.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                             cudaStreamCaptureModeRelaxed) == cudaSuccess;
  if (ok) {
    cublasSetStream(hb, cap);
    const bool enq = enqueue_step(d, st, hb, cap, emb, w_gates, b_gates, w_out, b_out, cond, 1, kProfSteps);
    cudaGraph_t body = nullptr;
    ok = cudaStreamEndCapture(cap, &body) == cudaSuccess && enq;
  }
  if (ok) ok = cudaGraphInstantiate(&exec, g, 0) == cudaSuccess;
  if (cap) cudaStreamDestroy(cap);
  if (g) cudaGraphDestroy(g);
  cudaGetLastError();   // a failed build falls back to the host-driven loop
  if (!ok) return nullptr;
  if (g_ngraphs == kGraphCache) {
    cudaGraphExecDestroy(g_graphs[0].exec);
    memmove(g_graphs, g_graphs + 1, sizeof(GraphEntry) * (kGraphCache - 1));
    --g_ngraphs;
  }
  GraphEntry& e = g_graphs[g_ngraphs++];
  e.d = *d;
  memcpy(e.ptrs, key, sizeof(key));
  e.tc = tc;
  e.exec = exec;
  return exec;
}

int g_last_mode = 0;   // 1 = conditional graph, 0 = host-driven loop

}  // namespace

extern "C" int skb_decode_last_mode(void) { return g_last_mode; }

extern "C" skb_status skb_decode(const skb_decode_shape* d, const float* h0, const float* c0, const float* emb,
                                 const float* w_gates, const float* b_gates, const float* w_out, const float* b_out,
                                 int32_t* tokens_out, float* scores_out, int32_t* lengths_out, int32_t* steps_out,
                                 void* workspace, void* stream) {
  if (!d || d->beam < 1 || d->beam > KMAX || d->sentences < 1 || d->vocab < d->beam || d->max_len < 0 ||
      (d->cell != SKB_CELL_LSTM && d->cell != SKB_CELL_RNN_TANH) || d->eos < 0 || d->eos >= d->vocab)
    return SKB_ERR_INVALID;
  cudaStream_t cs = (cudaStream_t)stream;
  DecodeState st;
  layout(*d, &st, (uint8_t*)workspace);
  const int S = d->sentences, K = d->beam, R = S * K, H = d->hidden, LT = d->max_len + 1;
  cublasHandle_t hb = handle_for(stream);
  if (!hb) return SKB_ERR_CUDA;
  static int32_t* host_word = nullptr;   // pinned poll / result word, allocated once
  if (!host_word && cudaMallocHost(&host_word, sizeof(int32_t) * 2) != cudaSuccess) return SKB_ERR_CUDA;
  dec_init<<<148 * 8, 256, 0, cs>>>(st, h0, c0, S, K, H, LT, d->max_len);
  if (dec_tc(*d)) {   // engine operands: K-major, gate-interleaved weights
    dec_prep_gates<<<148 * 8, 256, 0, cs>>>(w_gates, b_gates, st.wgT, st.bg, d->embed + H, H);
    const int Vp = dec_vp(d->vocab);
    dec_prep_out<<<dim3((Vp + 31) / 32, (H + 31) / 32), dim3(32, 8), 0, cs>>>(w_out, b_out, st.woT, st.bo, H, d->vocab, Vp);
  }
  cudaGraphExec_t exec = nullptr;
  if (d->max_len > 0 && !g_dprof && d->poll >= 0)
    exec = decode_graph(d, st, hb, workspace, emb, w_gates, b_gates, w_out, b_out);
  cublasSetStream(hb, cs);
  g_last_mode = exec ? 1 : 0;
  if (exec) {
    if (cudaGraphLaunch(exec, cs) != cudaSuccess) return SKB_ERR_CUDA;
  } else {
    // host-driven loop (profiling, or no conditional graphs): the same kernels,
    // the host polls the device stop flag every `poll` steps
    const int poll = d->poll > 0 ? d->poll : 4;
    for (int t = 0; t < d->max_len; ++t) {
      if (!enqueue_step(d, st, hb, cs, emb, w_gates, b_gates, w_out, b_out, cudaGraphConditionalHandle(), 0, t))
        return SKB_ERR_CUDA;
      if ((t + 1) % poll == 0 || t + 1 == d->max_len) {
        cudaMemcpyAsync(host_word, st.active + t + 1, sizeof(int32_t), cudaMemcpyDeviceToHost, cs);
        if (cudaStreamSynchronize(cs) != cudaSuccess) return SKB_ERR_CUDA;
        g_dsteps = t + 1 < kProfSteps ? t + 1 : kProfSteps;
        if (host_word[0] == 0) break;
      }
    }
  }
  dec_output<<<148 * 8, 256, 0, cs>>>(st, R, LT, tokens_out, scores_out, lengths_out);
  cudaMemcpyAsync(host_word, st.tstep, sizeof(int32_t), cudaMemcpyDeviceToHost, cs);
  if (cudaStreamSynchronize(cs) != cudaSuccess) return SKB_ERR_CUDA;
  if (steps_out) *steps_out = host_word[0];
  return skb_check_launch();
}

// Per-phase timing of the next skb_decode calls: enable != 0 turns it on.
extern "C" int skb_decode_profile(int enable) {
  if (enable && !g_dinit) {
    for (int i = 0; i < kProfSteps; ++i)
      for (int k = 0; k <= P_N; ++k)
        if (cudaEventCreate(&g_dev[i][k]) != cudaSuccess) return SKB_ERR_CUDA;
    g_dinit = true;
  }
  g_dprof = enable != 0;
  g_dsteps = 0;
  return SKB_OK;
}

// ms_out[4] = summed ms of {gather (+ idle), gate GEMM + cell, cell->logits GEMM, beam_select}
// over the steps the last skb_decode launched; returns the step count.
extern "C" int skb_decode_profile_read(float* ms_out) {
  for (int k = 0; k < P_N; ++k) ms_out[k] = 0.f;
  if (!g_dinit) return 0;
  for (int i = 0; i < g_dsteps; ++i) {
    if (cudaEventSynchronize(g_dev[i][P_N]) != cudaSuccess) return -1;
    for (int k = 0; k < P_N; ++k) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, g_dev[i][k], g_dev[i][k + 1]) != cudaSuccess) return -1;
      ms_out[k] += ms;
    }
  }
  return g_dsteps;
}
