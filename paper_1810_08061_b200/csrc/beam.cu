// beam.cu — staged seq2seq decoder with a data-dependent EOS stop (BASELINE
// config C3): the greedy program of SURVEY App. F (oracle/programs/greedy.msl,
// a `break` on EOS lowered into the While test) generalised to beam search.
//
// One decode step for R = sentences x beam rows:
//   dec_gather   xh = [emb[tok], h]                      (tensor.py:420-430 Index)
//   GEMM         gates = xh @ W_gates       (cuBLAS; fp32 exact or TF32 tensor cores)
//   dec_cell     rnn: h' = tanh(gates); lstm: i,f,g,o -> c', h'   (tensor.py:391-407)
//   GEMM         logits = h' @ W_out                     (cuBLAS, same math)
//   beam_select  ONE pass over the logits per sentence: per beam row a warp keeps
//                an online max / sum-exp (log-softmax) and a per-lane top-K with
//                warp-shuffle merges; the sentence's K x K candidates are ranked
//                (score desc, flat index asc — the oracle's tie-break), then the
//                CTA reindexes h, c, scores, tokens, lengths and history from the
//                chosen parents and counts unfinished sentences.
// Every kernel of step t+1 reads that count and exits when it is zero, so the
// stop is decided on the device; the host only polls the counter every few
// steps to stop launching.  Semantics: oracle/beam.py (pinned against the
// reference's greedy program at beam 1).
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include "skb_internal.h"

namespace {

constexpr int KMAX = 8;          // largest beam
constexpr int SEL_THREADS = 256;  // beam_select CTA: 8 warps, warp w handles rows w, w+8, ...

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
};

__device__ __forceinline__ float sigmoidf_ref(float x) {   // reference tensor.py:403-407 (two branches)
  if (x >= 0.f) return 1.f / (1.f + expf(-x));
  const float e = expf(x);
  return e / (1.f + e);
}

__global__ void dec_gather(const float* __restrict__ emb, const float* __restrict__ h, const int32_t* __restrict__ tok,
                           float* __restrict__ xh, int R, int E, int H, const int32_t* __restrict__ active, int t) {
  if (active[t] == 0) return;
  const int W = E + H;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < (long long)R * W;
       i += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(i / W), k = (int)(i % W);
    xh[i] = k < E ? emb[(long long)tok[r] * E + k] : h[(long long)r * H + (k - E)];
  }
}

__global__ void dec_cell(int cell, const float* __restrict__ gates, const float* __restrict__ bias,
                         const float* __restrict__ c, float* __restrict__ hn, float* __restrict__ cn, int R, int H,
                         const int32_t* __restrict__ active, int t) {
  if (active[t] == 0) return;
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

template <int K>
__global__ void __launch_bounds__(SEL_THREADS) beam_select(DecodeState st, int S, int V, int H, int LT, int eos,
                                                           const float* __restrict__ b_out, int t, int cur) {
  if (st.active[t] == 0) return;
  __shared__ float row_v[KMAX][KMAX];
  __shared__ int row_i[KMAX][KMAX];
  __shared__ float row_lse[KMAX];
  __shared__ int sel_par[KMAX], sel_tok[KMAX];
  __shared__ double sel_score[KMAX];
  const int s = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nxt = cur ^ 1;
  for (int b = warp; b < K; b += SEL_THREADS / 32) {
    const int r = s * K + b;
    if (st.fin[cur][r]) continue;   // finished beams offer only (EOS, score) below
    const float* L = st.logits + (long long)r * V;
    float mx = -INFINITY, sum = 0.f;
    float tv[K];
    int ti[K];
#pragma unroll
    for (int k = 0; k < K; ++k) { tv[k] = -INFINITY; ti[k] = 0x7fffffff; }
    for (int v = lane; v < V; v += 32) {
      const float x = L[v] + (b_out ? b_out[v] : 0.f);
      if (x > mx) { sum = sum * expf(mx - x) + 1.f; mx = x; } else { sum += expf(x - mx); }   // online softmax
      topk_insert<K>(tv, ti, x, v);
    }
    // warp: combine (max, sum) pairs, then merge the 32 sorted lists K times
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, mx, o), s2 = __shfl_xor_sync(0xffffffffu, sum, o);
      const float m = fmaxf(mx, m2);
      sum = (mx == -INFINITY ? 0.f : sum * expf(mx - m)) + (m2 == -INFINITY ? 0.f : s2 * expf(m2 - m));
      mx = m;
    }
    for (int k = 0; k < K; ++k) {
      float bv = tv[0];
      int bi = ti[0], bl = lane;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o), ol = __shfl_xor_sync(0xffffffffu, bl, o);
        if (better(ov, oi, bv, bi)) { bv = ov; bi = oi; bl = ol; }
      }
      if (lane == 0) { row_v[b][k] = bv; row_i[b][k] = bi; }
      if (lane == bl) {   // pop the winner's head
#pragma unroll
        for (int q = 0; q < K - 1; ++q) { tv[q] = tv[q + 1]; ti[q] = ti[q + 1]; }
        tv[K - 1] = -INFINITY; ti[K - 1] = 0x7fffffff;
      }
    }
    if (lane == 0) row_lse[b] = mx + logf(sum);
  }
  __syncthreads();
  if (warp == 0) {
    // candidates: K per live row (score + logit - lse), one (EOS, score) per finished row
    double cs[2];
    int ci[2];   // flat index b*V + v
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int slot = lane + 32 * q;   // K*K <= 64
      cs[q] = -INFINITY; ci[q] = 0x7fffffff;
      if (slot < K * K) {
        const int b = slot / K, k = slot % K, r = s * K + b;
        const double sc = st.score[cur][r];
        if (st.fin[cur][r]) {
          if (k == 0) { cs[q] = sc; ci[q] = b * V + eos; }
        } else if (sc != -INFINITY && row_i[b][k] != 0x7fffffff) {
          cs[q] = sc + ((double)row_v[b][k] - (double)row_lse[b]);
          ci[q] = b * V + row_i[b][k];
        } else if (row_i[b][k] != 0x7fffffff) {
          ci[q] = b * V + row_i[b][k];
        }
      }
    }
    for (int j = 0; j < K; ++j) {
      double bv = cs[0];
      int bi = ci[0], bq = 0;
      if (better_d(cs[1], ci[1], bv, bi)) { bv = cs[1]; bi = ci[1]; bq = 1; }
      int bl = lane;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        const int ol = __shfl_xor_sync(0xffffffffu, bl, o), oq = __shfl_xor_sync(0xffffffffu, bq, o);
        if (better_d(ov, oi, bv, bi)) { bv = ov; bi = oi; bl = ol; bq = oq; }
      }
      if (lane == 0) { sel_score[j] = bv; sel_par[j] = bi / V; sel_tok[j] = bi % V; }
      if (lane == bl) { cs[bq] = -INFINITY; ci[bq] = 0x7fffffff; }
    }
  }
  __syncthreads();
  // reindex: beam j of the next step continues parent p = sel_par[j]
  for (int j = warp; j < K; j += SEL_THREADS / 32) {
    const int p = sel_par[j], rp = s * K + p, rj = s * K + j;
    const bool pfin = st.fin[cur][rp] != 0;
    const float* hs = pfin ? st.h[cur] + (long long)rp * H : st.hn + (long long)rp * H;
    const float* cs = pfin ? st.c[cur] + (long long)rp * H : st.cn + (long long)rp * H;
    for (int k = lane; k < H; k += 32) {
      st.h[nxt][(long long)rj * H + k] = hs[k];
      st.c[nxt][(long long)rj * H + k] = cs[k];
    }
    for (int k = lane; k <= t; k += 32) st.hist[nxt][(long long)rj * LT + k] = st.hist[cur][(long long)rp * LT + k];
    if (lane == 0) {
      const int v = sel_tok[j];
      st.hist[nxt][(long long)rj * LT + t + 1] = v;
      st.tok[rj] = v;
      st.score[nxt][rj] = sel_score[j];
      st.fin[nxt][rj] = (pfin || v == eos) ? 1 : 0;
      st.len[nxt][rj] = st.len[cur][rp] + (pfin ? 0 : 1);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int live = 0;
    for (int j = 0; j < K; ++j) live |= st.fin[nxt][s * K + j] == 0;
    if (live) atomicAdd(&st.active[t + 1], 1);
  }
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
  }
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t <= max_len; t += gridDim.x * blockDim.x)
    st.active[t] = t == 0 ? S : 0;
}

__global__ void dec_output(DecodeState st, int R, int LT, int side, int32_t* tokens, float* scores,
                           int32_t* lengths) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < (long long)R * LT;
       i += (long long)gridDim.x * blockDim.x)
    tokens[i] = st.hist[side][i];
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < R; r += gridDim.x * blockDim.x) {
    scores[r] = (float)st.score[side][r];
    lengths[r] = st.len[side][r];
  }
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
  const int S = d->sentences, K = d->beam, R = S * K, E = d->embed, H = d->hidden, V = d->vocab;
  const int G = d->cell == SKB_CELL_LSTM ? 4 * H : H, LT = d->max_len + 1;
  cublasHandle_t hb = handle_for(stream);
  if (!hb) return SKB_ERR_CUDA;
  const int ew = 148 * 8;
  dec_init<<<ew, 256, 0, cs>>>(st, h0, c0, S, K, H, LT, d->max_len);
  int32_t* active_host = nullptr;
  cudaMallocHost(&active_host, sizeof(int32_t) * 2);
  int t = 0, cur = 0;
  const int poll = d->poll > 0 ? d->poll : 4;
  for (; t < d->max_len; ++t) {
    dec_gather<<<ew, 256, 0, cs>>>(emb, st.h[cur], st.tok, st.xh, R, E, H, st.active, t);
    if (!gemm(hb, d->math, st.xh, w_gates, st.gates, R, G, E + H)) return SKB_ERR_CUDA;
    dec_cell<<<ew, 256, 0, cs>>>(d->cell, st.gates, b_gates, st.c[cur], st.hn, st.cn, R, H, st.active, t);
    if (!gemm(hb, d->math, st.hn, w_out, st.logits, R, V, H)) return SKB_ERR_CUDA;
    switch (K) {
#define SKB_SEL(k) case k: beam_select<k><<<S, SEL_THREADS, 0, cs>>>(st, S, V, H, LT, d->eos, b_out, t, cur); break;
      SKB_SEL(1) SKB_SEL(2) SKB_SEL(3) SKB_SEL(4) SKB_SEL(5) SKB_SEL(6) SKB_SEL(7) SKB_SEL(8)
#undef SKB_SEL
    }
    cur ^= 1;
    if ((t + 1) % poll == 0 || t + 1 == d->max_len) {   // stop launching once the device says done
      cudaMemcpyAsync(active_host, st.active + t + 1, sizeof(int32_t), cudaMemcpyDeviceToHost, cs);
      if (cudaStreamSynchronize(cs) != cudaSuccess) { cudaFreeHost(active_host); return SKB_ERR_CUDA; }
      if (active_host[0] == 0) { ++t; break; }
    }
  }
  // the device state after the last step that ran: steps = first t with active[t] == 0
  int launched = t;
  int32_t* act = (int32_t*)malloc(sizeof(int32_t) * (launched + 1));
  cudaMemcpyAsync(act, st.active, sizeof(int32_t) * (launched + 1), cudaMemcpyDeviceToHost, cs);
  if (cudaStreamSynchronize(cs) != cudaSuccess) { free(act); cudaFreeHost(active_host); return SKB_ERR_CUDA; }
  int steps = launched;
  for (int k = 0; k <= launched; ++k)
    if (act[k] == 0) { steps = k; break; }
  free(act);
  cudaFreeHost(active_host);
  const int side = steps & 1;   // step k writes side (k+1)&1; steps executed = `steps`
  dec_output<<<ew, 256, 0, cs>>>(st, R, LT, side, tokens_out, scores_out, lengths_out);
  if (steps_out) *steps_out = steps;
  return skb_check_launch();
}
