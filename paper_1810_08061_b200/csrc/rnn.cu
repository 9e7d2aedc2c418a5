// rnn.cu — persistent, cluster-resident execution of a staged dynamic-length
// recurrent `While` region (LSTM or tanh-RNN cell) on sm_100a.
//
// Reference semantics (pkg/src/stagekit):
//   graph/execute.py:218-238  _eval_while: test `idx < reduce_max(seq_len)`
//                             before every iteration, body, state <- outputs
//   graph/tensor.py:302-319   matmul (x_t W + h U), :274-287 binop (+ b),
//                             :391-407 tanh / stable sigmoid,
//                             :356-377 where (rank-1 cond = row select),
//                             :420-430 index (x_tm[t]), :322-332 transpose
//   graph/execute.py:153-185  ListAppend / ListStack of the masked h
// Here the loop lives on the device: no host round trip per iteration, each
// batch row runs to its own length, rows past their length keep the frozen
// state (the reference's Where), and the stacked, transposed output
// [B, max_len, H] is written directly.
//
// Mapping: a thread-block cluster of C CTAs owns one tile
// of NT batch rows; CTA q owns U hidden units, i.e. 128 gate rows of the
// concatenated weight [W;U]^T, resident in shared memory for the whole
// kernel.  Per step each CTA issues tcgen05.mma  D[128 x NT] (TMEM) =
// Wcat_q[128 x K] * [x_t ; h_{t-1}]^T, the epilogue warps read D with
// tcgen05.ld, apply bias + gate nonlinearities + the c/h update + mask in
// registers, write h_t (fp32) to the output sequence and broadcast the fp16
// h_t slice to every CTA of the cluster with bulk DSMEM copies that complete
// on the receivers' mbarriers.  The x_t part of the next step's MMA is
// issued before h_t arrives (it does not depend on the recurrence).
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <climits>
#include <cstdlib>
#include "sm100.cuh"
#include "skb_internal.h"

using namespace skb;

namespace {

// Block: EW epilogue warps (warp w covers TMEM lane quarter w&3 and batch-column
// slice w>>2), an x loader warp and an MMA-issuer warp (+ TMEM alloc).
// EW = 16 halves each epilogue thread's share of a step (the recurrence's
// critical path); SKB_RNN_EW=8 selects the narrower variant.
inline int env_flag(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}
inline int rnn_ew() {
  static int ew = 0;
  if (!ew) {
    const char* e = getenv("SKB_RNN_EW");
    ew = (e && atoi(e) == 8) ? 8 : 16;
  }
  return ew;
}
// LSTM gate activations: 1 (default) = tanh.approx, one MUFU op per gate (the
// epilogue's MUFU/FMA work is on the recurrence's critical path; C1 step -18%,
// accuracy vs the f64 oracle unchanged within the fp16-operand error, see
// tools/c1_err.py); SKB_RNN_ACT=0 = ex2 + Newton reciprocal (rel. err ~1e-7).
// SKB_RNN_ACT=2: the CTA-pair kernel evaluates activations with tanh.approx.f16x2
// (measured slower: sm_100 issues it as two MUFU.TANH.F16, plus the conversions).
inline int rnn_act() {
  static int act = -1;
  if (act < 0) {
    const char* e = getenv("SKB_RNN_ACT");
    act = e ? (atoi(e) == 0 ? 0 : (atoi(e) == 2 ? 2 : 1)) : 1;
  }
  return act;
}
constexpr int kMaxClusterDim = 8;
int g_last_clusters = 0;   // clusters of the last recurrent-kernel launch (skb_rnn_last_clusters)
int g_last_kernel = 0;     // which recurrent kernel it was (skb_rnn_last_kernel)
constexpr int kGS = 36;   // sG row stride (floats): 32 units + 4 pad, conflict-free LDS.128

struct RnnGeom {
  int cell, H, F, T, Bp, P, R;
  int G;        // gates per unit
  int U;        // hidden units per CTA
  int C;        // CTAs per cluster
  int Kx, Kh, K;
};

__host__ __device__ inline int round_up(int a, int b) { return (a + b - 1) / b * b; }

inline bool make_geom(const skb_rnn_shape* s, RnnGeom* g) {
  if (!s || s->hidden <= 0 || s->input <= 0 || s->time < 0 || s->rows_per_problem <= 0 ||
      s->problems <= 0)
    return false;
  g->cell = s->cell;
  if (s->cell == SKB_CELL_LSTM || s->cell == SKB_CELL_GRU) g->G = 4;
  else if (s->cell == SKB_CELL_RNN_TANH) g->G = 1;
  else return false;
  g->H = s->hidden; g->F = s->input; g->T = s->time;
  g->Bp = s->rows_per_problem; g->P = s->problems;
  g->R = s->rows_per_problem * s->problems;
  g->U = 128 / g->G;
  int hp = round_up(g->H, 16);
  if (hp < g->U) g->U = hp;
  g->C = (g->H + g->U - 1) / g->U;
  g->Kx = round_up(g->F, 16);
  g->Kh = g->C * g->U;
  g->K = g->Kx + g->Kh;
  if (g->C > kMaxClusterDim) return false;
  if (g->K > 512) return false;   // weights must fit TMEM columns [256, 512)
  return true;
}

template <int NT>
inline size_t smem_bytes(const RnnGeom& g) {
  return (size_t)2 * NT * g.Kx * 2 + (size_t)2 * NT * g.Kh * 2 +
         (g.G == 4 ? (size_t)4 * NT * kGS * 4 : 0) + 1024;
}

struct RnnArgs {
  const void* x;
  const float* h0;
  const float* c0;
  const int64_t* lens;
  const int32_t* perm;
  const int32_t* pmax;
  const uint8_t* wpack;
  const float* bpack;
  float* out;
  float* hT;
  float* cT;
  const uint8_t* ximg; // [ntiles][T][NT x Kx] fp16 core-matrix images of x_t
  uint8_t* hscratch;   // per cluster: 2 x [NT x Kh] fp16 h_t exchange buffers (L2)
  int32_t* err;
  const int32_t* xflag; // pair4 kernel with the concurrent packer: [ntiles][T] image-ready flags, else null
  int32_t* tdone;       // pair4 kernel with the concurrent filler: [ntiles] CTAs that published h_T, else null
  int x_f64;
  int fill_inkernel;   // pair4 kernel: write the frozen tails itself (no fill pass)
  int R, T, F, H, Kx, Kh, K, U, C, Bp, ntiles;
};

// Optional per-step event trace of CTA 0 (debug only; set by skb_debug_rnn_trace).
__device__ long long* g_trace = nullptr;
__device__ int g_trace_steps = 0;
#ifdef SKB_TRACE_ENABLED
__device__ long long* g_ttrace = nullptr;   // per-tile events of CTA 0: [tile_iter][8]
__device__ int g_ttrace_n = 0;
#define SKB_TTRACE(it_, slot_)                                                             \
  do {                                                                                     \
    if (g_ttrace != nullptr && blockIdx.x == 0 && threadIdx.x == 0 && (it_) < g_ttrace_n)  \
      g_ttrace[(size_t)(it_) * 8 + (slot_)] = clock64();                                   \
  } while (0)
#define SKB_TRACE(step_, slot_)                                                            \
  do {                                                                                     \
    if (g_trace != nullptr && blockIdx.x == 0 && (int)(step_) < g_trace_steps)             \
      g_trace[(size_t)(step_) * 16 + (slot_)] = clock64();                                 \
  } while (0)
#define SKB_TRACE_CTA(cta_, step_, slot_)                                                  \
  do {                                                                                     \
    if (g_trace != nullptr && blockIdx.x == (cta_) && (int)(step_) < g_trace_steps)        \
      g_trace[(size_t)(step_) * 16 + (slot_)] = clock64();                                 \
  } while (0)
#else   // production build: trace points compile to nothing
#define SKB_TTRACE(it_, slot_) do {} while (0)
#define SKB_TRACE(step_, slot_) do {} while (0)
#define SKB_TRACE_CTA(cta_, step_, slot_) do {} while (0)
#endif

SKB_DEV void set_err(int32_t* err, int code, int problem, int t) {
  if (atomicCAS(err, 0, code) == 0) { err[1] = problem; err[2] = t; }
}

// Handoff from the concurrent x packer (pack_x_stream_kernel): the packer's image
// stores, a gpu-scope release of the (tile, t) flag; the loader polls with ld.acquire
// and orders its bulk (async-proxy) read after them with a proxy fence.  The packer
// never waits on anything, so the wait always ends; it is still bounded (a lost flag
// would be a bug: the launch reports SKB_ERR_HANDOFF instead of hanging).
SKB_DEV int ld_acquire_gpu(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
SKB_DEV void st_release_gpu(int32_t* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
SKB_DEV unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
SKB_DEV void red_release_gpu_add(int32_t* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
// Wait for *p >= want.  A timed-out wait marks the launch (err = SKB_ERR_HANDOFF) and
// every later wait of the launch gives up at once, so a lost producer costs one timeout.
SKB_DEV bool wait_flag(const int32_t* p, int want, int32_t* err) {
  if (ld_acquire_gpu(p) >= want) return true;
  const unsigned long long t0 = globaltimer_ns();
  while (ld_acquire_gpu(p) < want) {
    if (*reinterpret_cast<volatile int32_t*>(err) == SKB_ERR_HANDOFF) return false;
    __nanosleep(64);
    if (globaltimer_ns() - t0 > 200000000ull) {
      atomicExch(err, SKB_ERR_HANDOFF);
      return false;
    }
  }
  return true;
}

SKB_DEV float sel4(float a, float b, float c, float d, int i) {
  return i == 0 ? a : i == 1 ? b : i == 2 ? c : d;
}

SKB_DEV bool fp16_overflow(float v) { return isfinite(v) && fabsf(v) > 65504.f; }

// 1/d for d in [1, 1e30] on the FMA pipe (the MUFU pipe is the epilogue's
// bottleneck): bit-trick seed, three Newton steps, rel. err < 1e-7.
SKB_DEV float rcp_nr(float d) {
  float y = __int_as_float(0x7EF311C3 - __float_as_int(d));
  y = y * fmaf(-d, y, 2.f);
  y = y * fmaf(-d, y, 2.f);
  y = y * fmaf(-d, y, 2.f);
  return y;
}
SKB_DEV float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// 1/(1 + 2^a): one MUFU op (ex2) + the reciprocal on the FMA pipe.
SKB_DEV float inv1pexp2(float a) { return rcp_nr(1.f + fminf(ex2_approx(a), 1e30f)); }
// 1/(1 + e^{k x}) (kept for the RNN path)
SKB_DEV float inv1pexp(float kx) { return inv1pexp2(kx * 1.4426950408889634f); }

SKB_DEV void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" :: "l"(p)); }
// L2 prefetch of one x row (bytes rounded down to 16; the bulk form needs 16-byte alignment)
SKB_DEV void prefetch_l2_bulk_row(const void* p, int bytes) {
  if ((reinterpret_cast<uintptr_t>(p) & 15) == 0 && bytes >= 16) bulk_prefetch_l2(p, (uint32_t)(bytes & ~15));
  else prefetch_l2(p);
}
SKB_DEV float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
SKB_DEV float tanh_acc(float x) {
  // 1 - 2/(1+e^{2x}): saturates correctly at both ends, |err| ~ 1e-7.
  return fmaf(-2.f, inv1pexp2(x * 2.8853900817779268f), 1.f);
}

// Load 8 consecutive x elements (k0..k0+7) of one row/time step, zero past F.
template <typename XT>
SKB_DEV void load_x8(const XT* __restrict__ p, int k0, int F, float (&v)[8]) {
#pragma unroll
  for (int e = 0; e < 8; ++e) v[e] = (k0 + e < F) ? (float)__ldg(p + k0 + e) : 0.f;
}
template <>
SKB_DEV void load_x8<float>(const float* __restrict__ p, int k0, int F, float (&v)[8]) {
  if (k0 + 8 <= F && ((reinterpret_cast<uintptr_t>(p + k0) & 15) == 0)) {
    float4 a = __ldg(reinterpret_cast<const float4*>(p + k0));
    float4 b = __ldg(reinterpret_cast<const float4*>(p + k0 + 4));
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  } else {
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = (k0 + e < F) ? __ldg(p + k0 + e) : 0.f;
  }
}
template <>
SKB_DEV void load_x8<double>(const double* __restrict__ p, int k0, int F, float (&v)[8]) {
  if (k0 + 8 <= F && ((reinterpret_cast<uintptr_t>(p + k0) & 15) == 0)) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      double2 a = __ldg(reinterpret_cast<const double2*>(p + k0) + e);
      v[2 * e] = (float)a.x; v[2 * e + 1] = (float)a.y;
    }
  } else {
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = (k0 + e < F) ? (float)__ldg(p + k0 + e) : 0.f;
  }
}

// LSTM gate activations.  ACT 0: act = mul / (1 + 2^(kl*z + kb)) + add with ex2 and a
// Newton reciprocal (tanh(x) = 2 sigmoid(2x) - 1 for the g gate).  ACT 1: one MUFU
// op per gate, act = mul * tanh(kl*z + kb) + add (sigmoid(y) = 0.5 tanh(y/2) + 0.5).
template <int ACT>
SKB_DEV void gate_consts(int gate, float bias, float& kl, float& kb, float& mul, float& add) {
  if (ACT) {
    kl = (gate == 2) ? 1.f : 0.5f;
    mul = kl;
    add = (gate == 2) ? 0.f : 0.5f;
  } else {
    kl = (gate == 2) ? -2.8853900817779268f : -1.4426950408889634f;
    mul = (gate == 2) ? 2.f : 1.f;
    add = (gate == 2) ? -1.f : 0.f;
  }
  kb = kl * bias;
}
template <int ACT>
SKB_DEV float gate_act(float z, float kl, float kb, float mul, float add) {
  return ACT ? fmaf(mul, tanh_approx(fmaf(z, kl, kb)), add) : fmaf(mul, inv1pexp2(fmaf(z, kl, kb)), add);
}
template <int ACT>
SKB_DEV float cell_tanh(float c) { return ACT ? tanh_approx(c) : tanh_acc(c); }

// Four-gate-block cells (LSTM i,f,g,o; GRU z,r,n_x,n_h): the gate phase of TMEM
// lane quarter qw (warp-uniform).  GRU: z and r are sigmoids, n_x / n_h stay
// affine (+ bias) until the cell phase combines them.
template <int CELL, int ACT>
struct GateAct {
  float kl, kb, mul, add, bias;
  bool affine;
  SKB_DEV GateAct(int qw, float b) : bias(b) {
    affine = (CELL == SKB_CELL_GRU) && qw >= 2;
    gate_consts<ACT>(CELL == SKB_CELL_GRU ? 0 : qw, b, kl, kb, mul, add);
  }
  SKB_DEV float operator()(float z) const { return affine ? z + bias : gate_act<ACT>(z, kl, kb, mul, add); }
};

// The cell update from the four activated blocks, masked by `live` (the reference's Where).
//   LSTM: c' = f*c + i*g, h' = o*tanh(c')
//   GRU : n = tanh(n_x + r*n_h), h' = (1-z)*n + z*h = n + z*(h - n)
template <int CELL, int ACT>
SKB_DEV void cell_update(float g0, float g1, float g2, float g3, float& c, float& h, bool live) {
  if constexpr (CELL == SKB_CELL_GRU) {
    const float n = cell_tanh<ACT>(fmaf(g1, g3, g2));
    const float h2 = fmaf(g0, h - n, n);
    h = live ? h2 : h;
  } else {
    const float c2 = fmaf(g1, c, g0 * g2);
    const float h2 = g3 * cell_tanh<ACT>(c2);
    c = live ? c2 : c;
    h = live ? h2 : h;
  }
}

template <int CELL, int NT, typename XT, int EW, int ACT = 0>
__global__ void __launch_bounds__(EW * 32 + 64, 1) rnn_fwd_kernel(const RnnArgs a) {
  // EW epilogue warps (8 or 16), then the x loader warp and the MMA warp.
  constexpr int kEpi = EW * 32, kThreads = kEpi + 64;
  constexpr int NCOL = NT / (EW / 4);            // batch columns per epilogue warp
  constexpr int UG = (EW >= 16) ? 4 : 8;         // LSTM units per cell-phase item
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ uint64_t xfull[2], xempty[2], hfull[2], mdone[2], dfree[2];
  __shared__ uint32_t tmem_s;
  __shared__ int s_row[NT], s_len[NT], s_tmax[NT];
  __shared__ int s_trip;

  uint8_t* smem = smem_raw;   // (no pointer re-alignment: keeps the shared address space visible to the compiler)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t q = cluster_ctarank();
  const int C = a.C, U = a.U, H = a.H, T = a.T;
  const uint32_t xbytes = NT * a.Kx * 2, hbytes = NT * a.Kh * 2, sbytes = NT * U * 2;
  uint8_t* sX = smem;                      // 2 x [NT x Kx] fp16, core-matrix layout
  uint8_t* sH = sX + 2 * xbytes;           // 2 x [NT x Kh] fp16
  float* sG = reinterpret_cast<float*>(sH + 2 * hbytes);   // LSTM gates [4][NT][kGS] (padded rows)
  constexpr uint32_t b_lbo = NT * 16, b_sbo = 128;    // activations: K-chunk / row-group stride
  constexpr uint32_t kWCol = 256;                     // TMEM column of the weight operand
  constexpr bool two_chains = false;                  // (a second h accumulator costs more TMEM reads than it saves)

  if (tid == 0) {
    for (int j = 0; j < 2; ++j) {
      mbar_init(&xfull[j], 1);
      mbar_init(&xempty[j], 1);
      mbar_init(&hfull[j], 1);
      mbar_init(&mdone[j], 1);
      mbar_init(&dfree[j], kEpi / 32);
    }
    fence_mbar_init();
  }
  if (warp == EW + 1) tmem_alloc<512>(&tmem_s);
  for (uint32_t i = tid; i < (2 * xbytes + 2 * hbytes) / 16; i += kThreads)
    reinterpret_cast<uint4*>(sX)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_s;
  // Weights -> TMEM (A operand of every MMA): lane = gate row, column c holds
  // K elements (2c, 2c+1).  Epilogue warp w fills lanes [32w, 32w+32).
  float bias = 0.f;
  if (warp < 4) {
    const uint32_t* src = reinterpret_cast<const uint32_t*>(a.wpack + ((size_t)q * 128 + tid) * a.K * 2);
    for (int c0 = 0; c0 < a.K / 2; c0 += 8) {
      uint32_t r[8];
      const uint4 lo = __ldg(reinterpret_cast<const uint4*>(src + c0));
      const uint4 hi = __ldg(reinterpret_cast<const uint4*>(src + c0 + 4));
      r[0] = lo.x; r[1] = lo.y; r[2] = lo.z; r[3] = lo.w; r[4] = hi.x; r[5] = hi.y; r[6] = hi.z; r[7] = hi.w;
      tmem_st8(tmem + ((uint32_t)(warp * 32) << 16) + kWCol + c0, r);
    }
    tmem_st_wait();
  }
  if (warp < EW) bias = a.bpack[q * 128 + (warp & 3) * 32 + lane];
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  cluster_sync();   // every CTA's barriers are initialised before any remote traffic

  // Epilogue ownership (kEpi threads; warp w reads TMEM lane quarter qw = w&3 and
  // batch-column half ch = w>>2).
  //   LSTM: TMEM lane l = 32*g + u (gate g = qw, unit u = lane).  After the gate
  //         exchange through sG, thread tid owns "pairs" idx = tid + kEpi*p: batch
  //         column n = idx / G8 and the 8 consecutive units u8*8.. of that column
  //         (G8 = U/8 unit groups per CTA), so h/c/out/stage are 16/32-byte vectors.
  //   RNN : unit = 32*qw + lane; the thread owns the NT/2 columns of its half.
  const int qw = warp & 3, ch = warp >> 2;
  constexpr bool kGated = CELL == SKB_CELL_LSTM || CELL == SKB_CELL_GRU;   // four gate blocks
  constexpr int NP = kGated ? (NT * (32 / UG) + kEpi - 1) / kEpi : 1;   // max items per thread
  constexpr int NCELL = kGated ? NP * UG : NCOL;
  const int G8 = U / UG;
  int pn[NP], pu[NP];
  bool pv[NP];
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    const int idx = tid + kEpi * p;
    pn[p] = G8 ? idx / G8 : 0;
    pu[p] = G8 ? (idx % G8) * UG : 0;
    pv[p] = kGated && tid < kEpi && idx < NT * G8;
  }
  const int rnn_u = qw * 32 + lane;
  const int rnn_unit = (int)q * U + rnn_u;
  const bool rnn_valid = !kGated && (warp < EW) && (rnn_u < U) && (rnn_unit < H);
  float hp[NCELL], cc[NCELL];
  uint8_t* gscr = a.hscratch + (size_t)cluster_id_x() * 2 * hbytes;   // this cluster's h_t exchange buffers

  uint32_t step = 0;
  uint32_t hwait[2] = {0u, 0u};
  bool hfull_armed = false;
  const int nclusters = (int)nclusters_x();
  int tile_iter = 0;
  // Row metadata of a tile (thread tid < NT owns row tid): loaded one tile
  // ahead, and the next tile's h0/c0 rows prefetched into L2, so a tile's
  // setup does not wait on dependent global loads.
  static_assert(NT == 64, "the tile metadata reduction assumes 64-row tiles");
  auto tile_meta = [&](int tl, int& r, int& len, int& tmax) {
    r = -1; len = 0; tmax = 0;
    if (tl < a.ntiles && tid < NT) {
      r = a.perm[tl * NT + tid];
      if (r >= 0) {
        tmax = max(0, min(a.pmax[r / a.Bp], T));
        const long long L = a.lens[r];
        len = (int)max(0LL, min(L, (long long)tmax));
      }
    }
  };
  int m_r, m_len, m_tmax;
  tile_meta((int)cluster_id_x(), m_r, m_len, m_tmax);
  for (int tile = (int)cluster_id_x(); tile < a.ntiles; tile += nclusters, ++tile_iter) {
    SKB_TTRACE(tile_iter, 0);
    // No cluster barrier between tiles: a peer's first h exchange of the next tile
    // targets hbuf[s0&1], whose last reader (this CTA's MMA of step s0-2) has
    // completed before this CTA's step s0-2 h slice -- which the peer needed to
    // finish step s0-1 -- was sent; every other buffer and barrier phase is
    // per-CTA and carried across tiles.
    __syncthreads();   // this CTA's previous tile retired (s_row/s_len are rewritten below)
    SKB_TTRACE(tile_iter, 4);
    if (tid < NT) { s_row[tid] = m_r; s_len[tid] = m_len; s_tmax[tid] = m_tmax; }
    __syncthreads();
    if (warp == 0) {
      int m = max(s_len[lane], s_len[lane + 32]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (lane == 0) s_trip = m;
    }
    SKB_TTRACE(tile_iter, 5);
    SKB_TTRACE(tile_iter, 6);
    fence_proxy_async_smem();
    __syncthreads();
    const int trip = s_trip;
    SKB_TTRACE(tile_iter, 1);
#ifdef SKB_TRACE_ENABLED
    if (threadIdx.x == 0 && g_ttrace != nullptr && blockIdx.x == 0 && tile_iter < g_ttrace_n)
      g_ttrace[(size_t)tile_iter * 8 + 3] = trip;
#endif

    if (warp < EW) {
      // ======================= epilogue =======================
      if (tid < NT) {   // next tile's metadata (consumed next iteration) and its h0/c0 rows -> L2, off the critical path
        tile_meta(tile + nclusters, m_r, m_len, m_tmax);
        if (m_r >= 0) {
          const char* h0n = reinterpret_cast<const char*>(a.h0 + (size_t)m_r * H);
          const char* c0n = a.c0 ? reinterpret_cast<const char*>(a.c0 + (size_t)m_r * H) : nullptr;
          for (int off = 0; off < H * 4; off += 128) {
            prefetch_l2(h0n + off);
            if (c0n) prefetch_l2(c0n + off);
          }
        }
      }
      if constexpr (kGated) {
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          const int r = pv[p] ? s_row[pn[p]] : -1;
          const int unit0 = (int)q * U + pu[p];
          float hv[8], cv[8];
          if (r >= 0) {
            load_x8<float>(a.h0 + (size_t)r * H, unit0, H, hv);
            if (a.c0) {
              load_x8<float>(a.c0 + (size_t)r * H, unit0, H, cv);
            } else {
#pragma unroll
              for (int e = 0; e < 8; ++e) cv[e] = 0.f;
            }
          } else {
#pragma unroll
            for (int e = 0; e < 8; ++e) hv[e] = cv[e] = 0.f;
          }
#pragma unroll
          for (int e = 0; e < UG; ++e) { hp[p * UG + e] = hv[e]; cc[p * UG + e] = cv[e]; }
        }
      } else {
#pragma unroll
        for (int i = 0; i < NCOL; ++i) {
          const int r = s_row[ch * NCOL + i];
          hp[i] = (rnn_valid && r >= 0) ? a.h0[(size_t)r * H + rnn_unit] : 0.f;
        }
      }
      if (trip > 0) {   // h0 reaches every CTA's hbuf[step&1] like any h_t: own fp16 slice -> L2 -> multicast
        uint8_t* gs0 = gscr + (step & 1) * hbytes + q * sbytes;
        if constexpr (kGated) {
#pragma unroll
          for (int p = 0; p < NP; ++p) {
            if (!pv[p]) continue;
            uint32_t hw[UG / 2];
#pragma unroll
            for (int e = 0; e < UG / 2; ++e) {
              __half2 h2 = __floats2half2_rn(hp[p * UG + 2 * e], hp[p * UG + 2 * e + 1]);
              hw[e] = *reinterpret_cast<uint32_t*>(&h2);
            }
            uint8_t* dst = gs0 + cm_offset(pn[p], pu[p], b_lbo, b_sbo);
            if constexpr (UG == 8) *reinterpret_cast<uint4*>(dst) = make_uint4(hw[0], hw[1], hw[2], hw[3 % (UG / 2)]);
            else *reinterpret_cast<uint2*>(dst) = make_uint2(hw[0], hw[1 % (UG / 2)]);
          }
        } else if (rnn_u < U) {
#pragma unroll
          for (int i = 0; i < NCOL; ++i)
            *reinterpret_cast<__half*>(gs0 + cm_offset(ch * NCOL + i, rnn_u, b_lbo, b_sbo)) = __float2half_rn(hp[i]);
        }
        fence_proxy_async_global();
        named_bar_sync(1, kEpi);
        if (tid == 0)
          bulk_g2s_multicast(sH + (step & 1) * hbytes + q * sbytes, gs0, sbytes, &hfull[step & 1],
                             (uint16_t)((1u << C) - 1));
      }
      for (int t = 0; t < trip; ++t) {
        const uint32_t s = step + t, j = s & 1, use = s >> 1;
        const uint32_t nb = (s + 1) & 1;
        uint8_t* gslice = gscr + nb * hbytes + q * sbytes;   // where our h_t slice goes
        mbar_wait(&mdone[j], use & 1);
        if (tid == 0) SKB_TRACE(s, 4);
        tc_fence_after();
        const uint32_t trow = tmem + ((uint32_t)(qw * 32) << 16) + j * 2 * NT + ch * NCOL;
        if constexpr (kGated) {
          // gate g = warp (warp-uniform): sigmoid for i, f, o; tanh(x) = 2*sigmoid(2x)-1 for g.
          // act = mul / (1 + 2^(kl*z + kb)) + add, z = pre-activation without bias
          const GateAct<CELL, ACT> act(qw, bias);
          float* g_out = sG + (qw * NT + ch * NCOL) * kGS + lane;
#pragma unroll
          for (int c16 = 0; c16 < NCOL / 16; ++c16) {
            float v[16], v2[16];
            tmem_ld16(trow + c16 * 16, v);
            if (two_chains) tmem_ld16(trow + NT + c16 * 16, v2);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] += two_chains ? v2[i] : 0.f;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              g_out[(c16 * 16 + i) * kGS] = act(v[i]);
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&dfree[j]);
          named_bar_sync(2, kEpi);
          if (tid == 0) SKB_TRACE(s, 10);
#pragma unroll
          for (int p = 0; p < NP; ++p) {
            if (!pv[p]) continue;
            const int n = pn[p];
            float g4[4][UG];
#pragma unroll
            for (int g = 0; g < 4; ++g) {
              const float4* src = reinterpret_cast<const float4*>(sG + (g * NT + n) * kGS + pu[p]);
#pragma unroll
              for (int v4 = 0; v4 < UG / 4; ++v4) {
                const float4 x0 = src[v4];
                g4[g][4 * v4] = x0.x; g4[g][4 * v4 + 1] = x0.y; g4[g][4 * v4 + 2] = x0.z; g4[g][4 * v4 + 3] = x0.w;
              }
            }
            const bool live = t < s_len[n];
            uint32_t hw[UG / 2];
#pragma unroll
            for (int e = 0; e < UG; ++e)
              cell_update<CELL, ACT>(g4[0][e], g4[1][e], g4[2][e], g4[3][e], cc[p * UG + e], hp[p * UG + e], live);
#pragma unroll
            for (int e = 0; e < UG / 2; ++e) {
              __half2 h2 = __floats2half2_rn(hp[p * UG + 2 * e], hp[p * UG + 2 * e + 1]);
              hw[e] = *reinterpret_cast<uint32_t*>(&h2);
            }
            if (t + 1 < trip) {
              uint8_t* dst = gslice + cm_offset(n, pu[p], b_lbo, b_sbo);
              if constexpr (UG == 8) *reinterpret_cast<uint4*>(dst) = make_uint4(hw[0], hw[1], hw[2], hw[3 % (UG / 2)]);
              else *reinterpret_cast<uint2*>(dst) = make_uint2(hw[0], hw[1 % (UG / 2)]);
            }
          }
        } else {
#pragma unroll
          for (int c16 = 0; c16 < NCOL / 16; ++c16) {
            float v[16], v2[16];
            tmem_ld16(trow + c16 * 16, v);
            if (two_chains) tmem_ld16(trow + NT + c16 * 16, v2);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const int n = ch * NCOL + c16 * 16 + i;
              v[i] += two_chains ? v2[i] : 0.f;
              const float h2 = tanh_acc(v[i] + bias);
              hp[c16 * 16 + i] = (t < s_len[n]) ? h2 : hp[c16 * 16 + i];
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&dfree[j]);
          if (t + 1 < trip && rnn_u < U) {
#pragma unroll
            for (int i = 0; i < NCOL; ++i)
              *reinterpret_cast<__half*>(gslice + cm_offset(ch * NCOL + i, rnn_u, b_lbo, b_sbo)) = __float2half_rn(hp[i]);
          }
        }
        if (tid == 0) SKB_TRACE(s, 6);
        // h_t exchange: every CTA wrote its fp16 slice to this cluster's L2
        // scratch; one thread multicasts it into hbuf[nb] of every CTA, the
        // bytes completing on each CTA's hfull[nb].
        fence_proxy_async_global();
        named_bar_sync(1, kEpi);   // also: sG is rewritten next step only after every read
        if (t + 1 < trip && tid == 0) {
          bulk_g2s_multicast(sH + nb * hbytes + q * sbytes, gslice, sbytes, &hfull[nb],
                             (uint16_t)((1u << C) - 1));
          if (tid == 0) SKB_TRACE(s, 7);
        }
        // output sequence (stacked + transposed layout [R, T, H]); off the
        // critical path: the h_t exchange is already in flight.
        if constexpr (kGated) {
#pragma unroll
          for (int p = 0; p < NP; ++p) {
            if (!pv[p]) continue;
            const int n = pn[p], r = s_row[n];
            if (r < 0 || t >= s_len[n]) continue;   // frozen steps: rnn_fill_frozen_kernel
            const int unit0 = (int)q * U + pu[p];
            float* o = a.out + ((size_t)r * T + t) * H + unit0;
            if (unit0 + UG <= H && (H & 3) == 0) {
#pragma unroll
              for (int v4 = 0; v4 < UG / 4; ++v4)
                reinterpret_cast<float4*>(o)[v4] = make_float4(hp[p * UG + 4 * v4], hp[p * UG + 4 * v4 + 1],
                                                               hp[p * UG + 4 * v4 + 2], hp[p * UG + 4 * v4 + 3]);
            } else {
#pragma unroll
              for (int e = 0; e < UG; ++e) if (unit0 + e < H) o[e] = hp[p * UG + e];
            }
          }
        } else if (rnn_valid) {
#pragma unroll
          for (int i = 0; i < NCOL; ++i) {
            const int n = ch * NCOL + i, r = s_row[n];
            if (r >= 0 && t < s_len[n]) a.out[((size_t)r * T + t) * H + rnn_unit] = hp[i];
          }
        }
      }
      SKB_TTRACE(tile_iter, 2);
      // final states (the frozen tail [len, max_len_p) of the output sequence is
      // written by rnn_fill_frozen_kernel from hT, off the recurrence)
      if constexpr (kGated) {
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          if (!pv[p]) continue;
          const int n = pn[p], r = s_row[n];
          if (r < 0) continue;
#pragma unroll
          for (int e = 0; e < UG; ++e) {
            const int unit = (int)q * U + pu[p] + e;
            if (unit >= H) continue;
            a.hT[(size_t)r * H + unit] = hp[p * UG + e];
            if (a.cT) a.cT[(size_t)r * H + unit] = cc[p * UG + e];
          }
        }
      } else if (rnn_valid) {
#pragma unroll
        for (int i = 0; i < NCOL; ++i) {
          const int r = s_row[ch * NCOL + i];
          if (r >= 0) a.hT[(size_t)r * H + rnn_unit] = hp[i];
        }
      }
    } else if (warp == EW) {
      // ======================= x_t loader =======================
      // x_t arrives pre-converted (fp16, core-matrix image, see pack_x_kernel):
      // one bulk async copy per step, prefetched two steps ahead.
      if (tid == kEpi) {
        const uint8_t* img = a.ximg + (size_t)tile * T * xbytes;
        for (int t = 0; t < trip; ++t) {
          const uint32_t s = step + t, j = s & 1, use = s >> 1;
          SKB_TRACE(s, 8);
          mbar_wait(&xempty[j], (use & 1) ^ 1);
          mbar_arrive_expect_tx(&xfull[j], xbytes);
          for (uint32_t off = 0; off < xbytes; off += 16384)
            bulk_g2s(sX + j * xbytes + off, img + (size_t)t * xbytes + off, min(16384u, xbytes - off), &xfull[j]);
          SKB_TRACE(s, 9);
        }
      }
    } else if (warp == EW + 1) {
      // ======================= MMA issuer (whole warp, elected lane issues) =======================
      const uint32_t idesc = idesc_f16_f32(128, NT);
      const uint32_t x_addr = smem_u32(sX), h_addr = smem_u32(sH);
      const int kx_steps = a.Kx / 16, kh_steps = a.Kh / 16;
      if (!hfull_armed) {   // arm the first phase of both exchange barriers
        if (lane == 0) {
          mbar_arrive_expect_tx(&hfull[0], C * sbytes);
          mbar_arrive_expect_tx(&hfull[1], C * sbytes);
        }
        hfull_armed = true;
      }
      for (int t = 0; t < trip; ++t) {
        const uint32_t s = step + t, j = s & 1, use = s >> 1;
        mbar_wait(&xfull[j], use & 1);
        if (lane == 0) SKB_TRACE(s, 0);
        mbar_wait(&dfree[j], (use & 1) ^ 1);
        if (lane == 0) SKB_TRACE(s, 1);
        tc_fence_after();
        const uint32_t d = tmem + j * 2 * NT;   // accumulator pair: d (x + even h steps), d + NT (odd h steps)
        const uint64_t xdesc0 = sdesc_kmajor_noswz(x_addr + j * xbytes, b_lbo, b_sbo);
#pragma unroll 4
        for (int ks = 0; ks < kx_steps; ++ks)   // +2*b_lbo bytes per K=16 step (>>4 in the descriptor)
          umma_f16_ts_warp(d, tmem + kWCol + ks * 8, xdesc0 + (uint64_t)(ks * 2 * b_lbo >> 4), idesc,
                           ks > 0 ? 1u : 0u);
        umma_commit_warp(&xempty[j]);
        {   // h_t (h0 at a tile's first step) from every CTA of the cluster
          const uint32_t hb = s & 1;
          mbar_wait(&hfull[hb], hwait[hb] & 1);
          ++hwait[hb];
          if (lane == 0) mbar_arrive_expect_tx(&hfull[hb], C * sbytes);   // arm its next phase
        }
        if (lane == 0) SKB_TRACE(s, 2);
        tc_fence_after();
        const uint64_t hdesc0 = sdesc_kmajor_noswz(h_addr + (s & 1) * hbytes, b_lbo, b_sbo);
        // Two independent accumulation chains so consecutive MMAs do not wait on
        // each other's accumulator (the h part is on the recurrence's critical path).
#pragma unroll 4
        for (int ks = 0; ks < kh_steps; ++ks)
          umma_f16_ts_warp(two_chains ? d + (ks & 1) * NT : d, tmem + kWCol + (kx_steps + ks) * 8,
                           hdesc0 + (uint64_t)(ks * 2 * b_lbo >> 4), idesc,
                           (two_chains && (ks & 1)) ? (ks > 1 ? 1u : 0u) : 1u);
        umma_commit_warp(&mdone[j]);
        if (lane == 0) SKB_TRACE(s, 3);
      }
    }
    __syncwarp();
    step += trip;
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == EW + 1) tmem_dealloc<512>(tmem);
}

// ------------------------------------------------------------------ dual-lane LSTM kernel
// Two independent recurrences ("lanes") per CTA, each a full 64-row tile with
// N = 64 MMAs: lane L runs tiles 2*cluster + L, 2*cluster + L + 2*nclusters, ...
// with its own 8 epilogue warps, x loader warp, MMA warp, TMEM accumulators,
// shared buffers and mbarriers; the [W;U] slice in TMEM is shared.  While one
// lane's epilogue turns its gates into h_t and exchanges it across the cluster,
// the other lane's MMAs run on the tensor pipe, so the serial MMA -> epilogue ->
// exchange chain of one recurrence overlaps the other's (with N = 64 MMAs, unlike
// the ping-pong halves above).  Shared memory per lane: one x_t image, one h_t
// image, the gate exchange; a single h buffer is safe because a lane only
// multicasts h_{t+1} after every CTA's MMA of step t has retired (hempty: one
// remote arrival per CTA per step).
template <typename XT, int ACT = 1, int CELL = SKB_CELL_LSTM>
__global__ void __launch_bounds__(20 * 32, 1) rnn_fwd_dl_kernel(const RnnArgs a) {
  constexpr int NT = 64, EWL = 8, kEpiL = EWL * 32, NCOL = NT / (EWL / 4), UG = 8;   // NT == kNT
  constexpr int kLoad0 = 16, kMma0 = 18;   // warps: 0-15 epilogue (lane = warp >> 3), 16-17 loaders, 18-19 MMA
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ uint64_t xfull[2], xempty[2], hfull[2], hempty[2][2], mdone[2][2], dfree[2][2];
  __shared__ uint32_t tmem_s;
  __shared__ int s_row[2][NT], s_len[2][NT];
  __shared__ int s_trip[2];

  uint8_t* smem = smem_raw;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int L = warp < kLoad0 ? (warp >> 3) : (warp < kMma0 ? warp - kLoad0 : warp - kMma0);
  const uint32_t q = cluster_ctarank();
  const int C = a.C, U = a.U, H = a.H, T = a.T;
  const uint32_t xbytes = NT * a.Kx * 2, hbytes = NT * a.Kh * 2, sbytes = NT * U * 2;
  const uint32_t gbytes = 4 * NT * kGS * 4, lane_bytes = xbytes + hbytes + gbytes;
  uint8_t* sX = smem + L * lane_bytes;     // [NT x Kx] fp16, core-matrix layout
  uint8_t* sH = sX + xbytes;               // [NT x Kh] fp16
  float* sG = reinterpret_cast<float*>(sH + hbytes);   // gates [4][NT][kGS]
  constexpr uint32_t b_lbo = NT * 16, b_sbo = 128;
  constexpr uint32_t kWCol = 256;          // TMEM: lane L's D pair at L*128 + j*64, weights at 256

  if (tid == 0) {
    for (int l = 0; l < 2; ++l) {
      mbar_init(&xfull[l], 1);
      mbar_init(&xempty[l], 1);
      mbar_init(&hfull[l], 1);
      for (int j = 0; j < 2; ++j) {
        mbar_init(&hempty[l][j], C);
        mbar_init(&mdone[l][j], 1);
        mbar_init(&dfree[l][j], EWL);
      }
    }
    fence_mbar_init();
  }
  if (warp == kMma0) tmem_alloc<512>(&tmem_s);
  for (uint32_t i = tid; i < 2 * lane_bytes / 16; i += 20 * 32)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_s;
  float bias = 0.f;
  if (warp < 4) {
    const uint32_t* src = reinterpret_cast<const uint32_t*>(a.wpack + ((size_t)q * 128 + tid) * a.K * 2);
    for (int c0 = 0; c0 < a.K / 2; c0 += 8) {
      uint32_t r[8];
      const uint4 lo = __ldg(reinterpret_cast<const uint4*>(src + c0));
      const uint4 hi = __ldg(reinterpret_cast<const uint4*>(src + c0 + 4));
      r[0] = lo.x; r[1] = lo.y; r[2] = lo.z; r[3] = lo.w; r[4] = hi.x; r[5] = hi.y; r[6] = hi.z; r[7] = hi.w;
      tmem_st8(tmem + ((uint32_t)(warp * 32) << 16) + kWCol + c0, r);
    }
    tmem_st_wait();
  }
  if (warp < kLoad0) bias = a.bpack[q * 128 + (warp & 3) * 32 + lane];
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  cluster_sync();   // every CTA's barriers are initialised before any remote traffic

  // epilogue thread e (0..255 within the lane): gate phase = warp quarter qw, column
  // half ch; cell phase = row n = e / G8, units pu..pu+7 (G8 = U / 8 = 4)
  const int wl = warp & 7, qw = wl & 3, ch = wl >> 2, e = tid & (kEpiL - 1);
  const int G8 = U / UG;
  const int pn = e / G8, pu = (e % G8) * UG;
  float hp[UG], cc[UG];
  uint8_t* gslice = a.hscratch + ((size_t)cluster_id_x() * 2 + L) * hbytes + q * sbytes;   // our h slice (lane L)
  const uint32_t tile_bar = 5 + L, xch_bar = 1 + 2 * L, gate_bar = 2 + 2 * L;   // named barriers of lane L
  constexpr uint32_t kLaneThreads = kEpiL + 64;

  uint32_t step = 0;
  const int nclusters = (int)nclusters_x();
  const int stride = 2 * nclusters;
  int m_r = -1, m_len = 0;
  auto tile_meta = [&](int tl) {
    m_r = -1; m_len = 0;
    if (tl < a.ntiles) {
      m_r = a.perm[tl * NT + e];
      if (m_r >= 0) {
        const int tmax = max(0, min(a.pmax[m_r / a.Bp], T));
        m_len = (int)max(0LL, min((long long)a.lens[m_r], (long long)tmax));
      }
    }
  };
  // Tiles are sorted longest first; round k hands out tiles [k*stride, (k+1)*stride) in
  // snake order (reversed on odd rounds), so no lane or cluster always takes the longer tile.
  const int pos = 2 * (int)cluster_id_x() + L;
  auto tile_of = [&](int k) { return k * stride + ((k & 1) ? stride - 1 - pos : pos); };
  const int tile0 = tile_of(0);
  if (warp < kLoad0 && e < NT) tile_meta(tile0);
  if (warp == kMma0 + L && lane == 0) mbar_arrive_expect_tx(&hfull[L], C * sbytes);   // arm phase 0

  for (int round = 0, tile = tile0; tile < a.ntiles || round * stride < a.ntiles; tile = tile_of(++round)) {
    if (tile >= a.ntiles) continue;   // a partial last round
    named_bar_sync(tile_bar, kLaneThreads);   // this lane's previous tile retired (s_row/s_len rewritten)
    if (warp < kLoad0 && e < NT) { s_row[L][e] = m_r; s_len[L][e] = m_len; }
    named_bar_sync(tile_bar, kLaneThreads);
    if (warp == 8 * L) {
      int m = max(s_len[L][lane], s_len[L][lane + 32]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (lane == 0) s_trip[L] = m;
    }
    named_bar_sync(tile_bar, kLaneThreads);
    const int trip = s_trip[L];

    if (warp < kLoad0) {
      // ======================= epilogue (lane L) =======================
      if (e < NT) {   // next tile's metadata and its h0/c0 rows -> L2
        tile_meta(tile_of(round + 1));
        if (m_r >= 0) {
          const char* h0n = reinterpret_cast<const char*>(a.h0 + (size_t)m_r * H);
          const char* c0n = a.c0 ? reinterpret_cast<const char*>(a.c0 + (size_t)m_r * H) : nullptr;
          for (int off = 0; off < H * 4; off += 128) {
            prefetch_l2(h0n + off);
            if (c0n) prefetch_l2(c0n + off);
          }
        }
      }
      {
        const int r = s_row[L][pn];
        const int unit0 = (int)q * U + pu;
        float hv[8], cv[8];
        if (r >= 0) {
          load_x8<float>(a.h0 + (size_t)r * H, unit0, H, hv);
          if (a.c0) {
            load_x8<float>(a.c0 + (size_t)r * H, unit0, H, cv);
          } else {
#pragma unroll
            for (int k = 0; k < 8; ++k) cv[k] = 0.f;
          }
        } else {
#pragma unroll
          for (int k = 0; k < 8; ++k) hv[k] = cv[k] = 0.f;
        }
#pragma unroll
        for (int k = 0; k < UG; ++k) { hp[k] = hv[k]; cc[k] = cv[k]; }
      }
      // write h (fp16) for step u into our L2 slice and multicast it into every CTA's sH
      // once every CTA's MMA of step u-1 (the buffer's last reader) has retired
      auto send_h = [&](uint32_t u) {
        uint32_t hw[UG / 2];
#pragma unroll
        for (int k = 0; k < UG / 2; ++k) {
          __half2 h2 = __floats2half2_rn(hp[2 * k], hp[2 * k + 1]);
          hw[k] = *reinterpret_cast<uint32_t*>(&h2);
        }
        *reinterpret_cast<uint4*>(gslice + cm_offset(pn, pu, b_lbo, b_sbo)) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
        fence_proxy_async_global();
        named_bar_sync(xch_bar, kEpiL);
        if (e == 0) {
          if (L == 0 && u > 0) SKB_TRACE(u - 1, 6);
          if (u > 0) mbar_wait_cluster(&hempty[L][(u - 1) & 1], ((u - 1) >> 1) & 1);
          if (L == 0 && u > 0) SKB_TRACE(u - 1, 11);
          bulk_g2s_multicast(sH + q * sbytes, gslice, sbytes, &hfull[L], (uint16_t)((1u << C) - 1));
          if (L == 0 && u > 0) SKB_TRACE(u - 1, 7);
        }
      };
      if (trip > 0) send_h(step);
      const GateAct<CELL, ACT> act(qw, bias);
      for (int t = 0; t < trip; ++t) {
        const uint32_t s = step + t, j = s & 1, use = s >> 1;
        mbar_wait(&mdone[L][j], use & 1);
        if (e == 0 && L == 0) SKB_TRACE(s, 4);
        tc_fence_after();
        const uint32_t trow = tmem + ((uint32_t)(qw * 32) << 16) + L * 128 + j * NT + ch * NCOL;
        float* g_out = sG + (qw * NT + ch * NCOL) * kGS + lane;
#pragma unroll
        for (int c16 = 0; c16 < NCOL / 16; ++c16) {
          float v[16];
          tmem_ld16(trow + c16 * 16, v);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) g_out[(c16 * 16 + i) * kGS] = act(v[i]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&dfree[L][j]);
        named_bar_sync(gate_bar, kEpiL);
        if (e == 0 && L == 0) SKB_TRACE(s, 10);
        {
          float g4[4][UG];
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            const float4* src = reinterpret_cast<const float4*>(sG + (g * NT + pn) * kGS + pu);
#pragma unroll
            for (int v4 = 0; v4 < UG / 4; ++v4) {
              const float4 x0 = src[v4];
              g4[g][4 * v4] = x0.x; g4[g][4 * v4 + 1] = x0.y; g4[g][4 * v4 + 2] = x0.z; g4[g][4 * v4 + 3] = x0.w;
            }
          }
          const bool live = t < s_len[L][pn];
#pragma unroll
          for (int k = 0; k < UG; ++k) cell_update<CELL, ACT>(g4[0][k], g4[1][k], g4[2][k], g4[3][k], cc[k], hp[k], live);
        }
        if (t + 1 < trip) send_h(s + 1);
        else named_bar_sync(xch_bar, kEpiL);   // sG is rewritten next step only after every read
        // output sequence [R, T, H] (frozen tails: rnn_fill_frozen_kernel)
        {
          const int r = s_row[L][pn];
          if (r >= 0 && t < s_len[L][pn]) {
            float* o = a.out + ((size_t)r * T + t) * H + (int)q * U + pu;
            reinterpret_cast<float4*>(o)[0] = make_float4(hp[0], hp[1], hp[2], hp[3]);
            reinterpret_cast<float4*>(o)[1] = make_float4(hp[4], hp[5], hp[6], hp[7]);
          }
        }
      }
      {
        const int r = s_row[L][pn];
        if (r >= 0) {
          float* hT = a.hT + (size_t)r * H + (int)q * U + pu;
          reinterpret_cast<float4*>(hT)[0] = make_float4(hp[0], hp[1], hp[2], hp[3]);
          reinterpret_cast<float4*>(hT)[1] = make_float4(hp[4], hp[5], hp[6], hp[7]);
          if (a.cT) {
            float* cT = a.cT + (size_t)r * H + (int)q * U + pu;
            reinterpret_cast<float4*>(cT)[0] = make_float4(cc[0], cc[1], cc[2], cc[3]);
            reinterpret_cast<float4*>(cT)[1] = make_float4(cc[4], cc[5], cc[6], cc[7]);
          }
        }
      }
    } else if (warp < kMma0) {
      // ======================= x_t loader (lane L): one buffer, filled once x-part(s-1) retired
      if (lane == 0) {
        const uint8_t* img = a.ximg + (size_t)tile * T * xbytes;
        for (int t = 0; t < trip; ++t) {
          const uint32_t s = step + t;
          mbar_wait(&xempty[L], (s & 1) ^ 1);
          mbar_arrive_expect_tx(&xfull[L], xbytes);
          for (uint32_t off = 0; off < xbytes; off += 16384)
            bulk_g2s(sX + off, img + (size_t)t * xbytes + off, min(16384u, xbytes - off), &xfull[L]);
        }
      }
    } else {
      // ======================= MMA issuer (lane L)
      // order: x-part(s0); then per step h-part(s), x-part(s+1) -- a late x_{s+1}
      // (single buffer) never holds back the h-part on the recurrence's critical path
      const uint32_t idesc = idesc_f16_f32(128, NT);
      const uint32_t x_addr = smem_u32(sX), h_addr = smem_u32(sH);
      const int kx_steps = a.Kx / 16, kh_steps = a.Kh / 16;
      const uint64_t xdesc0 = sdesc_kmajor_noswz(x_addr, b_lbo, b_sbo);
      const uint64_t hdesc0 = sdesc_kmajor_noswz(h_addr, b_lbo, b_sbo);
      auto x_part = [&](uint32_t s) {
        const uint32_t j = s & 1, use = s >> 1;
        mbar_wait(&xfull[L], s & 1);
        if (lane == 0 && L == 0) SKB_TRACE(s, 0);
        mbar_wait(&dfree[L][j], (use & 1) ^ 1);
        if (lane == 0 && L == 0) SKB_TRACE(s, 1);
        tc_fence_after();
        const uint32_t d = tmem + L * 128 + j * NT;
#pragma unroll 4
        for (int ks = 0; ks < kx_steps; ++ks)
          umma_f16_ts_warp(d, tmem + kWCol + ks * 8, xdesc0 + (uint64_t)(ks * 2 * b_lbo >> 4), idesc, ks > 0 ? 1u : 0u);
        umma_commit_warp(&xempty[L]);
      };
      if (trip > 0) x_part(step);
      for (int t = 0; t < trip; ++t) {
        const uint32_t s = step + t, j = s & 1;
        const uint32_t d = tmem + L * 128 + j * NT;
        mbar_wait(&hfull[L], s & 1);
        if (lane == 0 && L == 0) SKB_TRACE(s, 2);
        if (lane == 0) mbar_arrive_expect_tx(&hfull[L], C * sbytes);   // arm the next phase
        tc_fence_after();
#pragma unroll 4
        for (int ks = 0; ks < kh_steps; ++ks)
          umma_f16_ts_warp(d, tmem + kWCol + (kx_steps + ks) * 8, hdesc0 + (uint64_t)(ks * 2 * b_lbo >> 4), idesc, 1u);
        umma_commit_warp(&mdone[L][j]);
        // the retirement of this CTA's MMAs of step s (the last reader of sH) is
        // counted on hempty[s&1] of every CTA of the cluster
        umma_commit_warp_multicast(&hempty[L][j], (uint16_t)((1u << C) - 1));
        if (lane == 0 && L == 0) SKB_TRACE(s, 3);
        if (t + 1 < trip) x_part(s + 1);
      }
    }
    __syncwarp();
    step += trip;
  }

  // Every CTA's tcgen05.commit of a lane's last step arrives (multicast) on this CTA's
  // hempty: wait for that phase, so no arrival is in flight to this CTA's shared memory
  // when it exits.
  if (warp < kLoad0 && e == 0 && step > 0) {
    const uint32_t last = step - 1;
    mbar_wait_cluster(&hempty[L][last & 1], (last >> 1) & 1);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == kMma0) tmem_dealloc<512>(tmem);
}

// ------------------------------------------------------------------ CTA-pair kernel
// The default LSTM/GRU kernel for 32-unit CTA slices with an even CTA count
// (H = 64, 128, 192, 256).  Measured on the dual-lane kernel: a 128x64x16
// tcgen05.mma costs ~60 cycles, about half the per-SM rate of N >= 128
// (profiles/r01_umma_rate.txt), and its shared-memory gate exchange sits on the
// recurrence's critical path.  Here
//   * CTAs 2p, 2p+1 of the cluster form a CTA pair; the even CTA issues M=256
//     cta_group::2 MMAs: A = the pair's 256 gate rows (each CTA's 128 [W;U] rows
//     resident in its own TMEM), B = x_t / h_t of a 128-row tile, 64 rows per CTA
//     in shared memory, D = 128 gate rows x 128 tile rows in each CTA's TMEM:
//     N = 128 per instruction at the shared-memory footprint of a 64-row tile.
//   * TMEM lane quarter w holds units 8w..8w+7 of the CTA's 32-unit slice with the
//     four gate blocks at lanes +0/+8/+16/+24, so two 16x256b tcgen05.ld hand each
//     epilogue thread all four gates of one unit for 16 batch rows: no gate
//     exchange, and c/h stay in registers for the whole tile.
//   * h_t is double-buffered in shared memory, so nothing waits for "buffer free":
//     h_{t+1} exists only after every CTA of the cluster consumed h_{t-1}.  Each CTA
//     writes its fp16 slice for rows 0-63 / 64-127 to L2 and multicasts it to the
//     even / odd CTAs.
//   * Two independent 128-row recurrences ("lanes") per CTA interleave on the
//     tensor pipe.  TMEM columns: D of lane 0 [0,128), lane 1 [128,256), weights
//     [256,512).
//   * The odd CTA's MMA warp relays its local "x_t landed" / "h_t landed" phases to
//     the leader (remote mbarrier arrivals); the epilogue warps of both CTAs release
//     D on the leader's dfree barrier.
SKB_DEV float2 tanh2_approx(float a, float b) {   // two tanh in one MUFU op (fp16 precision, ~2^-11)
  __half2 x = __floats2half2_rn(a, b);
  uint32_t r;
  asm("tanh.approx.f16x2 %0, %1;" : "=r"(r) : "r"(*reinterpret_cast<uint32_t*>(&x)));
  return __half22float2(*reinterpret_cast<__half2*>(&r));
}
// Gate activations of two cells (ACT 2: tanh.approx.f16x2; otherwise per cell via pact)
template <int CELL, int ACT, int G>
SKB_DEV float2 pact2(float z0, float z1, float kb);
// Cell update of two cells from their activated gate pairs (ACT 2: tanh(c) / tanh(n) in f16x2)
template <int CELL, int ACT>
SKB_DEV void cell_update2(float2 g0, float2 g1, float2 g2, float2 g3, float& c0, float& c1, float& h0, float& h1,
                          bool live0, bool live1) {
  if constexpr (ACT == 2) {
    if constexpr (CELL == SKB_CELL_GRU) {
      const float2 n = tanh2_approx(fmaf(g1.x, g3.x, g2.x), fmaf(g1.y, g3.y, g2.y));
      const float a0 = fmaf(g0.x, h0 - n.x, n.x), a1 = fmaf(g0.y, h1 - n.y, n.y);
      h0 = live0 ? a0 : h0;
      h1 = live1 ? a1 : h1;
    } else {
      const float ca = fmaf(g1.x, c0, g0.x * g2.x), cb = fmaf(g1.y, c1, g0.y * g2.y);
      const float2 th = tanh2_approx(ca, cb);
      const float ha = g3.x * th.x, hb = g3.y * th.y;
      c0 = live0 ? ca : c0;
      c1 = live1 ? cb : c1;
      h0 = live0 ? ha : h0;
      h1 = live1 ? hb : h1;
    }
  } else {
    cell_update<CELL, ACT>(g0.x, g1.x, g2.x, g3.x, c0, h0, live0);
    cell_update<CELL, ACT>(g0.y, g1.y, g2.y, g3.y, c1, h1, live1);
  }
}

template <int CELL, int ACT, int G>
SKB_DEV float pact(float z, float kb) {
  if constexpr (CELL == SKB_CELL_GRU && G >= 2) {
    return z + kb;   // GRU n_x / n_h stay affine (+ bias) until the cell combines them
  } else {
    constexpr bool th = (CELL != SKB_CELL_GRU) && G == 2;   // LSTM g gate: tanh; the rest sigmoid
    if constexpr (ACT != 0) {
      constexpr float kl = th ? 1.f : 0.5f, add = th ? 0.f : 0.5f;
      return fmaf(kl, tanh_approx(fmaf(z, kl, kb)), add);
    } else {
      constexpr float kl = th ? -2.8853900817779268f : -1.4426950408889634f;
      constexpr float mul = th ? 2.f : 1.f, add = th ? -1.f : 0.f;
      return fmaf(mul, inv1pexp2(fmaf(z, kl, kb)), add);
    }
  }
}
template <int CELL, int ACT, int G>
SKB_DEV float pact_kb(float bias) {
  if constexpr (CELL == SKB_CELL_GRU && G >= 2) {
    return bias;
  } else {
    constexpr bool th = (CELL != SKB_CELL_GRU) && G == 2;
    if constexpr (ACT != 0) return (th ? 1.f : 0.5f) * bias;
    else return (th ? -2.8853900817779268f : -1.4426950408889634f) * bias;
  }
}

template <int CELL, int ACT, int G>
SKB_DEV float2 pact2(float z0, float z1, float kb) {
  if constexpr (ACT != 2 || (CELL == SKB_CELL_GRU && G >= 2)) {
    return make_float2(pact<CELL, ACT, G>(z0, kb), pact<CELL, ACT, G>(z1, kb));
  } else {
    constexpr bool th = (CELL != SKB_CELL_GRU) && G == 2;
    constexpr float kl = th ? 1.f : 0.5f, add = th ? 0.f : 0.5f;
    const float2 t = tanh2_approx(fmaf(z0, kl, kb), fmaf(z1, kl, kb));
    return th ? t : make_float2(fmaf(kl, t.x, add), fmaf(kl, t.y, add));
  }
}

template <typename XT, int ACT = 1, int CELL = SKB_CELL_LSTM>
__global__ void __launch_bounds__(20 * 32, 1) rnn_fwd_pair_kernel(const RnnArgs a) {
  constexpr int NT = 128, NH = 64, EWL = 8, kEpiL = EWL * 32;
  constexpr int kLoad0 = 16, kMma0 = 18;   // warps: 0-15 epilogue (lane = warp >> 3), 16-17 loaders, 18-19 MMA / relay
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ uint64_t xfull[2], xempty[2], hfull[2][2], mdone[2], dfree[2];
  __shared__ uint32_t tmem_s;
  __shared__ int2 s_meta[2][NT];   // (row, clamped length) of the lane's tile rows
  __shared__ int s_trip[2][3];     // [lane]: tile trip, trip of rows 0-63, trip of rows 64-127

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int L = warp < kLoad0 ? (warp >> 3) : (warp < kMma0 ? warp - kLoad0 : warp - kMma0);
  const uint32_t q = cluster_ctarank(), odd = q & 1u, peer = q ^ 1u;
  const bool leader = odd == 0;
  const int C = a.C, H = a.H, T = a.T;
  const uint32_t xbytes = NH * a.Kx * 2, hbytes = NH * a.Kh * 2;
  constexpr uint32_t sbytes = NH * 32 * 2;   // one CTA's h slice of one 64-row half (4 KB)
  const uint32_t lane_bytes = xbytes + 2 * hbytes;
  uint8_t* sX = smem_raw + L * lane_bytes;   // [NH x Kx] fp16, core-matrix layout
  uint8_t* sH = sX + xbytes;                 // 2 x [NH x Kh] fp16
  constexpr uint32_t b_lbo = NH * 16, b_sbo = 128;
  constexpr uint32_t kWCol = 256;
  const uint16_t pair_mask = (uint16_t)(3u << (q & ~1u));
  uint16_t even_mask = 0;
  for (int i = 0; i < C; i += 2) even_mask |= (uint16_t)(1u << i);
  const uint16_t odd_mask = (uint16_t)(even_mask << 1);

  if (tid == 0) {
    for (int l = 0; l < 2; ++l) {
      mbar_init(&xfull[l], leader ? 2 : 1);      // own loader (+ the odd CTA's relay)
      mbar_init(&xempty[l], 1);
      mbar_init(&hfull[l][0], leader ? 2 : 1);   // own arm (+ relay)
      mbar_init(&hfull[l][1], leader ? 2 : 1);
      mbar_init(&mdone[l], 1);
      mbar_init(&dfree[l], 2 * EWL);             // epilogue warps of both CTAs (leader's copy is used)
    }
    fence_mbar_init();
  }
  if (warp == kMma0) tmem_alloc_pair<512>(&tmem_s);
  for (uint32_t i = tid; i < 2 * lane_bytes / 16; i += 20 * 32)
    reinterpret_cast<uint4*>(smem_raw)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_s;
  if (warp < 4) {
    // TMEM lane l = 32w + 8g + u <- packed slab row 32g + 8w + u (gate g of unit 8w + u)
    const int srow = ((tid & 31) >> 3) * 32 + warp * 8 + (tid & 7);
    const uint32_t* src = reinterpret_cast<const uint32_t*>(a.wpack + ((size_t)q * 128 + srow) * a.K * 2);
    for (int c0 = 0; c0 < a.K / 2; c0 += 8) {
      uint32_t r[8];
      const uint4 lo = __ldg(reinterpret_cast<const uint4*>(src + c0));
      const uint4 hi = __ldg(reinterpret_cast<const uint4*>(src + c0 + 4));
      r[0] = lo.x; r[1] = lo.y; r[2] = lo.z; r[3] = lo.w; r[4] = hi.x; r[5] = hi.y; r[6] = hi.z; r[7] = hi.w;
      tmem_st8(tmem + ((uint32_t)(warp * 32) << 16) + kWCol + c0, r);
    }
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  cluster_sync();   // every CTA's barriers and TMEM are initialised before any remote traffic

  // epilogue thread: TMEM lane quarter qw, column half ch (= tile rows 64ch..64ch+63),
  // unit uc = 8qw + lane/4 of the CTA's slice, rows 64ch + 8k + 2(lane%4) + {0,1}, k < 8
  const int wl = warp & 7, qw = wl & 3, ch = wl >> 2, cq = lane & 3, e = tid & (kEpiL - 1);
  const int uc = qw * 8 + (lane >> 2), unit = (int)q * 32 + uc;
  float kb0 = 0.f, kb1 = 0.f, kb2 = 0.f, kb3 = 0.f;
  if (warp < kLoad0) {
    const float* bp = a.bpack + q * 128 + uc;
    kb0 = pact_kb<CELL, ACT, 0>(bp[0]);
    kb1 = pact_kb<CELL, ACT, 1>(bp[32]);
    kb2 = pact_kb<CELL, ACT, 2>(bp[64]);
    kb3 = pact_kb<CELL, ACT, 3>(bp[96]);
  }
  float hh[16], cc[16];
  const uint32_t tile_bar = 5 + L;
  constexpr uint32_t kLaneThreads = kEpiL + 64;
  auto cell_row = [&](int ci) { return ch * 64 + (ci >> 3) * 32 + ((ci >> 1) & 3) * 8 + 2 * cq + (ci & 1); };

  uint32_t step = 0;
  const int nclusters = (int)nclusters_x();
  const int stride = 2 * nclusters;
  int2 m_meta = make_int2(-1, 0);
  auto tile_meta = [&](int tl) {
    m_meta = make_int2(-1, 0);
    if (tl < a.ntiles) {
      const int r = a.perm[tl * NT + e];
      if (r >= 0) {
        const int tmax = max(0, min(a.pmax[r / a.Bp], T));
        m_meta = make_int2(r, (int)max(0LL, min((long long)a.lens[r], (long long)tmax)));
      }
    }
  };
  const int pos = 2 * (int)cluster_id_x() + L;
  auto tile_of = [&](int k) { return k * stride + ((k & 1) ? stride - 1 - pos : pos); };
  const int tile0 = tile_of(0);
  if (warp < kLoad0 && e < NT) tile_meta(tile0);
  if (warp == kMma0 + L && lane == 0) {   // arm the h phases of steps 0 and 1
    mbar_arrive_expect_tx(&hfull[L][0], C * sbytes);
    mbar_arrive_expect_tx(&hfull[L][1], C * sbytes);
  }

  for (int round = 0, tile = tile0; tile < a.ntiles || round * stride < a.ntiles; tile = tile_of(++round)) {
    if (tile >= a.ntiles) continue;   // a partial last round
    named_bar_sync(tile_bar, kLaneThreads);   // this lane's previous tile retired (s_meta rewritten)
    if (warp < kLoad0 && e < NT) s_meta[L][e] = m_meta;
    named_bar_sync(tile_bar, kLaneThreads);
    if (warp == 8 * L) {
      int ma = max(s_meta[L][lane].y, s_meta[L][lane + 32].y);
      int mb = max(s_meta[L][lane + 64].y, s_meta[L][lane + 96].y);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        ma = max(ma, __shfl_xor_sync(0xffffffffu, ma, o));
        mb = max(mb, __shfl_xor_sync(0xffffffffu, mb, o));
      }
      if (lane == 0) { s_trip[L][0] = max(ma, mb); s_trip[L][1] = ma; s_trip[L][2] = mb; }
    }
    named_bar_sync(tile_bar, kLaneThreads);
    const int trip = s_trip[L][0];

    if (warp < kLoad0) {
      // ======================= epilogue (lane L)
      if (e < NT) {   // next tile's metadata and its h0/c0 rows -> L2
        tile_meta(tile_of(round + 1));
        if (m_meta.x >= 0) {
          const char* h0n = reinterpret_cast<const char*>(a.h0 + (size_t)m_meta.x * H);
          const char* c0n = a.c0 ? reinterpret_cast<const char*>(a.c0 + (size_t)m_meta.x * H) : nullptr;
          for (int off = 0; off < H * 4; off += 128) {
            prefetch_l2(h0n + off);
            if (c0n) prefetch_l2(c0n + off);
          }
        }
      }
#pragma unroll
      for (int ci = 0; ci < 16; ++ci) {
        const int r = s_meta[L][cell_row(ci)].x;
        hh[ci] = r >= 0 ? __ldg(a.h0 + (size_t)r * H + unit) : 0.f;
        cc[ci] = (r >= 0 && a.c0) ? __ldg(a.c0 + (size_t)r * H + unit) : 0.f;
      }
      // fp16 h slice for step u -> L2 -> multicast into sH[u&1] of the even (ch 0) or odd (ch 1) CTAs
      // Unit pairs: lanes l and l^4 hold units u, u^1 of the same rows; after one shuffle the
      // even-unit lane holds (h_u, h_u+1) of row 2cq and the odd-unit lane those of row 2cq+1
      // (within column group k), i.e. 2 consecutive units of one row per lane.
      const bool ueven = ((lane >> 2) & 1) == 0;
      const int ul = (lane >> 2) & ~1, er = ueven ? 0 : 1;
      auto unit_pair = [&](int k) {
        const int ci = (k >> 2) * 8 + (k & 3) * 2;
        const float send = ueven ? hh[ci + 1] : hh[ci];
        const float recv = __shfl_xor_sync(0xffffffffu, send, 4);
        return ueven ? make_float2(hh[ci], recv) : make_float2(recv, hh[ci + 1]);
      };
      // fp16 h slice for step u -> L2 -> multicast into sH[u&1] of the even (ch 0) or odd (ch 1) CTAs
      auto send_h = [&](uint32_t u) {
        uint8_t* gs = a.hscratch + (((size_t)cluster_id_x() * 2 + L) * 2 + (u & 1)) * (size_t)(NT * a.Kh * 2) +
                      (size_t)q * (NT * 64) + ch * sbytes;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float2 p = unit_pair(k);
          const int nl = k * 8 + 2 * cq + er;
          *reinterpret_cast<__half2*>(gs + qw * 1024 + (nl >> 3) * 128 + (nl & 7) * 16 + ul * 2) =
              __floats2half2_rn(p.x, p.y);
        }
        fence_proxy_async_global();
        named_bar_sync(1 + 2 * L + ch, 128);
        if (qw == 0 && lane == 0)
          bulk_g2s_multicast(sH + (u & 1) * hbytes + q * sbytes, gs, sbytes, &hfull[L][u & 1],
                             ch ? odd_mask : even_mask);
      };
      if (trip > 0) send_h(step);
      for (int t = 0; t < trip; ++t) {
        const uint32_t s = step + t;
        mbar_wait_sleep(&mdone[L], s & 1);
        if (e == 0 && L == 0) SKB_TRACE(s, 4);
        if (e == 0 && L == 0) SKB_TRACE_CTA(1, s, 11);
        tc_fence_after();
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          float ga[16], gb[16];
          const uint32_t col = tmem + L * 128 + ch * 64 + half * 32;
          tmem_ld_16x256b_x4(col + ((uint32_t)(qw * 32) << 16), ga);
          tmem_ld_16x256b_x4(col + ((uint32_t)(qw * 32 + 16) << 16), gb);
          tmem_ld_wait();
          if (e == 0 && L == 0) SKB_TRACE(s, 5 + 5 * half);
          if (e == 0 && L == 0 && half == 1) SKB_TRACE_CTA(1, s, 12);
          if (half == 1) {   // D fully read: the next step's x-part may overwrite it
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
              if (leader) mbar_arrive(&dfree[L]);
              else mbar_remote_arrive_relaxed(mapa(smem_u32(&dfree[L]), peer));   // no stores to publish
            }
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {   // cells ci, ci+1: same unit, tile rows r, r+1
            const int ci = half * 8 + j * 2;
            const bool live0 = t < s_meta[L][cell_row(ci)].y, live1 = t < s_meta[L][cell_row(ci + 1)].y;
            const float2 g0 = pact2<CELL, ACT, 0>(ga[4 * j], ga[4 * j + 1], kb0);
            const float2 g1 = pact2<CELL, ACT, 1>(ga[4 * j + 2], ga[4 * j + 3], kb1);
            const float2 g2 = pact2<CELL, ACT, 2>(gb[4 * j], gb[4 * j + 1], kb2);
            const float2 g3 = pact2<CELL, ACT, 3>(gb[4 * j + 2], gb[4 * j + 3], kb3);
            cell_update2<CELL, ACT>(g0, g1, g2, g3, cc[ci], cc[ci + 1], hh[ci], hh[ci + 1], live0, live1);
          }
        }
        if (e == 0 && L == 0) SKB_TRACE(s, 6);
        if (t + 1 < trip) send_h(s + 1);
        if (e == 0 && L == 0) SKB_TRACE(s, 7);
        if (e == 0 && L == 0) SKB_TRACE_CTA(1, s, 13);
        // output sequence [R, T, H], two units per store (frozen tails: rnn_fill_frozen_kernel)
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float2 p = unit_pair(k);
          const int2 m = s_meta[L][ch * 64 + k * 8 + 2 * cq + er];
          if (m.x >= 0 && t < m.y)
            *reinterpret_cast<float2*>(a.out + ((size_t)m.x * T + t) * H + (int)q * 32 + qw * 8 + ul) = p;
        }
        if (e == 0 && L == 0) SKB_TRACE(s, 9);
      }
#pragma unroll
      for (int ci = 0; ci < 16; ++ci) {
        const int r = s_meta[L][cell_row(ci)].x;
        if (r >= 0) {
          a.hT[(size_t)r * H + unit] = hh[ci];
          if (a.cT) a.cT[(size_t)r * H + unit] = cc[ci];
        }
      }
    } else if (warp < kMma0) {
      // ======================= x_t loader (lane L): this CTA's 64-row half of the tile
      if (lane == 0) {
        const int tself = s_trip[L][1 + odd];
        const uint8_t* img = a.ximg + (size_t)(2 * tile + (int)odd) * T * xbytes;
        for (int t = 0; t < trip; ++t) {
          const uint32_t s = step + t;
          mbar_wait_sleep(&xempty[L], (s & 1) ^ 1);
          if (t < tself) {
            mbar_arrive_expect_tx(&xfull[L], xbytes);
            for (uint32_t off = 0; off < xbytes; off += 16384)
              bulk_g2s(sX + off, img + (size_t)t * xbytes + off, min(16384u, xbytes - off), &xfull[L]);
          } else {
            mbar_arrive(&xfull[L]);   // every row of this half is past its length: stale (finite) image
          }
        }
      }
    } else if (leader) {
      // ======================= MMA issuer (lane L): x-part(s0); then per step h-part(s), x-part(s+1)
      const uint32_t idesc = idesc_f16_f32(256, NT);
      const int kx_steps = a.Kx / 16, kh_steps = a.Kh / 16;
      const uint64_t xdesc0 = sdesc_kmajor_noswz(smem_u32(sX), b_lbo, b_sbo);
      const uint32_t d = tmem + L * 128;
      auto x_part = [&](uint32_t s) {
        mbar_wait_sleep(&xfull[L], s & 1);
        if (lane == 0 && L == 0) SKB_TRACE(s, 0);
        mbar_wait_sleep(&dfree[L], (s & 1) ^ 1);
        if (lane == 0 && L == 0) SKB_TRACE(s, 1);
        tc_fence_after();
#pragma unroll 4
        for (int ks = 0; ks < kx_steps; ++ks)
          umma_f16_ts_pair_warp(d, tmem + kWCol + ks * 8, xdesc0 + (uint64_t)(ks * 2 * b_lbo >> 4), idesc,
                                ks > 0 ? 1u : 0u);
        umma_commit_pair_warp(&xempty[L], pair_mask);
      };
      if (trip > 0) x_part(step);
      for (int t = 0; t < trip; ++t) {
        const uint32_t s = step + t, j = s & 1;
        mbar_wait_sleep(&hfull[L][j], (s >> 1) & 1);
        if (lane == 0 && L == 0) SKB_TRACE(s, 2);
        if (lane == 0) mbar_arrive_expect_tx(&hfull[L][j], C * sbytes);   // arm step s+2
        tc_fence_after();
        const uint64_t hdesc0 = sdesc_kmajor_noswz(smem_u32(sH + j * hbytes), b_lbo, b_sbo);
#pragma unroll 4
        for (int ks = 0; ks < kh_steps; ++ks)
          umma_f16_ts_pair_warp(d, tmem + kWCol + (kx_steps + ks) * 8, hdesc0 + (uint64_t)(ks * 2 * b_lbo >> 4),
                                idesc, 1u);
        umma_commit_pair_warp(&mdone[L], pair_mask);
        if (lane == 0 && L == 0) SKB_TRACE(s, 3);
        if (t + 1 < trip) x_part(s + 1);
      }
    } else {
      // ======================= relay (odd CTA, lane L): local x_t / h_t phases -> the leader
      const uint32_t rx = mapa(smem_u32(&xfull[L]), peer);
      if (trip > 0) {
        mbar_wait_sleep(&xfull[L], step & 1);
        if (lane == 0) mbar_remote_arrive(rx);
      }
      for (int t = 0; t < trip; ++t) {
        const uint32_t s = step + t, j = s & 1;
        mbar_wait_sleep(&hfull[L][j], (s >> 1) & 1);
        if (lane == 0 && L == 0) SKB_TRACE_CTA(1, s, 14);
        if (lane == 0) {
          mbar_arrive_expect_tx(&hfull[L][j], C * sbytes);   // arm step s+2
          mbar_remote_arrive(mapa(smem_u32(&hfull[L][j]), peer));
        }
        if (t + 1 < trip) {
          mbar_wait_sleep(&xfull[L], (s + 1) & 1);
          if (lane == 0 && L == 0) SKB_TRACE_CTA(1, s + 1, 15);
          if (lane == 0) mbar_remote_arrive(rx);
        }
      }
    }
    __syncwarp();
    step += trip;
  }

  // Drain the asynchronous arrivals aimed at this CTA before it exits: the last
  // x-part's retire (xempty, both CTAs) and the peer's last D release (dfree, leader).
  if (step > 0 && lane == 0) {
    if (warp == kLoad0 + L) mbar_wait_sleep(&xempty[L], (step - 1) & 1);
    if (leader && warp == 8 * L) mbar_wait_sleep(&dfree[L], (step - 1) & 1);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == kMma0) tmem_dealloc_pair<512>(tmem);
}

// ------------------------------------------------------------------ CTA-pair kernel, four lanes
// Default for LSTM/GRU with 32-unit slices and an even CTA count.  The two-lane pair
// kernel above leaves the tensor pipe half idle: per 128-row step its chain
// (h-part MMAs -> MUFU-bound epilogue (~1.3 K cycles) -> L2 multicast exchange
// (~3 K cycles)) is ~7.7 K cycles against 2 x 2.1 K cycles of MMA (tools/trace_pair.py).
// A cta_group::2 MMA with N = 64 still runs at 89% of the N = 128 rate (36 vs 65
// cycles, profiles/r02_umma_pair.txt), so this kernel runs four independent 64-row
// recurrences per CTA pair in the same TMEM (D: 4 x 64 columns + weights) and shared
// memory (per lane: x_t 32 rows + 2 x h_t 32 rows): each lane's chain is ~half as
// long and four of them interleave on the tensor pipe.
//   * warps 0-15: epilogue, lane L = warp / 4, TMEM quarter = warp % 4; each thread
//     owns one unit x 16 rows (cols 0-31 of D = the even CTA's rows, 32-63 the odd's);
//   * warps 16-19: lane L's role warp: x_t loader (+ L2 prefetch of x_{t+2}) and, in
//     the even CTA, the MMA issuer; in the odd CTA the relay of its x_t / h_t phases.
//   * x_t images are packed per 32-row half ("halves" layout of the pack kernels).
//   * FW = 1 (SKB_RNN_FILLW=1): warp 20 is the fill warp.  At the end of each tile the lane's
//     epilogue hands the tile's rows (row, length, problem trip count) to it through a
//     two-slot shared-memory queue; it writes the frozen tails out[r, len <= t < tmax,
//     CTA slice] = h_T from the final states, off the recurrence's critical path (the
//     separate rnn_fill_frozen_kernel pass then does not run).
template <typename XT, int ACT = 1, int CELL = SKB_CELL_LSTM, int FW = 0>
__global__ void __launch_bounds__((20 + FW) * 32, 1) rnn_fwd_pair4_kernel(const RnnArgs a) {
  constexpr int NL = 4, NT = 64, NH = 32, EWL = 4, kEpiL = EWL * 32;
  constexpr int kRole0 = 16, kFill = 20;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ uint64_t xfull[NL], xempty[NL], hfull[NL][2], mdone[NL], dfree[NL];
  __shared__ uint64_t fq_full[NL][2], fq_empty[NL][2];   // fill queue (FW)
  __shared__ uint32_t tmem_s;
  __shared__ int2 s_meta[NL][NT];   // (row, clamped length) of the lane's tile rows
  __shared__ int s_trip[NL][3];     // [lane]: tile trip, trip of rows 0-31, trip of rows 32-63
  __shared__ int s_tmax[NL][NT];    // the row's problem trip count (its output rows)
  __shared__ int4 s_fq[FW ? NL : 1][2][NT];   // fill queue entries (row, length, tmax)

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int L = warp < kRole0 ? (warp >> 2) : (warp < kFill ? warp - kRole0 : 0);
  const uint32_t q = cluster_ctarank(), odd = q & 1u, peer = q ^ 1u;
  const bool leader = odd == 0;
  const int C = a.C, H = a.H, T = a.T;
  const uint32_t xbytes = NH * a.Kx * 2, hbytes = NH * a.Kh * 2;
  constexpr uint32_t sbytes = NH * 32 * 2;   // one CTA's h slice of one 32-row half (2 KB)
  const uint32_t lane_bytes = xbytes + 2 * hbytes;
  uint8_t* sX = smem_raw + L * lane_bytes;   // [NH x Kx] fp16, core-matrix layout
  uint8_t* sH = sX + xbytes;                 // 2 x [NH x Kh] fp16
  constexpr uint32_t b_lbo = NH * 16, b_sbo = 128;
  constexpr uint32_t kWCol = 256;
  const uint16_t pair_mask = (uint16_t)(3u << (q & ~1u));
  uint16_t even_mask = 0;
  for (int i = 0; i < C; i += 2) even_mask |= (uint16_t)(1u << i);
  const uint16_t odd_mask = (uint16_t)(even_mask << 1);

  if (tid == 0) {
    for (int l = 0; l < NL; ++l) {
      mbar_init(&xfull[l], leader ? 2 : 1);      // own bulk load (+ the odd CTA's relay)
      mbar_init(&xempty[l], 1);
      mbar_init(&hfull[l][0], leader ? 2 : 1);   // own arm (+ relay)
      mbar_init(&hfull[l][1], leader ? 2 : 1);
      mbar_init(&mdone[l], 1);
      mbar_init(&dfree[l], 2 * EWL);             // epilogue warps of both CTAs (leader's copy is used)
      if (FW) {
        mbar_init(&fq_full[l][0], kEpiL);
        mbar_init(&fq_full[l][1], kEpiL);
        mbar_init(&fq_empty[l][0], 1);
        mbar_init(&fq_empty[l][1], 1);
      }
    }
    fence_mbar_init();
  }
  if (warp == kRole0) tmem_alloc_pair<512>(&tmem_s);
  for (uint32_t i = tid; i < NL * lane_bytes / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem_raw)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_s;
  if (warp < 4) {
    // TMEM lane l = 32w + 8g + u <- packed slab row 32g + 8w + u (gate g of unit 8w + u)
    const int srow = ((tid & 31) >> 3) * 32 + warp * 8 + (tid & 7);
    const uint32_t* src = reinterpret_cast<const uint32_t*>(a.wpack + ((size_t)q * 128 + srow) * a.K * 2);
    for (int c0 = 0; c0 < a.K / 2; c0 += 8) {
      uint32_t r[8];
      const uint4 lo = __ldg(reinterpret_cast<const uint4*>(src + c0));
      const uint4 hi = __ldg(reinterpret_cast<const uint4*>(src + c0 + 4));
      r[0] = lo.x; r[1] = lo.y; r[2] = lo.z; r[3] = lo.w; r[4] = hi.x; r[5] = hi.y; r[6] = hi.z; r[7] = hi.w;
      tmem_st8(tmem + ((uint32_t)(warp * 32) << 16) + kWCol + c0, r);
    }
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  cluster_sync();   // every CTA's barriers and TMEM are initialised before any remote traffic

  // epilogue thread: TMEM quarter qw, unit uc = 8qw + lane/4 of the CTA's slice,
  // tile rows 32h + 8j + 2(lane%4) + e  (h: D column half = destination parity)
  const int qw = warp & 3, cq = lane & 3, e = tid & (kEpiL - 1);
  const int uc = qw * 8 + (lane >> 2), unit = (int)q * 32 + uc;
  float kb0 = 0.f, kb1 = 0.f, kb2 = 0.f, kb3 = 0.f;
  if (warp < kRole0) {
    const float* bp = a.bpack + q * 128 + uc;
    kb0 = pact_kb<CELL, ACT, 0>(bp[0]);
    kb1 = pact_kb<CELL, ACT, 1>(bp[32]);
    kb2 = pact_kb<CELL, ACT, 2>(bp[64]);
    kb3 = pact_kb<CELL, ACT, 3>(bp[96]);
  }
  float hh[16], cc[16];
  const uint32_t tile_bar = 1 + L, xch_bar = 1 + NL + L;
  constexpr uint32_t kLaneThreads = kEpiL + 32;
  auto cell_row = [&](int ci) { return (ci >> 3) * 32 + ((ci >> 1) & 3) * 8 + 2 * cq + (ci & 1); };

  uint32_t step = 0;
  const int nclusters = (int)nclusters_x();
  const int stride = NL * nclusters;
  int2 m_meta = make_int2(-1, 0);
  int m_tmax = 0;
  auto tile_meta = [&](int tl) {
    m_meta = make_int2(-1, 0);
    m_tmax = 0;
    if (tl < a.ntiles) {
      const int r = a.perm[tl * NT + e];
      if (r >= 0) {
        m_tmax = max(0, min(a.pmax[r / a.Bp], T));
        m_meta = make_int2(r, (int)max(0LL, min((long long)a.lens[r], (long long)m_tmax)));
      }
    }
  };
  // tiles sorted longest first; round k hands out [k*stride, (k+1)*stride) in snake order
  const int pos = NL * (int)cluster_id_x() + L;
  auto tile_of = [&](int k) { return k * stride + ((k & 1) ? stride - 1 - pos : pos); };
  const int tile0 = tile_of(0);
  if (warp < kRole0 && e < NT) tile_meta(tile0);
  if (warp == kRole0 + L && lane == 0) {   // arm the h phases of steps 0 and 1
    mbar_arrive_expect_tx(&hfull[L][0], C * sbytes);
    mbar_arrive_expect_tx(&hfull[L][1], C * sbytes);
  }

  if (FW && warp == kFill) {
    // ======================= fill warp: frozen tails of every finished tile of the CTA
    int cnt[NL], done[NL];
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      const int pl = NL * (int)cluster_id_x() + l;
      cnt[l] = 0;
      done[l] = 0;
      for (int k = 0; k * stride < a.ntiles; ++k)
        if (k * stride + ((k & 1) ? stride - 1 - pl : pl) < a.ntiles) ++cnt[l];
    }
    const int sub = lane & 7, grp = lane >> 3;
    for (;;) {
      bool more = false, any = false;
#pragma unroll
      for (int l = 0; l < NL; ++l) {
        if (done[l] >= cnt[l]) continue;
        more = true;
        const int slot = done[l] & 1;
        const uint32_t ph = (done[l] >> 1) & 1;
        const bool ready = __shfl_sync(0xffffffffu, mbar_try_wait(&fq_full[l][slot], ph) ? 1 : 0, 0) != 0;
        if (!ready) continue;
        mbar_wait(&fq_full[l][slot], ph);   // complete: acquire for every lane
        for (int i = grp; i < NT; i += 4) {
          const int4 m = s_fq[FW ? l : 0][slot][i];
          if (m.x >= 0 && m.z > m.y) {
            const float4 v = *(reinterpret_cast<const float4*>(a.hT + (size_t)m.x * H + (int)q * 32) + sub);
            float4* o = reinterpret_cast<float4*>(a.out + (size_t)m.x * T * H + (int)q * 32) + sub;
            for (int t = m.y; t < m.z; ++t) __stcs(o + (size_t)t * (H / 4), v);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&fq_empty[l][slot]);
        ++done[l];
        any = true;
      }
      if (!more) break;
      if (!any) __nanosleep(256);
    }
  } else
  for (int round = 0, tile = tile0, ntl = 0; tile < a.ntiles || round * stride < a.ntiles; tile = tile_of(++round)) {
    if (tile >= a.ntiles) continue;   // a partial last round
    named_bar_sync(tile_bar, kLaneThreads);   // this lane's previous tile retired (s_meta rewritten)
    if (warp < kRole0 && e < NT) { s_meta[L][e] = m_meta; s_tmax[L][e] = m_tmax; }
    named_bar_sync(tile_bar, kLaneThreads);
    if (warp == kRole0 + L) {
      int ma = s_meta[L][lane].y, mb = s_meta[L][lane + 32].y;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        ma = max(ma, __shfl_xor_sync(0xffffffffu, ma, o));
        mb = max(mb, __shfl_xor_sync(0xffffffffu, mb, o));
      }
      if (lane == 0) { s_trip[L][0] = max(ma, mb); s_trip[L][1] = ma; s_trip[L][2] = mb; }
    }
    named_bar_sync(tile_bar, kLaneThreads);
    const int trip = s_trip[L][0];

    if (warp < kRole0) {
      // ======================= epilogue (lane L)
      if (e < NT) {   // next tile's metadata and its h0/c0 rows -> L2
        tile_meta(tile_of(round + 1));
        if (m_meta.x >= 0) {
          const char* h0n = reinterpret_cast<const char*>(a.h0 + (size_t)m_meta.x * H);
          const char* c0n = a.c0 ? reinterpret_cast<const char*>(a.c0 + (size_t)m_meta.x * H) : nullptr;
          for (int off = 0; off < H * 4; off += 128) {
            prefetch_l2(h0n + off);
            if (c0n) prefetch_l2(c0n + off);
          }
        }
      }
#pragma unroll
      for (int ci = 0; ci < 16; ++ci) {
        const int r = s_meta[L][cell_row(ci)].x;
        hh[ci] = r >= 0 ? __ldg(a.h0 + (size_t)r * H + unit) : 0.f;
        cc[ci] = (r >= 0 && a.c0) ? __ldg(a.c0 + (size_t)r * H + unit) : 0.f;
      }
      // lanes l and l^4 hold units u, u^1 of the same rows: after one shuffle the even-unit
      // lane holds (h_u, h_u+1) of row 2cq, the odd-unit lane those of row 2cq+1 (group k)
      const bool ueven = ((lane >> 2) & 1) == 0;
      const int ul = (lane >> 2) & ~1, er = ueven ? 0 : 1;
      auto unit_pair = [&](int k) {
        const int ci = (k >> 2) * 8 + (k & 3) * 2;
        const float send = ueven ? hh[ci + 1] : hh[ci];
        const float recv = __shfl_xor_sync(0xffffffffu, send, 4);
        return ueven ? make_float2(hh[ci], recv) : make_float2(recv, hh[ci + 1]);
      };
      // fp16 h slices for step u -> L2 -> multicast: rows 0-31 into sH[u&1] of the even
      // CTAs, rows 32-63 into the odd CTAs'
      auto send_h = [&](uint32_t u) {
        uint8_t* gs = a.hscratch + (((size_t)cluster_id_x() * NL + L) * 2 + (u & 1)) * (size_t)(NT * a.Kh * 2) +
                      (size_t)q * (2 * sbytes);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float2 p = unit_pair(k);
          const int nl = (k & 3) * 8 + 2 * cq + er;   // row within the half k >> 2
          *reinterpret_cast<__half2*>(gs + (k >> 2) * sbytes + qw * (NH * 16) + (nl >> 3) * 128 + (nl & 7) * 16 +
                                      ul * 2) = __floats2half2_rn(p.x, p.y);
        }
        fence_proxy_async_global();
        named_bar_sync(xch_bar, kEpiL);
        if (qw < 2 && lane == 0)
          bulk_g2s_multicast(sH + (u & 1) * hbytes + q * sbytes, gs + qw * sbytes, sbytes, &hfull[L][u & 1],
                             qw ? odd_mask : even_mask);
      };
      if (trip > 0) send_h(step);
      for (int t = 0; t < trip; ++t) {
        const uint32_t s = step + t;
        mbar_wait_sleep(&mdone[L], s & 1);
        if (e == 0 && L == 0) SKB_TRACE(s, 4);
        tc_fence_after();
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          float ga[16], gb[16];
          const uint32_t col = tmem + L * NT + half * 32;
          tmem_ld_16x256b_x4(col + ((uint32_t)(qw * 32) << 16), ga);
          tmem_ld_16x256b_x4(col + ((uint32_t)(qw * 32 + 16) << 16), gb);
          tmem_ld_wait();
          if (half == 1) {   // D fully read: the next step's x-part may overwrite it
            if (e == 0 && L == 0) SKB_TRACE(s, 10);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
              if (leader) mbar_arrive(&dfree[L]);
              else mbar_remote_arrive_relaxed(mapa(smem_u32(&dfree[L]), peer));   // no stores to publish
            }
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {   // cells ci, ci+1: same unit, tile rows r, r+1
            const int ci = half * 8 + j * 2;
            const bool live0 = t < s_meta[L][cell_row(ci)].y, live1 = t < s_meta[L][cell_row(ci + 1)].y;
            const float2 g0 = pact2<CELL, ACT, 0>(ga[4 * j], ga[4 * j + 1], kb0);
            const float2 g1 = pact2<CELL, ACT, 1>(ga[4 * j + 2], ga[4 * j + 3], kb1);
            const float2 g2 = pact2<CELL, ACT, 2>(gb[4 * j], gb[4 * j + 1], kb2);
            const float2 g3 = pact2<CELL, ACT, 3>(gb[4 * j + 2], gb[4 * j + 3], kb3);
            cell_update2<CELL, ACT>(g0, g1, g2, g3, cc[ci], cc[ci + 1], hh[ci], hh[ci + 1], live0, live1);
          }
        }
        if (e == 0 && L == 0) SKB_TRACE(s, 6);
        if (t + 1 < trip) {
          send_h(s + 1);
          if (e == 0 && L == 0) SKB_TRACE(s, 7);
        }
        if (e == 0 && L == 0) SKB_TRACE(s, 8);
        // output sequence [R, T, H] for t < the problem's trip count (frozen rows repeat h),
        // two units per store
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float2 p = unit_pair(k);
          const int n = (k >> 2) * 32 + (k & 3) * 8 + 2 * cq + er;
          const int r = s_meta[L][n].x;
          if (r >= 0 && t < (a.fill_inkernel ? s_tmax[L][n] : s_meta[L][n].y))
            *reinterpret_cast<float2*>(a.out + ((size_t)r * T + t) * H + (int)q * 32 + qw * 8 + ul) = p;
        }
        if (e == 0 && L == 0) SKB_TRACE(s, 9);
      }
      // frozen tails past the tile's trip count: out[r, t, :] = h_T for trip <= t < tmax
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float2 p = unit_pair(k);
        const int n = (k >> 2) * 32 + (k & 3) * 8 + 2 * cq + er;
        const int r = s_meta[L][n].x, tm = s_tmax[L][n];
        if (r >= 0 && a.fill_inkernel) {
          float* o = a.out + ((size_t)r * T) * H + (int)q * 32 + qw * 8 + ul;
          for (int t = trip; t < tm; ++t) *reinterpret_cast<float2*>(o + (size_t)t * H) = p;
        }
      }
#pragma unroll
      for (int ci = 0; ci < 16; ++ci) {
        const int r = s_meta[L][cell_row(ci)].x;
        if (r >= 0) {
          a.hT[(size_t)r * H + unit] = hh[ci];
          if (a.cT) a.cT[(size_t)r * H + unit] = cc[ci];
        }
      }
      if (a.tdone) {   // concurrent filler: this CTA's h_T slice of the tile is published
        __threadfence();
        named_bar_sync(xch_bar, kEpiL);
        if (e == 0) red_release_gpu_add(a.tdone + tile, 1);
      }
      if constexpr (FW != 0) {   // hand the tile's rows and final states to the fill warp
        const int slot = ntl & 1;
        mbar_wait_sleep(&fq_empty[L][slot], ((ntl >> 1) & 1) ^ 1);
        if (e < NT) s_fq[L][slot][e] = make_int4(s_meta[L][e].x, s_meta[L][e].y, s_tmax[L][e], 0);
        mbar_arrive(&fq_full[L][slot]);   // release: the h_T stores and the entries
      }
    } else {
      // ======================= role warp (lane L): x_t image loads (pre-pass images), MMA
      // issuer (even CTA) / relay (odd CTA)
      const int tself = s_trip[L][1 + odd];
      const uint8_t* img = a.ximg + ((size_t)tile * T * 2 + odd) * xbytes;   // [tile][t][half] images
      auto bulk_x = [&](int t, uint32_t u) {   // slot free: x-part(u-1) retired
        mbar_wait_sleep(&xempty[L], (u & 1) ^ 1);
        if (lane == 0) {
          if (t < tself) {
            if (a.xflag) {   // concurrent packer: image (tile, t) published?
              wait_flag(a.xflag + (size_t)tile * T + t, 1, a.err);
              fence_proxy_async_global();
            }
            mbar_arrive_expect_tx(&xfull[L], xbytes);
            bulk_g2s(sX, img + (size_t)t * 2 * xbytes, xbytes, &xfull[L]);
            // the image two steps ahead -> L2 (an HBM miss here delays x-part(t+1) and with it
            // the h-part queued behind it: measured 1.2 vs 2.5 ms per launch)
            if (t + 2 < tself) bulk_prefetch_l2(img + (size_t)(t + 2) * 2 * xbytes, xbytes);
          } else {
            mbar_arrive(&xfull[L]);   // every row of this half is past its length: stale (finite) image
          }
        }
        __syncwarp();
      };
      if (leader) {
        const uint32_t idesc = idesc_f16_f32(256, NT);
        const int kx_steps = a.Kx / 16, kh_steps = a.Kh / 16;
        const uint64_t xdesc0 = sdesc_kmajor_noswz(smem_u32(sX), b_lbo, b_sbo);
        const uint32_t d = tmem + L * NT;
        auto x_part = [&](uint32_t s) {
          mbar_wait_sleep(&xfull[L], s & 1);
          if (lane == 0 && L == 0) SKB_TRACE(s, 0);
          mbar_wait_sleep(&dfree[L], (s & 1) ^ 1);
          if (lane == 0 && L == 0) SKB_TRACE(s, 1);
          tc_fence_after();
#pragma unroll 4
          for (int ks = 0; ks < kx_steps; ++ks)
            umma_f16_ts_pair_warp(d, tmem + kWCol + ks * 8, xdesc0 + (uint64_t)(ks * 2 * b_lbo >> 4), idesc,
                                  ks > 0 ? 1u : 0u);
          umma_commit_pair_warp(&xempty[L], pair_mask);
        };
        if (trip > 0) {
          if (tself > 1 && lane == 0) bulk_prefetch_l2(img + (size_t)2 * xbytes, xbytes);
          bulk_x(0, step);
          x_part(step);
        }
        for (int t = 0; t < trip; ++t) {
          const uint32_t s = step + t, j = s & 1;
          mbar_wait_sleep(&hfull[L][j], (s >> 1) & 1);
          if (lane == 0 && L == 0) SKB_TRACE(s, 2);
          if (lane == 0) mbar_arrive_expect_tx(&hfull[L][j], C * sbytes);   // arm step s+2
          tc_fence_after();
          const uint64_t hdesc0 = sdesc_kmajor_noswz(smem_u32(sH + j * hbytes), b_lbo, b_sbo);
#pragma unroll 4
          for (int ks = 0; ks < kh_steps; ++ks)
            umma_f16_ts_pair_warp(d, tmem + kWCol + (kx_steps + ks) * 8, hdesc0 + (uint64_t)(ks * 2 * b_lbo >> 4),
                                  idesc, 1u);
          umma_commit_pair_warp(&mdone[L], pair_mask);
          if (lane == 0 && L == 0) SKB_TRACE(s, 3);
          if (t + 1 < trip) {
            bulk_x(t + 1, s + 1);
            x_part(s + 1);
          }
        }
      } else {
        const uint32_t rx = mapa(smem_u32(&xfull[L]), peer);
        auto relay_x = [&](int t, uint32_t s) {
          bulk_x(t, s);
          mbar_wait_sleep(&xfull[L], s & 1);
          if (lane == 0) mbar_remote_arrive(rx);
        };
        if (trip > 0) relay_x(0, step);
        for (int t = 0; t < trip; ++t) {
          const uint32_t s = step + t, j = s & 1;
          mbar_wait_sleep(&hfull[L][j], (s >> 1) & 1);
          if (lane == 0) {
            mbar_arrive_expect_tx(&hfull[L][j], C * sbytes);   // arm step s+2
            mbar_remote_arrive(mapa(smem_u32(&hfull[L][j]), peer));
          }
          if (t + 1 < trip) relay_x(t + 1, s + 1);
        }
      }
    }
    __syncwarp();
    step += trip;
    ++ntl;
  }

  // Drain the asynchronous arrivals aimed at this CTA before it exits: the last
  // x-part's retire (xempty, both CTAs) and the peer's last D release (dfree, leader).
  if (step > 0 && lane == 0 && warp == kRole0 + L) {
    mbar_wait_sleep(&xempty[L], (step - 1) & 1);
    if (leader) mbar_wait_sleep(&dfree[L], (step - 1) & 1);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == kRole0) tmem_dealloc_pair<512>(tmem);
}

// ------------------------------------------------------------------ ping-pong LSTM kernel
// The rows of a 64-row tile form two independent 32-row recurrences (halves).
// The MMA warp alternates halves: while half A's epilogue (warps 0-7) turns
// its gates into h_t and exchanges it, half B's h-part MMA (N = 32) runs on
// the tensor pipe, and vice versa — the serial MMA -> epilogue -> exchange
// chain of one recurrence overlaps the other's.  Each half has its own TMEM
// accumulators, mbarriers, named barriers and contiguous h exchange buffers
// (core-matrix layout with LBO = 32*16 B); the x image is shared.
template <typename XT, int ACT = 0>
__global__ void __launch_bounds__(16 * 32 + 64, 1) rnn_fwd_pp_kernel(const RnnArgs a) {
  constexpr int NT = 64, NH = NT / 2, EW = 16, kEpi = EW * 32, kThreads = kEpi + 64, UG = 4;   // NT == kNT
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ uint64_t xfull[2], xempty[2], hfull[2][2], mdone[2][2], dfree[2][2];
  __shared__ uint32_t tmem_s;
  __shared__ int s_row[NT], s_len[NT], s_tmax[NT];
  __shared__ int s_trip;

  uint8_t* smem = smem_raw;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t q = cluster_ctarank();
  const int C = a.C, U = a.U, H = a.H, T = a.T;
  const uint32_t xbytes = NT * a.Kx * 2, hbytes = NT * a.Kh * 2, hhalf = hbytes / 2, shalf = NH * U * 2;
  uint8_t* sX = smem;
  uint8_t* sH = sX + 2 * xbytes;     // [buf][half][NH x Kh] fp16, LBO = NH*16
  float* sG = reinterpret_cast<float*>(sH + 2 * hbytes);
  constexpr uint32_t x_lbo = NT * 16, h_lbo = NH * 16, c_sbo = 128;
  constexpr uint32_t kWCol = 256;

  if (tid == 0) {
    for (int j = 0; j < 2; ++j) {
      mbar_init(&xfull[j], 1);
      mbar_init(&xempty[j], 1);
      for (int h = 0; h < 2; ++h) {
        mbar_init(&hfull[h][j], 1);
        mbar_init(&mdone[h][j], 1);
        mbar_init(&dfree[h][j], 8);
      }
    }
    fence_mbar_init();
  }
  if (warp == EW + 1) tmem_alloc<512>(&tmem_s);
  for (uint32_t i = tid; i < (2 * xbytes + 2 * hbytes) / 16; i += kThreads)
    reinterpret_cast<uint4*>(sX)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_s;
  float bias = 0.f;
  if (warp < 4) {
    const uint32_t* src = reinterpret_cast<const uint32_t*>(a.wpack + ((size_t)q * 128 + tid) * a.K * 2);
    for (int c0 = 0; c0 < a.K / 2; c0 += 8) {
      uint32_t r[8];
      const uint4 lo = __ldg(reinterpret_cast<const uint4*>(src + c0));
      const uint4 hi = __ldg(reinterpret_cast<const uint4*>(src + c0 + 4));
      r[0] = lo.x; r[1] = lo.y; r[2] = lo.z; r[3] = lo.w; r[4] = hi.x; r[5] = hi.y; r[6] = hi.z; r[7] = hi.w;
      tmem_st8(tmem + ((uint32_t)(warp * 32) << 16) + kWCol + c0, r);
    }
    tmem_st_wait();
  }
  if (warp < EW) bias = a.bpack[q * 128 + (warp & 3) * 32 + lane];
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  cluster_sync();

  // epilogue group hw = warp >> 3 owns rows [hw*NH, hw*NH + NH); within it warp
  // wl reads TMEM lane quarter qw = wl & 3 and columns ch*16.. of the half;
  // in the cell phase thread gt owns row nl = gt / G4 and units pu..pu+3.
  const int hw = warp >> 3, wl = warp & 7, qw = wl & 3, ch = wl >> 2, gt = tid & 255;
  const int G4 = U / UG;
  const int nl = G4 ? gt / G4 : 0, pu = G4 ? (gt % G4) * UG : 0;
  const bool pv = warp < EW && G4 && nl < NH;
  const int nrow = hw * NH + nl;
  float hp[UG], cc[UG];
  uint8_t* gscr = a.hscratch + (size_t)cluster_id_x() * 2 * hbytes;

  uint32_t step = 0;
  uint32_t hwait[2][2] = {{0u, 0u}, {0u, 0u}};
  bool hfull_armed = false;
  const int nclusters = (int)nclusters_x();
  for (int tile = (int)cluster_id_x(); tile < a.ntiles; tile += nclusters) {
    cluster_sync();
    if (tid < NT) {
      const int r = a.perm[tile * NT + tid];
      int len = 0, tmax = 0;
      if (r >= 0) {
        tmax = max(0, min(a.pmax[r / a.Bp], T));
        const long long L = a.lens[r];
        len = (int)max(0LL, min(L, (long long)tmax));
      }
      s_row[tid] = r; s_len[tid] = len; s_tmax[tid] = tmax;
    }
    __syncthreads();
    if (tid == 0) {
      int m = 0;
      for (int i = 0; i < NT; ++i) m = max(m, s_len[i]);
      s_trip = m;
    }
    {  // h0 -> hbuf[step&1] (both halves)
      uint8_t* hb = sH + (step & 1) * hbytes;
      const int kch = a.Kh / 8;
      for (int i = tid; i < NT * kch; i += kThreads) {
        const int n = i / kch, kc = i - n * kch;
        const int r = s_row[n];
        float v[8];
        if (r >= 0) load_x8<float>(a.h0 + (size_t)r * H, kc * 8, H, v);
        else {
#pragma unroll
          for (int e = 0; e < 8; ++e) v[e] = 0.f;
        }
        uint32_t w[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          __half2 h2 = __floats2half2_rn(v[2 * e], v[2 * e + 1]);
          w[e] = *reinterpret_cast<uint32_t*>(&h2);
        }
        *reinterpret_cast<uint4*>(hb + (n / NH) * hhalf + cm_offset(n % NH, kc * 8, h_lbo, c_sbo)) =
            make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
    fence_proxy_async_smem();
    __syncthreads();
    const int trip = s_trip;

    if (warp < EW) {
      // ======================= epilogue (half hw) =======================
      {
        const int r = pv ? s_row[nrow] : -1;
        float hv[8], cv[8];
        if (r >= 0) {
          load_x8<float>(a.h0 + (size_t)r * H, (int)q * U + pu, H, hv);
          load_x8<float>(a.c0 + (size_t)r * H, (int)q * U + pu, H, cv);
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e) hv[e] = cv[e] = 0.f;
        }
#pragma unroll
        for (int e = 0; e < UG; ++e) { hp[e] = hv[e]; cc[e] = cv[e]; }
      }
      float kl, kb, mul, add;
      gate_consts<ACT>(qw, bias, kl, kb, mul, add);
      const uint32_t bar_g = 1 + 2 * hw, bar_x = 2 + 2 * hw;   // named barriers of this half
      for (int t = 0; t < trip; ++t) {
        const uint32_t s = step + t, j = s & 1, use = s >> 1;
        const uint32_t nb = (s + 1) & 1;
        uint8_t* gslice = gscr + nb * hbytes + hw * hhalf + q * shalf;
        mbar_wait(&mdone[hw][j], use & 1);
        tc_fence_after();
        const uint32_t trow = tmem + ((uint32_t)(qw * 32) << 16) + j * 2 * NT + hw * NH + ch * 16;
        float* g_out = sG + (qw * NT + hw * NH + ch * 16) * kGS + lane;
        {
          float v[16];
          tmem_ld16(trow, v);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) g_out[i * kGS] = gate_act<ACT>(v[i], kl, kb, mul, add);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&dfree[hw][j]);
        named_bar_sync(bar_g, 256);
        if (pv) {
          float g4[4][UG];
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            const float4 x0 = *reinterpret_cast<const float4*>(sG + (g * NT + nrow) * kGS + pu);
            g4[g][0] = x0.x; g4[g][1] = x0.y; g4[g][2] = x0.z; g4[g][3] = x0.w;
          }
          const bool live = t < s_len[nrow];
#pragma unroll
          for (int e = 0; e < UG; ++e) {
            const float c2 = fmaf(g4[1][e], cc[e], g4[0][e] * g4[2][e]);
            const float h2 = g4[3][e] * cell_tanh<ACT>(c2);
            cc[e] = live ? c2 : cc[e];
            hp[e] = live ? h2 : hp[e];
          }
          if (t + 1 < trip) {
            __half2 h01 = __floats2half2_rn(hp[0], hp[1]), h23 = __floats2half2_rn(hp[2], hp[3]);
            *reinterpret_cast<uint2*>(gslice + cm_offset(nl, pu, h_lbo, c_sbo)) =
                make_uint2(*reinterpret_cast<uint32_t*>(&h01), *reinterpret_cast<uint32_t*>(&h23));
          }
        }
        fence_proxy_async_global();
        named_bar_sync(bar_x, 256);   // also: sG rows of this half are rewritten only after every read
        if (t + 1 < trip && gt == 0)
          bulk_g2s_multicast(sH + nb * hbytes + hw * hhalf + q * shalf, gslice, shalf, &hfull[hw][nb],
                             (uint16_t)((1u << C) - 1));
        if (pv) {   // output sequence [R, T, H] (live steps; the frozen tail is filled later)
          const int r = s_row[nrow];
          if (r >= 0 && t < s_len[nrow]) {
            const int unit0 = (int)q * U + pu;
            float* o = a.out + ((size_t)r * T + t) * H + unit0;
            if (unit0 + UG <= H && (H & 3) == 0) {
              *reinterpret_cast<float4*>(o) = make_float4(hp[0], hp[1], hp[2], hp[3]);
            } else {
#pragma unroll
              for (int e = 0; e < UG; ++e) if (unit0 + e < H) o[e] = hp[e];
            }
          }
        }
      }
      if (pv) {
        const int r = s_row[nrow];
        if (r >= 0) {
#pragma unroll
          for (int e = 0; e < UG; ++e) {
            const int unit = (int)q * U + pu + e;
            if (unit >= H) continue;
            a.hT[(size_t)r * H + unit] = hp[e];
            if (a.cT) a.cT[(size_t)r * H + unit] = cc[e];
          }
        }
      }
    } else if (warp == EW) {
      // ======================= x_t loader =======================
      if (lane == 0) {
        const uint8_t* img = a.ximg + (size_t)tile * T * xbytes;
        for (int t = 0; t < trip; ++t) {
          const uint32_t s = step + t, j = s & 1, use = s >> 1;
          mbar_wait(&xempty[j], (use & 1) ^ 1);
          mbar_arrive_expect_tx(&xfull[j], xbytes);
          for (uint32_t off = 0; off < xbytes; off += 16384)
            bulk_g2s(sX + j * xbytes + off, img + (size_t)t * xbytes + off, min(16384u, xbytes - off), &xfull[j]);
        }
      }
    } else {
      // ======================= MMA issuer (both halves) =======================
      const uint32_t idesc = idesc_f16_f32(128, NH);
      const uint32_t x_addr = smem_u32(sX), h_addr = smem_u32(sH);
      const int kx_steps = a.Kx / 16, kh_steps = a.Kh / 16;
      if (!hfull_armed) {
        if (lane == 0)
          for (int h = 0; h < 2; ++h)
            for (int b = 0; b < 2; ++b) mbar_arrive_expect_tx(&hfull[h][b], C * shalf);
        hfull_armed = true;
      }
      for (int t = 0; t < trip; ++t) {
        const uint32_t s = step + t, j = s & 1, use = s >> 1;
        mbar_wait(&xfull[j], use & 1);
        for (int h = 0; h < 2; ++h) {   // x parts (independent of the recurrence)
          mbar_wait(&dfree[h][j], (use & 1) ^ 1);
          tc_fence_after();
          const uint32_t d = tmem + j * 2 * NT + h * NH;
          const uint64_t xdesc0 = sdesc_kmajor_noswz(x_addr + j * xbytes + h * (NH / 8) * c_sbo, x_lbo, c_sbo);
#pragma unroll 4
          for (int ks = 0; ks < kx_steps; ++ks)
            umma_f16_ts_warp(d, tmem + kWCol + ks * 8, xdesc0 + (uint64_t)(ks * 2 * x_lbo >> 4), idesc,
                             ks > 0 ? 1u : 0u);
        }
        umma_commit_warp(&xempty[j]);
        for (int h = 0; h < 2; ++h) {   // h parts: each waits for its own half's exchange
          if (t > 0) {
            const uint32_t hb = s & 1;
            mbar_wait(&hfull[h][hb], hwait[h][hb] & 1);
            ++hwait[h][hb];
            if (lane == 0) mbar_arrive_expect_tx(&hfull[h][hb], C * shalf);
          }
          tc_fence_after();
          const uint32_t d = tmem + j * 2 * NT + h * NH;
          const uint64_t hdesc0 = sdesc_kmajor_noswz(h_addr + (s & 1) * hbytes + h * hhalf, h_lbo, c_sbo);
#pragma unroll 4
          for (int ks = 0; ks < kh_steps; ++ks)
            umma_f16_ts_warp(d, tmem + kWCol + (kx_steps + ks) * 8, hdesc0 + (uint64_t)(ks * 2 * h_lbo >> 4),
                             idesc, 1u);
          umma_commit_warp(&mdone[h][j]);
        }
      }
    }
    __syncwarp();
    step += trip;
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == EW + 1) tmem_dealloc<512>(tmem);
}

// ------------------------------------------------------------------ packing
struct PackArgs {
  const void* w[4];
  const void* u[4];
  const void* b[4];
  int f64;
  uint8_t* slab;
  float* bias;
  int32_t* err;
  int G, H, F, U, C, Kx, Kh, K;
};

SKB_DEV float ld_any(const void* p, size_t i, int f64) {
  return f64 ? (float)reinterpret_cast<const double*>(p)[i] : reinterpret_cast<const float*>(p)[i];
}

__global__ void rnn_pack_kernel(const PackArgs a) {
  const int kchunks = a.K / 8;
  const long long total = (long long)a.C * 128 * kchunks;
  bool bad = false;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int q = (int)(idx / (128 * kchunks));
    const int rem = (int)(idx - (long long)q * 128 * kchunks);
    const int row = rem % 128, kc = rem / 128;
    int g, ul;
    if (a.G == 4) { g = row >> 5; ul = row & 31; } else { g = 0; ul = row; }
    const int unit = q * a.U + ul;
    const bool valid = (ul < a.U) && (unit < a.H) && (g < a.G);
    __half hv[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int k = kc * 8 + e;
      float v = 0.f;
      if (valid) {
        if (k < a.F) v = a.w[g] ? ld_any(a.w[g], (size_t)k * a.H + unit, a.f64) : 0.f;   // NULL block: zeros (GRU n_h)
        else if (k >= a.Kx && k - a.Kx < a.H)
          v = a.u[g] ? ld_any(a.u[g], (size_t)(k - a.Kx) * a.H + unit, a.f64) : 0.f;   // (GRU n_x)
      }
      bad |= fp16_overflow(v);
      hv[e] = __float2half_rn(v);
    }
    // row-major [128][K] fp16 slab per CTA (copied into TMEM at kernel start)
    uint8_t* dst = a.slab + ((size_t)q * 128 + row) * a.K * 2 + kc * 16;
    *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<uint4*>(hv);
    if (kc == 0) a.bias[q * 128 + row] = valid ? ld_any(a.b[g], unit, a.f64) : 0.f;
  }
  if (bad) set_err(a.err, SKB_ERR_FP16_RANGE, -1, -1);
}

// ------------------------------------------------------------------ row schedule
// Per-problem max_len (= the While trip count, reference tensor.py:344-353),
// the reference's runtime errors for it, and a counting sort of rows by
// length (descending) so each tile's trip count is as short as possible.
struct SchedArgs {
  const int64_t* lens;
  int32_t* perm;      // [ntiles*NT]
  int32_t* pmax;      // [P]
  int32_t* hist;      // [T+1]
  int32_t* base;      // [T+1]
  int32_t* cursor;    // [T+1]
  int32_t* max_len_out;
  int32_t* err;
  int32_t* xflag;     // [nflags] concurrent-packer image flags, cleared here
  int32_t* tdone;     // [ntdone] concurrent-filler tile counters, cleared here
  int R, Bp, P, T, npad, nflags, ntdone;
};

__global__ void sched_init(const SchedArgs a) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int stride = gridDim.x * blockDim.x;
  for (int p = i; p < a.P; p += stride) a.pmax[p] = INT_MIN;
  for (int b = i; b <= a.T; b += stride) { a.hist[b] = 0; a.cursor[b] = 0; }
  for (int r = a.R + i; r < a.npad; r += stride) a.perm[r] = -1;
  for (int f = i; f < a.nflags; f += stride) a.xflag[f] = 0;
  for (int f = i; f < a.ntdone; f += stride) a.tdone[f] = 0;
}

SKB_DEV int len_bin(long long L, int T) { return (int)max(0LL, min(L, (long long)T)); }

__global__ void sched_hist(const SchedArgs a) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < a.R; r += gridDim.x * blockDim.x) {
    const long long L = a.lens[r];
    const int Lc = (int)max((long long)INT_MIN, min(L, (long long)INT_MAX));
    atomicMax(&a.pmax[r / a.Bp], Lc);
    atomicAdd(&a.hist[len_bin(L, a.T)], 1);
  }
}

__global__ void sched_scan(const SchedArgs a) {
  // base[b] = number of rows with bin > b  (descending order), single block
  __shared__ int part[1024];
  const int nb = a.T + 1;
  const int per = (nb + blockDim.x - 1) / blockDim.x;
  const int tid = threadIdx.x;
  // thread tid owns bins counted from the top: j = tid*per .. ; bin = T - j
  int s = 0;
  for (int j = tid * per; j < min(nb, (tid + 1) * per); ++j) s += a.hist[a.T - j];
  part[tid] = s;
  __syncthreads();
  for (int off = 1; off < (int)blockDim.x; off <<= 1) {
    const int v = tid >= off ? part[tid - off] : 0;
    __syncthreads();
    part[tid] += v;
    __syncthreads();
  }
  int run = tid > 0 ? part[tid - 1] : 0;
  for (int j = tid * per; j < min(nb, (tid + 1) * per); ++j) {
    a.base[a.T - j] = run;
    run += a.hist[a.T - j];
  }
  // per-problem checks, in the reference's evaluation order:
  //   Range(max_len) with max_len < 0 -> ShapeMismatch      (tensor.py:414-417)
  //   Index(x_tm, t) with t >= T      -> IndexOutOfRange    (tensor.py:420-430)
  //   ListStack of an empty list      -> EmptyPop           (execute.py:171-174)
  // The smallest failing problem index is reported.
  __shared__ int first_bad;
  if (tid == 0) first_bad = INT_MAX;
  __syncthreads();
  for (int p = tid; p < a.P; p += blockDim.x) {
    const int m = a.pmax[p];
    a.max_len_out[p] = m;
    if (m < 0 || m > a.T || m == 0) atomicMin(&first_bad, p);
  }
  __syncthreads();
  if (tid == 0 && first_bad != INT_MAX) {
    const int m = a.pmax[first_bad];
    const int code = m < 0 ? SKB_ERR_SHAPE_MISMATCH : (m > a.T ? SKB_ERR_INDEX_OUT_OF_RANGE : SKB_ERR_EMPTY_POP);
    if (atomicCAS(a.err, 0, code) == 0) { a.err[1] = first_bad; a.err[2] = m > a.T ? a.T : 0; a.err[3] = m; }
  }
}

__global__ void sched_scatter(const SchedArgs a) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < a.R; r += gridDim.x * blockDim.x) {
    const int b = len_bin(a.lens[r], a.T);
    a.perm[a.base[b] + atomicAdd(&a.cursor[b], 1)] = r;
  }
}

constexpr int kNT = 64;

// Pre-pass: gather each tile's rows (sorted order) and convert x[r, t, :] to the
// fp16 core-matrix image the recurrent kernel's MMA consumes, one image per
// (tile, t < tile trip count).  Rows past their length are zero.
template <typename XT>
__global__ void __launch_bounds__(256) pack_x_kernel(const XT* __restrict__ x, const int32_t* __restrict__ perm,
                              const int64_t* __restrict__ lens, const int32_t* __restrict__ pmax,
                              uint8_t* __restrict__ img, int32_t* err, int ntiles, int T, int F,
                              int Kx, int Bp, int halves) {
  // One block per (tile, t) image; item = (n, kc) with n fastest, so a warp reads
  // 32 rows x 32 B sectors and writes 512 contiguous bytes of image.  Row-steps
  // past the row's length are skipped (their MMA columns are masked).
  const int tile = blockIdx.x, t = blockIdx.y;
  const int r0 = perm[tile * kNT];
  if (r0 < 0) return;
  const int tm0 = min(max(pmax[r0 / Bp], 0), T);
  const long long L0 = lens[r0];
  if (t >= (L0 < tm0 ? L0 : tm0)) return;
  const int items = kNT * (Kx / 8);
  const uint32_t xbytes = kNT * Kx * 2;
  uint8_t* dst0 = img + ((size_t)tile * T + t) * xbytes;
  bool bad = false;
  constexpr int kB = 8;
  for (int i0 = threadIdx.x; i0 < items; i0 += 256 * kB) {
    float v[kB][8];
    bool ok[kB];
#pragma unroll
    for (int m = 0; m < kB; ++m) {
      const int i = i0 + m * 256;
      const int n = i % kNT, kc = i / kNT;
      ok[m] = false;
      if (i < items) {
        const int r = perm[tile * kNT + n];
        if (r >= 0 && t < lens[r]) {
          load_x8<XT>(x + ((size_t)r * T + t) * F, kc * 8, F, v[m]);
          ok[m] = true;
        }
      }
    }
#pragma unroll
    for (int m = 0; m < kB; ++m) {
      if (!ok[m]) continue;
      const int i = i0 + m * 256;
      const int n = i % kNT, kc = i / kNT;
      uint32_t w[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        bad |= fp16_overflow(v[m][2 * e]) || fp16_overflow(v[m][2 * e + 1]);
        __half2 h2 = __floats2half2_rn(v[m][2 * e], v[m][2 * e + 1]);
        w[e] = *reinterpret_cast<uint32_t*>(&h2);
      }
      const uint32_t off = halves ? (n >> 5) * (32 * Kx * 2) + cm_offset(n & 31, kc * 8, 32 * 16, 128)
                                  : cm_offset(n, kc * 8, kNT * 16, 128);
      *reinterpret_cast<uint4*>(dst0 + off) = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
  if (bad) set_err(err, SKB_ERR_FP16_RANGE, -1, -1);
}

// Coalesced variant for fp32 x with F % 128 == 0 (the C1 shape): one block per
// (tile, t) image.  Each warp reads whole 4*F-byte rows (lane k*4.., fully
// coalesced), converts to fp16 into a padded row-major shared tile, then all
// threads write the image in core-matrix order ([Kx/8][64 rows][8] halves) as
// contiguous 16-byte stores.  Rows past their length are written as zeros.
// One (tile, t) image; false (nothing written) when t is past the tile's trip count.
template <int NQ>
SKB_DEV bool pack_rows_item(const float* __restrict__ x, const int32_t* __restrict__ perm,
                            const int64_t* __restrict__ lens, const int32_t* __restrict__ pmax,
                            uint8_t* __restrict__ img, int32_t* err, int T, int Bp, int halves, int tile, int t,
                            uint8_t* srow) {
  constexpr int F = NQ * 128, kRow = F * 2 + 16;   // padded fp16 row: 16-byte reads of 8 lanes hit distinct banks
  const int r0 = perm[tile * kNT];
  if (r0 < 0) return false;
  const int tm0 = min(max(pmax[r0 / Bp], 0), T);
  const long long L0 = lens[r0];
  if (t >= (L0 < tm0 ? L0 : tm0)) return false;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  bool bad = false;
  float4 v[8][NQ];
  bool on[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int n = warp * 8 + i;
    const int r = perm[tile * kNT + n];
    on[i] = r >= 0 && t < lens[r];
    const float4* row = reinterpret_cast<const float4*>(x + ((size_t)(on[i] ? r : 0) * T + t) * F);
#pragma unroll
    for (int q = 0; q < NQ; ++q) v[i][q] = on[i] ? __ldcs(row + q * 32 + lane) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    uint8_t* dst = srow + (warp * 8 + i) * kRow;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const float4 a = v[i][q];
      bad |= fp16_overflow(a.x) || fp16_overflow(a.y) || fp16_overflow(a.z) || fp16_overflow(a.w);
      __half2 lo = __floats2half2_rn(a.x, a.y), hi = __floats2half2_rn(a.z, a.w);
      *reinterpret_cast<uint2*>(dst + (q * 128 + lane * 4) * 2) =
          make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
    }
  }
  __syncthreads();
  constexpr int kChunks = kNT * F / 8;   // 16-byte chunks of the image, row fastest
  uint4* out = reinterpret_cast<uint4*>(img + ((size_t)tile * T + t) * (kNT * F * 2));
#pragma unroll 4
  for (int o = threadIdx.x; o < kChunks; o += 256) {
    const int n = o % kNT, kc = o / kNT;
    out[halves ? (n >> 5) * (32 * F / 8) + kc * 32 + (n & 31) : o] =
        *reinterpret_cast<const uint4*>(srow + n * kRow + kc * 16);
  }
  if (bad) set_err(err, SKB_ERR_FP16_RANGE, -1, -1);
  return true;
}

template <int NQ>
__global__ void __launch_bounds__(256) pack_x_rows_kernel(const float* __restrict__ x, const int32_t* __restrict__ perm,
                                   const int64_t* __restrict__ lens, const int32_t* __restrict__ pmax,
                                   uint8_t* __restrict__ img, int32_t* err, int T, int Bp, int halves) {
  extern __shared__ __align__(16) uint8_t srow[];
  pack_rows_item<NQ>(x, perm, lens, pmax, img, err, T, Bp, halves, blockIdx.x, blockIdx.y, srow);
}

// Concurrent auxiliary grid of the pair4 kernel (default for fp32 x rows): a small
// persistent grid on the SMs the recurrent kernel's 8-CTA clusters leave idle.
//  1. packer: the x images, in the order the lanes consume them (round k of the
//     snake-order tile assignment, then t, then lane position); each (tile, t) image
//     is published with a gpu-scope release of its flag.  Never waits.
//  2. filler: the frozen tails out[r, len <= t < tmax, :] = h_T of each tile, as soon as
//     all C CTAs of the tile's cluster have published their h_T slices (tdone).
// Both flag arrays are cleared by sched_init.  Launched after the recurrent kernel on a
// lower-priority stream, preloaded (no lazy-loading stall while the recurrence waits).
struct AuxArgs {
  const float* x;
  const int32_t* perm;
  const int64_t* lens;
  const int32_t* pmax;
  uint8_t* img;
  int32_t* err;
  int32_t* xflag;        // null: no packing phase
  const int32_t* tdone;  // null: no filling phase
  float* out;
  const float* hT;
  int ntiles, T, H, Bp, stride, C;
};

template <int NQ>
__global__ void __launch_bounds__(256) rnn_aux_kernel(const AuxArgs a) {
  extern __shared__ __align__(16) uint8_t srow[];
  __shared__ int s_ok;
  const int rounds = (a.ntiles + a.stride - 1) / a.stride;
  if (a.xflag) {
    const long long items = (long long)rounds * a.T * a.stride;
    for (long long i = blockIdx.x; i < items; i += gridDim.x) {
      const int pos = (int)(i % a.stride);
      const long long kt = i / a.stride;
      const int t = (int)(kt % a.T), k = (int)(kt / a.T);
      const int tile = k * a.stride + ((k & 1) ? a.stride - 1 - pos : pos);
      if (tile >= a.ntiles) continue;
      if (!pack_rows_item<NQ>(a.x, a.perm, a.lens, a.pmax, a.img, a.err, a.T, a.Bp, 1, tile, t, srow)) continue;
      fence_proxy_async_global();   // the image is read by the consumer's bulk copies
      __syncthreads();              // every thread's image stores (and srow reads) are done
      if (threadIdx.x == 0) {
        __threadfence();
        st_release_gpu(a.xflag + (size_t)tile * a.T + t, 1);
      }
    }
  }
  if (a.tdone) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, H4 = a.H / 4;
    for (int j = blockIdx.x; j < rounds * a.stride; j += gridDim.x) {
      const int k = j / a.stride, pos = j % a.stride;
      const int tile = k * a.stride + ((k & 1) ? a.stride - 1 - pos : pos);
      if (tile >= a.ntiles) continue;
      __syncthreads();
      if (threadIdx.x == 0) s_ok = wait_flag(a.tdone + tile, a.C, a.err) ? 1 : 0;
      __syncthreads();
      if (!s_ok) return;
      for (int n = warp; n < kNT; n += 8) {
        const int r = a.perm[tile * kNT + n];
        if (r < 0) continue;
        const int tmax = min(max(a.pmax[r / a.Bp], 0), a.T);
        const long long L = a.lens[r];
        const int len = (int)(L < 0 ? 0 : (L < tmax ? L : tmax));
        if (len >= tmax) continue;
        float4* orow = reinterpret_cast<float4*>(a.out + (size_t)r * a.T * a.H);
        const float4* hrow = reinterpret_cast<const float4*>(a.hT + (size_t)r * a.H);
        for (int c = lane; c < H4; c += 32) {
          const float4 v = __ldcg(hrow + c);
          for (int t = len; t < tmax; ++t) __stcs(orow + (size_t)t * H4 + c, v);
        }
      }
    }
  }
}

struct Workspace {
  int32_t *perm, *pmax, *hist, *base, *cursor, *xflag, *tdone;
  uint8_t* hscratch;
  uint8_t* ximg;
  float* hT;
};

inline int max_clusters_bound(const RnnGeom& g) {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms / g.C + 1;
}

// 64-row x-image tiles, padded to an even count (the pair kernel's 128-row tiles)
inline int n_tiles64(const RnnGeom& g) { return round_up((g.R + kNT - 1) / kNT, 2); }

inline int64_t ws_layout(const RnnGeom& g, uint8_t* basep, Workspace* w) {
  const int ntiles = n_tiles64(g);
  int64_t off = 0;
  auto take = [&](int64_t n) { int64_t o = off; off += (n * 4 + 255) / 256 * 256; return o; };
  int64_t o_perm = take((int64_t)ntiles * kNT), o_pmax = take(g.P), o_hist = take(g.T + 1),
          o_base = take(g.T + 1), o_cur = take(g.T + 1);
  // h_t exchange scratch (int32 units for take()): per cluster 2 x [64 x Kh] fp16 (dual-lane
  // kernel) or 2 lanes x 2 step parities x [128 x Kh] fp16 (pair kernel)
  int64_t o_hs = take((int64_t)max_clusters_bound(g) * 4 * 2 * kNT * g.Kh * 2 / 4);
  int64_t o_x = take((int64_t)ntiles * g.T * kNT * g.Kx * 2 / 4);
  int64_t o_hT = take((int64_t)g.R * g.H);
  int64_t o_fl = take((int64_t)ntiles * g.T);
  int64_t o_td = take((int64_t)ntiles);
  if (w) {
    w->xflag = reinterpret_cast<int32_t*>(basep + o_fl);
    w->tdone = reinterpret_cast<int32_t*>(basep + o_td);
    w->perm = reinterpret_cast<int32_t*>(basep + o_perm);
    w->pmax = reinterpret_cast<int32_t*>(basep + o_pmax);
    w->hist = reinterpret_cast<int32_t*>(basep + o_hist);
    w->base = reinterpret_cast<int32_t*>(basep + o_base);
    w->cursor = reinterpret_cast<int32_t*>(basep + o_cur);
    w->hscratch = basep + o_hs;
    w->ximg = basep + o_x;
    w->hT = reinterpret_cast<float*>(basep + o_hT);
  }
  return off;
}

// Rows past their length carry the frozen state (the reference's Where):
// out[r, t, :] = hT[r, :] for len_r <= t < max_len_p.  Pure store stream.
__global__ void __launch_bounds__(256) rnn_fill_frozen_kernel(float* __restrict__ out, const float* __restrict__ hT,
                                       const int64_t* __restrict__ lens, const int32_t* __restrict__ pmax,
                                       int R, int T, int H, int Bp) {
  // one warp per row: out[r, t, :] = hT[r, :] for len_r <= t < max_len_p
  const int r = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= R) return;
  const int tmax = min(max(pmax[r / Bp], 0), T);
  const long long L = lens[r];
  const int len = (int)(L < 0 ? 0 : (L < tmax ? L : tmax));
  if (len >= tmax) return;
  float* orow = out + (size_t)r * T * H;
  const float* hrow = hT + (size_t)r * H;
  if ((H & 3) == 0) {
    const int h4 = H / 4;
    for (int j = lane; j < h4; j += 32) {
      const float4 v = reinterpret_cast<const float4*>(hrow)[j];
      for (int t = len; t < tmax; ++t) reinterpret_cast<float4*>(orow + (size_t)t * H)[j] = v;
    }
  } else {
    for (int j = lane; j < H; j += 32) {
      const float v = hrow[j];
      for (int t = len; t < tmax; ++t) orow[(size_t)t * H + j] = v;
    }
  }
}

// Kernel-only timing of the persistent recurrent kernel (bench.py's roofline):
// when armed, each launch is bracketed by a pair of CUDA events on its stream.
constexpr int kProfMax = 256;
cudaEvent_t g_prof_ev[2 * kProfMax];
int g_prof_cap = 0, g_prof_n = 0;

template <int CELL, typename XT, int EW, int ACT = 0>
int launch_main_ew(const RnnArgs& args, const RnnGeom& g, cudaStream_t stream) {
  auto kern = rnn_fwd_kernel<CELL, kNT, XT, EW, ACT>;
  g_last_kernel = SKB_RNN_KERNEL_SINGLE;
  constexpr int kThreads = EW * 32 + 64;
  const size_t smem = smem_bytes<kNT>(g);
  if (smem > 227 * 1024) return SKB_ERR_UNSUPPORTED;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return SKB_ERR_CUDA;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = g.C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.gridDim = dim3(g.C);
  int max_clusters = 0;
  if (cudaOccupancyMaxActiveClusters(&max_clusters, kern, &cfg) != cudaSuccess || max_clusters < 1)
    return SKB_ERR_CUDA;
  const int ncl = min(min(max_clusters, args.ntiles), max_clusters_bound(g) - 1);
  cfg.gridDim = dim3(g.C * max(ncl, 1));
  g_last_clusters = max(ncl, 1);
  const bool prof = g_prof_n < g_prof_cap;
  if (prof) cudaEventRecord(g_prof_ev[2 * g_prof_n], stream);
  if (cudaLaunchKernelEx(&cfg, kern, args) != cudaSuccess) return SKB_ERR_CUDA;
  if (prof) cudaEventRecord(g_prof_ev[2 * g_prof_n++ + 1], stream);
  return skb_check_launch();
}

// Ping-pong halves (LSTM) are opt-in (SKB_RNN_PP=1): measured slower on B200
// (1.89 vs 1.45 ms at C1) — two N=32 MMA chains cost as many tensor-pipe issue
// slots as two N=64 chains, so the MMA issue rate, not the epilogue, bounds a step.
inline bool rnn_pp() {
  static int pp = -1;
  if (pp < 0) {
    const char* e = getenv("SKB_RNN_PP");
    pp = (e && atoi(e) == 1) ? 1 : 0;
  }
  return pp == 1;
}

template <typename XT, int ACT>
int launch_pp(const RnnArgs& args, const RnnGeom& g, cudaStream_t stream) {
  auto kern = rnn_fwd_pp_kernel<XT, ACT>;
  g_last_kernel = SKB_RNN_KERNEL_PING_PONG;
  constexpr int kThreads = 16 * 32 + 64;
  const size_t smem = smem_bytes<kNT>(g);
  if (smem > 227 * 1024) return SKB_ERR_UNSUPPORTED;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return SKB_ERR_CUDA;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = g.C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.gridDim = dim3(g.C);
  int max_clusters = 0;
  if (cudaOccupancyMaxActiveClusters(&max_clusters, kern, &cfg) != cudaSuccess || max_clusters < 1)
    return SKB_ERR_CUDA;
  const int ncl = min(min(max_clusters, args.ntiles), max_clusters_bound(g) - 1);
  cfg.gridDim = dim3(g.C * max(ncl, 1));
  g_last_clusters = max(ncl, 1);
  const bool prof = g_prof_n < g_prof_cap;
  if (prof) cudaEventRecord(g_prof_ev[2 * g_prof_n], stream);
  if (cudaLaunchKernelEx(&cfg, kern, args) != cudaSuccess) return SKB_ERR_CUDA;
  if (prof) cudaEventRecord(g_prof_ev[2 * g_prof_n++ + 1], stream);
  return skb_check_launch();
}

// Dual-lane kernel (default for the LSTM when U == 32): SKB_RNN_DL=0 selects the
// single-lane kernel.
inline bool rnn_dl() {
  static int dl = -1;
  if (dl < 0) {
    const char* e = getenv("SKB_RNN_DL");
    dl = (e && atoi(e) == 0) ? 0 : 1;
  }
  return dl == 1;
}

template <typename XT, int ACT, int CELL = SKB_CELL_LSTM>
int launch_dl(const RnnArgs& args, const RnnGeom& g, cudaStream_t stream) {
  auto kern = rnn_fwd_dl_kernel<XT, ACT, CELL>;
  g_last_kernel = SKB_RNN_KERNEL_DUAL_LANE;
  constexpr int kThreads = 20 * 32;
  const size_t smem = (size_t)2 * (kNT * g.Kx * 2 + kNT * g.Kh * 2 + 4 * kNT * kGS * 4) + 1024;
  if (smem > 227 * 1024) return SKB_ERR_UNSUPPORTED;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return SKB_ERR_CUDA;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = g.C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.gridDim = dim3(g.C);
  int max_clusters = 0;
  if (cudaOccupancyMaxActiveClusters(&max_clusters, kern, &cfg) != cudaSuccess || max_clusters < 1)
    return SKB_ERR_CUDA;
  const int ncl = min(min(max_clusters, (args.ntiles + 1) / 2), max_clusters_bound(g) - 1);
  cfg.gridDim = dim3(g.C * max(ncl, 1));
  g_last_clusters = max(ncl, 1);
  const bool prof = g_prof_n < g_prof_cap;
  if (prof) cudaEventRecord(g_prof_ev[2 * g_prof_n], stream);
  if (cudaLaunchKernelEx(&cfg, kern, args) != cudaSuccess) return SKB_ERR_CUDA;
  if (prof) cudaEventRecord(g_prof_ev[2 * g_prof_n++ + 1], stream);
  return skb_check_launch();
}

// CTA-pair kernel (default for LSTM/GRU with 32-unit slices and an even CTA count;
// SKB_RNN_PAIR=0 selects the dual-lane kernel).
inline bool rnn_pair() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SKB_RNN_PAIR");
    v = (e && atoi(e) == 0) ? 0 : 1;
  }
  return v == 1;
}
inline size_t pair_smem(const RnnGeom& g) { return (size_t)2 * (64 * g.Kx * 2 + 2 * 64 * g.Kh * 2) + 1024; }
inline size_t pair4_smem(const RnnGeom& g) { return (size_t)4 * (32 * g.Kx * 2 + 2 * 32 * g.Kh * 2) + 1024; }
inline bool pair_ok(const RnnGeom& g) {
  return rnn_pair() && g.U == 32 && g.H == g.C * 32 && g.Kh == g.H && g.C % 2 == 0 && g.C >= 2 &&
         pair_smem(g) <= 227 * 1024;
}

template <typename XT, int ACT, int CELL = SKB_CELL_LSTM>
int launch_pair(RnnArgs args, const RnnGeom& g, cudaStream_t stream) {
  auto kern = rnn_fwd_pair_kernel<XT, ACT, CELL>;
  g_last_kernel = SKB_RNN_KERNEL_PAIR2;
  constexpr int kThreads = 20 * 32;
  const size_t smem = pair_smem(g);
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return SKB_ERR_CUDA;
  args.ntiles = (args.ntiles + 1) / 2;   // 128-row tiles = pairs of 64-row x-image tiles
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = g.C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.gridDim = dim3(g.C);
  int max_clusters = 0;
  if (cudaOccupancyMaxActiveClusters(&max_clusters, kern, &cfg) != cudaSuccess || max_clusters < 1)
    return SKB_ERR_CUDA;
  const int ncl = min(min(max_clusters, (args.ntiles + 1) / 2), max_clusters_bound(g) - 1);
  cfg.gridDim = dim3(g.C * max(ncl, 1));
  g_last_clusters = max(ncl, 1);
  const bool prof = g_prof_n < g_prof_cap;
  if (prof) cudaEventRecord(g_prof_ev[2 * g_prof_n], stream);
  if (cudaLaunchKernelEx(&cfg, kern, args) != cudaSuccess) return SKB_ERR_CUDA;
  if (prof) cudaEventRecord(g_prof_ev[2 * g_prof_n++ + 1], stream);
  return skb_check_launch();
}
// SKB_RNN_FILLW=1: the pair4 kernel's fill warp writes the frozen tails (measured slower:
// the 21st warp caps the kernel at 80 registers).
inline bool rnn_fill_warp() {
  static int v = -1;
  if (v < 0) v = env_flag("SKB_RNN_FILLW", 0) ? 1 : 0;
  return v == 1;
}
// SKB_RNN_XOVL=1: the pair4 kernel's x images are packed concurrently on the
// idle SMs (pack_x_stream_kernel) instead of by a pre-pass.
int g_overlap_off = 0;   // skb_rnn_set_overlap(0): no auxiliary grid (e.g. after a handoff timeout)
inline bool rnn_x_overlap() {
  static int v = -1;
  if (v < 0) v = env_flag("SKB_RNN_XOVL", 0) ? 1 : 0;
  return v == 1 && !g_overlap_off;
}

template <typename XT, int ACT, int CELL, int FW>
int launch_pair4_fw(RnnArgs args, const RnnGeom& g, cudaStream_t stream) {
  auto kern = rnn_fwd_pair4_kernel<XT, ACT, CELL, FW>;
  g_last_kernel = SKB_RNN_KERNEL_PAIR;
  constexpr int kThreads = (20 + FW) * 32;
  const size_t smem = pair4_smem(g);
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return SKB_ERR_CUDA;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = g.C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.gridDim = dim3(g.C);
  int max_clusters = 0;
  if (cudaOccupancyMaxActiveClusters(&max_clusters, kern, &cfg) != cudaSuccess || max_clusters < 1)
    return SKB_ERR_CUDA;
  const int ncl = min(min(max_clusters, (args.ntiles + 3) / 4), max_clusters_bound(g) - 1);
  cfg.gridDim = dim3(g.C * max(ncl, 1));
  g_last_clusters = max(ncl, 1);
  const bool prof = g_prof_n < g_prof_cap;
  if (prof) cudaEventRecord(g_prof_ev[2 * g_prof_n], stream);
  if (cudaLaunchKernelEx(&cfg, kern, args) != cudaSuccess) return SKB_ERR_CUDA;
  if (prof) cudaEventRecord(g_prof_ev[2 * g_prof_n++ + 1], stream);
  return skb_check_launch();
}
template <typename XT, int ACT, int CELL = SKB_CELL_LSTM>
int launch_pair4(RnnArgs args, const RnnGeom& g, cudaStream_t stream) {
  return args.fill_inkernel || !rnn_fill_warp() ? launch_pair4_fw<XT, ACT, CELL, 0>(args, g, stream)
                                                : launch_pair4_fw<XT, ACT, CELL, 1>(args, g, stream);
}


// Which recurrent kernel runs (SKB_RNN_KERNEL_*): the CTA-pair kernels for LSTM/GRU with
// 32-unit slices and an even CTA count (SKB_RNN_PAIR: 1 = four 64-row lanes, the default;
// 2 = two 128-row lanes; 0 = off), else the dual-lane / ping-pong / single kernels.
inline int rnn_pair_mode() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SKB_RNN_PAIR");
    v = e ? atoi(e) : 1;
    if (v < 0 || v > 2) v = 1;
  }
  return v;
}
inline int kernel_choice(const RnnGeom& g, bool has_c0) {
  const bool slices32 = g.U == 32 && g.H == g.C * 32 && g.Kh == g.H;
  const bool cell4 = g.cell == SKB_CELL_GRU || (g.cell == SKB_CELL_LSTM && has_c0);
  if (g.cell == SKB_CELL_LSTM || g.cell == SKB_CELL_GRU) {
    if (rnn_dl() && !rnn_pp() && rnn_ew() == 16 && cell4 && pair_ok(g) && rnn_pair_mode() != 0)
      return rnn_pair_mode() == 2 ? SKB_RNN_KERNEL_PAIR2 : SKB_RNN_KERNEL_PAIR;
    if (rnn_dl() && !rnn_pp() && rnn_ew() == 16 && slices32 && cell4) return SKB_RNN_KERNEL_DUAL_LANE;
    if (g.cell == SKB_CELL_LSTM && rnn_pp() && g.U == 32 && g.Kh == g.C * 32) return SKB_RNN_KERNEL_PING_PONG;
  }
  return SKB_RNN_KERNEL_SINGLE;
}

template <int CELL, typename XT>
int launch_main(const RnnArgs& args, const RnnGeom& g, cudaStream_t stream) {
  const int act = rnn_act();
  const int k = kernel_choice(g, args.c0 != nullptr);
  if constexpr (CELL == SKB_CELL_LSTM || CELL == SKB_CELL_GRU) {
    if (k == SKB_RNN_KERNEL_PAIR)
      return act == 2 ? launch_pair4<XT, 2, CELL>(args, g, stream)
                      : (act ? launch_pair4<XT, 1, CELL>(args, g, stream) : launch_pair4<XT, 0, CELL>(args, g, stream));
    if (k == SKB_RNN_KERNEL_PAIR2)
      return act == 2 ? launch_pair<XT, 2, CELL>(args, g, stream)
                      : (act ? launch_pair<XT, 1, CELL>(args, g, stream) : launch_pair<XT, 0, CELL>(args, g, stream));
    if (k == SKB_RNN_KERNEL_DUAL_LANE)
      return act ? launch_dl<XT, 1, CELL>(args, g, stream) : launch_dl<XT, 0, CELL>(args, g, stream);
  }
  if constexpr (CELL == SKB_CELL_LSTM) {
    if (k == SKB_RNN_KERNEL_PING_PONG)
      return act ? launch_pp<XT, 1>(args, g, stream) : launch_pp<XT, 0>(args, g, stream);
  }
  if constexpr (CELL == SKB_CELL_LSTM || CELL == SKB_CELL_GRU) {
    if (rnn_ew() == 8)
      return act ? launch_main_ew<CELL, XT, 8, 1>(args, g, stream) : launch_main_ew<CELL, XT, 8, 0>(args, g, stream);
    return act ? launch_main_ew<CELL, XT, 16, 1>(args, g, stream) : launch_main_ew<CELL, XT, 16, 0>(args, g, stream);
  }
  return rnn_ew() == 8 ? launch_main_ew<CELL, XT, 8>(args, g, stream) : launch_main_ew<CELL, XT, 16>(args, g, stream);
}

// SKB_RNN_FOVL=1: the pair4 kernel's frozen tails are written concurrently by
// the auxiliary grid on the idle SMs instead of by a pass after the kernel.
inline bool rnn_fill_overlap() {
  static int v = -1;
  if (v < 0) v = env_flag("SKB_RNN_FOVL", 0) ? 1 : 0;
  return v == 1 && !g_overlap_off;
}

// Force-load the auxiliary kernel before the recurrent kernel is queued: with CUDA's lazy
// module loading, loading a function while a kernel that waits on it is running stalls
// until that kernel ends (here: until its handoff waits time out).
int preload_aux(int nq, size_t smem) {
  static bool done[5] = {false, false, false, false, false};
  if (nq < 1 || nq > 4) return SKB_ERR_INVALID;
  if (!done[nq]) {
    cudaFuncAttributes fa;
    const void* f = nq == 1 ? (const void*)rnn_aux_kernel<1> : nq == 2 ? (const void*)rnn_aux_kernel<2>
                                                                      : (const void*)rnn_aux_kernel<4>;
    if (cudaFuncGetAttributes(&fa, f) != cudaSuccess) return SKB_ERR_CUDA;
    if (cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * (512 * 2 + 16)) != cudaSuccess)
      return SKB_ERR_CUDA;
    done[nq] = true;
  }
  (void)smem;
  return SKB_OK;
}

// Clusters the pair4 kernel launches with for `ntiles` tiles (as launch_pair4_fw computes it).
template <int FW>
int pair4_clusters(const RnnGeom& g, int ntiles) {
  auto kern = rnn_fwd_pair4_kernel<float, 1, SKB_CELL_LSTM, FW>;
  const size_t smem = pair4_smem(g);
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 0;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = g.C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3((20 + FW) * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.gridDim = dim3(g.C);
  int max_clusters = 0;
  if (cudaOccupancyMaxActiveClusters(&max_clusters, kern, &cfg) != cudaSuccess || max_clusters < 1) return 0;
  return max(1, min(min(max_clusters, (ntiles + 3) / 4), max_clusters_bound(g) - 1));
}

// Side streams of the concurrent-packer launch: the recurrent kernel on the
// highest-priority stream (its clusters are placed before the packer's CTAs), the
// packer on a lowest-priority one; fork/join through events on the caller's stream.
struct OverlapStreams {
  cudaStream_t hi = nullptr, pack = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_hi = nullptr, ev_pack = nullptr;
  bool ok = false;
};
OverlapStreams g_ovl[16];

OverlapStreams* overlap_streams() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 16) return nullptr;
  OverlapStreams& o = g_ovl[dev];
  if (!o.ok) {
    int least = 0, greatest = 0;
    if (cudaDeviceGetStreamPriorityRange(&least, &greatest) != cudaSuccess) return nullptr;
    if (cudaStreamCreateWithPriority(&o.hi, cudaStreamNonBlocking, greatest) != cudaSuccess ||
        cudaStreamCreateWithPriority(&o.pack, cudaStreamNonBlocking, least) != cudaSuccess ||
        cudaEventCreateWithFlags(&o.ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&o.ev_hi, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&o.ev_pack, cudaEventDisableTiming) != cudaSuccess)
      return nullptr;
    o.ok = true;
  }
  return &o;
}

int g_last_overlap = 0;

}  // namespace

extern "C" int skb_rnn_last_kernel(void) { return g_last_kernel; }
extern "C" int skb_rnn_last_overlap(void) { return g_last_overlap; }
extern "C" int skb_rnn_set_overlap(int enable) {
  g_overlap_off = enable ? 0 : 1;
  return SKB_OK;
}
extern "C" int skb_rnn_last_clusters(void) { return g_last_clusters; }

extern "C" int skb_profile_begin(int max_launches) {
  if (max_launches < 0 || max_launches > kProfMax) return SKB_ERR_INVALID;
  for (int i = g_prof_cap; i < max_launches; ++i) {
    if (cudaEventCreate(&g_prof_ev[2 * i]) != cudaSuccess) return SKB_ERR_CUDA;
    if (cudaEventCreate(&g_prof_ev[2 * i + 1]) != cudaSuccess) return SKB_ERR_CUDA;
  }
  if (max_launches > g_prof_cap) g_prof_cap = max_launches;
  g_prof_n = 0;
  return SKB_OK;
}

extern "C" int skb_profile_read(float* ms_out, int n) {
  int m = g_prof_n < n ? g_prof_n : n;
  for (int i = 0; i < m; ++i) {
    if (cudaEventSynchronize(g_prof_ev[2 * i + 1]) != cudaSuccess) return -1;
    if (cudaEventElapsedTime(&ms_out[i], g_prof_ev[2 * i], g_prof_ev[2 * i + 1]) != cudaSuccess) return -1;
  }
  g_prof_cap = g_prof_cap;  // events are kept for reuse
  return m;
}

extern "C" int skb_profile_end(void) {
  g_prof_n = 0;
  const int cap = g_prof_cap;
  g_prof_cap = 0;
  for (int i = 0; i < cap; ++i) { cudaEventDestroy(g_prof_ev[2 * i]); cudaEventDestroy(g_prof_ev[2 * i + 1]); }
  return SKB_OK;
}

extern "C" int skb_debug_rnn_tile_trace(long long* trace_dev, int tiles) {
#ifndef SKB_TRACE_ENABLED
  return trace_dev ? SKB_ERR_UNSUPPORTED : SKB_OK;   // build with SKB_TRACE=1
#else
  if (cudaMemcpyToSymbol(g_ttrace, &trace_dev, sizeof(trace_dev)) != cudaSuccess) return SKB_ERR_CUDA;
  if (cudaMemcpyToSymbol(g_ttrace_n, &tiles, sizeof(tiles)) != cudaSuccess) return SKB_ERR_CUDA;
  #endif
  return SKB_OK;
}

extern "C" int skb_debug_rnn_trace(long long* trace_dev, int steps) {
#ifndef SKB_TRACE_ENABLED
  return trace_dev ? SKB_ERR_UNSUPPORTED : SKB_OK;   // build with SKB_TRACE=1
#else
  if (cudaMemcpyToSymbol(g_trace, &trace_dev, sizeof(trace_dev)) != cudaSuccess) return SKB_ERR_CUDA;
  if (cudaMemcpyToSymbol(g_trace_steps, &steps, sizeof(steps)) != cudaSuccess) return SKB_ERR_CUDA;
  #endif
  return SKB_OK;
}

extern "C" int skb_rnn_plan(const skb_rnn_shape* shape, int32_t* clusters, int32_t* ctas_per_cluster,
                            int32_t* tile_rows) {
  RnnGeom g;
  if (!make_geom(shape, &g)) return SKB_ERR_INVALID;
  const size_t smem = smem_bytes<kNT>(g);
  if (smem > 227 * 1024) return SKB_ERR_UNSUPPORTED;
  auto kern = rnn_fwd_kernel<SKB_CELL_LSTM, kNT, float, 16>;
  const int kThreads = 16 * 32 + 64;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return SKB_ERR_CUDA;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = g.C; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(kThreads); cfg.dynamicSmemBytes = smem; cfg.attrs = attr; cfg.numAttrs = 1;
  cfg.gridDim = dim3(g.C);
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) return SKB_ERR_CUDA;
  if (clusters) *clusters = n;
  if (ctas_per_cluster) *ctas_per_cluster = g.C;
  if (tile_rows) *tile_rows = kNT;
  return SKB_OK;
}

extern "C" int64_t skb_rnn_packed_bytes(const skb_rnn_shape* shape) {
  RnnGeom g;
  if (!make_geom(shape, &g)) return -1;
  return (int64_t)g.C * 128 * g.K * 2 + (int64_t)g.C * 128 * 4;
}

extern "C" int64_t skb_rnn_workspace_bytes(const skb_rnn_shape* shape) {
  RnnGeom g;
  if (!make_geom(shape, &g)) return -1;
  return ws_layout(g, nullptr, nullptr);
}

extern "C" int skb_rnn_pack(const skb_rnn_shape* shape, const void* const* w_dev,
                            const void* const* u_dev, const void* const* b_dev, int f64,
                            void* packed_dev, int32_t* err_dev, void* stream) {
  RnnGeom g;
  if (!make_geom(shape, &g) || !packed_dev || !w_dev || !u_dev || !b_dev) return SKB_ERR_INVALID;
  PackArgs a = {};
  for (int i = 0; i < g.G; ++i) {
    a.w[i] = w_dev[i]; a.u[i] = u_dev[i]; a.b[i] = b_dev[i];
    const bool gru_zero_block = g.cell == SKB_CELL_GRU && ((i == 3 && !a.w[i]) || (i == 2 && !a.u[i]));
    if ((!a.w[i] || !a.u[i]) && !gru_zero_block) return SKB_ERR_INVALID;
    if (!a.b[i]) return SKB_ERR_INVALID;
  }
  a.f64 = f64;
  a.slab = reinterpret_cast<uint8_t*>(packed_dev);
  a.bias = reinterpret_cast<float*>(a.slab + (size_t)g.C * 128 * g.K * 2);
  a.err = err_dev;
  a.G = g.G; a.H = g.H; a.F = g.F; a.U = g.U; a.C = g.C; a.Kx = g.Kx; a.Kh = g.Kh; a.K = g.K;
  const long long total = (long long)g.C * 128 * (g.K / 8);
  const long long want = (total + 255) / 256;
  const int blocks = (int)(want < 4096 ? want : 4096);
  rnn_pack_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(a);
  return skb_check_launch();
}

extern "C" int skb_rnn_forward(const skb_rnn_shape* shape, const void* packed_dev, const void* x_dev,
                               int x_f64, const float* h0_dev, const float* c0_dev,
                               const int64_t* len_dev, float* out_dev, float* hT_dev, float* cT_dev,
                               int32_t* max_len_dev, int32_t* err_dev, void* workspace_dev,
                               void* stream) {
  RnnGeom g;
  if (!make_geom(shape, &g) || !packed_dev || !x_dev || !h0_dev || !len_dev || !out_dev ||
      !max_len_dev || !err_dev || !workspace_dev)
    return SKB_ERR_INVALID;
  if (g.cell == SKB_CELL_LSTM && !c0_dev) return SKB_ERR_INVALID;
  if (g.T > 1 << 20) return SKB_ERR_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  Workspace w;
  ws_layout(g, reinterpret_cast<uint8_t*>(workspace_dev), &w);
  const int ntiles = n_tiles64(g);
  // The four-lane pair kernel reads 32-row half images, packed by a pre-pass; its frozen
  // tails are filled by a pass after it.  Measured alternatives (each slower on the B200,
  // profiles/r02_c1_overlap.md): SKB_RNN_XOVL=1 / SKB_RNN_FOVL=1 pack / fill concurrently
  // on the idle SMs (the auxiliary grid); SKB_RNN_FILLW=1 fill warp in the kernel;
  // SKB_RNN_INFILL=1 fill from the epilogue.
  const bool pair4 = kernel_choice(g, c0_dev != nullptr) == SKB_RNN_KERNEL_PAIR;
  const bool infill = pair4 && env_flag("SKB_RNN_INFILL", 0);
  const bool fillw = pair4 && !infill && rnn_fill_warp();
  const bool rows_ok = !x_f64 && g.F == g.Kx && (reinterpret_cast<uintptr_t>(x_dev) & 15) == 0 &&
                       (g.F == 128 || g.F == 256 || g.F == 512) && !getenv("SKB_PACK_X_LEGACY");
  bool xovl = pair4 && rows_ok && rnn_x_overlap();
  bool fovl = pair4 && !infill && !fillw && rnn_fill_overlap();
  OverlapStreams* ovs = nullptr;
  int idle = 0;
  if (xovl || fovl) {   // only with enough idle SMs for the auxiliary grid (the kernel waits on it)
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int ncl = fillw ? pair4_clusters<1>(g, ntiles) : pair4_clusters<0>(g, ntiles);
    idle = sms - ncl * g.C;
    if (ncl > 0 && idle >= 16) ovs = overlap_streams();
  }
  if (!ovs) xovl = fovl = false;
  g_last_overlap = (xovl ? 1 : 0) | (fovl ? 2 : 0);
  SchedArgs sa = {len_dev, w.perm, w.pmax, w.hist, w.base, w.cursor, max_len_dev, err_dev, w.xflag, w.tdone,
                  g.R, g.Bp, g.P, g.T, ntiles * kNT, xovl ? ntiles * g.T : 0, fovl ? ntiles : 0};
  const int blocks = min(1184, max(1, (max(g.R, g.P) + 255) / 256));
  sched_init<<<blocks, 256, 0, st>>>(sa);
  sched_hist<<<blocks, 256, 0, st>>>(sa);
  sched_scan<<<1, 1024, 0, st>>>(sa);
  sched_scatter<<<blocks, 256, 0, st>>>(sa);
  if (int e = skb_check_launch()) return e;

  RnnArgs a = {};
  a.x = x_dev; a.h0 = h0_dev; a.c0 = c0_dev; a.lens = len_dev; a.perm = w.perm; a.pmax = w.pmax;
  a.wpack = reinterpret_cast<const uint8_t*>(packed_dev);
  a.bpack = reinterpret_cast<const float*>(a.wpack + (size_t)g.C * 128 * g.K * 2);
  a.out = out_dev; a.hT = hT_dev ? hT_dev : w.hT; a.cT = cT_dev; a.err = err_dev; a.x_f64 = x_f64;
  a.hscratch = w.hscratch;
  a.ximg = w.ximg;
  a.fill_inkernel = infill ? 1 : 0;
  a.R = g.R; a.T = g.T; a.F = g.F; a.H = g.H; a.Kx = g.Kx; a.Kh = g.Kh; a.K = g.K; a.U = g.U;
  a.C = g.C; a.Bp = g.Bp; a.ntiles = ntiles;
  if (!xovl) {   // pre-pass packer
    const dim3 pg(ntiles, g.T);
    const int halves = pair4 ? 1 : 0;
    if (x_f64)
      pack_x_kernel<double><<<pg, 256, 0, st>>>((const double*)x_dev, w.perm, len_dev, w.pmax, w.ximg,
                                                  err_dev, ntiles, g.T, g.F, g.Kx, g.Bp, halves);
    else if (rows_ok) {
      const size_t sm = (size_t)kNT * (g.F * 2 + 16);
      if (g.F == 128)
        pack_x_rows_kernel<1><<<pg, 256, sm, st>>>((const float*)x_dev, w.perm, len_dev, w.pmax, w.ximg, err_dev, g.T, g.Bp, halves);
      else if (g.F == 256)
        pack_x_rows_kernel<2><<<pg, 256, sm, st>>>((const float*)x_dev, w.perm, len_dev, w.pmax, w.ximg, err_dev, g.T, g.Bp, halves);
      else {
        static bool attr = false;
        if (!attr) {
          cudaFuncSetAttribute(pack_x_rows_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
          attr = true;
        }
        pack_x_rows_kernel<4><<<pg, 256, sm, st>>>((const float*)x_dev, w.perm, len_dev, w.pmax, w.ximg, err_dev, g.T, g.Bp, halves);
      }
    } else
      pack_x_kernel<float><<<pg, 256, 0, st>>>((const float*)x_dev, w.perm, len_dev, w.pmax, w.ximg,
                                                 err_dev, ntiles, g.T, g.F, g.Kx, g.Bp, halves);
    if (int e = skb_check_launch()) return e;
  }
  auto launch_rec = [&](cudaStream_t rs) {
    if (g.cell == SKB_CELL_LSTM)
      return x_f64 ? launch_main<SKB_CELL_LSTM, double>(a, g, rs) : launch_main<SKB_CELL_LSTM, float>(a, g, rs);
    if (g.cell == SKB_CELL_GRU)
      return x_f64 ? launch_main<SKB_CELL_GRU, double>(a, g, rs) : launch_main<SKB_CELL_GRU, float>(a, g, rs);
    return x_f64 ? launch_main<SKB_CELL_RNN_TANH, double>(a, g, rs) : launch_main<SKB_CELL_RNN_TANH, float>(a, g, rs);
  };
  if (ovs) {
    // fork: the recurrent kernel (high priority, placed first) and the auxiliary grid
    // (low priority, on the idle SMs); join on the caller's stream
    const int nq = xovl ? g.F / 128 : 1;
    const size_t sm = xovl ? (size_t)kNT * (g.F * 2 + 16) : 0;
    if (int e = preload_aux(nq, sm)) return e;
    a.xflag = xovl ? w.xflag : nullptr;
    a.tdone = fovl ? w.tdone : nullptr;
    cudaEventRecord(ovs->ev_fork, st);
    cudaStreamWaitEvent(ovs->hi, ovs->ev_fork, 0);
    cudaStreamWaitEvent(ovs->pack, ovs->ev_fork, 0);
    int rc = launch_rec(ovs->hi);
    if (rc == SKB_OK) {
      AuxArgs x = {(const float*)x_dev, w.perm, len_dev, w.pmax, w.ximg, err_dev, xovl ? w.xflag : nullptr, a.tdone, out_dev, a.hT,
                   ntiles, g.T, g.H, g.Bp, 4 * g_last_clusters, g.C};
      const int grid = 2 * idle;
      if (nq == 1) rnn_aux_kernel<1><<<grid, 256, sm, ovs->pack>>>(x);
      else if (nq == 2) rnn_aux_kernel<2><<<grid, 256, sm, ovs->pack>>>(x);
      else rnn_aux_kernel<4><<<grid, 256, sm, ovs->pack>>>(x);
      rc = skb_check_launch();
    }
    cudaEventRecord(ovs->ev_hi, ovs->hi);
    cudaEventRecord(ovs->ev_pack, ovs->pack);
    cudaStreamWaitEvent(st, ovs->ev_hi, 0);
    cudaStreamWaitEvent(st, ovs->ev_pack, 0);
    if (rc) return rc;
  } else if (int rc = launch_rec(st)) {
    return rc;
  }
  if (!fillw && !infill && !fovl)
    rnn_fill_frozen_kernel<<<(g.R + 7) / 8, 256, 0, st>>>(out_dev, a.hT, len_dev, w.pmax, g.R, g.T, g.H, g.Bp);
  return skb_check_launch();
}
