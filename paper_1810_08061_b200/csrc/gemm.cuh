// gemm.cuh — skb's own tcgen05 GEMM engine for sm_100a (no cuBLAS / CUTLASS).
//
// D[M x N] (fp32, TMEM) = A[M x K] · B[K x N] on the 5th-generation tensor cores:
//   * operands staged by TMA tensor maps (cp.async.bulk.tensor.2d, 128-byte swizzle) into
//     a ring of shared-memory stages (full/empty mbarriers);
//   * one elected thread issues tcgen05.mma (M = 128, N = BN, K = 32 bytes per
//     instruction) from shared-memory descriptors; completion is committed to the
//     stage's empty barrier (frees the slot) and, per tile, to a TMEM-full barrier;
//   * the fp32 accumulator lives in TMEM, double buffered (2 x BN columns), so the
//     epilogue of tile i (tcgen05.ld -> registers -> fused epilogue -> global) overlaps
//     the MMAs of tile i+1;
//   * persistent CTAs (one per SM) walk the tiles (x K-splits) in a fixed order.
// Element types: bf16 (kind::f16, bf16 x bf16 -> fp32) and tf32 (kind::tf32, fp32 in
// memory).  Each bf16 operand may be K-major or MN-major in memory (tf32: K-major only —
// kind::tf32 with an MN-major operand produced no result on the B200):
//   A: [M, K] row-major (K contiguous)  or  [K, M] row-major (M contiguous, "A^T")
//   B: [N, K] row-major (K contiguous)  or  [K, N] row-major (N contiguous)
// Canonical SW128 layouts (K-major: 8-row x 128-byte atoms, SBO = 1024 B; MN-major:
// 128-byte MN rows, 8 K-rows per atom, SBO = 1024 B, LBO = distance between 128-byte MN
// column blocks).  The encodings are pinned by tests/test_gpu_gemm.py against torch.
//
// Warp roles (64 + 128 EW threads): warp 0 TMA producer, warp 1 TMEM allocator + MMA
// issuer, warps 2 .. 2 + 4 EW epilogue: warp w reads TMEM lanes 32 (w % 4) .. +31 (tile
// rows) and column group (w - 2) / 4 of EW (BN / EW columns) — EW > 1 for the fused
// epilogues whose per-element math would otherwise run on one warp per SM sub-partition.
// The epilogue is a functor (per 16 consecutive columns of one row): plain stores,
// split-K partials and the fused LSTM cells of train.cu.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "sm100.cuh"

namespace skb {
namespace gemm {

enum Elem { kBF16 = 0, kTF32 = 1 };

// ---------------------------------------------------------------- device helpers
SKB_DEV void tma_load_2d(void* smem_dst, const CUtensorMap* tm, int c0, int c1, uint64_t* bar) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
               :: "r"(smem_u32(smem_dst)), "l"(tm), "r"(c0), "r"(c1), "r"(smem_u32(bar)) : "memory");
}
SKB_DEV void tma_prefetch_desc(const CUtensorMap* tm) {
  asm volatile("prefetch.tensormap [%0];" :: "l"(tm) : "memory");
}
// 128-byte-swizzle shared-memory matrix descriptor (layout type 2 at bits [61,64)).
SKB_DEV uint64_t sdesc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
// Instruction descriptor: fp32 accumulate, a/b format (kind::f16: BF16 = 1; kind::tf32:
// TF32 = 2), a/b major (1 = MN-major), N >> 3, M >> 4.
__host__ __device__ constexpr uint32_t idesc(int elem, int M, int N, bool a_mn, bool b_mn) {
  return (1u << 4) | ((elem == kBF16 ? 1u : 2u) << 7) | ((elem == kBF16 ? 1u : 2u) << 10) |
         ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}
template <int ELEM>
SKB_DEV void umma_ss(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t id, uint32_t accumulate) {
  if constexpr (ELEM == kBF16) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                 :: "r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(id), "r"(accumulate) : "memory");
  } else {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                 :: "r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(id), "r"(accumulate) : "memory");
  }
}

// ---------------------------------------------------------------- geometry
template <int ELEM, int BN, uint32_t OPB = 0, int BUDGET_KB = 212>
struct Geo {
  static constexpr int EB = ELEM == kBF16 ? 2 : 4;      // bytes per element
  static constexpr int BM = 128;
  static constexpr int BK = 128 / EB;                   // one 128-byte swizzle row of K
  static constexpr int UK = 32 / EB;                    // K per tcgen05.mma (32 bytes)
  static constexpr int MNB = 128 / EB;                  // MN elements per 128-byte row (MN-major)
  static constexpr int A_BYTES = BM * BK * EB;          // 16 KB
  static constexpr int B_BYTES = BN * BK * EB;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int S = ((BUDGET_KB * 1024 - (int)OPB) / STAGE) > 8 ? 8 : ((BUDGET_KB * 1024 - (int)OPB) / STAGE);
  static constexpr uint32_t TMEM_COLS = 2 * BN <= 32 ? 32 : 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128
                                      : 2 * BN <= 256 ? 256 : 512;
  static constexpr size_t SMEM = (size_t)S * STAGE + OPB + 1024;
};

// Address of 16-byte chunk `c16` of row `row` in a [rows][128 B] box written by TMA with
// the 128-byte swizzle (box base 1024-byte aligned): conflict-free row-per-thread reads.
SKB_DEV const uint8_t* sw128_at(const uint8_t* box, int row, int c16) {
  return box + row * 128 + ((c16 ^ (row & 7)) << 4);
}

struct Shape {
  int M, N, K;
  int ksplit;    // K split into this many contiguous ranges (work unit = tile x split)
  int ka;        // A2 kernels: k-blocks [0, ka) come from tmA, [ka, ..) from tmA2 (K-major)
};

// Tile t -> (tm, tn), N fastest: consecutive CTAs share the A row block (L2 reuse).
SKB_DEV void tile_coords(int u, int tiles_n, int ksplit, int& tm, int& tn, int& ks) {
  ks = u % ksplit;
  const int t = u / ksplit;
  tm = t / tiles_n;
  tn = t % tiles_n;
}

// Epilogue functor contract (const: the functor is a __grid_constant__ kernel parameter,
// so tensor maps it holds are usable by TMA; per-thread state lives in Epi::State):
//   skip()                    true: the whole grid exits at once (checked before any setup)
//   kOpBytes                  shared-memory bytes of per-tile epilogue operands (0: none)
//   prefetch(sop, tm, tn, bar) producer thread: TMA loads of the tile's operands into sop
//                             (completion counted on bar; issued before the tile's K loop,
//                             so they land while the MMAs run)
//   begin_tile / chunk / end_tile  per epilogue thread; chunk gets 16 accumulator columns
//                             [n0, n0+16) of row m, c = n0 - tile column 0, r = tile row
template <int ELEM, int BN, bool AMN, bool BMN, class Epi, bool A2 = false, int EW = 1>
__global__ void __launch_bounds__(64 + 128 * EW, 1) gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                                                      const __grid_constant__ CUtensorMap tmB,
                                                      const __grid_constant__ CUtensorMap tmA2, const Shape sh,
                                                      const __grid_constant__ Epi epi) {
  using G = Geo<ELEM, BN, Epi::kOpBytes>;
  if (epi.skip()) return;   // device-side predicate (e.g. a decode loop that has finished)
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sop = smem + G::S * G::STAGE;   // epilogue operands (1024-aligned: STAGE is)
  __shared__ uint64_t full[G::S], empty[G::S], tfull[2], tempty[2], opfull, opfree;
  __shared__ uint32_t tmem_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles_m = (sh.M + G::BM - 1) / G::BM, tiles_n = (sh.N + BN - 1) / BN;
  const int kblocks = (sh.K + G::BK - 1) / G::BK;
  const int units = tiles_m * tiles_n * sh.ksplit;

  if (threadIdx.x == 0) {
    for (int s = 0; s < G::S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 4 * EW); }
    mbar_init(&opfull, 1);
    mbar_init(&opfree, 4 * EW);
    fence_mbar_init();
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    if (A2) tma_prefetch_desc(&tmA2);
  }
  if (warp == 1) tmem_alloc<G::TMEM_COLS>(&tmem_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_s;
  // Programmatic dependent launch: the setup above overlaps the previous kernel's tail;
  // nothing it wrote is touched before this wait (a no-op without a prerequisite grid).
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  if (warp == 0) {
    // ===================== TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t ph = 0, oph = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        int tm, tn, ks;
        tile_coords(u, tiles_n, sh.ksplit, tm, tn, ks);
        const int kb0 = (int)((long long)kblocks * ks / sh.ksplit), kb1 = (int)((long long)kblocks * (ks + 1) / sh.ksplit);
        if constexpr (Epi::kOpBytes > 0) {   // the tile's epilogue operands, behind its MMAs
          mbar_wait_sleep(&opfree, oph ^ 1);
          if (epi.ops_on()) {
            mbar_arrive_expect_tx(&opfull, Epi::kOpBytes);
            epi.prefetch(sop, tm, tn, &opfull);
          } else {
            mbar_arrive(&opfull);
          }
          oph ^= 1;
        }
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait_sleep(&empty[stage], ph ^ 1);
          mbar_arrive_expect_tx(&full[stage], G::STAGE);
          uint8_t* sa = smem + stage * G::STAGE;
          uint8_t* sb = sa + G::A_BYTES;
          const int k0 = kb * G::BK;
          if constexpr (A2) {
            if (kb < sh.ka) tma_load_2d(sa, &tmA, k0, tm * G::BM, &full[stage]);
            else tma_load_2d(sa, &tmA2, k0 - sh.ka * G::BK, tm * G::BM, &full[stage]);
          } else if constexpr (!AMN) {
            tma_load_2d(sa, &tmA, k0, tm * G::BM, &full[stage]);
          } else {
#pragma unroll
            for (int h = 0; h < G::BM / G::MNB; ++h)
              tma_load_2d(sa + h * (G::BK * 128), &tmA, tm * G::BM + h * G::MNB, k0, &full[stage]);
          }
          if constexpr (!BMN) {
            tma_load_2d(sb, &tmB, k0, tn * BN, &full[stage]);
          } else {
#pragma unroll
            for (int h = 0; h < BN / G::MNB; ++h)
              tma_load_2d(sb + h * (G::BK * 128), &tmB, tn * BN + h * G::MNB, k0, &full[stage]);
          }
          if (++stage == G::S) { stage = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (one thread)
    if (lane == 0) {
      constexpr uint32_t id = idesc(ELEM, G::BM, BN, AMN, BMN);
      // per-instruction K advance: 32 bytes inside the swizzle row (K-major), or UK
      // 128-byte K rows (MN-major)
      constexpr uint32_t a_step = AMN ? G::UK * 128 : 32, b_step = BMN ? G::UK * 128 : 32;
      constexpr uint32_t a_lbo = AMN ? G::BK * 128 : 16, b_lbo = BMN ? G::BK * 128 : 16;
      int stage = 0, acc = 0;
      uint32_t ph = 0, aph = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        int tm, tn, ks;
        tile_coords(u, tiles_n, sh.ksplit, tm, tn, ks);
        const int kb0 = (int)((long long)kblocks * ks / sh.ksplit), kb1 = (int)((long long)kblocks * (ks + 1) / sh.ksplit);
        mbar_wait_sleep(&tempty[acc], aph ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait_sleep(&full[stage], ph);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * G::STAGE), sb = sa + G::A_BYTES;
#pragma unroll
          for (int k = 0; k < G::BK / G::UK; ++k)
            umma_ss<ELEM>(d, sdesc_sw128(sa + k * a_step, a_lbo, 1024), sdesc_sw128(sb + k * b_step, b_lbo, 1024), id,
                          (kb > kb0 || k > 0) ? 1u : 0u);
          umma_commit(&empty[stage]);   // the slot is free once these MMAs have read it
          if (++stage == G::S) { stage = 0; ph ^= 1; }
        }
        umma_commit(&tfull[acc]);       // accumulator complete
        if (++acc == 2) { acc = 0; aph ^= 1; }
      }
    }
  } else {
    // ===================== epilogue warps 2 .. 2 + 4 EW
    static_assert((BN / EW) % 16 == 0, "epilogue column groups are multiples of 16");
    const int q = warp & 3, r = q * 32 + lane, cg0 = ((warp - 2) >> 2) * (BN / EW);
    int acc = 0;
    uint32_t aph = 0, oph = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      int tm, tn, ks;
      tile_coords(u, tiles_n, sh.ksplit, tm, tn, ks);
      const int m = tm * G::BM + r;
      typename Epi::State st;
      epi.begin_tile(st, tm, tn, ks, m);
      mbar_wait_sleep(&tfull[acc], aph);
      tc_fence_after();
      if constexpr (Epi::kOpBytes > 0) mbar_wait_sleep(&opfull, oph);
      const int kb0 = (int)((long long)kblocks * ks / sh.ksplit), kb1 = (int)((long long)kblocks * (ks + 1) / sh.ksplit);
      const bool empty_k = kb1 <= kb0;   // no MMA ran: the accumulator is stale, the tile is zero
#pragma unroll 1
      for (int c = cg0; c < cg0 + BN / EW; c += 16) {
        float v[16];
        tmem_ld16(tmem + acc * BN + c + ((uint32_t)(q * 32) << 16), v);
        tmem_ld_wait();
        if (empty_k) {
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = 0.f;
        }
        const int n0 = tn * BN + c;
        if (n0 < sh.N) epi.chunk(st, sop, r, m, n0, c, ks, v, m < sh.M);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive_relaxed(&tempty[acc]);   // TMEM drained: nothing to publish
        if constexpr (Epi::kOpBytes > 0) mbar_arrive(&opfree);
      }
      oph ^= 1;
      epi.end_tile(st, tm, tn, ks, warp - 2, lane);   // slot: epilogue warp index
      if (++acc == 2) { acc = 0; aph ^= 1; }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<G::TMEM_COLS>(tmem);
}

// ---------------------------------------------------------------- CTA-pair kernel
// cta_group::2 tiles of 256 x BN: a cluster of two CTAs (a TPC pair); each CTA stages its own
// 128 rows of A and half of B's BN rows (the pair's tensor cores read B from both CTAs' shared
// memory), so per-CTA operand traffic drops from (16 KB + BN x 128 B) to (16 KB + BN x 64 B) per
// k-block.  Both CTAs' TMA loads complete on the LEADER's full barrier (the .cta_group::2 form
// of cp.async.bulk.tensor); the leader's single thread issues tcgen05.mma.cta_group::2 (M = 256)
// and commits, multicast, to both CTAs' empty / TMEM-full barriers; each CTA's epilogue reads
// its own 128 TMEM lanes and both arrive on the leader's TMEM-empty barrier.
SKB_DEV void tma_load_2d_pair(void* smem_dst, const CUtensorMap* tm, int c0, int c1, uint32_t leader_bar) {
  asm volatile("cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
               " [%0], [%1, {%2, %3}], [%4];"
               :: "r"(smem_u32(smem_dst)), "l"(tm), "r"(c0), "r"(c1), "r"(leader_bar) : "memory");
}
SKB_DEV void tma_load_3d_pair(void* smem_dst, const CUtensorMap* tm, int c0, int c1, int c2, uint32_t leader_bar) {
  asm volatile("cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
               " [%0], [%1, {%2, %3, %4}], [%5];"
               :: "r"(smem_u32(smem_dst)), "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(leader_bar) : "memory");
}
// Multicast form: the box lands at the same offset in every CTA of `mask`; each destination's
// bytes complete on its own pair leader's barrier (the .cta_group::2 signalling rule).
SKB_DEV void tma_load_3d_pair_mc(void* smem_dst, const CUtensorMap* tm, int c0, int c1, int c2, uint32_t leader_bar,
                                 uint16_t mask) {
  asm volatile("cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
               ".multicast::cluster [%0], [%1, {%2, %3, %4}], [%5], %6;"
               :: "r"(smem_u32(smem_dst)), "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(leader_bar), "h"(mask)
               : "memory");
}
template <int ELEM>
SKB_DEV void umma_ss_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t id, uint32_t accumulate) {
  if constexpr (ELEM == kBF16) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                 :: "r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(id), "r"(accumulate) : "memory");
  } else {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                 :: "r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(id), "r"(accumulate) : "memory");
  }
}
SKB_DEV void umma_commit_pair(uint64_t* bar, uint16_t mask = 3) {   // mask: the pair's cluster ranks
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
               :: "r"(smem_u32(bar)), "h"(mask) : "memory");
}

template <int ELEM, int BN, bool AMN, bool BMN, class Epi, int EW = 1>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(64 + 128 * EW, 1)
    gemm_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, const Shape sh,
                     const __grid_constant__ Epi epi) {
  using G = Geo<ELEM, BN / 2, Epi::kOpBytes>;   // per-CTA stage: A 128 rows + B BN / 2 rows
  static_assert(Epi::kOpBytes == 0, "pair kernel: epilogue operands not supported");
  static_assert((BN / EW) % 16 == 0, "epilogue column groups are multiples of 16");
  constexpr uint32_t TMEM_COLS = BN * 2 <= 256 ? 256 : 512;   // two BN-column accumulators
  if (epi.skip()) return;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[G::S], empty[G::S], tfull[2], tempty[2];
  __shared__ uint32_t tmem_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int pairs_m = (sh.M + 255) / 256, tiles_n = (sh.N + BN - 1) / BN;
  const int kblocks = (sh.K + G::BK - 1) / G::BK;
  const int units = pairs_m * tiles_n;
  const int npairs = gridDim.x / 2, pair = blockIdx.x / 2;

  if (threadIdx.x == 0) {
    for (int s = 0; s < G::S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 2 * 4 * EW); }
    fence_mbar_init();
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }
  if (warp == 1) tmem_alloc_pair<TMEM_COLS>(&tmem_s);
  tc_fence_before();
  __syncthreads();
  cluster_sync();   // both CTAs' barriers and TMEM ready before any cross-CTA traffic
  tc_fence_after();
  const uint32_t tmem = tmem_s;
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (warp == 0) {
    // ===================== TMA producer (both CTAs; completion on the leader's barrier)
    if (lane == 0) {
      int stage = 0;
      uint32_t ph = 0;
      for (int u = pair; u < units; u += npairs) {
        const int tm = u / tiles_n, tn = u % tiles_n;
        const int row0 = tm * 256 + (int)rank * 128, col0 = tn * BN + (int)rank * (BN / 2);
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait_sleep(&empty[stage], ph ^ 1);
          if (leader) mbar_arrive_expect_tx(&full[stage], 2 * G::STAGE);
          const uint32_t lbar = mapa(smem_u32(&full[stage]), 0);
          uint8_t* sa = smem + stage * G::STAGE;
          uint8_t* sb = sa + G::A_BYTES;
          const int k0 = kb * G::BK;
          if constexpr (!AMN) {
            tma_load_2d_pair(sa, &tmA, k0, row0, lbar);
          } else {
#pragma unroll
            for (int h = 0; h < G::BM / G::MNB; ++h)
              tma_load_2d_pair(sa + h * (G::BK * 128), &tmA, row0 + h * G::MNB, k0, lbar);
          }
          if constexpr (!BMN) {
            tma_load_2d_pair(sb, &tmB, k0, col0, lbar);
          } else {
#pragma unroll
            for (int h = 0; h < (BN / 2) / G::MNB; ++h)
              tma_load_2d_pair(sb + h * (G::BK * 128), &tmB, col0 + h * G::MNB, k0, lbar);
          }
          if (++stage == G::S) { stage = 0; ph ^= 1; }
        }
      }
      // drain: every slot's last commit has arrived here before the CTA may exit
      for (int i = 0; i < G::S; ++i) {
        mbar_wait_sleep(&empty[stage], ph ^ 1);
        if (++stage == G::S) { stage = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (leader CTA, one thread)
    if (leader && lane == 0) {
      constexpr uint32_t id = idesc(ELEM, 256, BN, AMN, BMN);
      constexpr uint32_t a_step = AMN ? G::UK * 128 : 32, b_step = BMN ? G::UK * 128 : 32;
      constexpr uint32_t a_lbo = AMN ? G::BK * 128 : 16, b_lbo = BMN ? G::BK * 128 : 16;
      int stage = 0, acc = 0;
      uint32_t ph = 0, aph = 0;
      for (int u = pair; u < units; u += npairs) {
        mbar_wait_sleep(&tempty[acc], aph ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * BN;
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait_sleep(&full[stage], ph);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * G::STAGE), sb = sa + G::A_BYTES;
#pragma unroll
          for (int k = 0; k < G::BK / G::UK; ++k)
            umma_ss_pair<ELEM>(d, sdesc_sw128(sa + k * a_step, a_lbo, 1024), sdesc_sw128(sb + k * b_step, b_lbo, 1024),
                               id, (kb > 0 || k > 0) ? 1u : 0u);
          umma_commit_pair(&empty[stage]);   // frees the slot in both CTAs
          if (++stage == G::S) { stage = 0; ph ^= 1; }
        }
        umma_commit_pair(&tfull[acc]);       // accumulator complete, in both CTAs
        if (++acc == 2) { acc = 0; aph ^= 1; }
      }
    }
  } else {
    // ===================== epilogue warps (each CTA: its 128 rows)
    const int q = warp & 3, r = q * 32 + lane, cg0 = ((warp - 2) >> 2) * (BN / EW);
    const uint32_t ltempty0 = mapa(smem_u32(&tempty[0]), 0), ltempty1 = mapa(smem_u32(&tempty[1]), 0);
    int acc = 0;
    uint32_t aph = 0;
    for (int u = pair; u < units; u += npairs) {
      const int tm = u / tiles_n, tn = u % tiles_n;
      const int m = tm * 256 + (int)rank * 128 + r;
      typename Epi::State st;
      epi.begin_tile(st, 2 * tm + (int)rank, tn, 0, m);
      mbar_wait_sleep(&tfull[acc], aph);
      tc_fence_after();
#pragma unroll 1
      for (int c = cg0; c < cg0 + BN / EW; c += 16) {
        float v[16];
        tmem_ld16(tmem + acc * BN + c + ((uint32_t)(q * 32) << 16), v);
        tmem_ld_wait();
        const int n0 = tn * BN + c;
        if (n0 < sh.N) epi.chunk(st, nullptr, r, m, n0, c, 0, v, m < sh.M);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_remote_arrive_relaxed(acc ? ltempty1 : ltempty0);
      epi.end_tile(st, 2 * tm + (int)rank, tn, 0, warp - 2, lane);
      if (++acc == 2) { acc = 0; aph ^= 1; }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();   // no CTA leaves while its peer may still signal its barriers
  tc_fence_after();
  if (warp == 1) tmem_dealloc_pair<TMEM_COLS>(tmem);
}

// ---------------------------------------------------------------- persistent step kernel
// A recurrence of `steps` dependent GEMMs D_s = A_s · B^T with the same B (weights) and
// tiling every step (BPTT, the forward While): one launch, one CTA per tile (all
// co-resident: cooperative launch), a grid-wide barrier between steps instead of a
// kernel boundary (no per-step launch, barrier init, TMEM allocation or descriptor
// fetch).  A_s is row block a_coord(s) of a 3-D tensor map [outer][rows][K] (time-major
// activations), B a 2-D K-major map.  Step s + 1 may load A only after every CTA's
// epilogue of step s has stored (the epilogue's global writes produce A_{s+1}): each
// epilogue warp publishes its tile with a fence + gpu-scope release add on `sync`; the
// producer acquires the count, orders its bulk reads after it with a proxy fence.
// Epi contract as above plus a_coord(s), k_empty(s) (no MMA at step s: D = 0), k_indep(s)
// (the leading K blocks of A_s that no earlier step writes: loaded and multiplied before the
// barrier) and the step index in begin_tile / chunk / end_tile / prefetch.  prefetch(st) may only read
// inputs and state written by this CTA's own epilogue (it is issued before the barrier).
SKB_DEV void tma_load_3d(void* smem_dst, const CUtensorMap* tm, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
               :: "r"(smem_u32(smem_dst)), "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)) : "memory");
}
SKB_DEV int ld_acquire_gpu_s32(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

struct StepShape {
  int M, N, K;
  int steps;
  const int* steps_dev;   // non-null: the step count is read from device memory (a device-side trip count)
  int* sync;      // zeroed before the launch
  long long* trace;   // optional: per-step globaltimer stamps of CTA trace_cta ([steps][8]), else null
  int trace_cta;
};
SKB_DEV void step_trace(const StepShape& sh, int st, int slot) {
  if (sh.trace && (int)blockIdx.x == sh.trace_cta) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    sh.trace[(long long)st * 8 + slot] = (long long)t;
  }
}

// KS = 2 or 4: every output tile is computed by KS CTAs of one cluster, each over 1/KS of K
// (fewer, wider tiles for the same CTA count: the activations / weights are re-read by fewer
// tiles).  The partial sums are reduce-scattered through distributed shared memory: each CTA
// writes every partner's BN / KS accumulator columns into that partner's receive buffer and
// runs the epilogue on its own columns (the epilogue functor sees tiles of BN / KS columns,
// tile index KS tn + ks).
// Step st + 1 arms its first stages with the weight (B) k-blocks before the grid
// barrier; the activation (A) halves follow once the barrier is passed.
// Steps-kernel geometry: behind the epilogue operands, KS > 1 keeps KS - 1 [128][BN / KS] fp32
// receive buffers for the partners' partial sums; the budget runs to the 227 KB limit.
template <int ELEM, int BN, class Epi, int KS>
using StepGeo = Geo<ELEM, BN, Epi::kOpBytes + 128u * (BN / KS) * 4u * (KS - 1), 224>;

template <int ELEM, int BN, class Epi, int EW, int KS = 1>
__global__ void __cluster_dims__(KS, 1, 1) __launch_bounds__(64 + 128 * EW, 1) gemm_steps_kernel(const __grid_constant__ CUtensorMap tmA,
                                                                     const __grid_constant__ CUtensorMap tmB,
                                                                     const StepShape sh,
                                                                     const __grid_constant__ Epi epi) {
  using G = StepGeo<ELEM, BN, Epi, KS>;
  constexpr int BNE = BN / KS;   // epilogue columns per CTA
  static_assert((BNE / EW) % 16 == 0, "epilogue column groups are multiples of 16");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sop = smem + G::S * G::STAGE;
  __shared__ uint64_t full[G::S], empty[G::S], tfull[2], tempty[2], opfull, opfree, xfull;
  __shared__ uint32_t tmem_s;
  // KS = 2: the partner CTA (the other K half of the tile, same cluster) writes its partial
  // sums of this CTA's columns straight into xrecv through distributed shared memory
  float* xrecv = reinterpret_cast<float*>(sop + Epi::kOpBytes);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles_n = (sh.N + BN - 1) / BN;
  const int kblocks = (sh.K + G::BK - 1) / G::BK;
  const int nunits = ((sh.M + G::BM - 1) / G::BM) * tiles_n * KS;
  const int per_step = nunits;   // barrier arrivals per step: one per unit (CTA tile)
  const int steps = sh.steps_dev ? *sh.steps_dev : sh.steps;

  if (threadIdx.x == 0) {
    for (int s = 0; s < G::S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 4 * EW); }
    mbar_init(&opfull, 1);
    mbar_init(&opfree, 4 * EW);
    mbar_init(&xfull, 1);   // KS > 1: one local expect_tx arrival per step; partners' st.async complete_tx
    fence_mbar_init();
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }
  if (warp == 1) tmem_alloc<G::TMEM_COLS>(&tmem_s);
  tc_fence_before();
  __syncthreads();
  if constexpr (KS > 1) cluster_sync();   // the partners' barriers exist before any DSMEM traffic
  tc_fence_after();
  const uint32_t tmem = tmem_s;

  if (warp == 0) {
    // ===================== TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t ph = 0, oph = 0;
      for (int st = 0; st < steps; ++st) {
        const int ac = epi.a_coord(st);
        const bool kz = epi.k_empty(st);
        for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
          const int t = u / KS, ks = u % KS, tm = t / tiles_n, tn = t % tiles_n;
          const int kb0 = kblocks * ks / KS, kb1 = kblocks * (ks + 1) / KS;
          const bool first = u == (int)blockIdx.x;
          if (first) step_trace(sh, st, 0);
          // before the grid barrier: the K blocks of A that do not depend on step st - 1
          // (epi.k_indep) in full -- their MMAs run while the previous step finishes --, then
          // the weights of the next blocks
          int npre = 0, nind = 0;
          int s0 = stage;
          if (st > 0 && first && !kz) {
            nind = max(0, min(kb1, epi.k_indep(st)) - kb0);
            for (int i = 0; i < nind; ++i) {
              mbar_wait_sleep(&empty[stage], ph ^ 1);
              mbar_arrive_expect_tx(&full[stage], G::STAGE);
              uint8_t* sa = smem + stage * G::STAGE;
              tma_load_3d(sa, &tmA, (kb0 + i) * G::BK, tm * G::BM, ac, &full[stage]);
              tma_load_2d(sa + G::A_BYTES, &tmB, (kb0 + i) * G::BK, tn * BN, &full[stage]);
              if (++stage == G::S) { stage = 0; ph ^= 1; }
            }
            s0 = stage;
            npre = min(G::S, kb1 - kb0 - nind);
            for (int i = 0; i < npre; ++i) {
              mbar_wait_sleep(&empty[stage], ph ^ 1);
              mbar_arrive_expect_tx(&full[stage], G::STAGE);
              tma_load_2d(smem + stage * G::STAGE + G::A_BYTES, &tmB, (kb0 + nind + i) * G::BK, tn * BN,
                          &full[stage]);
              if (++stage == G::S) { stage = 0; ph ^= 1; }
            }
          }
          if constexpr (Epi::kOpBytes > 0) {
            // the epilogue operands depend only on this CTA's own previous epilogue (its state
            // slice; opfree is arrived after its stores) and on inputs: no grid barrier needed
            mbar_wait_sleep(&opfree, oph ^ 1);
            fence_proxy_async_global();
            mbar_arrive_expect_tx(&opfull, Epi::kOpBytes);
            epi.prefetch(sop, st, tm, tn * KS + ks, &opfull);
            oph ^= 1;
          }
          if (st > 0 && first) {   // every unit of step st - 1 stored: A_st is ready
            const int want = st * per_step;
            while (ld_acquire_gpu_s32(sh.sync) < want) __nanosleep(64);
            fence_proxy_async_global();
          }
          if (first) step_trace(sh, st, 1);
          if (kz) continue;
          for (int kb = kb0 + nind; kb < kb1; ++kb) {
            const int i = kb - kb0 - nind;
            if (i < npre) {   // stage armed before the barrier: only its A half is missing
              const int sidx = (s0 + i) % G::S;
              tma_load_3d(smem + sidx * G::STAGE, &tmA, kb * G::BK, tm * G::BM, ac, &full[sidx]);
              continue;
            }
            mbar_wait_sleep(&empty[stage], ph ^ 1);
            mbar_arrive_expect_tx(&full[stage], G::STAGE);
            uint8_t* sa = smem + stage * G::STAGE;
            tma_load_3d(sa, &tmA, kb * G::BK, tm * G::BM, ac, &full[stage]);
            tma_load_2d(sa + G::A_BYTES, &tmB, kb * G::BK, tn * BN, &full[stage]);
            if (++stage == G::S) { stage = 0; ph ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (one thread)
    if (lane == 0) {
      constexpr uint32_t id = idesc(ELEM, G::BM, BN, false, false);
      int stage = 0, acc = 0;
      uint32_t ph = 0, aph = 0;
      for (int st = 0; st < steps; ++st) {
        const bool kz = epi.k_empty(st);
        for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
          const int ks = u % KS;
          const int kb0 = kblocks * ks / KS, kb1 = kblocks * (ks + 1) / KS;
          mbar_wait_sleep(&tempty[acc], aph ^ 1);
          tc_fence_after();
          const uint32_t d = tmem + acc * BN;
          if (!kz) {
            for (int kb = kb0; kb < kb1; ++kb) {
              mbar_wait_sleep(&full[stage], ph);
              if (kb == kb0) step_trace(sh, st, 2);
              tc_fence_after();
              const uint32_t sa = smem_u32(smem + stage * G::STAGE), sb = sa + G::A_BYTES;
#pragma unroll
              for (int k = 0; k < G::BK / G::UK; ++k)
                umma_ss<ELEM>(d, sdesc_sw128(sa + k * 32, 16, 1024), sdesc_sw128(sb + k * 32, 16, 1024), id,
                              (kb > kb0 || k > 0) ? 1u : 0u);
              umma_commit(&empty[stage]);
              if (++stage == G::S) { stage = 0; ph ^= 1; }
            }
          }
          step_trace(sh, st, 3);
          umma_commit(&tfull[acc]);
          if (++acc == 2) { acc = 0; aph ^= 1; }
        }
      }
    }
  } else {
    // ===================== epilogue warps
    const int q = warp & 3, r = q * 32 + lane, cg0 = ((warp - 2) >> 2) * (BNE / EW);
    int acc = 0;
    uint32_t aph = 0, oph = 0;
    typename Epi::State es;   // lives across steps: a CTA keeps its unit, so state may ride in registers
    for (int st = 0; st < steps; ++st) {
      const bool kz = epi.k_empty(st);
      for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
        const int t = u / KS, ks = u % KS, tm = t / tiles_n, tn = t % tiles_n, tv = tn * KS + ks;
        const int m = tm * G::BM + r;
        epi.begin_tile(es, st, tm, tv, m);
        mbar_wait_sleep(&tfull[acc], aph);
        if (warp == 2 && lane == 0) step_trace(sh, st, 4);
        tc_fence_after();
        const uint32_t dacc = tmem + acc * BN + ((uint32_t)(q * 32) << 16);
        if constexpr (KS > 1) {   // each partner's columns of the partial sums -> its xrecv (DSMEM)
          // (partner ks ^ o files this CTA's block in slot o - 1; cluster rank = ks).  st.async:
          // each 16-byte store completes its bytes on the receiver's xfull, whose one local
          // arrival per step announces the bytes to expect -- no release fence, no arrivals
          if (warp == 2 && lane == 0)
            mbar_arrive_expect_tx(&xfull, kz ? 0u : (uint32_t)((KS - 1) * 128 * BNE * 4));
          if (!kz) {   // (a step without MMAs still completes the phase: expect 0 bytes)
#pragma unroll 1
            for (int c = cg0; c < cg0 + BNE / EW; c += 16) {
              float v[KS - 1][16];
#pragma unroll
              for (int o = 1; o < KS; ++o) tmem_ld16(dacc + (ks ^ o) * BNE + c, v[o - 1]);   // all in flight
              tmem_ld_wait();
#pragma unroll
              for (int o = 1; o < KS; ++o) {
                const uint32_t peer = (uint32_t)(ks ^ o);
                const uint32_t xr = mapa(smem_u32(xrecv + ((o - 1) * 128 + r) * BNE), peer);
                const uint32_t xb = mapa(smem_u32(&xfull), peer);
#pragma unroll
                for (int i = 0; i < 16; i += 4) {   // 16-byte chunks XOR-swizzled by row: conflict-free
                  const uint32_t q = (uint32_t)((c + i) >> 2) ^ (uint32_t)(r & 7);
                  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];"
                               :: "r"(xr + q * 16), "f"(v[o - 1][i]), "f"(v[o - 1][i + 1]), "f"(v[o - 1][i + 2]),
                                  "f"(v[o - 1][i + 3]), "r"(xb) : "memory");
                }
              }
            }
          }
          mbar_wait_cluster(&xfull, st & 1);   // every partner's bytes landed
        }
        if constexpr (Epi::kOpBytes > 0) mbar_wait_sleep(&opfull, oph);
        if (warp == 2 && lane == 0) step_trace(sh, st, 5);
#pragma unroll 1
        for (int c = cg0; c < cg0 + BNE / EW; c += 16) {
          float v[16];
          tmem_ld16(dacc + ks * BNE + c, v);
          tmem_ld_wait();
          if (kz) {
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = 0.f;
          } else if constexpr (KS > 1) {
#pragma unroll
            for (int o = 1; o < KS; ++o) {   // partners in rank order ks ^ 1, ks ^ 2, ...
#pragma unroll
              for (int i = 0; i < 16; i += 4) {
                const uint32_t q = (uint32_t)((c + i) >> 2) ^ (uint32_t)(r & 7);
                const float4 p = *reinterpret_cast<const float4*>(xrecv + ((o - 1) * 128 + r) * BNE + q * 4);
                v[i] += p.x; v[i + 1] += p.y; v[i + 2] += p.z; v[i + 3] += p.w;
              }
            }
          }
          const int n0 = tn * BN + ks * BNE + c;
          if (n0 < sh.N) epi.chunk(es, sop, st, r, m, n0, c, v, m < sh.M);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive_relaxed(&tempty[acc]);   // TMEM drained: nothing to publish
          if constexpr (Epi::kOpBytes > 0) mbar_arrive(&opfree);
        }
        oph ^= 1;
        epi.end_tile(es, st, tm, tv, warp - 2, lane);
        if (warp == 2 && lane == 0) step_trace(sh, st, 6);
        // publish this CTA's stores of step st (the next step's A operand / state): one
        // arrival per CTA after the epilogue warps' named barrier
        // (no per-thread __threadfence: it is fence.sc.gpu + an L1 invalidate; the named barrier
        // orders every epilogue thread's stores before the single gpu-scope release below)
        named_bar_sync(1, 128 * EW);
        if (warp == 2 && lane == 0) {
          asm volatile("red.release.gpu.global.add.s32 [%0], %1;" :: "l"(sh.sync), "r"(1) : "memory");
          step_trace(sh, st, 7);
        }
        if (++acc == 2) { acc = 0; aph ^= 1; }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (KS > 1) cluster_sync();   // no CTA leaves while a partner may still write to it
  tc_fence_after();
  if (warp == 1) tmem_dealloc<G::TMEM_COLS>(tmem);
}

// CTA-pair form of gemm_steps_kernel: each pair of CTAs computes a 256 x BN tile of every
// step with cta_group::2 MMAs (the B = weights tile is split between the two CTAs: half the
// per-CTA weight traffic); the epilogue functor sees the CTA's own 128-row tile (tile row
// 2 tm + rank).  KS = 2: two pairs (one 4-CTA cluster) share each tile, pair ks taking the K
// blocks ks, ks + 2, ... (so both halves hold independent and dependent blocks), and the CTAs
// with the same rows reduce-scatter their partial sums through DSMEM (the functor then sees
// tiles of BN / 2 columns, index 2 tn + ks).  Cooperative launch with static cluster dims.
template <int ELEM, int BN, class Epi, int EW, int KS = 1>
using PairGeo = Geo<ELEM, BN / 2, Epi::kOpBytes + 128u * (BN / KS) * 4u * (KS - 1), (KS > 1 ? 224 : 212)>;

template <int ELEM, int BN, class Epi, int EW, int KS = 1, int MC = 1>
__global__ void __cluster_dims__(2 * KS * MC, 1, 1) __launch_bounds__(64 + 128 * EW, 1)
    gemm_steps_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                           const StepShape sh, const __grid_constant__ Epi epi) {
  using G = PairGeo<ELEM, BN, Epi, EW, KS>;
  static_assert(KS == 1 || MC == 1, "split-K and A multicast are separate variants");
  constexpr int BNE = BN / KS;   // epilogue columns per CTA
  static_assert((BNE / EW) % 16 == 0, "epilogue column groups are multiples of 16");
  constexpr uint32_t TMEM_COLS = BN * 2 <= 256 ? 256 : 512;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sop = smem + G::S * G::STAGE;
  float* xrecv = reinterpret_cast<float*>(sop + Epi::kOpBytes);   // KS = 2: the partner's partial sums
  __shared__ uint64_t full[G::S], empty[G::S], tfull[2], tempty[2], opfull, opfree, xfull;
  __shared__ uint32_t tmem_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = cluster_ctarank();
  const uint32_t rank = crank & 1u, base = crank & ~1u;   // rank in the pair; the pair's leader
  const int ks = KS > 1 ? (int)(crank >> 1) : 0;          // K share (0 when KS = 1)
  // MC = 2: two pairs (a 4-CTA cluster) on adjacent column tiles of the same rows; each CTA
  // loads half of its A box's rows and multicasts it to the CTA with the same rows in the
  // other pair, so every stage slot is refilled only after both pairs consumed it
  const int mcg = MC > 1 ? (int)(crank >> 1) : 0;
  const uint16_t amask = (uint16_t)((1u << crank) | (1u << (crank ^ 2u)));
  const bool leader = rank == 0;
  const int tiles_n = (sh.N + BN - 1) / BN;
  const int kblocks = (sh.K + G::BK - 1) / G::BK;
  const int nk = (kblocks - ks + KS - 1) / KS;   // this pair's K blocks: ks, ks + KS, ...
  const int tiles_c = tiles_n / MC;                            // column tiles per cluster
  const int units = ((sh.M + 255) / 256) * tiles_c;          // cluster tiles
  const int nclu = gridDim.x / (2 * KS * MC), clu = blockIdx.x / (2 * KS * MC);
  const int per_step = gridDim.x;   // one arrival per CTA per step
  const int steps = sh.steps_dev ? *sh.steps_dev : sh.steps;

  if (threadIdx.x == 0) {
    for (int s = 0; s < G::S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], MC); }
    for (int i = 0; i < 2; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 2 * 4 * EW); }
    mbar_init(&opfull, 1);
    mbar_init(&opfree, 4 * EW);
    mbar_init(&xfull, 1);   // KS = 2: one local expect_tx arrival per step; the partner's st.async bytes
    fence_mbar_init();
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }
  if (warp == 1) tmem_alloc_pair<TMEM_COLS>(&tmem_s);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = tmem_s;

  if (warp == 0) {
    // ===================== TMA producer (both CTAs; completion on the leader's barrier)
    if (lane == 0) {
      int stage = 0;
      uint32_t ph = 0, oph = 0;
      for (int st = 0; st < steps; ++st) {
        const int ac = epi.a_coord(st);
        const bool kz = epi.k_empty(st);
        for (int u = clu; u < units; u += nclu) {
          const int tm2 = u / tiles_c, tn = (u % tiles_c) * MC + mcg, tmv = 2 * tm2 + (int)rank;
          const int row0 = tmv * 128, col0 = tn * BN + (int)rank * (BN / 2);
          const bool first = u == clu;
          // A of K block kb into stage slot sa (completion on lbar): MC = 2 loads half the rows
          // and multicasts them to the same-rows CTA of the other pair
          auto load_a = [&](uint8_t* sa, int kb, uint32_t lbar) {
            if constexpr (MC > 1)
              tma_load_3d_pair_mc(sa + mcg * 64 * 128, &tmA, kb * G::BK, row0 + mcg * 64, ac, lbar, amask);
            else
              tma_load_3d_pair(sa, &tmA, kb * G::BK, row0, ac, lbar);
          };
          if (first) step_trace(sh, st, 0);
          int npre = 0, nind = 0;
          int s0 = stage;
          if (st > 0 && first && !kz) {   // independent A blocks in full, then weights (as above)
            const int kind = min(kblocks, epi.k_indep(st));
            nind = kind > ks ? min(nk, (kind - ks + KS - 1) / KS) : 0;
            for (int i = 0; i < nind; ++i) {
              const int kb = ks + KS * i;
              mbar_wait_sleep(&empty[stage], ph ^ 1);
              if (leader) mbar_arrive_expect_tx(&full[stage], 2 * G::STAGE);
              const uint32_t lbar = mapa(smem_u32(&full[stage]), base);
              uint8_t* sa = smem + stage * G::STAGE;
              load_a(sa, kb, lbar);
              tma_load_2d_pair(sa + G::A_BYTES, &tmB, kb * G::BK, col0, lbar);
              if (++stage == G::S) { stage = 0; ph ^= 1; }
            }
            s0 = stage;
            npre = min(G::S, nk - nind);
            for (int i = 0; i < npre; ++i) {
              mbar_wait_sleep(&empty[stage], ph ^ 1);
              if (leader) mbar_arrive_expect_tx(&full[stage], 2 * G::STAGE);
              tma_load_2d_pair(smem + stage * G::STAGE + G::A_BYTES, &tmB, (ks + KS * (nind + i)) * G::BK, col0,
                               mapa(smem_u32(&full[stage]), base));
              if (++stage == G::S) { stage = 0; ph ^= 1; }
            }
          }
          if constexpr (Epi::kOpBytes > 0) {   // CTA-local operands of this CTA's 128 rows
            mbar_wait_sleep(&opfree, oph ^ 1);
            fence_proxy_async_global();
            mbar_arrive_expect_tx(&opfull, Epi::kOpBytes);
            epi.prefetch(sop, st, tmv, tn * KS + ks, &opfull);
            oph ^= 1;
          }
          if (st > 0 && first) {
            const int want = st * per_step;
            while (ld_acquire_gpu_s32(sh.sync) < want) __nanosleep(64);
            fence_proxy_async_global();
          }
          if (first) step_trace(sh, st, 1);
          if (kz) continue;
          for (int i = nind; i < nk; ++i) {
            const int kb = ks + KS * i;
            if (i - nind < npre) {
              const int sidx = (s0 + i - nind) % G::S;
              load_a(smem + sidx * G::STAGE, kb, mapa(smem_u32(&full[sidx]), base));
              continue;
            }
            mbar_wait_sleep(&empty[stage], ph ^ 1);
            if (leader) mbar_arrive_expect_tx(&full[stage], 2 * G::STAGE);
            const uint32_t lbar = mapa(smem_u32(&full[stage]), base);
            uint8_t* sa = smem + stage * G::STAGE;
            load_a(sa, kb, lbar);
            tma_load_2d_pair(sa + G::A_BYTES, &tmB, kb * G::BK, col0, lbar);
            if (++stage == G::S) { stage = 0; ph ^= 1; }
          }
        }
      }
      for (int i = 0; i < G::S; ++i) {   // drain the last commits before the CTA may exit
        mbar_wait_sleep(&empty[stage], ph ^ 1);
        if (++stage == G::S) { stage = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (leader CTA, one thread)
    if (leader && lane == 0) {
      constexpr uint32_t id = idesc(ELEM, 256, BN, false, false);
      const uint16_t pmask = (uint16_t)(3u << base);   // commits reach both CTAs of this pair
      const uint16_t emask = MC > 1 ? (uint16_t)0xF : pmask;   // MC = 2: stage slots are shared by both pairs
      int stage = 0, acc = 0;
      uint32_t ph = 0, aph = 0;
      for (int st = 0; st < steps; ++st) {
        const bool kz = epi.k_empty(st);
        for (int u = clu; u < units; u += nclu) {
          mbar_wait_sleep(&tempty[acc], aph ^ 1);
          tc_fence_after();
          const uint32_t d = tmem + acc * BN;
          if (!kz) {
            for (int i = 0; i < nk; ++i) {
              mbar_wait_sleep(&full[stage], ph);
              if (i == 0) step_trace(sh, st, 2);
              tc_fence_after();
              const uint32_t sa = smem_u32(smem + stage * G::STAGE), sb = sa + G::A_BYTES;
#pragma unroll
              for (int k = 0; k < G::BK / G::UK; ++k)
                umma_ss_pair<ELEM>(d, sdesc_sw128(sa + k * 32, 16, 1024), sdesc_sw128(sb + k * 32, 16, 1024), id,
                                   (i > 0 || k > 0) ? 1u : 0u);
              umma_commit_pair(&empty[stage], emask);
              if (++stage == G::S) { stage = 0; ph ^= 1; }
            }
          }
          step_trace(sh, st, 3);
          umma_commit_pair(&tfull[acc], pmask);
          if (++acc == 2) { acc = 0; aph ^= 1; }
        }
      }
    }
  } else {
    // ===================== epilogue warps (each CTA: its 128 rows)
    const int q = warp & 3, r = q * 32 + lane, cg0 = ((warp - 2) >> 2) * (BNE / EW);
    const uint32_t ltempty0 = mapa(smem_u32(&tempty[0]), base), ltempty1 = mapa(smem_u32(&tempty[1]), base);
    int acc = 0;
    uint32_t aph = 0, oph = 0;
    typename Epi::State es;   // lives across steps: a pair keeps its unit, so state may ride in registers
    for (int st = 0; st < steps; ++st) {
      const bool kz = epi.k_empty(st);
      for (int u = clu; u < units; u += nclu) {
        const int tm2 = u / tiles_c, tn = (u % tiles_c) * MC + mcg, tmv = 2 * tm2 + (int)rank, tv = tn * KS + ks;
        const int m = tmv * 128 + r;
        epi.begin_tile(es, st, tmv, tv, m);
        mbar_wait_sleep(&tfull[acc], aph);
        if (warp == 2 && lane == 0) step_trace(sh, st, 4);
        tc_fence_after();
        const uint32_t dacc = tmem + acc * BN + ((uint32_t)(q * 32) << 16);
        if constexpr (KS == 2) {   // the other pair's columns of these rows -> its xrecv (DSMEM, st.async)
          const uint32_t peer = crank ^ 2u;
          if (warp == 2 && lane == 0) mbar_arrive_expect_tx(&xfull, kz ? 0u : (uint32_t)(128 * BNE * 4));
          if (!kz) {
            const uint32_t xr = mapa(smem_u32(xrecv + r * BNE), peer), xb = mapa(smem_u32(&xfull), peer);
#pragma unroll 1
            for (int c = cg0; c < cg0 + BNE / EW; c += 16) {
              float v[16];
              tmem_ld16(dacc + (ks ^ 1) * BNE + c, v);
              tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 16; i += 4) {   // 16-byte chunks XOR-swizzled by row: conflict-free
                const uint32_t qq = (uint32_t)((c + i) >> 2) ^ (uint32_t)(r & 7);
                asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];"
                             :: "r"(xr + qq * 16), "f"(v[i]), "f"(v[i + 1]), "f"(v[i + 2]), "f"(v[i + 3]), "r"(xb)
                             : "memory");
              }
            }
          }
          mbar_wait_cluster(&xfull, st & 1);   // the partner's bytes landed
        }
        if constexpr (Epi::kOpBytes > 0) mbar_wait_sleep(&opfull, oph);
        if (warp == 2 && lane == 0) step_trace(sh, st, 5);
#pragma unroll 1
        for (int c = cg0; c < cg0 + BNE / EW; c += 16) {
          float v[16];
          tmem_ld16(dacc + ks * BNE + c, v);
          tmem_ld_wait();
          if (kz) {
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = 0.f;
          } else if constexpr (KS == 2) {
#pragma unroll
            for (int i = 0; i < 16; i += 4) {
              const uint32_t qq = (uint32_t)((c + i) >> 2) ^ (uint32_t)(r & 7);
              const float4 p = *reinterpret_cast<const float4*>(xrecv + r * BNE + qq * 4);
              v[i] += p.x; v[i + 1] += p.y; v[i + 2] += p.z; v[i + 3] += p.w;
            }
          }
          const int n0 = tn * BN + ks * BNE + c;
          if (n0 < sh.N) epi.chunk(es, sop, st, r, m, n0, c, v, m < sh.M);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_remote_arrive_relaxed(acc ? ltempty1 : ltempty0);
          if constexpr (Epi::kOpBytes > 0) mbar_arrive(&opfree);
        }
        oph ^= 1;
        epi.end_tile(es, st, tmv, tv, warp - 2, lane);
        if (warp == 2 && lane == 0) step_trace(sh, st, 6);
        // (no per-thread __threadfence: it is fence.sc.gpu + an L1 invalidate; the named barrier
        // orders every epilogue thread's stores before the single gpu-scope release below)
        named_bar_sync(1, 128 * EW);
        if (warp == 2 && lane == 0) {
          asm volatile("red.release.gpu.global.add.s32 [%0], %1;" :: "l"(sh.sync), "r"(1) : "memory");
          step_trace(sh, st, 7);
        }
        if (++acc == 2) { acc = 0; aph ^= 1; }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  if (warp == 1) tmem_dealloc_pair<TMEM_COLS>(tmem);
}

// ---------------------------------------------------------------- epilogues
// C[m, n] (+)= D, fp32, row-major with ldc; with ksplit > 1 each split writes its own
// partial plane C + ks * split_stride (reduced by reduce_splits).
struct EpiStore {
  static constexpr uint32_t kOpBytes = 0;
  struct State {};
  float* C;
  long long ldc;
  long long split_stride;
  int beta;
  SKB_DEV bool skip() const { return false; }
  SKB_DEV bool ops_on() const { return false; }
  SKB_DEV void prefetch(uint8_t*, int, int, uint64_t*) const {}
  SKB_DEV void begin_tile(State&, int, int, int, int) const {}
  SKB_DEV void chunk(State&, const uint8_t*, int, int m, int n0, int, int ks, const float (&v)[16], bool row_ok) const {
    if (!row_ok) return;
    float* p = C + (long long)ks * split_stride + (long long)m * ldc + n0;
#pragma unroll
    for (int i = 0; i < 16; i += 4) {
      float4 o = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
      if (beta) {
        const float4 c = *reinterpret_cast<const float4*>(p + i);
        o.x += c.x; o.y += c.y; o.z += c.z; o.w += c.w;
      }
      *reinterpret_cast<float4*>(p + i) = o;
    }
  }
  SKB_DEV void end_tile(State&, int, int, int, int, int) const {}
};

// ---------------------------------------------------------------- host side
// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda symbol use).
bool encode_2d(CUtensorMap* tm, int elem, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld_elems,
               uint32_t box_inner, uint32_t box_outer);

// 3-D map [d2][d1][d0] (d0 contiguous; s1 / s2 element strides of d1 / d2), 128-byte swizzle.
bool encode_3d(CUtensorMap* tm, int elem, const void* ptr, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1_elems,
               uint64_t s2_elems, uint32_t b0, uint32_t b1, uint32_t b2);

// Launch configuration for a GEMM with the given operand layouts (see the header).
struct Problem {
  int elem;           // kBF16 / kTF32
  bool a_mn, b_mn;    // A stored [K, M] / B stored [K, N]
  const void* A; long long lda;
  const void* B; long long ldb;
  int M, N, K;
};

// Build the two tensor maps of a problem for tile width BN.
template <int ELEM, int BN>
bool make_maps(const Problem& p, CUtensorMap* ta, CUtensorMap* tb) {
  using G = Geo<ELEM, BN>;
  const bool oka = p.a_mn ? encode_2d(ta, ELEM, p.A, p.M, p.K, p.lda, G::MNB, G::BK)
                          : encode_2d(ta, ELEM, p.A, p.K, p.M, p.lda, G::BK, G::BM);
  const bool okb = p.b_mn ? encode_2d(tb, ELEM, p.B, p.N, p.K, p.ldb, G::MNB, G::BK)
                          : encode_2d(tb, ELEM, p.B, p.K, p.N, p.ldb, G::BK, BN);
  return oka && okb;
}

int num_sms();

// Launch gemm_kernel<ELEM, BN, AMN, BMN, Epi> persistent over min(units, SMs) CTAs.
template <int ELEM, int BN, bool AMN, bool BMN, class Epi, bool A2 = false, int EW = 1>
int launch(const CUtensorMap& ta, const CUtensorMap& tb, const Shape& sh, const Epi& epi, cudaStream_t st,
           int max_ctas = 0, const CUtensorMap* ta2 = nullptr, bool pdl = false) {
  using G = Geo<ELEM, BN, Epi::kOpBytes>;
  auto kern = gemm_kernel<ELEM, BN, AMN, BMN, Epi, A2, EW>;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM) != cudaSuccess)
      return 2;
    attr = true;
  }
  const int units = ((sh.M + G::BM - 1) / G::BM) * ((sh.N + BN - 1) / BN) * sh.ksplit;
  int grid = num_sms();
  if (max_ctas > 0 && max_ctas < grid) grid = max_ctas;
  if (units < grid) grid = units;
  if (grid < 1) return 0;
  if (!pdl) {
    kern<<<grid, 64 + 128 * EW, G::SMEM, st>>>(ta, tb, ta2 ? *ta2 : ta, sh, epi);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute lattr[1];
  lattr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  lattr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(64 + 128 * EW);
  cfg.dynamicSmemBytes = G::SMEM;
  cfg.stream = st;
  cfg.attrs = lattr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, ta, tb, ta2 ? *ta2 : ta, sh, epi) == cudaSuccess ? 0 : 2;
}

// Persistent CTA-pair GEMM: pairs over (256-row, BN-column) tiles.
template <int ELEM, int BN, bool AMN, bool BMN, class Epi, int EW = 1>
int launch_pair(const CUtensorMap& ta, const CUtensorMap& tb, const Shape& sh, const Epi& epi, cudaStream_t st) {
  using G = Geo<ELEM, BN / 2, Epi::kOpBytes>;
  auto kern = gemm_pair_kernel<ELEM, BN, AMN, BMN, Epi, EW>;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM) != cudaSuccess)
      return 2;
    attr = true;
  }
  const int units = ((sh.M + 255) / 256) * ((sh.N + BN - 1) / BN);
  int pairs = num_sms() / 2;
  if (units < pairs) pairs = units;
  if (pairs < 1) return 0;
  kern<<<2 * pairs, 64 + 128 * EW, G::SMEM, st>>>(ta, tb, sh, epi);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;
}

// Clusters of `kern` (launch shape `cfg`) that can be resident at once: the persistent step
// kernels need every cluster co-resident (cached per kernel; INT_MAX if the query fails).
template <class K>
int resident_clusters(K kern, const cudaLaunchConfig_t& cfg) {
  static const void* key[16];   // per kernel (instantiations of one signature share K)
  static int val[16], cnt = 0;
  for (int i = 0; i < cnt; ++i)
    if (key[i] == (const void*)kern) return val[i];
  cudaLaunchConfig_t q = cfg;
  q.attrs = nullptr;
  q.numAttrs = 0;
  int c = 0;
  const int n = cudaOccupancyMaxActiveClusters(&c, (void*)kern, &q) == cudaSuccess ? c : 0x7fffffff;
  cudaGetLastError();
  if (cnt < 16) { key[cnt] = (const void*)kern; val[cnt] = n; ++cnt; }
  return n;
}

// Cooperative launch of gemm_steps_pair_kernel: one CTA pair per 256-row tile, all resident.
template <int ELEM, int BN, class Epi, int EW, int KS = 1, int MC = 1>
int launch_steps_pair(const CUtensorMap& ta, const CUtensorMap& tb, const StepShape& sh, const Epi& epi,
                      cudaStream_t st) {
  using G = PairGeo<ELEM, BN, Epi, EW, KS>;
  auto kern = gemm_steps_pair_kernel<ELEM, BN, Epi, EW, KS, MC>;
  if (((sh.N + BN - 1) / BN) % MC) return 3;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM) != cudaSuccess)
      return 2;
    attr = true;
  }
  const int units = ((sh.M + 255) / 256) * ((sh.N + BN - 1) / BN);
  if (2 * KS * units > num_sms()) return 3;   // (units: pair tiles; MC pairs per cluster)
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute lattr[1];
  lattr[0].id = cudaLaunchAttributeCooperative;
  lattr[0].val.cooperative = 1;
  cfg.gridDim = dim3(2 * KS * units);
  cfg.blockDim = dim3(64 + 128 * EW);
  cfg.dynamicSmemBytes = G::SMEM;
  cfg.stream = st;
  cfg.attrs = lattr;
  cfg.numAttrs = 1;
  if (units / MC > resident_clusters(kern, cfg)) return 3;   // not all clusters co-resident
  return cudaLaunchKernelEx(&cfg, kern, ta, tb, sh, epi) == cudaSuccess ? 0 : 2;
}

// Cooperative launch of gemm_steps_kernel: one CTA per unit (tile x K half), all resident.
template <int ELEM, int BN, class Epi, int EW, int KS = 1>
int launch_steps(const CUtensorMap& ta, const CUtensorMap& tb, const StepShape& sh, const Epi& epi, cudaStream_t st) {
  using G = StepGeo<ELEM, BN, Epi, KS>;
  auto kern = gemm_steps_kernel<ELEM, BN, Epi, EW, KS>;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM) != cudaSuccess)
      return 2;
    attr = true;
  }
  const int nunits = ((sh.M + G::BM - 1) / G::BM) * ((sh.N + BN - 1) / BN) * KS;
  if (nunits > num_sms()) return 3;   // one resident CTA per unit
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute lattr[1];
  lattr[0].id = cudaLaunchAttributeCooperative;
  lattr[0].val.cooperative = 1;
  cfg.gridDim = dim3(nunits);
  cfg.blockDim = dim3(64 + 128 * EW);
  cfg.dynamicSmemBytes = G::SMEM;
  cfg.stream = st;
  cfg.attrs = lattr;
  cfg.numAttrs = 1;
  if (nunits / KS > resident_clusters(kern, cfg)) return 3;   // not all clusters co-resident
  return cudaLaunchKernelEx(&cfg, kern, ta, tb, sh, epi) == cudaSuccess ? 0 : 2;
}

}  // namespace gemm
}  // namespace skb
