// sm100.cuh — hand-written Blackwell (sm_100a) primitives used by every skb kernel.
//
// tcgen05 (UMMA issue, TMEM alloc/ld, commit), mbarrier, cluster/DSMEM and
// bulk-async-copy wrappers as inline PTX.  No CUTLASS/CuTe: the encodings
// below (instruction descriptor, shared-memory matrix descriptor, TMEM
// addressing) are written out by hand and pinned by the GPU self-test
// (`skb_diag_umma_gemm`, tests/test_gpu_kernels.py).
#pragma once
#include <cstdint>
#include <cuda_fp16.h>

#define SKB_DEV __device__ __forceinline__

namespace skb {

// ---------------------------------------------------------------- basics
SKB_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
SKB_DEV uint32_t lane_id() { uint32_t r; asm volatile("mov.u32 %0, %%laneid;" : "=r"(r)); return r; }
SKB_DEV uint32_t cluster_ctarank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
SKB_DEV uint32_t cluster_id_x() { uint32_t r; asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r)); return r; }
SKB_DEV uint32_t nclusters_x() { uint32_t r; asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r)); return r; }

SKB_DEV void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n"
               "barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
SKB_DEV void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" :: "r"(id), "r"(nthreads) : "memory");
}
// Map a local shared::cta address to the same offset in CTA `rank` of the cluster.
SKB_DEV uint32_t mapa(uint32_t local_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_addr), "r"(rank));
  return r;
}

// ---------------------------------------------------------------- mbarrier
SKB_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count) : "memory");
}
SKB_DEV void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
SKB_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(bar)) : "memory");
}
// A pure "done" signal (no memory to publish, e.g. TMEM drained after tcgen05.wait::ld +
// tcgen05.fence::before_thread_sync): no release fence, so it never waits on the thread's
// outstanding global stores.
SKB_DEV void mbar_arrive_relaxed(uint64_t* bar) {
  asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" :: "r"(smem_u32(bar)) : "memory");
}
SKB_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
               :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// Arrive (+expect_tx) on an mbarrier living in another CTA of the cluster.
SKB_DEV void mbar_remote_arrive_expect_tx(uint32_t cluster_bar_addr, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cluster.shared::cluster.b64 _, [%0], %1;"
               :: "r"(cluster_bar_addr), "r"(bytes) : "memory");
}
SKB_DEV void mbar_remote_arrive(uint32_t cluster_bar_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];"
               :: "r"(cluster_bar_addr) : "memory");
}
// Relaxed remote arrival: a pure "done" signal with nothing to publish (no
// release fence, so it never waits on the issuing thread's outstanding stores).
SKB_DEV void mbar_remote_arrive_relaxed(uint32_t cluster_bar_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];"
               :: "r"(cluster_bar_addr) : "memory");
}
SKB_DEV bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\t"
               "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
               "selp.u32 %0, 1, 0, p;\n\t}"
               : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}
SKB_DEV bool mbar_try_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\t"
               "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
               "selp.u32 %0, 1, 0, p;\n\t}"
               : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}
SKB_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {}
}
// try_wait with a long suspend-time hint: the waiting warp sleeps until the phase
// completes instead of re-polling (frees issue slots for the warps doing work).
SKB_DEV void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  do {
    asm volatile("{\n\t.reg .pred p;\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity), "r"(0x989680u) : "memory");
  } while (!ok);
}
SKB_DEV void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait_cluster(bar, parity)) {}
}

// ---------------------------------------------------------------- async proxy / bulk copies
SKB_DEV void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// global -> own shared memory, completion counted in bytes on `bar`.
SKB_DEV void bulk_g2s(void* smem_dst, const void* gmem_src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(smem_u32(smem_dst)), "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// own shared memory -> shared memory of a peer CTA (DSMEM), completion on the
// peer's mbarrier.  dst/bar are shared::cluster addresses (from mapa).
SKB_DEV void bulk_s2peer(uint32_t cluster_dst, const void* smem_src, uint32_t bytes, uint32_t cluster_bar) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(cluster_dst), "r"(smem_u32(smem_src)), "r"(bytes), "r"(cluster_bar) : "memory");
}
// global -> the same shared-memory offset in every CTA of `cta_mask`, completion
// counted on the mbarrier at the same offset in each destination CTA.
SKB_DEV void bulk_g2s_multicast(void* smem_dst, const void* gmem_src, uint32_t bytes, uint64_t* bar,
                                uint16_t cta_mask) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
               " [%0], [%1], %2, [%3], %4;"
               :: "r"(smem_u32(smem_dst)), "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar)), "h"(cta_mask)
               : "memory");
}
// Bulk prefetch of [gmem, gmem + bytes) into L2 (bytes a multiple of 16).
SKB_DEV void bulk_prefetch_l2(const void* gmem, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(gmem), "r"(bytes) : "memory");
}
SKB_DEV void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
SKB_DEV void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
SKB_DEV void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
SKB_DEV void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }

// ---------------------------------------------------------------- TMEM
// One full warp allocates `ncols` (power of two >= 32) columns and stores the
// base address to *dst_smem.
template <uint32_t NCOLS>
SKB_DEV void tmem_alloc(uint32_t* dst_smem) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
               :: "r"(smem_u32(dst_smem)), "n"(NCOLS) : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <uint32_t NCOLS>
SKB_DEV void tmem_dealloc(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(taddr), "n"(NCOLS) : "memory");
}
SKB_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
SKB_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[smem] * B[smem]^T   (kind::f16: fp16/bf16 in, fp32 accumulate)
SKB_DEV void umma_f16_ss(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile("{\n\t.reg .pred p;\n\t"
               "setp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
               :: "r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate) : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem]^T  (A operand resident in tensor memory)
SKB_DEV void umma_f16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile("{\n\t.reg .pred p;\n\t"
               "setp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
               :: "r"(tmem_d), "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate) : "memory");
}
// Warp-collective variants: every lane of the warp executes them with identical
// (warp-uniform) operands and one elected lane issues, so the compiler keeps
// descriptors in uniform registers instead of a per-lane R2UR loop.
SKB_DEV void umma_f16_ts_warp(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile("{\n\t.reg .pred p, e;\n\t.reg .b32 rx;\n\t"
               "elect.sync rx|e, 0xffffffff;\n\t"
               "setp.ne.b32 p, %4, 0;\n\t"
               "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
               :: "r"(tmem_d), "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate) : "memory");
}
SKB_DEV void umma_commit_warp(uint64_t* bar) {
  asm volatile("{\n\t.reg .pred e;\n\t.reg .b32 rx;\n\t"
               "elect.sync rx|e, 0xffffffff;\n\t"
               "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}"
               :: "r"(smem_u32(bar)) : "memory");
}
// The same, arriving on the mbarrier at this offset in every CTA of `cta_mask`.
SKB_DEV void umma_commit_warp_multicast(uint64_t* bar, uint16_t cta_mask) {
  asm volatile("{\n\t.reg .pred e;\n\t.reg .b32 rx;\n\t"
               "elect.sync rx|e, 0xffffffff;\n\t"
               "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}"
               :: "r"(smem_u32(bar)), "h"(cta_mask) : "memory");
}
// Warp-wide store of 8 consecutive 32-bit columns into the warp's 32 TMEM lanes.
SKB_DEV void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
               :: "r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]),
                  "r"(r[6]), "r"(r[7]) : "memory");
}
SKB_DEV void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// Arrive once on `bar` when all previously issued tcgen05.mma of this thread complete.
SKB_DEV void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
               :: "r"(smem_u32(bar)) : "memory");
}

// 32 lanes x 16 columns of 32-bit words: thread i of the warp receives TMEM
// lane (quarter*32 + i), columns [col, col+16).
SKB_DEV void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 "
               "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]),
                 "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
               : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
SKB_DEV void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// ---------------------------------------------------------------- CTA pairs (cta_group::2)
// A pair is two CTAs of a cluster with ranks 2p, 2p+1.  One M=256 MMA issued by the
// even (leader) CTA computes D[128 x N] in each CTA's TMEM: A rows [128r, 128r+128)
// come from CTA r's TMEM (same address in both), B columns [r*N/2, (r+1)*N/2) from
// CTA r's shared memory (same offset in both).  TMEM of a pair is allocated and freed
// by one warp of the same index in each CTA.
template <uint32_t NCOLS>
SKB_DEV void tmem_alloc_pair(uint32_t* dst_smem) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
               :: "r"(smem_u32(dst_smem)), "n"(NCOLS) : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
template <uint32_t NCOLS>
SKB_DEV void tmem_dealloc_pair(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" :: "r"(taddr), "n"(NCOLS) : "memory");
}
// Warp-collective pair MMA (leader CTA only), A from TMEM.
SKB_DEV void umma_f16_ts_pair_warp(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                   uint32_t accumulate) {
  asm volatile("{\n\t.reg .pred p, e;\n\t.reg .b32 rx;\n\t"
               "elect.sync rx|e, 0xffffffff;\n\t"
               "setp.ne.b32 p, %4, 0;\n\t"
               "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
               :: "r"(tmem_d), "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate) : "memory");
}
// Completion of the leader's previously issued pair MMAs, arriving on the mbarrier at
// this offset in every CTA of `cta_mask`.
SKB_DEV void umma_commit_pair_warp(uint64_t* bar, uint16_t cta_mask) {
  asm volatile("{\n\t.reg .pred e;\n\t.reg .b32 rx;\n\t"
               "elect.sync rx|e, 0xffffffff;\n\t"
               "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}"
               :: "r"(smem_u32(bar)), "h"(cta_mask) : "memory");
}
// 16 TMEM lanes x 256 bits, .x2 (16 columns): thread i receives lanes base + i/4 and
// base + 8 + i/4, columns 2(i%4), 2(i%4)+1 and 8 + 2(i%4), 9 + 2(i%4):
//   v[0] (l, c0)  v[1] (l, c0+1)  v[2] (l+8, c0)  v[3] (l+8, c0+1)
//   v[4] (l, c0+8) v[5] (l, c0+9) v[6] (l+8, c0+8) v[7] (l+8, c0+9)
SKB_DEV void tmem_ld_16x256b_x2(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
// .x4: 32 columns; v[4j..4j+3] as .x2's v[0..3] for columns 8j + ...
SKB_DEV void tmem_ld_16x256b_x4(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x4.b32 "
               "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]),
                 "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
               : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// ---------------------------------------------------------------- descriptors
// Instruction descriptor, kind::f16, fp16 x fp16 -> fp32, both operands K-major.
//   bits [4,6) c_format (1 = F32), [7,10) a_format (0 = F16), [10,13) b_format,
//   [15] a_major, [16] b_major (0 = K), [17,23) N>>3, [24,29) M>>4.
__host__ __device__ constexpr uint32_t idesc_f16_f32(uint32_t M, uint32_t N) {
  return (1u << 4) | (0u << 7) | (0u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

// Shared-memory matrix descriptor for a K-major operand without swizzle
// ("interleaved" canonical layout): the operand is tiled into 8x8 core
// matrices (8 rows x 16 bytes, rows 16 B apart, 128 B contiguous).
//   lbo = byte distance between core matrices adjacent along K
//   sbo = byte distance between core matrices adjacent along M/N
//   bits [0,14) addr>>4, [16,30) lbo>>4, [32,46) sbo>>4, [46,48) version=1 (sm100),
//   [49,52) base offset 0, [52] lbo mode 0, [61,64) layout 0 (SWIZZLE_NONE).
SKB_DEV uint64_t sdesc_kmajor_noswz(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

// Byte offset of element (r, k) of a K-major fp16 operand in the core-matrix
// layout used throughout skb: core matrix (k/8, r/8) at (k/8)*lbo + (r/8)*sbo.
SKB_DEV uint32_t cm_offset(uint32_t r, uint32_t k, uint32_t lbo, uint32_t sbo) {
  return (k >> 3) * lbo + (r >> 3) * sbo + (r & 7) * 16 + (k & 7) * 2;
}

// ---------------------------------------------------------------- math
SKB_DEV float sigmoid_f(float x) {
  // Same branch structure as the reference's stable sigmoid
  // (reference pkg/src/stagekit/graph/tensor.py:403-407), in fp32.
  if (x >= 0.f) return 1.f / (1.f + __expf(-x));
  float e = __expf(x);
  return e / (1.f + e);
}
SKB_DEV float tanh_f(float x) { return tanhf(x); }

}  // namespace skb
