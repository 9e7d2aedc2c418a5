// stream.cu — vector-stream region executor: staged While/Cond programs whose
// tensors are scalars or vectors of one large shape (L-BFGS, SGD loops,
// element-wise iterative solvers; BASELINE config C4).
//
// The generic region VM (vm.cu) separates every instruction with a grid
// barrier.  Here the execution model is split by value class instead:
//
//  * Scalars, lists and control flow are executed REDUNDANTLY by lane 0 of
//    warp 0 in every CTA, on a private copy of the scalar/list state kept in
//    shared memory (`W`, one int64 word per scalar slot, buffer ids for vector
//    slots, [len, items...] for list slots).  Every CTA computes the same
//    values and takes the same branches, so loop predicates are decided on
//    chip with no host round trip and no grid barrier.
//  * Vector values are immutable, reference-counted HBM buffers.  Element e of
//    every vector always belongs to the same thread (tile e/1024 -> CTA
//    (e/1024) % grid), so element-wise instructions never need a barrier: a
//    thread only ever reads elements it wrote itself.
//  * A fused element-wise group (VEXEC, compiled by stream.py from a chain of
//    reference nodes) streams its vector operands through shared memory with a
//    3-stage cp.async pipeline, evaluates a small stack program per element
//    with the top of stack in registers, stores its materialised results and
//    accumulates its reductions.
//  * A reduction is the only cross-CTA exchange: per-CTA partials, one grid
//    arrival, then every CTA combines the partials in the same fixed order
//    (RFIN) and so holds a bit-identical scalar.
//
// Semantics follow the reference kernels (pkg/src/stagekit/graph/tensor.py):
// f64/i64/bool words, `/` always f64 (tensor.py:269-270), Python floor-mod,
// DivisionByZero on a zero divisor even for floats (tensor.py:235-241),
// stable sigmoid (:403-407), scalar-condition whole-tensor Where (:367-368),
// list indexing with negative wrap and IndexOutOfRange (execute.py:240-249),
// max_iterations checked after a true test (execute.py:232-234).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include "skb_internal.h"


namespace {

constexpr int TPB = 512;
// A CTA owns whole 4096-element units of every vector (unit u -> CTA u mod grid).
// A group processes a unit as one tile of 8 elements per thread (32 KB per
// operand per stage) when two such stages fit in shared memory, else as two
// 2048-element tiles of 4 per thread, so its stage ring still holds two stages.
constexpr int UNIT = TPB * 8;
constexpr int TILE = UNIT;          // largest tile (spill-slot size)
constexpr int kMaxStages = 8;
constexpr long long kSmemBudget = 220 * 1024;   // dynamic shared memory the kernel may use
constexpr int kMaxInstr = 256;      // vector instructions per fused group
constexpr int RMAX = 4;             // reductions per fused group (D_RSUM cases cover 0..3)
constexpr int kMaxGroupPtrs = 32;   // staged operands / stores per fused group

enum Dt : int { DT_F64 = 0, DT_I64 = 1, DT_BOOL = 2 };
enum BinK : int { B_ADD, B_SUB, B_MUL, B_DIV, B_MOD, B_LT, B_GT, B_LE, B_GE, B_EQ, B_NE };
enum UnK : int { U_NEG, U_NOT, U_TANH, U_SIGMOID };

// scalar-phase opcodes (stream.py SOP)
enum SOp : int {
  S_HALT = 0, S_BIN = 1, S_UN = 2, S_SEL = 3, S_MOV = 4, S_SELREF = 5, S_LNEW = 6, S_LAPPEND = 7,
  S_LPOP = 8, S_LGET = 9, S_LSET = 10, S_JMP = 11, S_JZ = 12, S_ITER = 13, S_SETI = 14, S_ASSERT = 15,
  S_RAISE = 16, S_ALLOC = 17, S_VEXEC = 18, S_RFIN = 19
};
// vector-phase opcodes
enum VOp : int { V_PUSH = 1, V_BIN = 2, V_UN = 3, V_SEL = 4, V_STORE = 5, V_RED = 6, V_SAVE = 7, V_POP = 8 };
enum Src : int { SRC_STACK = 0, SRC_VEC = 1, SRC_SCALAR = 2, SRC_TEMP = 3 };
// slot kinds for MOV / list items
enum Kind : int { K_SCALAR = 0, K_VEC = 1, K_LIST_S = 2, K_LIST_V = 3 };

enum { E_INDEX = 10, E_EMPTY = 11, E_SHAPE = 12, E_DIV0 = 13, E_LIMIT = 14, E_ASSERT = 15,
       E_DTYPE = 16, E_POOL = 30, E_STEPS = 31, E_CAP = 32, E_INTERNAL = 33 };

struct SIns { int32_t op, uid, a[6]; };

struct StreamCtl {               // device control block (host-zeroed)
  unsigned long long err;        // (pc << 16) | code, min over reporters
  long long detail;
  long long steps;
  long long barriers;
  unsigned int arrive;           // grid-arrival counter (monotonic)
  unsigned int pad;
  long long max_live;            // buffer-pool high-water mark
  long long t_scalar, t_rfin, t_vec, t_sync;   // CTA 0 clock64 totals (SKB_STREAM_TIMING builds only)
};
#ifdef SKB_STREAM_TIMING
#define SKB_T0(v) const long long v = clock64()
#define SKB_TADD(field, t0) do { if (blockIdx.x == 0 && threadIdx.x == 0) a.ctl->field += clock64() - (t0); } while (0)
#else
#define SKB_T0(v) do {} while (0)
#define SKB_TADD(field, t0) do {} while (0)
#endif

struct StreamArgs {
  const SIns* prog;
  const int32_t* extra;
  const long long* w_init;       // initial W image
  long long* w_out;              // final W image (written by CTA 0)
  const long long* bufptr;       // buffer id -> device address
  const int32_t* rc_init;        // initial reference counts (feeds pinned)
  long long* part;               // [2][RMAX][grid] reduction partials
  StreamCtl* ctl;
  long long n;                   // elements per vector
  int nwords;
  int nbuf;
  int max_stack;                 // spill depth
  int max_temp;
  int max_ops;                   // staged operands per group
  long long smem;                // dynamic shared memory bytes of the launch
  long long max_steps;
  int nprog;                     // scalar instructions (copied into shared memory when they fit)
};

struct Smem {                    // carved from dynamic shared memory
  long long* W;
  int32_t* rc;
  int32_t* freel;
  long long* stage;              // [stages][nops][TILE] for the running group
  long long stage_bytes;
  long long* gptr;               // [kMaxGroupPtrs operands | kMaxGroupPtrs stores] addresses
  int4* gins;                    // the running group's vector instructions
  uint64_t* bars;                // "full" mbarrier per stage (bulk-copy bytes landed)
  uint64_t* empty;               // "empty" mbarrier per stage (all warps done with it)
  long long* stk;                // [max_stack][TILE] spilled stack entries
  uint32_t* uses;                // completed phases per stage mbarrier
  long long* red;                // [TPB/32][RMAX]
  const SIns* prog;              // the scalar program (shared-memory copy, or global)
};
constexpr int kProgSmemMax = 32 * 1024;   // scalar programs up to this size run from shared memory

struct Ctl {                     // per-CTA scalar-phase state (shared)
  int pc, halt, nfree, barrier_gen;
  long long steps, live, max_live;
};

__device__ __forceinline__ double as_f(long long w) { return __longlong_as_double(w); }
__device__ __forceinline__ long long as_w(double d) { return __double_as_longlong(d); }
__device__ __forceinline__ double num(long long w, int dt) { return dt == DT_F64 ? as_f(w) : (double)w; }

__device__ double sigmoid_ref(double x) {   // reference tensor.py:403-407
  if (x >= 0) return 1.0 / (1.0 + exp(-x));
  const double e = exp(x);
  return e / (1.0 + e);
}
__device__ __forceinline__ double py_fmod(double a, double b) {
  double r = fmod(a, b);
  if (r != 0.0 && ((r < 0.0) != (b < 0.0))) r += b;
  return r;
}
__device__ __forceinline__ long long py_imod(long long a, long long b) {
  long long r = a % b;
  if (r != 0 && ((r < 0) != (b < 0))) r += b;
  return r;
}

// One reference binop on words (tensor.py:227-287).  `dts` = dta | dtb << 4 | dto << 8.
__device__ __forceinline__ long long binop_w(int op, int dts, long long a, long long b, bool& div0) {
  const int dta = dts & 15, dtb = (dts >> 4) & 15, dto = (dts >> 8) & 15;
  if (op >= B_LT) {
    bool r;
    if (dta == DT_F64 || dtb == DT_F64) {
      const double x = num(a, dta), y = num(b, dtb);
      r = op == B_LT ? x < y : op == B_GT ? x > y : op == B_LE ? x <= y : op == B_GE ? x >= y
        : op == B_EQ ? x == y : x != y;
    } else {
      r = op == B_LT ? a < b : op == B_GT ? a > b : op == B_LE ? a <= b : op == B_GE ? a >= b
        : op == B_EQ ? a == b : a != b;
    }
    return r ? 1 : 0;
  }
  if (dto == DT_F64) {
    const double x = num(a, dta), y = num(b, dtb);
    double r;
    switch (op) {
      case B_ADD: r = x + y; break;
      case B_SUB: r = x - y; break;
      case B_MUL: r = x * y; break;
      case B_DIV: if (y == 0.0) { div0 = true; r = 0.0; } else r = x / y; break;
      default:    if (y == 0.0) { div0 = true; r = 0.0; } else r = py_fmod(x, y); break;
    }
    return as_w(r);
  }
  switch (op) {
    case B_ADD: return a + b;
    case B_SUB: return a - b;
    case B_MUL: return a * b;
    default:
      if (b == 0) { div0 = true; return 0; }
      return py_imod(a, b);
  }
}

__device__ __forceinline__ long long unop_w(int op, int dts, long long a) {
  const int dta = dts & 15;
  switch (op) {
    case U_NEG: return dta == DT_F64 ? as_w(-as_f(a)) : -a;
    case U_NOT: return a ? 0 : 1;
    case U_TANH: return as_w(tanh(num(a, dta)));
    default: return as_w(sigmoid_ref(num(a, dta)));
  }
}

__device__ __forceinline__ unsigned int ld_acquire(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// ------------------------------------------------------------ scalar phase
struct Scalar {
  const StreamArgs& a;
  Smem& s;
  Ctl& c;

  __device__ void ref(long long id) const { if (id >= 0) s.rc[id]++; }
  __device__ void rel(long long id) const {
    if (id >= 0 && --s.rc[id] == 0) { s.freel[c.nfree++] = (int)id; c.live--; }
  }
  __device__ long long alloc() const {
    if (c.nfree == 0) return -1;
    const int id = s.freel[--c.nfree];
    s.rc[id] = 1;
    if (++c.live > c.max_live) c.max_live = c.live;
    return id;
  }
  // release the contents of a list slot of vectors
  __device__ void rel_list(int off, int kind) const {
    if (kind == K_LIST_V) {
      const long long n = s.W[off];
      for (long long i = 0; i < n; ++i) rel(s.W[off + 1 + i]);
    }
  }
  __device__ void set_vec(int dst, long long id) const {   // ref-before-rel
    ref(id);
    rel(s.W[dst]);
    s.W[dst] = id;
  }
  // dst <- src for any kind (MOV / VIEW / loop-state copies)
  __device__ void mov(int dst, int src, int kind) const {
    if (dst == src) return;
    if (kind == K_SCALAR) { s.W[dst] = s.W[src]; return; }
    if (kind == K_VEC) { set_vec(dst, s.W[src]); return; }
    const long long n = s.W[src];
    if (kind == K_LIST_V)
      for (long long i = 0; i < n; ++i) ref(s.W[src + 1 + i]);
    rel_list(dst, kind);
    s.W[dst] = n;
    for (long long i = 0; i < n; ++i) s.W[dst + 1 + i] = s.W[src + 1 + i];
  }
  __device__ bool list_index(int list, long long i, long long& out) const {   // execute.py:240-245
    const long long n = s.W[list];
    if (!(-n <= i && i < n)) return false;
    out = i < 0 ? i + n : i;
    return true;
  }
};

__device__ void report(StreamCtl* ctl, int pc, int code, long long detail) {
  const unsigned long long w = ((unsigned long long)pc << 16) | (unsigned long long)code;
  const unsigned long long old = atomicMin(&ctl->err, w);
  if (w < old) ctl->detail = detail;
}

// Runs lane 0's scalar instructions from c.pc until a VEXEC, RFIN or HALT.
// Returns the opcode it stopped at (c.pc points at it).
__device__ int scalar_run(const StreamArgs& a, Smem& s, Ctl& c) {
  Scalar S{a, s, c};
  long long* W = s.W;
  int pc = c.pc;               // program counter and step count in registers; written back on exit
  long long steps = c.steps;
  for (;;) {
    const SIns in = s.prog[pc];
    if (++steps > a.max_steps) {
      c.pc = pc; c.steps = steps;
      report(a.ctl, pc, E_STEPS, steps); c.halt = 1; return S_HALT;
    }
    int next = pc + 1;
    int fail = 0;
    long long detail = 0;
    switch (in.op) {
      case S_HALT: c.pc = pc; c.steps = steps; return S_HALT;
      case S_VEXEC: c.pc = pc; c.steps = steps; return S_VEXEC;
      case S_RFIN: c.pc = pc; c.steps = steps; return S_RFIN;
      case S_BIN: {
        bool d0 = false;
        W[in.a[0]] = binop_w(in.a[3], in.a[4], W[in.a[1]], W[in.a[2]], d0);
        if (d0) fail = E_DIV0;
        break;
      }
      case S_UN: W[in.a[0]] = unop_w(in.a[2], in.a[3], W[in.a[1]]); break;
      case S_SEL: W[in.a[0]] = W[in.a[1]] ? W[in.a[2]] : W[in.a[3]]; break;
      case S_MOV: S.mov(in.a[0], in.a[1], in.a[2]); break;
      case S_SELREF: S.set_vec(in.a[0], W[in.a[1]] ? W[in.a[2]] : W[in.a[3]]); break;
      case S_ALLOC: {
        const long long id = S.alloc();
        if (id < 0) { fail = E_POOL; break; }
        S.rel(W[in.a[0]]);
        W[in.a[0]] = id;
        break;
      }
      case S_LNEW: {   // a0 dst, a1 extra off (n, item offsets), a2 kind (list), a3 cap
        const int32_t* ex = a.extra + in.a[1];
        const int n = ex[0];
        if (n > in.a[3]) { fail = E_CAP; break; }
        if (in.a[2] == K_LIST_V)
          for (int i = 0; i < n; ++i) S.ref(W[ex[1 + i]]);
        S.rel_list(in.a[0], in.a[2]);
        W[in.a[0]] = n;
        for (int i = 0; i < n; ++i) W[in.a[0] + 1 + i] = W[ex[1 + i]];
        break;
      }
      case S_LAPPEND: {   // a0 dst, a1 list, a2 item, a3 kind, a4 cap
        const long long n = W[in.a[1]];
        if (n + 1 > in.a[4]) { fail = E_CAP; break; }
        S.mov(in.a[0], in.a[1], in.a[3]);
        if (in.a[3] == K_LIST_V) S.ref(W[in.a[2]]);
        W[in.a[0] + 1 + n] = W[in.a[2]];
        W[in.a[0]] = n + 1;
        break;
      }
      case S_LPOP: {      // a0 dst list, a1 dst item, a2 list, a3 kind
        const long long n = W[in.a[2]];
        if (n == 0) { fail = E_EMPTY; break; }
        const long long item = W[in.a[2] + n];
        if (in.a[3] == K_LIST_V) S.set_vec(in.a[1], item); else W[in.a[1]] = item;
        S.mov(in.a[0], in.a[2], in.a[3]);
        if (in.a[3] == K_LIST_V) S.rel(W[in.a[0] + n]);
        W[in.a[0]] = n - 1;
        break;
      }
      case S_LGET: {      // a0 dst, a1 list, a2 idx slot, a3 kind
        long long i;
        if (!S.list_index(in.a[1], W[in.a[2]], i)) { fail = E_INDEX; detail = W[in.a[2]]; break; }
        const long long item = W[in.a[1] + 1 + i];
        if (in.a[3] == K_LIST_V) S.set_vec(in.a[0], item); else W[in.a[0]] = item;
        break;
      }
      case S_LSET: {      // a0 dst, a1 list, a2 idx, a3 value, a4 kind
        long long i;
        if (!S.list_index(in.a[1], W[in.a[2]], i)) { fail = E_INDEX; detail = W[in.a[2]]; break; }
        const long long v = W[in.a[3]];
        S.mov(in.a[0], in.a[1], in.a[4]);
        if (in.a[4] == K_LIST_V) { S.ref(v); S.rel(W[in.a[0] + 1 + i]); }
        W[in.a[0] + 1 + i] = v;
        break;
      }
      case S_JMP: next = in.a[0]; break;
      case S_JZ: if (!W[in.a[0]]) next = in.a[1]; break;
      case S_ITER: {
        const long long it = W[in.a[0]];
        if (it >= in.a[1]) { fail = E_LIMIT; detail = it; break; }
        W[in.a[0]] = it + 1;
        break;
      }
      case S_SETI: W[in.a[0]] = in.a[1]; break;
      case S_ASSERT: if (!W[in.a[0]]) fail = E_ASSERT; break;
      case S_RAISE: fail = in.a[0]; detail = in.a[1]; break;
      default: fail = E_DTYPE + 100; break;
    }
    if (fail) { c.pc = pc; c.steps = steps; report(a.ctl, pc, fail, detail); c.halt = 1; return S_HALT; }
    pc = next;
  }
}

// ------------------------------------------------------------ vector phase
struct Group {
  int nops, nstores, nred, ninstr;
  const int32_t* op_slots;
  const int32_t* store_slots;
  const int32_t* red_kd;
  const int32_t* ins;
};

__device__ __forceinline__ Group decode(const int32_t* g) {
  Group G;
  G.nops = g[0]; G.nstores = g[1]; G.nred = g[2]; G.ninstr = g[3];
  G.op_slots = g + 4;
  G.store_slots = G.op_slots + G.nops;
  G.red_kd = G.store_slots + G.nstores;
  G.ins = G.red_kd + G.nred;
  return G;
}

// Element j (0..EPT-1) of this thread within a tile: pair j>>1 of the thread
// sits at (j>>1)*(2*TPB) + 2*tid, so every 16-byte access of a warp is one
// contiguous 512-byte run (coalesced HBM stores, conflict-free LDS.128).
__device__ __forceinline__ int elem_of(int j) { return (j >> 1) * (2 * TPB) + threadIdx.x * 2 + (j & 1); }
// (the pair layout is the same for both tile sizes: an 8-per-thread tile is
//  two 4-per-thread tiles back to back)

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
               :: "r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  const uint32_t addr = (uint32_t)__cvta_generic_to_shared(bar);
  while (!ok) {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(addr), "r"(parity) : "memory");
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes),
                  "r"((uint32_t)__cvta_generic_to_shared(bar)) : "memory");
}

// One elected thread stages every vector operand of `tile` into stage `st`
// (one 1-D bulk copy per operand, completion counted in bytes on the stage's
// mbarrier).  The last tile is rounded up to 16 bytes; buffers are padded.
template <int TL>
__device__ __forceinline__ void issue_tile(const StreamArgs& a, const Smem& s, const Group& G, long long base, int st,
                                           int nops) {
  const long long left = a.n - base;
  const long long cnt = left < 0 ? 0 : (left < TL ? left : TL);
  const uint32_t bytes = (uint32_t)((cnt * 8 + 15) & ~15ll);
  uint64_t* bar = s.bars + st;
  mbar_expect_tx(bar, bytes * G.nops);
  if (bytes == 0) return;
  for (int k = 0; k < G.nops; ++k) {
    const long long* src = reinterpret_cast<const long long*>(s.gptr[k]) + base;
    bulk_g2s(s.stage + ((long long)st * nops + k) * TL, src, bytes, bar);
  }
}

__device__ __forceinline__ long long red_identity(int kd) {
  const int kind = kd & 15, dt = kd >> 4;
  if (kind == 0) return dt == DT_F64 ? as_w(0.0) : 0;
  return dt == DT_F64 ? as_w(-INFINITY) : LLONG_MIN;
}
__device__ __forceinline__ long long red_combine(int kd, long long x, long long y) {
  const int kind = kd & 15, dt = kd >> 4;
  if (dt == DT_F64) {
    const double a = as_f(x), b = as_f(y);
    return as_w(kind == 0 ? a + b : (b > a ? b : a));
  }
  return kind == 0 ? x + y : (y > x ? y : x);
}

// This thread's EPT elements of a tile-sized shared-memory vector (stage,
// temporary or spill slot): two LDS.128 / STS.128, bank-conflict free.
template <int EPT>
__device__ __forceinline__ void lds_lane(const long long* p, long long (&v)[EPT]) {
#pragma unroll
  for (int j = 0; j < EPT; j += 2) {
    const longlong2 t = *reinterpret_cast<const longlong2*>(p + elem_of(j));
    v[j] = t.x; v[j + 1] = t.y;
  }
}
template <int EPT>
__device__ __forceinline__ void sts_lane(long long* p, const long long (&v)[EPT]) {
#pragma unroll
  for (int j = 0; j < EPT; j += 2) *reinterpret_cast<longlong2*>(p + elem_of(j)) = make_longlong2(v[j], v[j + 1]);
}

// Device encoding of the fused group's stack program (stream.py emits it):
// the operand source is folded into the opcode so one switch dispatches.
// Values a group both stores and reuses are recomputed from staged operands
// by the compiler, so there are no temporaries: only the top of stack lives
// in registers and rare spills go to a shared-memory stack.
enum DOp : int {
  D_PUSH_VEC = 1, D_PUSH_SCALAR = 2, D_BIN_VEC = 4, D_BIN_SCALAR = 5, D_BIN_STACK = 7, D_UN = 8,
  D_SEL = 9, D_STORE = 10, D_RED = 11, D_POP = 13,
  // f64 fast forms (no per-element dtype / operand-order decisions):
  // D_FV + 2*op + rev: TOS = TOS op vec (rev: vec op TOS), op in {add, sub, mul}
  D_FV = 20, D_FS = 30,           // ... same with a broadcast scalar operand
  D_FK = 40,                      // D_FK + op: TOS = popped op TOS
  D_RSUM = 50                     // D_RSUM + r: f64 sum reduction r (0..RMAX-1)
};

__device__ __forceinline__ void lds2(uint32_t addr, long long& x, long long& y) {
  asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(x), "=l"(y) : "r"(addr));
}
__device__ __forceinline__ void sts2(uint32_t addr, long long x, long long y) {
  asm volatile("st.shared.v2.u64 [%0], {%1, %2};" :: "r"(addr), "l"(x), "l"(y) : "memory");
}
// This thread's EPT elements of a tile-sized shared-memory vector at `addr`.
template <int EPT>
__device__ __forceinline__ void lds_lane(uint32_t addr, long long (&v)[EPT]) {
#pragma unroll
  for (int j = 0; j < EPT; j += 2) lds2(addr + 8u * elem_of(j), v[j], v[j + 1]);
}
template <int EPT>
__device__ __forceinline__ void sts_lane(uint32_t addr, const long long (&v)[EPT]) {
#pragma unroll
  for (int j = 0; j < EPT; j += 2) sts2(addr + 8u * elem_of(j), v[j], v[j + 1]);
}

// TOS <- (TOS op val) or (val op TOS); the operation is uniform, so the
// branch on it sits outside the element loop.
template <int EPT>
__device__ __forceinline__ void bin_lane(long long (&tos)[EPT], const long long (&val)[EPT], int bz, int dts,
                                         bool tos_left, long long base, long long n, int q, int& div0_q) {
  const int bop = bz & 255;
  if (dts == (DT_F64 | DT_F64 << 4 | DT_F64 << 8) && bop <= B_MUL) {
    double l[EPT], r[EPT];
#pragma unroll
    for (int j = 0; j < EPT; ++j) {
      l[j] = as_f(tos_left ? tos[j] : val[j]);
      r[j] = as_f(tos_left ? val[j] : tos[j]);
    }
    if (bop == B_ADD) {
#pragma unroll
      for (int j = 0; j < EPT; ++j) tos[j] = as_w(l[j] + r[j]);
    } else if (bop == B_SUB) {
#pragma unroll
      for (int j = 0; j < EPT; ++j) tos[j] = as_w(l[j] - r[j]);
    } else {
#pragma unroll
      for (int j = 0; j < EPT; ++j) tos[j] = as_w(l[j] * r[j]);
    }
    return;
  }
#pragma unroll
  for (int j = 0; j < EPT; ++j) {
    const long long l = tos_left ? tos[j] : val[j], r = tos_left ? val[j] : tos[j];
    bool d = false;
    tos[j] = binop_w(bop, dts, l, r, d);
    if (d && base + elem_of(j) < n && q < div0_q) div0_q = q;
  }
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"((uint32_t)__cvta_generic_to_shared(bar))
               : "memory");
}

// The fused group over this CTA's tiles.  Operands arrive by bulk copy into a
// ring of S stages (full[st]: bytes landed; empty[st]: every warp is done with
// the stage), the stack program runs over EPT elements per thread, results are
// stored straight to HBM and reductions end in one per-CTA partial + arrival.
template <int EPT>
__device__ __forceinline__ void vector_run(const StreamArgs& a, Smem& s, Ctl& c, const Group& G, int pc) {
  constexpr int TL = TPB * EPT, SUB = UNIT / TL;   // tile elements, tiles per owned unit
  const long long nunits = (a.n + UNIT - 1) / UNIT;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nops = G.nops < 1 ? 1 : G.nops;
  int S = (int)(s.stage_bytes / ((long long)nops * TL * 8));   // deepest pipeline the operands allow
  if (S > kMaxStages) S = kMaxStages;
  auto tile_base = [&](long long i) {   // i-th tile of this CTA
    return (blockIdx.x + (i / SUB) * gridDim.x) * UNIT + (i % SUB) * TL;
  };
  int div0_q = 1 << 30;   // first vector instruction that divided by zero
  long long racc[RMAX];
#pragma unroll
  for (int r = 0; r < RMAX; ++r) racc[r] = r < G.nred ? red_identity(G.red_kd[r]) : 0;
  const int nmy = blockIdx.x < nunits ? (int)((nunits - 1 - blockIdx.x) / gridDim.x + 1) * SUB : 0;
  if (tid == 0) {
    asm volatile("fence.proxy.async.global;" ::: "memory");   // generic stores -> bulk-copy reads
    for (int st = 0; st < S - 1 && st < nmy; ++st) issue_tile<TL>(a, s, G, tile_base(st), st, nops);
  }
  const int4* ins = s.gins;
  const uint32_t stage0 = (uint32_t)__cvta_generic_to_shared(s.stage);
  const uint32_t stk0 = (uint32_t)__cvta_generic_to_shared(s.stk);
  int st = 0, round = 0;        // stage of tile i, and how many times it was used before in this group
  int pst = S - 1, pround = 0;  // producer: stage / round of tile i + S - 1
  for (int i = 0; i < nmy; ++i) {
    if (tid == 0 && i + S - 1 < nmy) {
      if (pround > 0)   // wait until every warp released this stage's previous tile
        mbar_wait(s.empty + pst, (s.uses[pst] + (uint32_t)pround - 1) & 1);
      issue_tile<TL>(a, s, G, tile_base(i + S - 1), pst, nops);
    }
    if (++pst == S) { pst = 0; ++pround; }
    mbar_wait(s.bars + st, (s.uses[st] + (uint32_t)round) & 1);   // uses[] advance after the loop
    const long long base = tile_base(i);
    const bool full = base + TL <= a.n;
    const uint32_t stage = stage0 + (uint32_t)(st * nops * TL * 8);
    long long tos[EPT], val[EPT];
    int sp = 0;
    int4 wn = ins[0];
    for (int q = 0; q < G.ninstr; ++q) {
      const int4 w = wn;
      wn = ins[q + 1];   // next dispatch word in flight while this one executes (gins is padded)
      switch (w.x) {
        case D_PUSH_VEC:
          if (w.z) sts_lane(stk0 + (uint32_t)(sp++ * TL * 8), tos);
          lds_lane(stage + (uint32_t)(w.y * TL * 8), tos);
          break;
        case D_PUSH_SCALAR: {
          if (w.z) sts_lane(stk0 + (uint32_t)(sp++ * TL * 8), tos);
          const long long v = s.W[w.y];
#pragma unroll
          for (int j = 0; j < EPT; ++j) tos[j] = v;
          break;
        }
        case D_BIN_VEC:
          lds_lane(stage + (uint32_t)(w.y * TL * 8), val);
          bin_lane(tos, val, w.z, w.w, !((w.z >> 8) & 1), base, a.n, q, div0_q);
          break;
        case D_BIN_SCALAR: {
          const long long v = s.W[w.y];
#pragma unroll
          for (int j = 0; j < EPT; ++j) val[j] = v;
          bin_lane(tos, val, w.z, w.w, !((w.z >> 8) & 1), base, a.n, q, div0_q);
          break;
        }
        case D_BIN_STACK:   // left = popped value, right = TOS
          lds_lane(stk0 + (uint32_t)(--sp * TL * 8), val);
          bin_lane(tos, val, w.z, w.w, false, base, a.n, q, div0_q);
          break;
        case D_UN:
#pragma unroll
          for (int j = 0; j < EPT; ++j) tos[j] = unop_w(w.y, w.w, tos[j]);
          break;
        case D_SEL: {   // c, x spilled (c deeper), TOS = y
          long long x[EPT];
          lds_lane(stk0 + (uint32_t)(--sp * TL * 8), x);
          lds_lane(stk0 + (uint32_t)(--sp * TL * 8), val);
#pragma unroll
          for (int j = 0; j < EPT; ++j) tos[j] = val[j] ? x[j] : tos[j];
          break;
        }
        case D_STORE: {
          long long* dst = reinterpret_cast<long long*>(s.gptr[kMaxGroupPtrs + w.y]) + base;
          if (full) {
#pragma unroll
            for (int j = 0; j < EPT; j += 2)
              *reinterpret_cast<longlong2*>(dst + elem_of(j)) = make_longlong2(tos[j], tos[j + 1]);
          } else {
#pragma unroll
            for (int j = 0; j < EPT; ++j)
              if (base + elem_of(j) < a.n) dst[elem_of(j)] = tos[j];
          }
          break;
        }
        case D_RED: {
          const int kd = G.red_kd[w.y];
#pragma unroll
          for (int rr = 0; rr < RMAX; ++rr) {
            if (rr != w.y) continue;
#pragma unroll
            for (int j = 0; j < EPT; ++j)
              if (full || base + elem_of(j) < a.n) racc[rr] = red_combine(kd, racc[rr], tos[j]);
          }
          break;
        }
#define SKB_FAST(OPC, EXPR)                                                       \
  case OPC: {                                                                     \
    _Pragma("unroll") for (int j = 0; j < EPT; ++j) {                             \
      const double t_ = as_f(tos[j]), v_ = as_f(val[j]);                          \
      tos[j] = as_w(EXPR);                                                        \
    }                                                                             \
    break;                                                                        \
  }
#define SKB_FAST_SET(BASE)                                                        \
  SKB_FAST(BASE + 0, t_ + v_) SKB_FAST(BASE + 1, v_ + t_)                         \
  SKB_FAST(BASE + 2, t_ - v_) SKB_FAST(BASE + 3, v_ - t_)                         \
  SKB_FAST(BASE + 4, t_ * v_) SKB_FAST(BASE + 5, v_ * t_)
        case D_FV: case D_FV + 1: case D_FV + 2: case D_FV + 3: case D_FV + 4: case D_FV + 5:
          lds_lane(stage + (uint32_t)(w.y * TL * 8), val);
          switch (w.x) { SKB_FAST_SET(D_FV) }
          break;
        case D_FS: case D_FS + 1: case D_FS + 2: case D_FS + 3: case D_FS + 4: case D_FS + 5: {
          const long long v = s.W[w.y];
#pragma unroll
          for (int j = 0; j < EPT; ++j) val[j] = v;
          switch (w.x) { SKB_FAST_SET(D_FS) }
          break;
        }
        case D_FK: case D_FK + 1: case D_FK + 2:   // left = popped value (val), right = TOS
          lds_lane(stk0 + (uint32_t)(--sp * TL * 8), val);
          switch (w.x) {
            SKB_FAST(D_FK + 0, v_ + t_) SKB_FAST(D_FK + 1, v_ - t_) SKB_FAST(D_FK + 2, v_ * t_)
          }
          break;
#undef SKB_FAST_SET
#undef SKB_FAST
#define SKB_RSUM(R)                                                               \
  case D_RSUM + R: {                                                              \
    double acc_ = as_f(racc[R]);                                                  \
    if (full) {                                                                   \
      _Pragma("unroll") for (int j = 0; j < EPT; ++j) acc_ += as_f(tos[j]);       \
    } else {                                                                      \
      _Pragma("unroll") for (int j = 0; j < EPT; ++j)                             \
        if (base + elem_of(j) < a.n) acc_ += as_f(tos[j]);                        \
    }                                                                             \
    racc[R] = as_w(acc_);                                                         \
    break;                                                                        \
  }
        SKB_RSUM(0) SKB_RSUM(1) SKB_RSUM(2) SKB_RSUM(3)
#undef SKB_RSUM
        default:   // D_POP
          lds_lane(stk0 + (uint32_t)(--sp * TL * 8), tos);
          break;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(s.empty + st);   // this warp is done with stage `st`
    if (++st == S) { st = 0; ++round; }
  }
  __syncthreads();
  if (tid == 0)
    for (int k = 0; k < S; ++k) s.uses[k] += (uint32_t)(nmy > k ? (nmy - 1 - k) / S + 1 : 0);
  if (__syncthreads_or(div0_q != (1 << 30))) {
    __shared__ int first_q;
    if (tid == 0) first_q = 1 << 30;
    __syncthreads();
    if (div0_q != (1 << 30)) atomicMin(&first_q, div0_q);
    __syncthreads();
    if (tid == 0) report(a.ctl, pc, E_DIV0, first_q);   // host maps (pc, q) -> node
  }
  if (G.nred > 0) {
    // block reduce in a fixed order, then one arrival per CTA
#pragma unroll
    for (int r = 0; r < RMAX; ++r) {
      if (r >= G.nred) break;
      long long v = racc[r];
      for (int o = 16; o; o >>= 1) v = red_combine(G.red_kd[r], v, __shfl_xor_sync(0xffffffffu, v, o));
      if (lane == 0) s.red[warp * RMAX + r] = v;
    }
    __syncthreads();
    if (tid == 0) {
      const int gen = c.barrier_gen;
      for (int r = 0; r < G.nred; ++r) {
        long long v = s.red[r];
        for (int w = 1; w < TPB / 32; ++w) v = red_combine(G.red_kd[r], v, s.red[w * RMAX + r]);
        a.part[((long long)(gen & 1) * RMAX + r) * gridDim.x + blockIdx.x] = v;
      }
      __threadfence();
      atomicAdd(&a.ctl->arrive, 1u);
      c.barrier_gen = gen + 1;
    }
  }
}

__global__ void __launch_bounds__(TPB, 1) stream_kernel(StreamArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ Ctl c;
  Smem s;
  {
    unsigned char* p = smem_raw;
    auto take = [&](size_t bytes) { unsigned char* r = p; p += (bytes + 15) & ~size_t(15); return r; };
    s.bars = reinterpret_cast<uint64_t*>(take(sizeof(uint64_t) * kMaxStages));
    s.empty = reinterpret_cast<uint64_t*>(take(sizeof(uint64_t) * kMaxStages));
    s.stk = reinterpret_cast<long long*>(take(sizeof(long long) * a.max_stack * TILE));
    s.uses = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * kMaxStages));
    s.gins = reinterpret_cast<int4*>(take(sizeof(int4) * (kMaxInstr + 1)));
    s.W = reinterpret_cast<long long*>(take(sizeof(long long) * a.nwords));
    s.gptr = reinterpret_cast<long long*>(take(sizeof(long long) * 2 * kMaxGroupPtrs));
    s.red = reinterpret_cast<long long*>(take(sizeof(long long) * (TPB / 32) * RMAX));
    // the scalar program from shared memory: the interpreter's instruction fetches sit on the
    // serial path between vector groups (one thread, every L-BFGS iteration)
    const size_t prog_bytes = sizeof(SIns) * (size_t)a.nprog;
    s.prog = prog_bytes <= (size_t)kProgSmemMax ? reinterpret_cast<const SIns*>(take(prog_bytes)) : a.prog;
    s.rc = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * a.nbuf));
    s.freel = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * a.nbuf));
    // everything left of the budget stages the running group's operands
    p = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(p) + 127) & ~uintptr_t(127));
    s.stage = reinterpret_cast<long long*>(p);
    s.stage_bytes = a.smem - (long long)(p - smem_raw);
  }
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (s.prog != a.prog) {
    int4* dst = const_cast<int4*>(reinterpret_cast<const int4*>(s.prog));
    const int4* src = reinterpret_cast<const int4*>(a.prog);
    for (int i = tid; i < a.nprog * (int)(sizeof(SIns) / sizeof(int4)); i += TPB) dst[i] = src[i];
  }
  for (int i = tid; i < a.nwords; i += TPB) s.W[i] = a.w_init[i];
  for (int i = tid; i < a.nbuf; i += TPB) s.rc[i] = a.rc_init[i];
  if (tid == 0) {
    c.pc = 0; c.halt = 0; c.barrier_gen = 0; c.steps = 0;
    int nf = 0, live = 0;
    for (int i = a.nbuf - 1; i >= 0; --i) {   // lowest id allocated first
      if (a.rc_init[i] == 0) s.freel[nf++] = i; else ++live;
    }
    c.nfree = nf; c.live = live; c.max_live = live;
    for (int st = 0; st < kMaxStages; ++st) {
      mbar_init(s.bars + st, 1);
      mbar_init(s.empty + st, TPB / 32);
      s.uses[st] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  for (;;) {
    if (warp == 0) {
      for (;;) {
        int stop = S_HALT;
        SKB_T0(ts0);
        if (lane == 0) stop = scalar_run(a, s, c);
        SKB_TADD(t_scalar, ts0);
        stop = __shfl_sync(0xffffffffu, stop, 0);
        __syncwarp();
        if (stop != S_RFIN) break;
        // RFIN: a0 dst word, a1 reduction index, a2 kind|dt<<4, a3 wait flag
        const SIns in = s.prog[c.pc];
        if (in.a[3]) {
          if (lane == 0) {
            const unsigned int target = (unsigned int)(c.barrier_gen) * gridDim.x;
            SKB_T0(tr0);
            while (ld_acquire(&a.ctl->arrive) < target) {}
            SKB_TADD(t_rfin, tr0);
          }
          __syncwarp();
          const unsigned long long e = *reinterpret_cast<volatile unsigned long long*>(&a.ctl->err);
          if (e != ~0ull) {
            if (lane == 0) c.halt = 1;
            __syncwarp();
            break;
          }
        }
        const int kd = in.a[2];
        const long long* part = a.part + ((long long)((c.barrier_gen - 1) & 1) * RMAX + in.a[1]) * gridDim.x;
        long long acc = red_identity(kd);
        for (int i = lane; i < (int)gridDim.x; i += 32) acc = red_combine(kd, acc, __ldcg(part + i));
#pragma unroll
        for (int o = 16; o; o >>= 1) acc = red_combine(kd, acc, __shfl_xor_sync(0xffffffffu, acc, o));
        if (lane == 0) { s.W[in.a[0]] = acc; c.pc++; }
        __syncwarp();
      }
    }
    __syncthreads();
    if (c.halt || s.prog[c.pc].op == S_HALT) break;
    // VEXEC: a0 = group offset in extra
    const int pc = c.pc;
    const Group G = decode(a.extra + s.prog[pc].a[0]);
    bool bad = false;
    if (tid < G.nops + G.nstores) {
      const int slot = tid < G.nops ? G.op_slots[tid] : G.store_slots[tid - G.nops];
      const long long id = s.W[slot];
      if (id < 0 || id >= a.nbuf) {
        bad = true;
        report(a.ctl, pc, E_INTERNAL, ((long long)slot << 32) | (id & 0xffffffffll));
      } else {
        s.gptr[tid < G.nops ? tid : kMaxGroupPtrs + tid - G.nops] = a.bufptr[id];
      }
    }
    for (int q = tid; q < 4 * G.ninstr; q += TPB) reinterpret_cast<int*>(s.gins)[q] = G.ins[q];
    if (__syncthreads_or(bad)) break;   // identical in every CTA: all stop here
    // 8 elements per thread when two stages of full-unit tiles fit, else half tiles
    SKB_T0(tv0);
    if (2ll * (G.nops < 1 ? 1 : G.nops) * UNIT * 8 <= s.stage_bytes) vector_run<8>(a, s, c, G, pc);
    else vector_run<4>(a, s, c, G, pc);
    SKB_TADD(t_vec, tv0);
    if (tid == 0) c.pc = pc + 1;
    __syncthreads();
  }
  if (blockIdx.x == 0) {
    __syncthreads();
    for (int i = tid; i < a.nwords; i += TPB) a.w_out[i] = s.W[i];
    if (tid == 0) {
      a.ctl->steps = c.steps;
      a.ctl->barriers = c.barrier_gen;
      a.ctl->max_live = c.max_live;
    }
  }
}

size_t fixed_bytes(int max_stack, int max_temp, int nwords, int nbuf) {
  auto r = [](size_t b) { return (b + 15) & ~size_t(15); };
  (void)max_temp;   // groups recompute reused values: no temporaries
  return r(8ull * max_stack * TILE) + r(16ull * kMaxStages) + r(4ull * kMaxStages) +
         r(16ull * (kMaxInstr + 1)) + r(8ull * nwords) + r(8ull * 2 * kMaxGroupPtrs) + r(8ull * (TPB / 32) * RMAX) +
         2 * r(4ull * nbuf) + 128;
}

// The whole budget when the widest group still gets a double-buffered pipeline.
size_t smem_bytes(int max_ops, int max_stack, int max_temp, int nwords, int nbuf) {
  if (max_ops < 1) max_ops = 1;
  if (max_stack < 1) max_stack = 1;
  if (max_temp < 1) max_temp = 1;
  const size_t fixed = fixed_bytes(max_stack, max_temp, nwords, nbuf);
  const size_t need = fixed + 2ull * max_ops * (TILE / 2) * 8;   // two stages of half tiles at least
  return need > (size_t)kSmemBudget ? need : (size_t)kSmemBudget;
}

}  // namespace

extern "C" int skb_stream_tile_elems(void) { return UNIT; }   // elements per CTA-owned unit

extern "C" int64_t skb_stream_smem_bytes(int max_ops, int max_stack, int max_temp, int nwords, int nbuf) {
  return (int64_t)smem_bytes(max_ops, max_stack, max_temp, nwords, nbuf);
}

// Grid size the cooperative stream kernel will use for this shared-memory
// footprint (co-resident CTAs on all SMs), or <= 0 if it does not fit.
extern "C" int skb_stream_grid(int64_t smem) {
  int dev = 0, sms = 0, per = 0, optin = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (smem > optin) return 0;
  if (cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return -1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, stream_kernel, TPB, (size_t)smem) != cudaSuccess)
    return -1;
  return sms * per;
}

extern "C" int skb_stream_run(const void* prog, const int32_t* extra, const int64_t* w_init, int64_t* w_out,
                              const int64_t* bufptr, const int32_t* rc_init, int64_t* part, void* ctl,
                              int64_t n, int nwords, int nbuf, int max_ops, int max_stack, int max_temp,
                              int64_t max_steps, int nprog, int grid, int64_t smem, void* stream) {
  if (grid <= 0 || n <= 0 || max_stack > 3) return SKB_ERR_INVALID;
  StreamArgs a;
  a.prog = reinterpret_cast<const SIns*>(prog);
  a.extra = extra;
  a.w_init = reinterpret_cast<const long long*>(w_init);
  a.w_out = reinterpret_cast<long long*>(w_out);
  a.bufptr = reinterpret_cast<const long long*>(bufptr);
  a.rc_init = rc_init;
  a.part = reinterpret_cast<long long*>(part);
  a.ctl = reinterpret_cast<StreamCtl*>(ctl);
  a.n = n;
  a.nwords = nwords;
  a.nbuf = nbuf;
  a.max_ops = max_ops < 1 ? 1 : max_ops;
  a.max_stack = max_stack < 1 ? 1 : max_stack;
  a.max_temp = max_temp < 1 ? 1 : max_temp;
  a.max_steps = max_steps;
  a.nprog = nprog;
  a.smem = smem;
  if ((size_t)smem < fixed_bytes(a.max_stack, a.max_temp, nwords, nbuf) + 2ull * a.max_ops * (TILE / 2) * 8)
    return SKB_ERR_INVALID;
  if (cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return SKB_ERR_CUDA;
  void* params[] = {&a};
  if (cudaLaunchCooperativeKernel((void*)stream_kernel, dim3(grid), dim3(TPB), params, (size_t)smem,
                                  (cudaStream_t)stream) != cudaSuccess)
    return SKB_ERR_CUDA;
  return skb_check_launch();
}
