// vm.cu — device-resident region VM: executes an arbitrary staged graph
// (every op of the reference IR, reference pkg/src/stagekit/graph/ir.py:19-27)
// with its While/Cond control flow decided on the GPU.
//
// The host compiler (paper_1810_08061_b200/vm.py) flattens the graph's frames
// into a linear bytecode (jumps for While/Cond, inlined FuncCalls) over value
// slots.  This kernel is an SPMD interpreter: every thread of every CTA walks
// the same bytecode; metadata (shapes, allocation, program counter) is computed
// redundantly and identically by all threads, element loops are spread over
// the whole grid, and a grid barrier separates instructions.  Control
// decisions read device values written before the barrier, so all threads take
// the same path without any host round trip.  One CTA is launched for small
// programs (barrier = __syncthreads); large tensors get a cooperative grid.
//
// Semantics follow the reference kernels (graph/tensor.py, graph/execute.py):
// f64/i64/bool values, trailing-dim broadcasting, `/` always f64, Python
// floor-mod, DivisionByZero on a zero divisor, k-ordered matmul accumulation,
// stable sigmoid, leading-axis Where row selection, functional lists, and the
// reference's error kinds (tensor.py:160-430, execute.py:148-202).
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <climits>
#include <math.h>
#include <stdint.h>
#include "skb_internal.h"

namespace cg = cooperative_groups;

namespace {

enum Dt : int32_t { DT_F64 = 0, DT_I64 = 1, DT_BOOL = 2, DT_LIST = 3, DT_TREE = 4 };
constexpr int kMaxRank = 6;

struct VmVal {            // slot descriptor (also a list item)
  int64_t view;           // arena byte offset of the current data (list: item array)
  int64_t own;            // arena byte offset of the slot's own storage, -1 if none
  int64_t own_cap;        // bytes of own storage
  int64_t numel;          // tensor: elements; list: item count; tree: node index
  int32_t dtype;
  int32_t rank;
  int32_t shape[kMaxRank];
};
static_assert(sizeof(VmVal) == 64, "VmVal layout");

struct VmIns { int32_t op, uid, a[6]; };

enum Op : int32_t {
  OP_HALT = 0, OP_COPY = 2, OP_BINOP = 3, OP_UNARY = 4, OP_MATMUL = 5, OP_TRANSPOSE = 6,
  OP_REDUCE = 7, OP_WHERE = 8, OP_SHAPE = 9, OP_RANGE = 10, OP_INDEX = 11, OP_LIST_NEW = 12,
  OP_LIST_APPEND = 13, OP_LIST_POP = 14, OP_LIST_GET = 15, OP_LIST_SET = 16, OP_LIST_STACK = 17,
  OP_JMP = 18, OP_JZ = 19, OP_ITER = 20, OP_PRINT = 21, OP_ASSERT = 22, OP_TREE = 23,
  OP_VIEW = 24, OP_SET_I64 = 25, OP_RAISE = 26, OP_SWAP = 27, OP_CALL = 28, OP_RET = 29
};
enum BinK : int32_t { B_ADD, B_SUB, B_MUL, B_DIV, B_MOD, B_LT, B_GT, B_LE, B_GE, B_EQ, B_NE };
enum UnK : int32_t { U_NEG, U_NOT, U_TANH, U_SIGMOID };

// error codes (include/skb.h) + VM-only kinds
enum { E_INDEX = 10, E_EMPTY = 11, E_SHAPE = 12, E_DIV0 = 13, E_LIMIT = 14, E_ASSERT = 15,
       E_DTYPE = 16, E_TYPE = 17, E_ARENA = 30, E_DEPTH = 32, E_OVERFLOW = 33 };
constexpr int kMaxCallDepth = 1 << 16;

struct VmCtl {            // device control block
  int32_t err, err_uid;
  int64_t err_detail;
  int64_t arena_used;     // high-water mark of the bump allocator (reported)
  int64_t log_count;      // print events recorded
  int64_t steps;          // instructions executed
};

struct VmArgs {
  const VmIns* prog;
  const int32_t* extra;
  VmVal* slots;
  uint8_t* arena;
  int64_t arena_bytes;
  int64_t arena_start;    // first free byte (constants / feeds live below)
  double* scratch;        // per-CTA reduction partials (gridDim.x * 2 doubles)
  const double* tree_val; // tree node table: value, left, right (-1 = empty)
  const int32_t* tree_left;
  const int32_t* tree_right;
  int64_t* log;           // print log: records of (instr uid, slot snapshot offsets)
  int64_t log_cap;
  VmCtl* ctl;
  int64_t max_steps;
  int nslots;             // slots per CTA: every CTA of a grid keeps its own copy of the table
};

struct Sync {
  bool grid;
  __device__ void operator()() const {
    if (grid) cg::this_grid().sync();
    else __syncthreads();
  }
};

__device__ __forceinline__ bool leader() { return blockIdx.x == 0 && threadIdx.x == 0; }
__device__ __forceinline__ int64_t gtid() { return (int64_t)blockIdx.x * blockDim.x + threadIdx.x; }
__device__ __forceinline__ int64_t gstride() { return (int64_t)gridDim.x * blockDim.x; }

__device__ __forceinline__ double ld_num(const uint8_t* base, int64_t i, int32_t dt) {
  const int64_t w = reinterpret_cast<const int64_t*>(base)[i];
  return dt == DT_F64 ? __longlong_as_double(w) : (double)w;
}
__device__ __forceinline__ int64_t ld_i(const uint8_t* base, int64_t i) {
  return reinterpret_cast<const int64_t*>(base)[i];
}
__device__ __forceinline__ double ld_f(const uint8_t* base, int64_t i) {
  return __longlong_as_double(reinterpret_cast<const int64_t*>(base)[i]);
}
__device__ __forceinline__ void st_f(uint8_t* base, int64_t i, double v) {
  reinterpret_cast<int64_t*>(base)[i] = __double_as_longlong(v);
}
__device__ __forceinline__ void st_i(uint8_t* base, int64_t i, int64_t v) {
  reinterpret_cast<int64_t*>(base)[i] = v;
}

__device__ double sigmoid_ref(double x) {   // reference tensor.py:403-407
  if (x >= 0) return 1.0 / (1.0 + exp(-x));
  const double e = exp(x);
  return e / (1.0 + e);
}

__device__ double py_fmod(double a, double b) {   // Python float %: sign of the divisor
  double r = fmod(a, b);
  if (r != 0.0 && ((r < 0.0) != (b < 0.0))) r += b;
  return r;
}
// i64 arithmetic with overflow detection: the reference's ints are unbounded
// Python ints (tensor.py), so a result outside int64 cannot be represented on
// the device — it is reported (E_OVERFLOW), never wrapped.
__device__ __forceinline__ bool add_ovf(int64_t x, int64_t y, int64_t& r) {
  r = (int64_t)((uint64_t)x + (uint64_t)y);
  return ((x ^ r) & (y ^ r)) < 0;
}
__device__ __forceinline__ bool sub_ovf(int64_t x, int64_t y, int64_t& r) {
  r = (int64_t)((uint64_t)x - (uint64_t)y);
  return ((x ^ y) & (x ^ r)) < 0;
}
__device__ __forceinline__ bool mul_ovf(int64_t x, int64_t y, int64_t& r) {
  r = (int64_t)((uint64_t)x * (uint64_t)y);
  return __mul64hi(x, y) != (r >> 63);
}

__device__ int64_t py_imod(int64_t a, int64_t b) {
  int64_t r = a % b;
  if (r != 0 && ((r < 0) != (b < 0))) r += b;
  return r;
}

// The interpreter's per-thread view of the machine state.
struct Vm {
  VmArgs a;
  Sync sync;
  int64_t bump;           // identical in every thread

  // Slot descriptors: a private copy per CTA (every CTA computes the same values), so an
  // op's descriptor reads only race with its own CTA's commit (block barrier, not grid).
  __device__ VmVal& S(int i) const { return a.slots[(int64_t)blockIdx.x * a.nslots + i]; }
  __device__ uint8_t* P(int64_t off) const { return a.arena + off; }

  __device__ void fail(int code, int uid, int64_t detail) const {
    if (atomicCAS(&a.ctl->err, 0, code) == 0) { a.ctl->err_uid = uid; a.ctl->err_detail = detail; }
  }
  // Deterministic bump allocation (every thread computes the same offset).
  __device__ int64_t alloc(int64_t bytes) {
    const int64_t off = bump;
    bump += (bytes + 255) & ~int64_t(255);
    return off;
  }
  // Make sure slot `d` owns >= bytes; returns the data offset.  Only the leader
  // writes the descriptor; everyone gets the same answer.
  // The instruction's inputs (x0..x2) must not live in that storage: threads
  // write output elements while others still read input elements (matmul,
  // transpose, broadcasts, scalars), so an aliased input gets fresh storage.
  __device__ int64_t own_storage(int d, int64_t bytes, VmVal& nv, const VmVal* x0 = nullptr,
                                 const VmVal* x1 = nullptr, const VmVal* x2 = nullptr) {
    const VmVal cur = S(d);
    int64_t off = cur.own;
    int64_t cap = cur.own_cap;
    auto aliased = [&](const VmVal* x) {
      return x != nullptr && x->dtype != DT_LIST && x->dtype != DT_TREE && off >= 0 && x->view >= off &&
             x->view < off + cap;
    };
    if (off < 0 || cap < bytes || aliased(x0) || aliased(x1) || aliased(x2)) {
      cap = bytes < 64 ? 64 : bytes;
      off = alloc(cap);
    }
    nv.own = off;
    nv.own_cap = cap;
    nv.view = off;
    // Every thread has read this instruction's slot descriptors (inputs, and S(d) above)
    // before its CTA's leader commits the output descriptor at the end of the op: without
    // this barrier a lagging thread could read the new descriptor, take the other
    // allocation branch and desynchronise the replicated bump allocator.  (Tables are
    // per CTA, so a block barrier suffices in grid mode too.)
    __syncthreads();
    return off;
  }
  __device__ void commit(int d, const VmVal& nv) const {
    if (threadIdx.x == 0) S(d) = nv;   // each CTA's own table
  }
};

__device__ int64_t numel_of(const int32_t* shape, int rank) {
  int64_t n = 1;
  for (int i = 0; i < rank; ++i) n *= shape[i];
  return n;
}

// Broadcast-index helper: offset of output element `i` in an operand.
struct BIdx {
  int rank;
  int64_t ostride[kMaxRank];   // output strides
  int64_t istride[kMaxRank];   // operand strides (0 on broadcast dims)
  __device__ int64_t map(int64_t i) const {
    int64_t off = 0;
    for (int d = 0; d < rank; ++d) {
      const int64_t c = i / ostride[d];
      i -= c * ostride[d];
      off += c * istride[d];
    }
    return off;
  }
};

__device__ void make_bidx(BIdx& b, const int32_t* oshape, int orank, const VmVal& v) {
  b.rank = orank;
  int64_t acc = 1;
  for (int d = orank - 1; d >= 0; --d) { b.ostride[d] = acc; acc *= oshape[d]; }
  int64_t iacc = 1;
  for (int d = orank - 1; d >= 0; --d) {
    const int k = d - (orank - v.rank);
    if (k < 0) { b.istride[d] = 0; continue; }
    const int dim = v.shape[k];
    b.istride[d] = dim == 1 ? 0 : iacc;
    iacc *= dim;
  }
}

// ---------------------------------------------------------------- handlers
__device__ void op_copy(Vm& vm, const VmIns& in) {
  const int d = in.a[0], s = in.a[1];
  const VmVal src = vm.S(s);
  VmVal nv = vm.S(d);
  if (src.dtype == DT_LIST || src.dtype == DT_TREE) {   // descriptor copy (lists are COW)
    VmVal c = src;
    c.own = nv.own;
    c.own_cap = nv.own_cap;
    vm.commit(d, c);
    return;
  }
  const int64_t off = vm.own_storage(d, src.numel * 8, nv, &src);
  nv.numel = src.numel; nv.dtype = src.dtype; nv.rank = src.rank;
  for (int i = 0; i < kMaxRank; ++i) nv.shape[i] = src.shape[i];
  const int64_t* sp = reinterpret_cast<const int64_t*>(vm.P(src.view));
  int64_t* dp = reinterpret_cast<int64_t*>(vm.P(off));
  for (int64_t i = gtid(); i < src.numel; i += gstride()) dp[i] = sp[i];
  vm.commit(d, nv);
}

__device__ void op_binop(Vm& vm, const VmIns& in) {
  const int d = in.a[0], kind = in.a[3], out_dt = in.a[4];
  const VmVal A = vm.S(in.a[1]), B = vm.S(in.a[2]);
  // broadcast shapes (reference tensor.py:160-181)
  int32_t shape[kMaxRank];
  const int rank = A.rank > B.rank ? A.rank : B.rank;
  for (int i = 0; i < rank; ++i) {
    const int ia = A.rank - 1 - i, ib = B.rank - 1 - i;
    const int da = ia >= 0 ? A.shape[ia] : 1, db = ib >= 0 ? B.shape[ib] : 1;
    int o;
    if (da == 1) o = db;
    else if (db == 1) o = da;
    else if (da == db) o = da;
    else { vm.fail(E_SHAPE, in.uid, 0); return; }
    shape[rank - 1 - i] = o;
  }
  const int64_t n = numel_of(shape, rank);
  VmVal nv = vm.S(d);
  const int64_t off = vm.own_storage(d, n * 8, nv, &A, &B);
  nv.numel = n; nv.dtype = out_dt; nv.rank = rank;
  for (int i = 0; i < kMaxRank; ++i) nv.shape[i] = i < rank ? shape[i] : 0;
  BIdx ba, bb;
  make_bidx(ba, shape, rank, A);
  make_bidx(bb, shape, rank, B);
  const uint8_t* pa = vm.P(A.view);
  const uint8_t* pb = vm.P(B.view);
  uint8_t* po = vm.P(off);
  const bool fa = A.dtype == DT_F64, fb = B.dtype == DT_F64;
  const bool fl = fa || fb;
  for (int64_t i = gtid(); i < n; i += gstride()) {
    const int64_t ia = ba.map(i), ib = bb.map(i);
    if (kind <= B_MOD) {
      if (kind == B_DIV || (kind == B_MOD && fl)) {
        const double x = ld_num(pa, ia, A.dtype), y = ld_num(pb, ib, B.dtype);
        if (y == 0.0) { vm.fail(E_DIV0, in.uid, 0); continue; }
        st_f(po, i, kind == B_DIV ? x / y : py_fmod(x, y));
      } else if (fl) {
        const double x = ld_num(pa, ia, A.dtype), y = ld_num(pb, ib, B.dtype);
        st_f(po, i, kind == B_ADD ? x + y : kind == B_SUB ? x - y : x * y);
      } else {
        const int64_t x = ld_i(pa, ia), y = ld_i(pb, ib);
        int64_t r;
        if (kind == B_MOD) {
          if (y == 0) { vm.fail(E_DIV0, in.uid, 0); continue; }
          r = py_imod(x, y);
        } else {
          const bool ovf = kind == B_ADD ? add_ovf(x, y, r) : kind == B_SUB ? sub_ovf(x, y, r) : mul_ovf(x, y, r);
          if (ovf) { vm.fail(E_OVERFLOW, in.uid, 0); continue; }
        }
        st_i(po, i, r);
      }
    } else {
      bool r;
      if (A.dtype == DT_BOOL || B.dtype == DT_BOOL || !fl) {
        const int64_t x = ld_i(pa, ia), y = ld_i(pb, ib);
        r = kind == B_LT ? x < y : kind == B_GT ? x > y : kind == B_LE ? x <= y : kind == B_GE ? x >= y
          : kind == B_EQ ? x == y : x != y;
      } else {
        const double x = ld_num(pa, ia, A.dtype), y = ld_num(pb, ib, B.dtype);
        r = kind == B_LT ? x < y : kind == B_GT ? x > y : kind == B_LE ? x <= y : kind == B_GE ? x >= y
          : kind == B_EQ ? x == y : x != y;
      }
      st_i(po, i, r ? 1 : 0);
    }
  }
  vm.commit(d, nv);
}

__device__ void op_unary(Vm& vm, const VmIns& in) {
  const int d = in.a[0], kind = in.a[2], out_dt = in.a[3];
  const VmVal A = vm.S(in.a[1]);
  VmVal nv = vm.S(d);
  const int64_t off = vm.own_storage(d, A.numel * 8, nv);
  nv.numel = A.numel; nv.dtype = out_dt; nv.rank = A.rank;
  for (int i = 0; i < kMaxRank; ++i) nv.shape[i] = A.shape[i];
  const uint8_t* pa = vm.P(A.view);
  uint8_t* po = vm.P(off);
  for (int64_t i = gtid(); i < A.numel; i += gstride()) {
    if (kind == U_NEG) {
      if (A.dtype == DT_F64) st_f(po, i, -ld_f(pa, i));
      else st_i(po, i, -ld_i(pa, i));
    } else if (kind == U_NOT) {
      st_i(po, i, ld_i(pa, i) ? 0 : 1);
    } else {
      const double x = ld_num(pa, i, A.dtype);
      st_f(po, i, kind == U_TANH ? tanh(x) : sigmoid_ref(x));
    }
  }
  vm.commit(d, nv);
}

__device__ void op_matmul(Vm& vm, const VmIns& in) {   // reference tensor.py:302-319
  const int d = in.a[0], out_dt = in.a[3];
  const VmVal A = vm.S(in.a[1]), B = vm.S(in.a[2]);
  if (A.rank != 2 || B.rank != 2) { vm.fail(E_SHAPE, in.uid, 0); return; }
  const int n = A.shape[0], k = A.shape[1], m = B.shape[1];
  if (B.shape[0] != k) { vm.fail(E_SHAPE, in.uid, 1); return; }
  VmVal nv = vm.S(d);
  const int64_t off = vm.own_storage(d, (int64_t)n * m * 8, nv, &A, &B);
  nv.numel = (int64_t)n * m; nv.dtype = out_dt; nv.rank = 2;
  nv.shape[0] = n; nv.shape[1] = m;
  for (int i = 2; i < kMaxRank; ++i) nv.shape[i] = 0;
  const uint8_t* pa = vm.P(A.view);
  const uint8_t* pb = vm.P(B.view);
  uint8_t* po = vm.P(off);
  for (int64_t e = gtid(); e < (int64_t)n * m; e += gstride()) {
    const int64_t i = e / m, j = e - i * m;
    if (out_dt == DT_F64) {
      double acc = 0.0;
      for (int t = 0; t < k; ++t)
        acc = __dadd_rn(acc, __dmul_rn(ld_num(pa, i * k + t, A.dtype), ld_num(pb, (int64_t)t * m + j, B.dtype)));
      st_f(po, e, acc);
    } else {
      int64_t acc = 0;
      for (int t = 0; t < k; ++t) acc += ld_i(pa, i * k + t) * ld_i(pb, (int64_t)t * m + j);
      st_i(po, e, acc);
    }
  }
  vm.commit(d, nv);
}

__device__ void op_transpose(Vm& vm, const VmIns& in) {   // reference tensor.py:322-332
  const int d = in.a[0];
  const int32_t* perm = vm.a.extra + in.a[2];
  const int prank = in.a[3];
  const VmVal A = vm.S(in.a[1]);
  if (prank != A.rank) { vm.fail(E_SHAPE, in.uid, 0); return; }
  int32_t shape[kMaxRank];
  for (int i = 0; i < A.rank; ++i) shape[i] = A.shape[perm[i]];
  VmVal nv = vm.S(d);
  const int64_t off = vm.own_storage(d, A.numel * 8, nv, &A);
  nv.numel = A.numel; nv.dtype = A.dtype; nv.rank = A.rank;
  for (int i = 0; i < kMaxRank; ++i) nv.shape[i] = i < A.rank ? shape[i] : 0;
  int64_t sstride[kMaxRank], ostride[kMaxRank];
  int64_t acc = 1;
  for (int i = A.rank - 1; i >= 0; --i) { sstride[i] = acc; acc *= A.shape[i]; }
  acc = 1;
  for (int i = A.rank - 1; i >= 0; --i) { ostride[i] = acc; acc *= shape[i]; }
  const int64_t* pa = reinterpret_cast<const int64_t*>(vm.P(A.view));
  int64_t* po = reinterpret_cast<int64_t*>(vm.P(off));
  for (int64_t e = gtid(); e < A.numel; e += gstride()) {
    int64_t r = e, src = 0;
    for (int ax = 0; ax < A.rank; ++ax) {
      const int64_t c = r / ostride[ax];
      r -= c * ostride[ax];
      src += c * sstride[perm[ax]];
    }
    po[e] = pa[src];
  }
  vm.commit(d, nv);
}

__device__ void op_reduce(Vm& vm, const VmIns& in) {   // reference tensor.py:335-353
  const int d = in.a[0], is_max = in.a[2];
  const VmVal A = vm.S(in.a[1]);
  if (is_max && A.numel == 0) { vm.fail(E_SHAPE, in.uid, 0); return; }
  VmVal nv = vm.S(d);
  const int64_t off = vm.own_storage(d, 8, nv, &A);
  nv.numel = 1; nv.dtype = A.dtype; nv.rank = 0;
  for (int i = 0; i < kMaxRank; ++i) nv.shape[i] = 0;
  const uint8_t* pa = vm.P(A.view);
  uint8_t* po = vm.P(off);
  // Sequential (reference order) for small inputs; two-level otherwise.
  if (A.numel <= 4096 || gridDim.x == 1) {
    if (leader()) {
      if (A.dtype == DT_F64) {
        double acc = is_max ? ld_f(pa, 0) : 0.0;
        for (int64_t i = is_max ? 1 : 0; i < A.numel; ++i) {
          const double v = ld_f(pa, i);
          acc = is_max ? (v > acc ? v : acc) : acc + v;
        }
        st_f(po, 0, acc);
      } else {
        int64_t acc = is_max ? ld_i(pa, 0) : 0;
        for (int64_t i = is_max ? 1 : 0; i < A.numel; ++i) {
          const int64_t v = ld_i(pa, i);
          acc = is_max ? (v > acc ? v : acc) : acc + v;
        }
        st_i(po, 0, acc);
      }
    }
    vm.commit(d, nv);
    return;
  }
  __shared__ double red_f[32];
  __shared__ long long red_i[32];
  double af = is_max ? -INFINITY : 0.0;
  long long ai = is_max ? LLONG_MIN : 0;
  for (int64_t i = gtid(); i < A.numel; i += gstride()) {
    if (A.dtype == DT_F64) { const double v = ld_f(pa, i); af = is_max ? fmax(af, v) : af + v; }
    else { const long long v = ld_i(pa, i); ai = is_max ? (v > ai ? v : ai) : ai + v; }
  }
  for (int o = 16; o; o >>= 1) {
    const double of = __shfl_xor_sync(0xffffffffu, af, o);
    const long long oi = __shfl_xor_sync(0xffffffffu, ai, o);
    af = is_max ? fmax(af, of) : af + of;
    ai = is_max ? (oi > ai ? oi : ai) : ai + oi;
  }
  if ((threadIdx.x & 31) == 0) { red_f[threadIdx.x >> 5] = af; red_i[threadIdx.x >> 5] = ai; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double bf = red_f[0];
    long long bi = red_i[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      bf = is_max ? fmax(bf, red_f[w]) : bf + red_f[w];
      bi = is_max ? (red_i[w] > bi ? red_i[w] : bi) : bi + red_i[w];
    }
    vm.a.scratch[2 * blockIdx.x] = bf;
    reinterpret_cast<long long*>(vm.a.scratch)[2 * blockIdx.x + 1] = bi;
  }
  vm.sync();
  if (leader()) {
    double bf = vm.a.scratch[0];
    long long bi = reinterpret_cast<long long*>(vm.a.scratch)[1];
    for (int b = 1; b < (int)gridDim.x; ++b) {
      const double f = vm.a.scratch[2 * b];
      const long long i = reinterpret_cast<long long*>(vm.a.scratch)[2 * b + 1];
      bf = is_max ? fmax(bf, f) : bf + f;
      bi = is_max ? (i > bi ? i : bi) : bi + i;
    }
    if (A.dtype == DT_F64) st_f(po, 0, bf);
    else st_i(po, 0, bi);
  }
  vm.commit(d, nv);
}

__device__ void op_where(Vm& vm, const VmIns& in) {   // reference tensor.py:356-377
  const int d = in.a[0];
  const VmVal Cn = vm.S(in.a[1]), A = vm.S(in.a[2]), B = vm.S(in.a[3]);
  if (A.rank != B.rank) { vm.fail(E_SHAPE, in.uid, 0); return; }
  for (int i = 0; i < A.rank; ++i)
    if (A.shape[i] != B.shape[i]) { vm.fail(E_SHAPE, in.uid, 0); return; }
  bool same = Cn.rank == A.rank;
  for (int i = 0; same && i < A.rank; ++i) same = Cn.shape[i] == A.shape[i];
  int mode;   // 0 elementwise, 1 scalar, 2 row select
  if (same) mode = 0;
  else if (Cn.rank == 0) mode = 1;
  else if (Cn.rank == 1 && A.rank >= 1 && Cn.shape[0] == A.shape[0]) mode = 2;
  else { vm.fail(E_SHAPE, in.uid, 1); return; }
  VmVal nv = vm.S(d);
  const int64_t off = vm.own_storage(d, A.numel * 8, nv, &Cn, &A, &B);
  nv.numel = A.numel; nv.dtype = A.dtype; nv.rank = A.rank;
  for (int i = 0; i < kMaxRank; ++i) nv.shape[i] = A.shape[i];
  const int64_t row = mode == 2 ? (A.shape[0] ? A.numel / A.shape[0] : 0) : 1;
  const int64_t* pc = reinterpret_cast<const int64_t*>(vm.P(Cn.view));
  const int64_t* pa = reinterpret_cast<const int64_t*>(vm.P(A.view));
  const int64_t* pb = reinterpret_cast<const int64_t*>(vm.P(B.view));
  int64_t* po = reinterpret_cast<int64_t*>(vm.P(off));
  for (int64_t e = gtid(); e < A.numel; e += gstride()) {
    const int64_t c = mode == 0 ? pc[e] : mode == 1 ? pc[0] : pc[e / row];
    po[e] = c ? pa[e] : pb[e];
  }
  vm.commit(d, nv);
}

__device__ void set_scalar_i(Vm& vm, int d, int64_t v, int dt) {
  VmVal nv = vm.S(d);
  const int64_t off = vm.own_storage(d, 8, nv);
  nv.numel = 1; nv.dtype = dt; nv.rank = 0;
  for (int i = 0; i < kMaxRank; ++i) nv.shape[i] = 0;
  if (leader()) st_i(vm.P(off), 0, v);
  vm.commit(d, nv);
}

__device__ void op_shape(Vm& vm, const VmIns& in) {
  const int d = in.a[0];
  const VmVal A = vm.S(in.a[1]);
  VmVal nv = vm.S(d);
  const int64_t off = vm.own_storage(d, 8 * (A.rank ? A.rank : 1), nv);
  nv.numel = A.rank; nv.dtype = DT_I64; nv.rank = 1;
  nv.shape[0] = A.rank;
  for (int i = 1; i < kMaxRank; ++i) nv.shape[i] = 0;
  if (leader()) for (int i = 0; i < A.rank; ++i) st_i(vm.P(off), i, A.shape[i]);
  vm.commit(d, nv);
}

__device__ void op_range(Vm& vm, const VmIns& in) {   // reference tensor.py:414-417
  const int d = in.a[0];
  const VmVal N = vm.S(in.a[1]);
  const int64_t n = ld_i(vm.P(N.view), 0);
  if (n < 0) { vm.fail(E_SHAPE, in.uid, n); return; }
  VmVal nv = vm.S(d);
  const int64_t off = vm.own_storage(d, n * 8, nv, &N);
  nv.numel = n; nv.dtype = DT_I64; nv.rank = 1;
  nv.shape[0] = (int32_t)n;
  for (int i = 1; i < kMaxRank; ++i) nv.shape[i] = 0;
  for (int64_t i = gtid(); i < n; i += gstride()) st_i(vm.P(off), i, i);
  vm.commit(d, nv);
}

__device__ void op_index(Vm& vm, const VmIns& in) {   // reference tensor.py:420-430
  const int d = in.a[0];
  const VmVal A = vm.S(in.a[1]), I = vm.S(in.a[2]);
  if (A.rank == 0) { vm.fail(E_INDEX, in.uid, 0); return; }
  int64_t i = ld_i(vm.P(I.view), 0);
  const int64_t n = A.shape[0];
  if (!(-n <= i && i < n)) { vm.fail(E_INDEX, in.uid, i); return; }
  if (i < 0) i += n;
  const int64_t row = n ? A.numel / n : 0;
  VmVal nv = vm.S(d);
  const int64_t off = vm.own_storage(d, row * 8, nv, &A, &I);
  nv.numel = row; nv.dtype = A.dtype; nv.rank = A.rank - 1;
  for (int k = 0; k < kMaxRank; ++k) nv.shape[k] = k + 1 < A.rank ? A.shape[k + 1] : 0;
  const int64_t* pa = reinterpret_cast<const int64_t*>(vm.P(A.view)) + i * row;
  int64_t* po = reinterpret_cast<int64_t*>(vm.P(off));
  for (int64_t e = gtid(); e < row; e += gstride()) po[e] = pa[e];
  vm.commit(d, nv);
}

// Lists: view -> item array of VmVal, preceded by a 16-byte header {cap, hw}.
// Items are immutable once written; appends write in place only at the
// high-water mark (copy-on-write otherwise), so aliased list values never see
// each other's later elements.
__device__ int64_t list_alloc(Vm& vm, int64_t cap) {
  const int64_t off = vm.alloc(16 + cap * (int64_t)sizeof(VmVal)) + 16;
  if (leader()) {
    int64_t* h = reinterpret_cast<int64_t*>(vm.P(off - 16));
    h[0] = cap; h[1] = 0;
  }
  return off;
}
__device__ VmVal* items_of(Vm& vm, int64_t view) { return reinterpret_cast<VmVal*>(vm.P(view)); }

// Copy a tensor value into fresh immutable storage, returning its item descriptor.
__device__ VmVal snapshot(Vm& vm, const VmVal& v) {
  VmVal it = v;
  if (v.dtype == DT_LIST || v.dtype == DT_TREE) { it.own = -1; it.own_cap = 0; return it; }
  const int64_t off = vm.alloc(v.numel * 8 > 0 ? v.numel * 8 : 8);
  const int64_t* sp = reinterpret_cast<const int64_t*>(vm.P(v.view));
  int64_t* dp = reinterpret_cast<int64_t*>(vm.P(off));
  for (int64_t e = gtid(); e < v.numel; e += gstride()) dp[e] = sp[e];
  it.view = off; it.own = -1; it.own_cap = 0;
  return it;
}

__device__ void op_list_new(Vm& vm, const VmIns& in) {
  const int d = in.a[0];
  const int32_t* ex = vm.a.extra + in.a[1];
  const int n = ex[0];
  const int64_t cap = n < 8 ? 8 : 2 * n;
  const int64_t arr = list_alloc(vm, cap);
  for (int k = 0; k < n; ++k) {
    const VmVal it = snapshot(vm, vm.S(ex[1 + k]));
    if (leader()) items_of(vm, arr)[k] = it;
  }
  if (leader()) reinterpret_cast<int64_t*>(vm.P(arr - 16))[1] = n;
  VmVal nv = vm.S(d);
  nv.view = arr; nv.numel = n; nv.dtype = DT_LIST; nv.rank = 0;
  vm.commit(d, nv);
}

__device__ void op_list_append(Vm& vm, const VmIns& in) {   // reference execute.py:153-156
  const int d = in.a[0];
  const VmVal L = vm.S(in.a[1]);
  // Every thread must see the header before the leader bumps its high-water mark below,
  // or threads disagree on copy-on-write and their bump allocators diverge.
  const int64_t* hdr = reinterpret_cast<const int64_t*>(vm.P(L.view - 16));
  const int64_t cap = hdr[0], hw = hdr[1];
  const VmVal item = snapshot(vm, vm.S(in.a[2]));
  vm.sync();
  int64_t arr = L.view;
  if (L.numel != hw || L.numel >= cap) {   // copy-on-write / grow
    const int64_t ncap = L.numel + 1 > cap ? 2 * cap : cap;
    arr = list_alloc(vm, ncap);
    const VmVal* src = items_of(vm, L.view);
    VmVal* dst = items_of(vm, arr);
    for (int64_t k = gtid(); k < L.numel; k += gstride()) dst[k] = src[k];
  }
  if (leader()) {
    items_of(vm, arr)[L.numel] = item;
    reinterpret_cast<int64_t*>(vm.P(arr - 16))[1] = L.numel + 1;
  }
  VmVal nv = vm.S(d);
  nv.view = arr; nv.numel = L.numel + 1; nv.dtype = DT_LIST; nv.rank = 0;
  vm.commit(d, nv);
}

__device__ void op_list_get(Vm& vm, const VmIns& in) {
  const int d = in.a[0];
  const VmVal L = vm.S(in.a[1]);
  int64_t i = ld_i(vm.P(vm.S(in.a[2]).view), 0);
  const int64_t n = L.numel;
  if (!(-n <= i && i < n)) { vm.fail(E_INDEX, in.uid, i); return; }
  if (i < 0) i += n;
  VmVal it = items_of(vm, L.view)[i];
  const VmVal cur = vm.S(d);
  it.own = cur.own; it.own_cap = cur.own_cap;   // a view of the immutable item
  vm.commit(d, it);
}

__device__ void op_list_set(Vm& vm, const VmIns& in) {
  const int d = in.a[0];
  const VmVal L = vm.S(in.a[1]);
  int64_t i = ld_i(vm.P(vm.S(in.a[2]).view), 0);
  const int64_t n = L.numel;
  if (!(-n <= i && i < n)) { vm.fail(E_INDEX, in.uid, i); return; }
  if (i < 0) i += n;
  const VmVal item = snapshot(vm, vm.S(in.a[3]));
  const int64_t arr = list_alloc(vm, n < 8 ? 8 : n);
  const VmVal* src = items_of(vm, L.view);
  VmVal* dst = items_of(vm, arr);
  for (int64_t k = gtid(); k < n; k += gstride()) dst[k] = k == i ? item : src[k];
  if (leader()) reinterpret_cast<int64_t*>(vm.P(arr - 16))[1] = n;
  VmVal nv = vm.S(d);
  nv.view = arr; nv.numel = n; nv.dtype = DT_LIST; nv.rank = 0;
  vm.commit(d, nv);
}

__device__ void op_list_pop(Vm& vm, const VmIns& in) {
  const int dl = in.a[0], di = in.a[1];
  const VmVal L = vm.S(in.a[2]);
  if (L.numel == 0) { vm.fail(E_EMPTY, in.uid, 0); return; }
  VmVal it = items_of(vm, L.view)[L.numel - 1];
  VmVal nl = vm.S(dl);
  nl.view = L.view; nl.numel = L.numel - 1; nl.dtype = DT_LIST; nl.rank = 0;
  const VmVal cur = vm.S(di);
  it.own = cur.own; it.own_cap = cur.own_cap;
  if (threadIdx.x == 0) { vm.S(dl) = nl; vm.S(di) = it; }
}

__device__ void op_list_stack(Vm& vm, const VmIns& in) {   // reference execute.py:171-184
  const int d = in.a[0];
  const VmVal L = vm.S(in.a[1]);
  if (L.numel == 0) { vm.fail(E_EMPTY, in.uid, 0); return; }
  const VmVal* items = items_of(vm, L.view);
  const VmVal f = items[0];
  for (int64_t k = 1; k < L.numel; ++k) {
    bool ok = items[k].dtype == f.dtype && items[k].rank == f.rank;
    for (int r = 0; ok && r < f.rank; ++r) ok = items[k].shape[r] == f.shape[r];
    if (!ok) { vm.fail(E_SHAPE, in.uid, k); return; }
  }
  if (f.rank + 1 > kMaxRank) { vm.fail(E_SHAPE, in.uid, -1); return; }
  const int64_t tot = L.numel * f.numel;
  VmVal nv = vm.S(d);
  const int64_t off = vm.own_storage(d, tot * 8, nv);
  nv.numel = tot; nv.dtype = f.dtype; nv.rank = f.rank + 1;
  nv.shape[0] = (int32_t)L.numel;
  for (int r = 1; r < kMaxRank; ++r) nv.shape[r] = r - 1 < f.rank ? f.shape[r - 1] : 0;
  int64_t* po = reinterpret_cast<int64_t*>(vm.P(off));
  for (int64_t e = gtid(); e < tot; e += gstride()) {
    const int64_t k = f.numel ? e / f.numel : 0, j = e - k * f.numel;
    po[e] = reinterpret_cast<const int64_t*>(vm.P(items[k].view))[j];
  }
  vm.commit(d, nv);
}

__device__ void op_tree(Vm& vm, const VmIns& in) {   // reference execute.py:136-146
  const int d = in.a[0], kind = in.a[2];
  const VmVal Tr = vm.S(in.a[1]);
  const int64_t node = Tr.numel;
  const bool empty = node < 0 || isnan(vm.a.tree_val[node]);
  if (kind == 0) { set_scalar_i(vm, d, empty ? 1 : 0, DT_BOOL); return; }
  if (empty) { vm.fail(E_TYPE, in.uid, 0); return; }
  if (kind == 3) {
    VmVal nv = vm.S(d);
    const int64_t off = vm.own_storage(d, 8, nv);
    nv.numel = 1; nv.dtype = DT_F64; nv.rank = 0;
    for (int i = 0; i < kMaxRank; ++i) nv.shape[i] = 0;
    if (leader()) st_f(vm.P(off), 0, vm.a.tree_val[node]);
    vm.commit(d, nv);
    return;
  }
  VmVal nv = vm.S(d);
  nv.dtype = DT_TREE; nv.rank = 0;
  nv.numel = kind == 1 ? vm.a.tree_left[node] : vm.a.tree_right[node];
  vm.commit(d, nv);
}

// Recursive FuncCall (reference graph/execute.py:191-193): a device call stack of
// arena frame records.  Record at `rec`: a shared header (written identically by
// every CTA) {prev fp, return pc, call-site extra, per-CTA bytes, lo, n}, then one
// portion per CTA: the n saved slot descriptors of the callee's range [lo, lo+n)
// followed by a scratch area for the call's arguments / results.  Only thread 0
// of a CTA touches its CTA's slot table; the instruction barrier publishes it.
__device__ void op_call(Vm& vm, const VmIns& in, int pc, int64_t& fp, int& depth) {
  const int lo = in.a[2], n = in.a[3] - in.a[2];
  const int32_t* ex = vm.a.extra + in.a[1];
  const int nargs = ex[0], ndest = ex[1 + nargs];
  const int32_t* px = vm.a.extra + in.a[4];
  const int64_t per = (int64_t)(n + (nargs > ndest ? nargs : ndest)) * (int64_t)sizeof(VmVal);
  const int64_t rec = vm.alloc(64 + per * gridDim.x);
  if (vm.bump > vm.a.arena_bytes) return;   // E_ARENA is raised by the loop
  if (threadIdx.x == 0) {
    int64_t* hdr = reinterpret_cast<int64_t*>(vm.P(rec));
    hdr[0] = fp; hdr[1] = pc + 1; hdr[2] = in.a[1]; hdr[3] = per; hdr[4] = lo; hdr[5] = n;
    VmVal* saved = reinterpret_cast<VmVal*>(vm.P(rec + 64 + per * blockIdx.x));
    VmVal* tmp = saved + n;
    for (int i = 0; i < n; ++i) saved[i] = vm.S(lo + i);
    for (int k = 0; k < nargs; ++k) tmp[k] = vm.S(ex[1 + k]);
    for (int i = 0; i < n; ++i) { vm.S(lo + i).own = -1; vm.S(lo + i).own_cap = 0; }   // fresh storage
    for (int k = 0; k < px[0] && k < nargs; ++k) {
      VmVal v = tmp[k];
      v.own = -1; v.own_cap = 0;
      vm.S(px[1 + k]) = v;
    }
  }
  fp = rec;
  ++depth;
}

__device__ int op_ret(Vm& vm, const VmIns& in, int64_t& fp, int& depth) {
  const int64_t* hdr = reinterpret_cast<const int64_t*>(vm.P(fp));
  const int64_t prev = hdr[0], per = hdr[3];
  const int ret = (int)hdr[1], lo = (int)hdr[4], n = (int)hdr[5];
  const int32_t* ex = vm.a.extra + hdr[2];
  const int nargs = ex[0], ndest = ex[1 + nargs];
  const int32_t* dest = ex + 2 + nargs;
  const int32_t* rx = vm.a.extra + in.a[0];
  if (threadIdx.x == 0) {
    VmVal* saved = reinterpret_cast<VmVal*>(vm.P(fp + 64 + per * blockIdx.x));
    VmVal* tmp = saved + n;
    for (int k = 0; k < rx[0] && k < ndest; ++k) tmp[k] = vm.S(rx[1 + k]);
    for (int i = 0; i < n; ++i) vm.S(lo + i) = saved[i];
    for (int k = 0; k < rx[0] && k < ndest; ++k) {
      VmVal v = tmp[k];
      const VmVal cur = vm.S(dest[k]);
      v.own = cur.own; v.own_cap = cur.own_cap;
      vm.S(dest[k]) = v;
    }
  }
  fp = prev;
  --depth;
  return ret;
}

__global__ void __launch_bounds__(256) vm_kernel(VmArgs a, int grid_sync) {
  Vm vm;
  vm.a = a;
  vm.sync.grid = grid_sync != 0;
  vm.bump = a.arena_start;
  int pc = 0;
  int64_t steps = 0;
  int64_t fp = 0;   // current call frame record (0: main)
  int depth = 0;
  for (;;) {
    const VmIns in = a.prog[pc];
    int next = pc + 1;
    if (++steps > a.max_steps) { vm.fail(E_ARENA + 1, in.uid, steps); break; }
    switch (in.op) {
      case OP_HALT: next = -1; break;
      case OP_COPY: op_copy(vm, in); break;
      case OP_VIEW: {
        VmVal v = vm.S(in.a[1]);
        const VmVal cur = vm.S(in.a[0]);
        v.own = cur.own; v.own_cap = cur.own_cap;
        vm.commit(in.a[0], v);
        break;
      }
      case OP_SWAP: {
        const VmVal x = vm.S(in.a[0]), y = vm.S(in.a[1]);
        if (threadIdx.x == 0) { vm.S(in.a[0]) = y; vm.S(in.a[1]) = x; }
        break;
      }
      case OP_BINOP: op_binop(vm, in); break;
      case OP_UNARY: op_unary(vm, in); break;
      case OP_MATMUL: op_matmul(vm, in); break;
      case OP_TRANSPOSE: op_transpose(vm, in); break;
      case OP_REDUCE: op_reduce(vm, in); break;
      case OP_WHERE: op_where(vm, in); break;
      case OP_SHAPE: op_shape(vm, in); break;
      case OP_RANGE: op_range(vm, in); break;
      case OP_INDEX: op_index(vm, in); break;
      case OP_LIST_NEW: op_list_new(vm, in); break;
      case OP_LIST_APPEND: op_list_append(vm, in); break;
      case OP_LIST_POP: op_list_pop(vm, in); break;
      case OP_LIST_GET: op_list_get(vm, in); break;
      case OP_LIST_SET: op_list_set(vm, in); break;
      case OP_LIST_STACK: op_list_stack(vm, in); break;
      case OP_TREE: op_tree(vm, in); break;
      case OP_JMP: next = in.a[0]; break;
      case OP_JZ: {
        const int64_t p = ld_i(vm.P(vm.S(in.a[0]).view), 0);
        if (!p) next = in.a[1];
        break;
      }
      case OP_SET_I64: set_scalar_i(vm, in.a[0], in.a[1], DT_I64); break;
      case OP_ITER: {   // reference execute.py:232-234: limit checked after a true test
        const int64_t c = ld_i(vm.P(vm.S(in.a[0]).view), 0);
        if (c >= in.a[1]) { vm.fail(E_LIMIT, in.uid, c); break; }
        vm.sync();
        if (leader()) st_i(vm.P(vm.S(in.a[0]).view), 0, c + 1);
        break;
      }
      case OP_PRINT: {   // snapshot the printed values; the host formats the log
        const int32_t* ex = a.extra + in.a[0];
        const int n = ex[0];
        const int64_t base = a.ctl->log_count;   // read before the leader bumps it (synced below)
        vm.sync();
        if (base + 1 + n <= a.log_cap) {
          for (int k = 0; k < n; ++k) {
            const VmVal it = snapshot(vm, vm.S(ex[1 + k]));
            if (leader()) reinterpret_cast<VmVal*>(a.log)[base + 1 + k] = it;
          }
          if (leader()) {
            VmVal h = {};
            h.numel = n; h.dtype = in.uid;
            reinterpret_cast<VmVal*>(a.log)[base] = h;
            a.ctl->log_count = base + 1 + n;
          }
        } else if (leader()) {
          a.ctl->log_count = a.log_cap + 1;   // overflow marker
        }
        break;
      }
      case OP_ASSERT: {
        const int64_t p = ld_i(vm.P(vm.S(in.a[0]).view), 0);
        if (!p) vm.fail(E_ASSERT, in.uid, 0);
        break;
      }
      case OP_RAISE: vm.fail(in.a[0], in.uid, in.a[1]); break;
      case OP_CALL:
        if (depth >= kMaxCallDepth) { vm.fail(E_DEPTH, in.uid, depth); break; }
        __syncthreads();   // every thread read the slot table of the previous instruction
        op_call(vm, in, pc, fp, depth);
        next = in.a[0];
        break;
      case OP_RET:
        __syncthreads();
        next = op_ret(vm, in, fp, depth);
        break;
      default: vm.fail(E_TYPE + 100, in.uid, in.op); break;
    }
    if (vm.bump > a.arena_bytes) vm.fail(E_ARENA, in.uid, vm.bump);
    vm.sync();
    if (a.ctl->err != 0 || next < 0) break;
    pc = next;
  }
  if (leader()) { a.ctl->arena_used = vm.bump; a.ctl->steps = steps; }
}

}  // namespace

extern "C" int skb_vm_run(const void* prog, const int32_t* extra, void* slots, void* arena,
                          int64_t arena_bytes, int64_t arena_start, double* scratch,
                          const double* tree_val, const int32_t* tree_left, const int32_t* tree_right,
                          int64_t* log, int64_t log_cap, void* ctl, int64_t max_steps, int ctas,
                          int nslots, void* stream) {
  VmArgs a;
  a.prog = reinterpret_cast<const VmIns*>(prog);
  a.extra = extra;
  a.slots = reinterpret_cast<VmVal*>(slots);
  a.arena = reinterpret_cast<uint8_t*>(arena);
  a.arena_bytes = arena_bytes;
  a.arena_start = arena_start;
  a.scratch = scratch;
  a.tree_val = tree_val; a.tree_left = tree_left; a.tree_right = tree_right;
  a.log = log; a.log_cap = log_cap;
  a.ctl = reinterpret_cast<VmCtl*>(ctl);
  a.max_steps = max_steps;
  a.nslots = nslots;
  cudaStream_t st = (cudaStream_t)stream;
  if (ctas <= 1) {
    vm_kernel<<<1, 256, 0, st>>>(a, 0);
    return skb_check_launch();
  }
  int grid_sync = 1;
  void* params[] = {&a, &grid_sync};
  if (cudaLaunchCooperativeKernel((void*)vm_kernel, dim3(ctas), dim3(256), params, 0, st) != cudaSuccess)
    return SKB_ERR_CUDA;
  return skb_check_launch();
}

extern "C" int skb_vm_max_ctas(void) {
  int dev = 0, sms = 0, per = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, vm_kernel, 256, 0) != cudaSuccess) return -1;
  return sms * per;
}
