/* skb.h — C ABI of libskb, the B200 (sm_100a) execution backend for staged
 * control-flow graphs produced by the stagekit conversion API
 * (reference: pkg/src/stagekit, arXiv 1810.08061 re-creation).
 *
 * The reference executes staged graphs with a pure-Python interpreter,
 * `execute(graph, feeds, check=True)` (reference pkg/src/stagekit/graph/execute.py:27-36),
 * whose hot loop is `_Session._eval_while` (execute.py:218-238) calling the
 * per-element kernels of pkg/src/stagekit/graph/tensor.py.  The reference has
 * no FFI of its own; these entry points are what its `execute` seam binds to
 * (see INTEGRATION.md for the ctypes binding a stagekit maintainer adds).
 *
 * Conventions: plain pointers and sizes only; every pointer argument named
 * `*_dev` is device memory; `stream` is a cudaStream_t passed as void*.
 * Every function returns an skb_status.  Runtime graph failures detected on
 * the device are reported through a device-resident error word
 * (`skb_err_word`, 4 x int32: code, problem index, time step, detail) that the
 * host copies back after the stream synchronises; codes map 1:1 onto the
 * reference's RuntimeGraphError.cause_kind strings (errors.py:155-174).
 */
#ifndef SKB_H
#define SKB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int skb_status;

enum {
  SKB_OK = 0,
  SKB_ERR_INVALID = 1,      /* bad argument / unsupported shape              */
  SKB_ERR_CUDA = 2,         /* CUDA runtime failure (launch, config)         */
  SKB_ERR_UNSUPPORTED = 3,  /* configuration not compiled into this library  */
  /* device-detected runtime errors (cause_kind of the reference)            */
  SKB_ERR_INDEX_OUT_OF_RANGE = 10, /* "IndexOutOfRange" tensor.py:420-430     */
  SKB_ERR_EMPTY_POP = 11,          /* "EmptyPop"        execute.py:171-174    */
  SKB_ERR_SHAPE_MISMATCH = 12,     /* "ShapeMismatch"   tensor.py:344-353,414 */
  SKB_ERR_DIVISION_BY_ZERO = 13,   /* "DivisionByZero"  tensor.py:235-241     */
  SKB_ERR_ITERATION_LIMIT = 14,    /* "IterationLimitExceeded" execute.py:232 */
  SKB_ERR_ASSERTION_FAILED = 15,   /* "AssertionFailed" execute.py:198-202    */
  SKB_ERR_FP16_RANGE = 20,         /* input outside the fp16 tensor-core range */
  SKB_ERR_HANDOFF = 21             /* internal: a producer/consumer handoff between
                                      concurrent kernels timed out (never expected) */
};

/* Cell kinds recognised by the lowering of a staged `While` region. */
enum {
  SKB_CELL_LSTM = 1,      /* i,f,g,o gates; c' = f*c + i*g; h' = o*tanh(c')  */
  SKB_CELL_RNN_TANH = 2,  /* h' = tanh(x W + h U + b)  (corpus/dynamic_rnn.msl) */
  SKB_CELL_GRU = 3        /* z,r = sigmoid(x W + h U + b); n = tanh(x Wn + bn + r*(h Un + bhn));
                             h' = (1-z)*n + z*h  (oracle/programs/gru.msl).  Packed as four
                             gate blocks z, r, n_x = [Wn | 0], n_h = [0 | Un] (biases bz, br,
                             bn, bhn): pass w = {Wz, Wr, Wn, NULL}, u = {Uz, Ur, NULL, Un}. */
};

/* Library / device information. */
const char* skb_version(void);
int skb_device_sm_count(void);
int skb_last_cuda_error(void); /* cudaError_t of the last SKB_ERR_CUDA */

/* ---------------------------------------------------------------------------
 * Dynamic-length recurrent loop.
 *
 * Replaces, for a `While` whose body is an RNN/LSTM cell with a per-row
 * `Where(t < seq_len, new, old)` mask and a `ListAppend` of h:
 *   execute.py:218-238 (_eval_while) + tensor.py:302-319 (matmul),
 *   :274-287 (binop), :391-407 (tanh/sigmoid), :356-377 (where),
 *   :420-430 (index), :322-332 (the two Transposes) and execute.py:153-185
 *   (ListAppend/ListStack).
 * The loop predicate (t < reduce_max(seq_len)) is evaluated on the device;
 * every row exits at its own trip count; rows past their length carry the
 * frozen state exactly as the reference's Where does.
 * ------------------------------------------------------------------------- */
typedef struct skb_rnn_shape {
  int32_t cell;               /* SKB_CELL_* (LSTM, RNN_TANH, GRU)              */
  int32_t hidden;             /* H                                            */
  int32_t input;              /* F                                            */
  int32_t time;               /* T: time extent of x (leading dim after the transpose) */
  int32_t rows_per_problem;   /* batch rows of one execute() problem          */
  int32_t problems;           /* independent problems batched in this launch  */
} skb_rnn_shape;

/* Bytes of device scratch the packed weights need (fp16 slabs + fp32 bias). */
int64_t skb_rnn_packed_bytes(const skb_rnn_shape* shape);
/* Bytes of device scratch skb_rnn_forward needs for its row schedule. */
int64_t skb_rnn_workspace_bytes(const skb_rnn_shape* shape);
/* Launch plan of the persistent kernel on the current device: co-resident
 * clusters, CTAs per cluster and batch rows per tile. */
skb_status skb_rnn_plan(const skb_rnn_shape* shape, int32_t* clusters, int32_t* ctas_per_cluster,
                        int32_t* tile_rows);

/* Pack per-gate weights into the per-CTA tensor-core slabs.
 * w_dev[g]: [F,H], u_dev[g]: [H,H], b_dev[g]: [H]; gate order i,f,g,o for
 * LSTM, a single gate for RNN_TANH.  `f64` selects double (1) or float (0)
 * element type.  Sets SKB_ERR_FP16_RANGE in err_dev if |w| > 65504. */
skb_status skb_rnn_pack(const skb_rnn_shape* shape, const void* const* w_dev,
                        const void* const* u_dev, const void* const* b_dev, int f64,
                        void* packed_dev, int32_t* err_dev, void* stream);

/* Run the staged loop for shape->problems independent problems.
 *   x_dev:    [R, T, F] (R = problems*rows_per_problem), batch-major as fed
 *             (the reference's Transpose(1,0,2) is folded into addressing)
 *   x_f64:    1 if x is double, 0 if float
 *   h0_dev:   [R, H] float;  c0_dev: [R, H] float (LSTM) or NULL
 *   len_dev:  [R] int64 sequence lengths
 *   out_dev:  [R, T, H] float; problem p's result is out[p*rows : (p+1)*rows, :max_len_p, :]
 *   hT_dev/cT_dev: optional [R, H] final states (NULL to skip)
 *   max_len_dev: [problems] int32, receives max_len_p (the While trip count)
 *   err_dev:  skb_err_word (4 x int32), must be zeroed by the caller
 *   workspace_dev: skb_rnn_workspace_bytes() bytes */
skb_status skb_rnn_forward(const skb_rnn_shape* shape, const void* packed_dev,
                           const void* x_dev, int x_f64, const float* h0_dev,
                           const float* c0_dev, const int64_t* len_dev, float* out_dev,
                           float* hT_dev, float* cT_dev, int32_t* max_len_dev,
                           int32_t* err_dev, void* workspace_dev, void* stream);

/* ---------------------------------------------------------------------------
 * Region VM: any staged graph, its While/Cond
 * control flow evaluated on the device.  Replaces the whole of
 * graph/execute.py:27-238 for graphs without a fused kernel.  The bytecode,
 * slot table and arena layout are produced by paper_1810_08061_b200/vm.py:
 *   prog_dev:  int32[n][8] instructions {op, node uid, a0..a5}
 *   extra_dev: int32 side table (perms, list items, print operands)
 *   slots_dev: 64-byte value descriptors, feeds/constants pre-initialised
 *   arena_dev: arena_bytes; bytes [0, arena_start) hold feeds and constants
 *   scratch_dev: 2*ctas doubles;  tree_*: tree node table (NaN value = empty)
 *   log_dev: print records (log_cap x 64 bytes);  ctl_dev: 8 x int64 control
 *            block {err | uid<<32, detail, arena_used, log_count, steps}
 * ctas == 1 runs one CTA (block barriers); > 1 a cooperative grid.  slots_dev holds one copy of
 * the nslots descriptors per CTA (ctas x nslots; results are read from copy 0). */
skb_status skb_vm_run(const void* prog_dev, const int32_t* extra_dev, void* slots_dev, void* arena_dev,
                      int64_t arena_bytes, int64_t arena_start, double* scratch_dev,
                      const double* tree_val_dev, const int32_t* tree_left_dev,
                      const int32_t* tree_right_dev, int64_t* log_dev, int64_t log_cap, void* ctl_dev,
                      int64_t max_steps, int ctas, int nslots, void* stream);
/* Largest cooperative grid (CTAs) the VM kernel can use on this device. */
int skb_vm_max_ctas(void);

/* ---------------------------------------------------------------------------
 * Staged decoder with a data-dependent EOS stop (BASELINE config C3; csrc/beam.cu).
 *
 * The reference can stage greedy decoding (a `break` on EOS
 * lowered into the While test, runtime/dispatch.py:275-387 +
 * transforms/lowering.py:95-115, executed by graph/execute.py:218-238) but its
 * IR has no log-softmax / top-k (graph/ir.py:19-27), so beam search is this
 * extension entry; semantics in oracle/beam.py, pinned at beam 1 against the
 * reference's greedy program.  All matrices row-major fp32:
 *   h0 [S,H], c0 [S,H] (LSTM) or NULL, emb [V,E],
 *   w_gates [(E+H), G] with G = 4H (LSTM, gate order i,f,g,o) or H (RNN_TANH:
 *   [w_in; u]), b_gates [G] or NULL, w_out [H,V], b_out [V] or NULL.
 * Outputs (device): tokens [S,K,max_len+1] (position 0 = BOS 0), scores [S,K]
 * (sum of log-probabilities, best first), lengths [S,K]; steps_out (host) =
 * decode steps executed (<= max_len; fewer when every beam hit EOS).
 * ------------------------------------------------------------------------- */
typedef struct skb_decode_shape {
  int32_t cell;        /* SKB_CELL_LSTM or SKB_CELL_RNN_TANH */
  int32_t sentences;   /* S */
  int32_t beam;        /* K, 1..8 (1 = greedy) */
  int32_t vocab;       /* V */
  int32_t embed;       /* E */
  int32_t hidden;      /* H */
  int32_t max_len;
  int32_t eos;
  int32_t math;        /* 0: fp32 GEMMs (no TF32), 1: TF32 tensor-core GEMMs */
  int32_t poll;        /* host polls the device stop flag every `poll` steps (0 = 4) */
} skb_decode_shape;
int64_t skb_decode_workspace_bytes(const skb_decode_shape* shape);
/* Byte offset, inside the decode workspace, of the float[sentences*beam] array
 * that holds, for beam 1 (greedy), each sentence's smallest top-1 minus top-2
 * logit gap over the decode (+inf if it never chose).  A gap within fp32
 * rounding means the reference's f64 argmax could differ (reference
 * graph/tensor.py matmul in f64; argmax_row sums tied ids). */
int64_t skb_decode_margin_offset(const skb_decode_shape* shape);
/* Per-phase CUDA-event timing of subsequent skb_decode calls (bench/profiling):
 * read returns the steps timed and ms_out[4] = {embedding gather, gate GEMM +
 * cell, logits GEMM, beam_select} summed over them. */
int skb_decode_profile(int enable);
/* 1 if the last skb_decode ran as one conditional-WHILE CUDA graph launch (the
 * loop decided on the device), 0 if it used the host-polled loop. */
int skb_decode_last_mode(void);
int skb_decode_profile_read(float* ms_out);
skb_status skb_decode(const skb_decode_shape* shape, const float* h0_dev, const float* c0_dev,
                      const float* emb_dev, const float* w_gates_dev, const float* b_gates_dev,
                      const float* w_out_dev, const float* b_out_dev, int32_t* tokens_dev, float* scores_dev,
                      int32_t* lengths_dev, int32_t* steps_out, void* workspace_dev, void* stream);

/* ---------------------------------------------------------------------------
 * Batched level-by-level TreeLSTM (BASELINE config C5; csrc/tree.cu).
 *
 * Replaces the reference's recursive evaluation of the TreeLSTM program
 * (FuncCall / TreeLeft / TreeRight / TreeValue, graph/
 * execute.py:136-146, 191-194) for a whole forest.  The host schedule
 * (paper_1810_08061_b200/tree.py) numbers the forest's nodes, lists leaves,
 * orders internal nodes by height (order[], level_off_host[nlevels+1]) and
 * gives each node the X row of its parent: dest[n] = 2*row + side, -1 = root.
 *   value [nnodes] (leaf values), wc [H], U [2H, 5H] (gate blocks i|f_l|f_r|o|u,
 *   rows 0..H-1 multiply h_left, H..2H-1 h_right), bias [5H] (bf repeated)
 *   h_out/c_out [nnodes, H] (every node's state), math 0 fp32 / 1 TF32.
 * ------------------------------------------------------------------------- */
int64_t skb_tree_workspace_bytes(int nnodes, int ninternal, int hidden);
int skb_tree_last_mode(void);   /* 1 = the last skb_tree_lstm replayed a captured CUDA graph */
/* Host-side forest schedule (native, O(nodes)): heights, height-sorted internal
 * nodes with level offsets, leaf list and parent-row destinations (see tree.cu).
 * Returns the maximum height, or -1 for a node with exactly one child. */
int skb_tree_schedule(int64_t nnodes, const int64_t* left, const int64_t* right, int32_t* height,
                      int32_t* order, int32_t* level_off, int32_t* leaves, int32_t* dest);
/* Forest form: concatenated trees with tree-local child indices; writes global int32 child ids.
 * Replaces the per-tree recursion of the reference's Tree values (graph/execute.py:136-146). */
int skb_forest_schedule(int64_t ntrees, const int64_t* sizes, const int64_t* left, const int64_t* right,
                        int32_t* left_out, int32_t* right_out, int32_t* height, int32_t* order,
                        int32_t* level_off, int32_t* leaves, int32_t* dest);
skb_status skb_tree_lstm(int nnodes, int nleaves, int ninternal, int hidden, int nlevels, const int32_t* leaves_dev,
                         const int32_t* order_dev, const int32_t* level_off_host, const int32_t* left_dev,
                         const int32_t* right_dev, const int32_t* dest_dev, const float* value_dev,
                         const float* wc_dev, const float* u_dev, const float* bias_dev, int math, float* h_out_dev,
                         float* c_out_dev, void* workspace_dev, void* stream);

/* ---------------------------------------------------------------------------
 * Dynamic-length LSTM training step (BASELINE config C2; csrc/train.cu).
 *
 * Replaces the reference's hand-derived staged BPTT program (forward While
 * storing states + reverse While, oracle/programs/lstm_bptt.msl; executed by
 * graph/execute.py:218-238 — the reference cannot differentiate a While,
 * graph/grad.py:159-161) for one shard of `rows` sequences:
 *   x [rows,time,input], y [rows,time,hidden] fp32 batch-major, lens [rows] int64,
 *   h0/c0 [rows,hidden] or NULL (zeros), params = W [input,4H] | U [H,4H] | b [4H]
 *   (gate order i,f,g,o), grads (same layout, overwritten), loss (device fp32).
 * loss = inv_batch * sum_{b, t < len_b} <h_{b,t}, y_{b,t}>; max_len = max(lens)
 * (the While trip count).  graph != 0 captures the step once per (max_len,
 * buffers) and replays it as one CUDA graph launch.  The cross-GPU gradient
 * allreduce (NCCL) runs between this call and skb_sgd_update.
 * ------------------------------------------------------------------------- */
typedef struct skb_train_shape {
  int32_t rows, time, input, hidden;
  int32_t math;        /* 0 fp32 GEMMs, 1 TF32 tensor cores, 2 bf16 operands / fp32 accumulate */
  int32_t graph;       /* 1: capture/replay the step as a CUDA graph */
  float inv_batch;     /* 1 / global batch (loss normalisation) */
} skb_train_shape;
int64_t skb_train_workspace_bytes(const skb_train_shape* shape);
skb_status skb_lstm_train_step(const skb_train_shape* shape, const float* x_dev, const float* y_dev,
                               const int64_t* lens_dev, const float* h0_dev, const float* c0_dev,
                               const float* params_dev, float* grads_dev, float* loss_dev, int max_len,
                               void* workspace_dev, void* stream);
/* 1 if skb_lstm_train_step runs on skb's tcgen05 engine for this shape (bf16 math); then
 * max_len = -1 lets the device determine the While trip count (reduce_max of the lengths). */
int skb_train_uses_engine(const skb_train_shape* shape);
/* Debug: with SKB_TC_TRACE=1, copy the last forward (which = 0) or backward (1) step kernel's
 * per-step globaltimer stamps of CTA 0 ([steps][8] int64: step start, barrier passed, first
 * stage, last MMA, TMEM full, operands, epilogue done, published); returns steps or -1. */
int skb_train_tc_trace(long long* host_out, int steps, int which);
int skb_train_last_mode(void);   /* 1 = the last step replayed a CUDA graph */
skb_status skb_sgd_update(float* params_dev, const float* grads_dev, int64_t n, float lr, void* stream);

/* ---------------------------------------------------------------------------
 * MAML sinusoid meta-gradient (BASELINE config C5; csrc/maml.cu).
 *
 * Replaces executing the reference's gradient() (graph/grad.py:35-70) of the
 * staged one-task program oracle/programs/maml.msl once per task: MLP
 * 1-H-H-1 ReLU, one inner SGD step (alpha), query MSE; second-order
 * meta-gradient g_q - alpha * H_s g_q.  theta: w1[H] | b1[H] | w2[H*H] | b2[H]
 * | w3[H] | b3 (P = H*H + 4H + 1 floats); xs/ys/xq/yq [tasks, shots] fp32.
 * meta_grad [P] and mean_loss [1] are task means (fixed summation order).
 * ------------------------------------------------------------------------- */
int64_t skb_maml_workspace_bytes(int hidden, int tasks);
skb_status skb_maml_meta_grad(int hidden, int shots, int tasks, const float* theta_dev, const float* xs_dev,
                              const float* ys_dev, const float* xq_dev, const float* yq_dev, float alpha,
                              float* meta_grad_dev, float* mean_loss_dev, void* workspace_dev, void* stream);

/* ---------------------------------------------------------------------------
 * Vector-stream region executor (csrc/stream.cu; compiler stream.py).
 *
 * Replaces `execute` (graph/execute.py:27-36) for staged programs whose
 * tensors are scalars or vectors of one shape (L-BFGS, in-graph SGD: BASELINE
 * config C4): `_eval_while`/`_eval_cond` (execute.py:205-238) run on chip,
 * element-wise nodes (tensor.py:227-300, 356-407) are fused into HBM streams
 * and ReduceSum/ReduceMax (tensor.py:335-353) are the only grid exchanges.
 *   prog_dev:  int32[n][8] scalar-phase instructions {op, uid, a0..a5}
 *   extra_dev: fused-group descriptors and list item tables
 *   w_init_dev / w_out_dev: int64[nwords] scalar/list state image in / out
 *   bufptr_dev: int64[nbuf] device address of every vector buffer (feeds first)
 *   rc_init_dev: int32[nbuf] initial reference counts (0 = free pool buffer)
 *   part_dev: int64[2*8*grid] reduction partials;  ctl_dev: 8 x int64
 *            {err = pc<<16|code (host sets -1), detail, steps, barriers,
 *             arrive counter, max live buffers}
 *   n: elements per vector; grid from skb_stream_grid(smem). */
int64_t skb_stream_smem_bytes(int max_ops, int max_stack, int max_temp, int nwords, int nbuf);
int skb_stream_grid(int64_t smem_bytes);
int skb_stream_tile_elems(void);   /* vector elements per CTA tile (grid sizing) */
skb_status skb_stream_run(const void* prog_dev, const int32_t* extra_dev, const int64_t* w_init_dev,
                          int64_t* w_out_dev, const int64_t* bufptr_dev, const int32_t* rc_init_dev,
                          int64_t* part_dev, void* ctl_dev, int64_t n, int nwords, int nbuf, int max_ops,
                          int max_stack, int max_temp, int64_t max_steps, int nprog, int grid,
                          int64_t smem_bytes, void* stream);   /* nprog: scalar instructions in prog_dev */

/* ---------------------------------------------------------------------------
 * Multi-GPU collective (SURVEY §8(b) skb_comm_init / skb_allreduce_f32; csrc/comm.cu).
 * One rank per GPU; the training configs (C2 BPTT, C5 MAML) sum per-shard
 * gradients with one NCCL allreduce over NVLink / NVSwitch, enqueued on the
 * caller's stream.  NCCL is resolved at run time: the copy already loaded in
 * the process (PyTorch's), else `nccl_path` of skb_comm_load, else the system
 * libnccl.so.2.  The host exchanges the 128-byte unique id out of band.
 * Replaces the reference's nothing: stagekit is single-process; these back the
 * data-parallel trainers that replace its per-graph gradient() runs
 * (graph/grad.py:35-70) and the hand BPTT program (oracle/programs/lstm_bptt.msl).
 * ------------------------------------------------------------------------- */
enum { SKB_DT_F32 = 0, SKB_DT_F64 = 1, SKB_DT_I32 = 2, SKB_DT_I64 = 3 };
enum { SKB_OP_SUM = 0, SKB_OP_MAX = 1 };
skb_status skb_comm_load(const char* nccl_path);      /* optional: NULL = default search */
const char* skb_comm_last_error(void);
int skb_comm_nccl_version(void);                       /* e.g. 22809, or -1 */
skb_status skb_comm_unique_id(uint8_t* uid_out128);    /* rank 0 creates, host broadcasts */
skb_status skb_comm_init(int rank, int world, const uint8_t* uid128, void** comm_out);
skb_status skb_comm_allreduce(void* comm, void* buf_dev, int64_t n, int dtype, int op, void* stream);
skb_status skb_allreduce_f32(void* comm, float* buf_dev, int64_t n, void* stream);   /* in place, sum */
skb_status skb_allreduce_f64(void* comm, double* buf_dev, int64_t n, void* stream);
skb_status skb_comm_destroy(void* comm);

/* ---------------------------------------------------------------------------
 * Diagnostics (GPU self-tests of the tcgen05 / DSMEM building blocks).
 * ------------------------------------------------------------------------- */
skb_status skb_diag_umma_gemm(const void* a_dev, const void* b_dev, void* d_dev, int n, int k,
                              int swap_lbo_sbo, long long* cycles_dev, void* stream);
/* CTA-pair (cta_group::2) MMA with A from TMEM: D[256 x n] = reps * A[256 x k] B[n x k]^T,
 * read back through 32x32b (d_dev) and 16x256b (d2_dev) TMEM loads; cycles of the chain. */
skb_status skb_diag_umma_pair(const void* a_dev, const void* b_dev, void* d_dev, void* d2_dev, int n, int k,
                              int reps, long long* cycles_dev, void* stream);
/* Accurate tier of the same recurrent While (csrc/rnn_f32.cu): FP32 FFMA with
 * fp32 weights / state and accurate activations, within rtol 1e-4 of the
 * reference's float64 (north_star's fp32 bound).  One CTA per 32-row tile,
 * thread = hidden unit (H <= 256, (F+H) % 4 == 0).  Same arguments and error
 * contract as skb_rnn_forward; packing from the same per-gate weights. */
/* Which recurrent kernel the last skb_rnn_forward launched, and its cluster count. */
enum {
  SKB_RNN_KERNEL_SINGLE = 1,      /* one 64-row recurrence per cluster */
  SKB_RNN_KERNEL_PING_PONG = 2,   /* two 32-row halves (SKB_RNN_PP=1) */
  SKB_RNN_KERNEL_DUAL_LANE = 3,   /* two 64-row recurrences per CTA (SKB_RNN_PAIR=0) */
  SKB_RNN_KERNEL_PAIR = 4,        /* CTA pairs, M=256 cta_group::2 MMAs, four 64-row lanes (default) */
  SKB_RNN_KERNEL_PAIR2 = 5        /* CTA pairs, two 128-row lanes (SKB_RNN_PAIR=2) */
};
int skb_rnn_last_kernel(void);
int skb_rnn_last_clusters(void);
/* Concurrency of the last skb_rnn_forward: bit 0 = x images packed, bit 1 = frozen tails
 * filled by the auxiliary grid on the SMs the pair4 kernel's clusters leave idle, while
 * the recurrent kernel runs (on a high-priority side stream; joined on the caller's). */
int skb_rnn_last_overlap(void);
/* enable = 0: never use the auxiliary grid (pre-pass packer + fill pass), e.g. after a
 * launch reported SKB_ERR_HANDOFF; 1: as selected by SKB_RNN_XOVL / SKB_RNN_FOVL (both
 * default 0: measured slower than the sequential passes). */
int skb_rnn_set_overlap(int enable);
int64_t skb_rnn_f32_packed_bytes(const skb_rnn_shape* shape);
int64_t skb_rnn_f32_workspace_bytes(const skb_rnn_shape* shape);
skb_status skb_rnn_pack_f32(const skb_rnn_shape* shape, const void* const* w_dev, const void* const* u_dev,
                            const void* const* b_dev, int f64, void* packed_dev, void* stream);
skb_status skb_rnn_forward_f32(const skb_rnn_shape* shape, const void* packed_dev, const void* x_dev, int x_f64,
                               const float* h0_dev, const float* c0_dev, const int64_t* len_dev, float* out_dev,
                               float* hT_dev, float* cT_dev, int32_t* max_len_dev, int32_t* err_dev,
                               void* workspace_dev, void* stream);
/* Kernel-only timing: for the next `max_launches` skb_rnn_forward calls the
 * persistent recurrent kernel is bracketed by CUDA events on its stream;
 * skb_profile_read returns how many were recorded and their durations (ms). */
skb_status skb_profile_begin(int max_launches);
int skb_profile_read(float* ms_out, int n);
skb_status skb_profile_end(void);
/* Record clock64() role events of CTA 0 for the first `steps` loop steps into
 * trace_dev[steps*16] on subsequent skb_rnn_forward calls (NULL disables). */
skb_status skb_debug_rnn_trace(long long* trace_dev, int steps);
/* Per-tile events of CTA 0 (setup start, loop start, loop end, trip count). */
skb_status skb_debug_rnn_tile_trace(long long* trace_dev, int tiles);
/* gscratch_dev == NULL: bulk DSMEM copies; else slices go through L2 and are
 * multicast to the cluster (gscratch_dev: 2 x cluster x slice_bytes per cluster). */
skb_status skb_diag_cluster_exchange(int cluster, int slice_bytes, int rounds,
                                     long long* cycles_dev, int* errors_dev, void* gscratch_dev,
                                     void* stream);


/* ---------------------------------------------------------------------------
 * skb's own tcgen05 GEMM engine (csrc/gemm.cuh): C[M,N] (+)= op(A) op(B), fp32 out.
 *   elem 0: bf16 operands (kind::f16), 1: fp32 operands on tf32 tensor cores (K-major
 *   operands only: a_mn = b_mn = 0, else SKB_ERR_UNSUPPORTED)
 *   A: [M,K] row-major (a_mn = 0) or [K,M] row-major (a_mn = 1), leading dim lda
 *   B: [N,K] row-major (b_mn = 0) or [K,N] row-major (b_mn = 1), leading dim ldb
 *   beta 0/1 (accumulate into C), bn tile width 64/128/256 (0 = auto; -128 / -256: CTA-pair
 *   cta_group::2 tiles of 256 x |bn|, the two CTAs of a cluster sharing the B tile),
 *   ksplit > 1: deterministic split-K through workspace (skb_gemm_workspace_bytes).
 * Operand rows must be 16-byte aligned; N % 16 == 0.  Replaces the cuBLAS calls the
 * reference-free configs used in round 1 (C2 training GEMMs). */
int64_t skb_gemm_workspace_bytes(int M, int N, int ksplit);
skb_status skb_gemm(int elem, int a_mn, int b_mn, int M, int N, int K, const void* A, int64_t lda,
                    const void* B, int64_t ldb, float* C, int64_t ldc, int beta, int bn, int ksplit,
                    void* workspace, void* stream);


/* Host-to-device copy of the valid prefix of each row of a [rows, T, step] PINNED host
 * array: row r moves min(max(lens[r], 0), T) * step_bytes bytes, read by a device-pull
 * gather kernel on `stream` (lens_dev: the device copy of the row lengths).  Used by the
 * host-to-host C1 pipeline: the padded timesteps of a dynamic-length batch are never read
 * by the kernels.  SKB_ERR_INVALID for pageable memory (the caller copies the block). */
int skb_h2d_rows(void* dst_dev, const void* src_host, int64_t row_bytes, const int64_t* lens_dev,
                 int64_t rows, int64_t step_bytes, int T, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SKB_H */
