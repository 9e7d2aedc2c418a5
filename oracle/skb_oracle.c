/* skb_oracle.c — TEST INFRASTRUCTURE ONLY (checker / CPU baseline).
 *
 * A plain-C float64 restatement of the reference executor's arithmetic for
 * the staged dynamic-length recurrent program.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this library; the product path never does.
 *
 * Every kernel follows the reference operation order so results are bit-for-
 * bit the reference's (Python floats are IEEE doubles; math.tanh/math.exp are
 * libm's tanh/exp).  Compile with -ffp-contract=off: no fused multiply-add.
 *
 *   oracle_matmul   reference pkg/src/stagekit/graph/tensor.py:302-319
 *                   (acc starts at 0.0, adds a[i,t]*b[t,j] for t = 0..k-1)
 *   oracle_sigmoid  reference tensor.py:397-407 (stable two-branch form)
 *   binop / where   reference tensor.py:274-287, :356-377 (row select)
 *   oracle_rnn_program
 *                   the traced program (reference runtime/dispatch.py:326-468
 *                   builds it; graph/execute.py:218-238 runs it):
 *                   max_len = reduce_max(seq_len)            tensor.py:344-353
 *                   range(max_len) (negative -> ShapeMismatch) tensor.py:414-417
 *                   while idx < max_len: [limit check]        execute.py:227-237
 *                     x_t = transpose(x)[idx] (t >= T -> IndexOutOfRange) tensor.py:420-430
 *                     LSTM: i = sigmoid((x_t@Wi + h@Ui) + bi) ... c' = f*c + i*g;
 *                           h' = o*tanh(c')            (SURVEY App. A op order)
 *                     RNN:  h' = tanh((x_t@Wx + h@Wh) + b)     corpus/dynamic_rnn.msl
 *                     GRU:  z = sigmoid((x_t@Wz + h@Uz) + bz); r likewise;
 *                           n = tanh((x_t@Wn + bn) + r*(h@Un + bhn));
 *                           h' = (1.0 - z)*n + z*h         oracle/programs/gru.msl
 *                     h = where(idx < len, h', h) ...; outputs.append(h)
 *                   stack(outputs) (empty -> EmptyPop)  execute.py:171-174
 *                   transpose(stack, [1,0,2])
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { OK = 0, ERR_INDEX = 10, ERR_EMPTY = 11, ERR_SHAPE = 12, ERR_LIMIT = 14 };
enum { CELL_LSTM = 1, CELL_RNN = 2, CELL_GRU = 3 };

/* out[n,m] = a[n,k] @ b[k,m]; per element: acc = 0.0; acc += a*b in t order.
 * The j-inner loop keeps that per-element order while vectorising. */
void oracle_matmul(const double* a, const double* b, double* out, int n, int k, int m) {
  for (int i = 0; i < n; ++i) {
    double* o = out + (size_t)i * m;
    for (int j = 0; j < m; ++j) o[j] = 0.0;
    for (int t = 0; t < k; ++t) {
      const double av = a[(size_t)i * k + t];
      const double* brow = b + (size_t)t * m;
      for (int j = 0; j < m; ++j) {
        double p = av * brow[j];
        o[j] = o[j] + p;
      }
    }
  }
}

double oracle_sigmoid(double x) {
  if (x >= 0) return 1.0 / (1.0 + exp(-x));
  double e = exp(x);
  return e / (1.0 + e);
}

static void affine_gate(const double* xt, const double* h, const double* W, const double* U,
                        const double* b, double* tmp1, double* tmp2, int B, int F, int H) {
  /* tmp1 = (xt @ W + h @ U) + b   (reference: Add(Add(MatMul, MatMul), b)) */
  oracle_matmul(xt, W, tmp1, B, F, H);
  oracle_matmul(h, U, tmp2, B, H, H);
  for (int i = 0; i < B * H; ++i) tmp1[i] = tmp1[i] + tmp2[i];
  for (int r = 0; r < B; ++r)
    for (int j = 0; j < H; ++j) tmp1[(size_t)r * H + j] = tmp1[(size_t)r * H + j] + b[j];
}

/* Returns an error code (0 = ok).  out: [B, min(max_len, T), H] (batch-major, i.e.
 * after the final transpose); *max_len_out receives reduce_max(seq_len).
 * max_iterations < 0 means no limit. */
int oracle_rnn_program(int cell, int B, int T, int F, int H, const double* x, const double* h0,
                       const double* c0, const int64_t* lens, const double* const* W,
                       const double* const* U, const double* const* bias, long long max_iterations,
                       double* out, int64_t* max_len_out) {
  if (B <= 0) return ERR_SHAPE; /* reduce_max of an empty tensor */
  int64_t m = lens[0];
  for (int r = 1; r < B; ++r)
    if (lens[r] > m) m = lens[r];
  *max_len_out = m;
  if (m < 0) return ERR_SHAPE; /* Range(max_len) */
  const int G = cell == CELL_LSTM ? 4 : cell == CELL_GRU ? 3 : 1;
  const int64_t mo = m < T ? m : T; /* row stride of out (== max_len whenever there is no error) */
  double* h = malloc(sizeof(double) * B * H);
  double* c = malloc(sizeof(double) * B * H);
  double* xt = malloc(sizeof(double) * B * (F > 0 ? F : 1));
  double* gates = malloc(sizeof(double) * G * B * H);
  double* tmp = malloc(sizeof(double) * B * H);
  double* nh = malloc(sizeof(double) * B * H);
  double* nc = malloc(sizeof(double) * B * H);
  memcpy(h, h0, sizeof(double) * B * H);
  if (cell == CELL_LSTM) memcpy(c, c0, sizeof(double) * B * H);
  int rc = OK;
  for (int64_t t = 0; t < m; ++t) {
    if (max_iterations >= 0 && t >= max_iterations) { rc = ERR_LIMIT; break; }
    if (t >= T) { rc = ERR_INDEX; break; }
    for (int r = 0; r < B; ++r)
      memcpy(xt + (size_t)r * F, x + ((size_t)r * T + t) * F, sizeof(double) * F);
    for (int g = 0; g < G && cell != CELL_GRU; ++g) {
      double* z = gates + (size_t)g * B * H;
      affine_gate(xt, h, W[g], U[g], bias[g], z, tmp, B, F, H);
      const int is_tanh = (cell == CELL_RNN) || (g == 2);
      for (int i = 0; i < B * H; ++i) z[i] = is_tanh ? tanh(z[i]) : oracle_sigmoid(z[i]);
    }
    if (cell == CELL_GRU) {
      double *gz = gates, *gr = gates + (size_t)B * H, *gn = gates + (size_t)2 * B * H;
      for (int g = 0; g < 2; ++g) {
        double* z = gates + (size_t)g * B * H;
        affine_gate(xt, h, W[g], U[g], bias[g], z, tmp, B, F, H);
        for (int i = 0; i < B * H; ++i) z[i] = oracle_sigmoid(z[i]);
      }
      /* n = tanh((x@Wn + bn) + r * (h@Un + bhn)) */
      oracle_matmul(xt, W[2], gn, B, F, H);
      oracle_matmul(h, U[2], tmp, B, H, H);
      for (int r = 0; r < B; ++r)
        for (int j = 0; j < H; ++j) {
          const size_t i = (size_t)r * H + j;
          double a = gn[i] + bias[2][j];
          double hn = tmp[i] + bias[3][j];
          double rh = gr[i] * hn;
          gn[i] = tanh(a + rh);
        }
      for (int i = 0; i < B * H; ++i) {
        double one_minus = 1.0 - gz[i];
        double p1 = one_minus * gn[i];
        double p2 = gz[i] * h[i];
        nh[i] = p1 + p2;
      }
    } else if (cell == CELL_LSTM) {
      const double *gi = gates, *gf = gates + (size_t)B * H, *gg = gates + (size_t)2 * B * H,
                   *go = gates + (size_t)3 * B * H;
      for (int i = 0; i < B * H; ++i) {
        double fc = gf[i] * c[i];
        double ig = gi[i] * gg[i];
        nc[i] = fc + ig;
        nh[i] = go[i] * tanh(nc[i]);
      }
    } else {
      memcpy(nh, gates, sizeof(double) * B * H);
    }
    for (int r = 0; r < B; ++r) {
      if (t < lens[r]) {
        memcpy(h + (size_t)r * H, nh + (size_t)r * H, sizeof(double) * H);
        if (cell == CELL_LSTM) memcpy(c + (size_t)r * H, nc + (size_t)r * H, sizeof(double) * H);
      }
      memcpy(out + ((size_t)r * mo + t) * H, h + (size_t)r * H, sizeof(double) * H);
    }
  }
  if (rc == OK && m == 0) rc = ERR_EMPTY; /* ListStack of an empty list */
  free(h); free(c); free(xt); free(gates); free(tmp); free(nh); free(nc);
  return rc;
}

/* ------------------------------------------------------------------ CPU baseline
 * P independent problems (one batch each, shared weights) over `threads`
 * POSIX threads: the multi-core CPU executor the bench reports beside the GPU.
 * out_p is [B, T, H] per problem (only [:max_len] written). */
typedef struct {
  int cell, B, T, F, H, P, first, step;
  const double *x, *h0, *c0;
  const int64_t* lens;
  const double* const* W;
  const double* const* U;
  const double* const* bias;
  double* out;
  int64_t* max_len;
  int* status;
} many_args;

static void* many_worker(void* p) {
  many_args* a = (many_args*)p;
  for (int i = a->first; i < a->P; i += a->step) {
    const size_t rows = (size_t)i * a->B;
    a->status[i] = oracle_rnn_program(
        a->cell, a->B, a->T, a->F, a->H, a->x + rows * a->T * a->F, a->h0 + rows * a->H,
        a->cell == CELL_LSTM ? a->c0 + rows * a->H : NULL, a->lens + rows, a->W, a->U, a->bias, -1,
        a->out + rows * a->T * a->H, a->max_len + i);
  }
  return NULL;
}

int oracle_rnn_many(int cell, int B, int T, int F, int H, int P, const double* x, const double* h0,
                    const double* c0, const int64_t* lens, const double* const* W,
                    const double* const* U, const double* const* bias, double* out,
                    int64_t* max_len, int* status, int threads) {
  if (threads < 1) threads = 1;
  pthread_t* tid = malloc(sizeof(pthread_t) * threads);
  many_args* args = malloc(sizeof(many_args) * threads);
  for (int k = 0; k < threads; ++k) {
    many_args a = {cell, B, T, F, H, P, k, threads, x, h0, c0, lens, W, U, bias, out, max_len, status};
    args[k] = a;
    pthread_create(&tid[k], NULL, many_worker, &args[k]);
  }
  for (int k = 0; k < threads; ++k) pthread_join(tid[k], NULL);
  free(tid);
  free(args);
  return 0;
}
