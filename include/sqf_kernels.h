/* sqf_kernels.h — C ABI of the B200 (sm_100a) kernels behind the training
 * step of the seqforge reference (/root/reference/proj). Plain pointers, sizes
 * and a CUDA stream passed as void*; every entry returns 0 on success or a
 * negative SFK_E* code, never allocates device memory, never throws, and
 * launches asynchronously on the given stream.
 *
 * Each entry replaces one compute site of the reference's CPU tape
 * (src/tape.cpp, src/kernels.cpp); the comment on each names the site.
 * All matrices are row-major with an explicit leading dimension (elements).
 * dtype: SFK_F32 (fp32 parity mode), SFK_F16 (the reference's emulated-FP16
 * mode, here real binary16 storage: every store rounds to the binary16 grid
 * exactly as the reference's quantize_fp16 does), SFK_BF16.
 */
#ifndef SQF_KERNELS_H
#define SQF_KERNELS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum sfk_dtype { SFK_F32 = 0, SFK_F16 = 1, SFK_BF16 = 2 };

enum sfk_status {
  SFK_OK = 0,
  SFK_EINVAL = -1,   /* bad shape / pointer / alignment */
  SFK_ECUDA = -2,    /* launch or driver failure; see sfk_last_error() */
  SFK_EUNSUP = -3    /* combination not supported (e.g. tensor-core GEMM in fp32) */
};

const char* sfk_last_error(void);
/* number of SMs of the current device (grid sizing); <0 on failure */
int sfk_num_sms(void);

/* ------------------------------------------------------------------ GEMM
 * C[m x n] (op)= epilogue( sum_k A(i,k) * B(j,k) ), fp32 accumulate.
 * A(i,k) = a[i*lda + k] when a_kmajor else a[k*lda + i]
 * B(j,k) = b[j*ldb + k] when b_kmajor else b[k*ldb + j]
 * Covers the three layouts of Tape::matmul_nt (tape.cpp:182-189, 324-346):
 *   forward  Y = X W^T      : a_kmajor=1, b_kmajor=1
 *   dgrad    dX = dY W      : a_kmajor=1, b_kmajor=0
 *   wgrad    dW += dY^T X   : a_kmajor=0, b_kmajor=0
 * Epilogue flags, applied in this order (q() = round to the storage grid):
 *   SFK_EPI_PREROUND  v = q(acc)            (matmul node output, tape.cpp:292)
 *   SFK_EPI_BIAS      v = q(v + bias[j])    (add_bias, tape.cpp:190-197)
 *   SFK_EPI_RELU      v = max(v, 0)         (relu, tape.cpp:207-210)
 *   SFK_EPI_MASK      v = mask(i,j) > 0 ? q(v) : 0   (relu backward, tape.cpp:376-382)
 *   SFK_EPI_RESIDUAL  v = q(res(i,j) + v)   (residual add, tape.cpp:198-202)
 *   SFK_EPI_ACCUM     v = q(c(i,j) + acc)   (gradient accumulation into c)
 * dtype F16/BF16 runs on tcgen05 tensor cores (TMA -> smem -> UMMA -> TMEM);
 * F32 runs a SIMT fp32 kernel (true fp32, no TF32, for the 1e-4 parity mode).
 */
enum sfk_epi_flags {
  SFK_EPI_PREROUND = 1,
  SFK_EPI_BIAS = 2,
  SFK_EPI_RELU = 4,
  SFK_EPI_MASK = 8,
  SFK_EPI_RESIDUAL = 16,
  SFK_EPI_ACCUM = 32
};

typedef struct sfk_gemm_args {
  int m, n, k;
  int dtype;
  const void* a; int64_t lda; int a_kmajor;
  const void* b; int64_t ldb; int b_kmajor;
  void* c; int64_t ldc;
  const void* bias;               /* [n]            (SFK_EPI_BIAS)     */
  const void* res; int64_t ldr;   /* [m x n]        (SFK_EPI_RESIDUAL) */
  const void* mask; int64_t ldm;  /* [m x n]        (SFK_EPI_MASK)     */
  int flags;
  int force_simt;                 /* testing: run the SIMT kernel for any dtype */
  int tile_n;                     /* tuning: force the tcgen05 tile width (64/128/256), 0 = auto,
                                     < 0 = auto, CTA-pair tiles narrow only past -tile_n % gain */
  int pair;                       /* tuning: 1 = CTA-pair (cta_group::2) 256-row tiles, -1 = single-CTA, 0 = auto */
  /* stream-K (optional): with a workspace of >= 2*SMs*128*256 floats and
   * zeroed counters (>= tiles; re-armed to 0 by the kernel) the 128x256
   * kernel may split the k-loop of the last wave's tiles across all SMs;
   * the parts are summed in k order by the last arriving CTA (deterministic).
   * Concurrent launches need distinct workspaces and counters. */
  float* workspace; int64_t workspace_floats;
  int32_t* counters; int n_counters;
  int stream_k;                   /* 0 = auto, -1 = off, 1 = force when possible */
  /* weight-gradient layout only (a_kmajor = 0, 16-bit): also accumulate the
   * bias gradient of the layer, bias_grad[i] = q(bias_grad[i] + sum_k A(i,k))
   * (add_bias backward, tape.cpp:347-358), summed from the A tiles already in
   * shared memory by the epilogue warps -- no second pass over dY. */
  void* bias_grad;
  /* scheduling: at most this many SMs for the persistent tile loop (0 = all);
   * leaves SMs to kernels of concurrent streams */
  int max_sms;
} sfk_gemm_args;

int sfk_gemm(const sfk_gemm_args* g, void* stream);

/* -------------------------------------------------------- embeddings (a8)
 * out[r] = q( q( q(E[ids[r]]) * scale ) + q(pe[r % width]) )
 * (embedding_lookup + scale + position leaf + add, model.cpp:204-207 /
 * tape.cpp:174-181, 203-206, 25-32, 198-202). pe is an fp32 table
 * [max_positions x d] computed on the host with model.cpp:12-19's libm calls.
 */
int sfk_embed_fwd(int dtype, const int32_t* ids, int rows, int width, int d,
                  const void* table, const float* pe, float scale, void* out,
                  void* stream);

/* Embedding backward (tape.cpp:311-323 with the scale node 370-375 folded in):
 * for each unique id u (uniq[u]), rows seg_rows[seg_off[u]..seg_off[u+1]) in
 * recording order: grad[u] = q( grad[u] + sum_r q(scale * dx[r]) ).
 * Deterministic (no atomics); the host builds the segments. */
int sfk_embed_bwd(int dtype, const int32_t* uniq, const int32_t* seg_off,
                  const int32_t* seg_rows, int nuniq, int d, const void* dx,
                  float scale, void* grad_table, void* stream);
/* The same sums with the segments cut into chunks of <= 16 rows so a
 * frequent id (eos, pad, a Zipf head) no longer serialises one block:
 * chunks[4*c..] = {id, s0, s1, slot} over seg_rows[s0..s1); slot < 0: the id's
 * only chunk, grad[id] = q(grad[id] + sum) directly; slot >= 0: the chunk sum
 * goes to scratch[slot*d..], and multi[4*m..] = {id, first_slot, nslots, 0}
 * folds grad[id] = q(grad[id] + sum over its slots in order). Deterministic
 * (fixed association). 16-bit dtypes, d % 8 == 0; scratch >= nslots*d floats. */
int sfk_embed_bwd_chunked(int dtype, const int32_t* chunks, int nchunks, const int32_t* multi,
                          int nmulti, const int32_t* seg_rows, int d, const void* dx, float scale,
                          float* scratch, void* grad_table, void* stream);

/* ------------------------------------------------------ dropout (a15)
 * Tape::dropout (tape.cpp:109-121, 223-228, 419-425) with the mask stream of
 * model.cpp:156-163: element i keeps factor float(1/(1-p)) unless
 * RngStream(seed, stream_id) draw number i is < p; the mask is recomputed
 * from the counter-based RNG (rng.cpp:10-31), never stored.
 * fwd: out = q(res + q(x*m)), or q(x*m) when res == NULL;
 * bwd: dx = q(g*m), or q(dx + g*m) when accumulate. */
int sfk_dropout_fwd(int dtype, const void* x, const void* res, void* out, int64_t n, float p,
                    uint64_t seed, uint64_t stream_id, void* stream);
int sfk_dropout_bwd(int dtype, const void* g, void* dx, int64_t n, float p, uint64_t seed,
                    uint64_t stream_id, int accumulate, void* stream);

/* ------------------------------------------------------ layer norm (a14)
 * kernels.cpp:30-45 / tape.cpp:211-222: two-pass mean/biased var,
 * rstd = 1/sqrt(var + 1e-5); y = q((x-mean)*rstd*g + b); stats[r] = {mean, rstd}.
 * x, y row stride = d. */
int sfk_layernorm_fwd(int dtype, const void* x, int rows, int d, const void* gamma,
                      const void* beta, void* y, float* stats, void* stream);
/* tape.cpp:383-418: dx = q(dx + rstd*(dxh - mean(dxh) - xh*mean(dxh*xh)))
 * when accumulate, else dx = q(...) ; column partial sums of dy*xh and dy are
 * written to part[2][nblk][d] (fp32) and folded into dgamma/dbeta by
 * sfk_colsum_finish. Returns nblk (<= 592) through *nparts; part holds
 * >= 2*592*d floats. */
int sfk_layernorm_bwd(int dtype, const void* x, const void* dy, int rows, int d,
                      const void* gamma, const float* stats, void* dx, int accumulate,
                      float* part, int* nparts, void* stream);

/* Complete LN backward: dx as above plus dgamma = q(dgamma + sum dy*xh),
 * dbeta = q(dbeta + sum dy), the column partials folded in a fixed order
 * (deterministic) by one fold kernel for both vectors.
 * part: >= 2*592*d floats scratch; counter: reserved (may be NULL). */
int sfk_layernorm_bwd_fused(int dtype, const void* x, const void* dy, int rows, int d,
                            const void* gamma, const float* stats, void* dx, int accumulate,
                            float* part, int32_t* counter, void* dgamma, void* dbeta, void* stream);

/* The same backward split for the B200 schedule (16-bit data, d % 8 == 0,
 * SFK_EUNSUP otherwise): the activation gradient alone (one warp per row, on
 * the critical path) and the gamma/beta gradients alone (column reduction
 * over rows, parameter work; part >= 2*256*d floats). Same formulas and
 * rounding points as sfk_layernorm_bwd_fused. */
int sfk_layernorm_bwd_dx(int dtype, const void* x, const void* dy, int rows, int d,
                         const void* gamma, const float* stats, void* dx, int accumulate,
                         void* stream);
/* The activation gradient with an explicit accumulation source:
 * dx = q(acc + contribution) (acc == NULL: dx = q(contribution); acc may be dx
 * itself or another buffer, so an accumulation need not wait for a reader of
 * the old gradient on another stream). */
int sfk_layernorm_bwd_dx_acc(int dtype, const void* x, const void* dy, int rows, int d,
                             const void* gamma, const float* stats, const void* acc, void* dx,
                             void* stream);
int sfk_layernorm_bwd_params(int dtype, const void* x, const void* dy, int rows, int d,
                             const float* stats, float* part, int32_t* counters, void* dgamma,
                             void* dbeta, void* stream);
/* The activation gradient plus per-block gamma/beta column partials in one
 * pass over x and dy (16 rows per block, warp-order combine): part[2][nblk][d]
 * (*nparts = nblk = ceil(rows/16)); sfk_layernorm_bwd_fold then folds them in
 * block order into dgamma = q(dgamma + sum), dbeta = q(dbeta + sum). */
int sfk_layernorm_bwd_dx_part(int dtype, const void* x, const void* dy, int rows, int d,
                              const void* gamma, const float* stats, void* dx, int accumulate,
                              float* part, int* nparts, void* stream);
int sfk_layernorm_bwd_fold(int dtype, const float* part, int nparts, int d, void* dgamma,
                           void* dbeta, void* stream);
/* gamma/beta gradients in two steps, so the per-node work is one lean pass and
 * the folds of many LayerNorm nodes share one launch:
 * sfk_layernorm_bwd_params_partial: block b of *nparts (<= 148) sums its row
 * chunk of dy*xhat and dy into part[b][0|1][d] (fixed order); part holds
 * >= 2*148*d floats. sfk_layernorm_bwd_params_fold: for every job, in block
 * order, dgamma = q(dgamma + sum_b part[b][0]), dbeta = q(dbeta + sum_b part[b][1]). */
int sfk_layernorm_bwd_params_partial(int dtype, const void* x, const void* dy, int rows, int d,
                                     const float* stats, float* part, int* nparts, void* stream);
typedef struct {
  const float* part;
  void* dgamma;
  void* dbeta;
  int nparts;
  int d;
} sfk_ln_fold_job;
enum { SFK_LN_FOLD_MAX_JOBS = 48 };
int sfk_layernorm_bwd_params_fold(int dtype, const sfk_ln_fold_job* jobs, int njobs, void* stream);
/* (counters: >= ceil(d/256) zeroed int32 slots, re-armed to 0 by the kernel,
 * selects the single-launch form; NULL falls back to partial + fold launches) */

/* ------------------------------------------- column sums (bias grad, a11)
 * tape.cpp:347-358: db = q(db + sum_rows dy). Two deterministic passes:
 * sfk_colsum_partial writes part[nblk][n]; sfk_colsum_finish folds nblk
 * partials in order into out = q(out + sum) (out dtype = dtype). */
int sfk_colsum_partial(int dtype, const void* x, int rows, int n, int64_t ld,
                       float* part, int* nparts, void* stream);
int sfk_colsum_finish(int dtype, const float* part, int nparts, int n, void* out,
                      void* stream);
/* Both passes in one call: out = q(out + sum_rows x). part: >= min(512*n, 4M)
 * floats scratch; counters: >= ceil(n/256) zeroed int32 slots (re-armed to 0 by
 * the kernel) for the single-launch form, or NULL for partial + fold launches. */
int sfk_colsum(int dtype, const void* x, int rows, int n, int64_t ld, float* part,
               int32_t* counters, void* out, void* stream);

/* --------------------------------------------------- attention (a16/a17)
 * Multi-head attention over ragged per-sentence key spans (tape.cpp:229-258,
 * 426-480; spans model.cpp:168-187, 241-249). Query row r = b*q_width + t
 * attends keys b*k_width + j for j < (causal ? t+1 : k_len[b]).
 * q/k/v/o are column slices: element (row, h*dh + c) at ptr[row*ld + h*dh + c].
 * stats[(row*heads + h)] = {max, 1/sum} of the fp32 softmax (saved for bwd).
 * sm_scale = 1/sqrt(dh) applied after the dot, as the reference does. */
typedef struct sfk_attn_args {
  int dtype;
  int batch, q_width, k_width, heads, dh, causal;
  const int32_t* k_len;            /* [batch] (ignored when causal) */
  const void* q; int64_t ldq;
  const void* k; int64_t ldk;
  const void* v; int64_t ldv;
  void* o; int64_t ldo;
  float* stats;                    /* [batch*q_width*heads] float2 */
  /* backward only */
  const void* dout; int64_t lddo;
  void* dq; int64_t lddq;
  void* dk; int64_t lddk;
  void* dv; int64_t lddv;
  float* scratch;                  /* [batch*q_width*heads] floats (row dots) */
} sfk_attn_args;
int sfk_attention_fwd(const sfk_attn_args* a, void* stream);
/* dq/dk/dv are written (not accumulated): each is the attention node's sole
 * contribution to its input gradient. */
int sfk_attention_bwd(const sfk_attn_args* a, void* stream);
/* n attention problems of one pass (the parts of a multi-part batch, each
 * with its own widths, lengths and pointers; heads, dh, causality and
 * strides shared): the same results as n single calls, with the parts of one
 * width class served by one launch. */
int sfk_attention_fwd_parts(const sfk_attn_args* a, int n, void* stream);
int sfk_attention_bwd_parts(const sfk_attn_args* a, int n, void* stream);
/* kernels launched by the calling thread's last sfk_attention_* call */
int sfk_attention_last_launches(void);

/* ---------------------------------- fused label-smoothed xent (a18 + a19)
 * tape.cpp:259-290 + 481-502 + criterions.cpp:10-36 in one pass per row:
 * for active rows (gold != pad): lse, nll = lse - l_gold, correct = argmax==gold
 * (first max), loss = (1-eps)*nll + eps/V * sum_v(lse - l_v) (stored q()'d);
 * dlogits = q(seed * (softmax - target)) written in place over logits when
 * dlogits == logits; inactive rows get zero gradient.
 * row_out[r] = {loss, nll, correct, active}. */
int sfk_xent_fwd_bwd(int dtype, void* logits, int rows, int vocab, int64_t ld,
                     const int32_t* gold, int pad_id, float eps, float seed,
                     void* dlogits, float* row_out, void* stream);
/* ordered reduction of row_out into acc[4] (double: loss, nll, ntokens,
 * ncorrect), accumulated: acc += sums (criterions.cpp:28-34, trainer.cpp:233-236) */
int sfk_xent_reduce(const float* row_out, int rows, double* acc, void* stream);

/* ------------------------------------------------ optimizer (a25, a27, a28)
 * flag[0] |= any non-finite in g[0..n) (trainer.cpp:247-253) */
int sfk_nonfinite(int dtype, const void* g, int64_t n, int32_t* flag, void* stream);
/* Adam (optim.cpp:48-66) fused with the trainer's unscale and 1/ntokens
 * (trainer.cpp:260-265): per element in double math exactly as the reference:
 *   g = float(grad); if (inv_scale_on) g = g / scale (float); g = g / ntok (float)
 *   m = b1*m + (1-b1)*g; v = b2*v + (1-b2)*g*g  (stored float)
 *   p = float(p - lr*(m/bc1)/(sqrt(v/bc2)+eps)); shadow = q(p)
 * Skipped entirely when *skip != 0 (device-side overflow decision). */
int sfk_adam(int grad_dtype, float* master, void* shadow, int shadow_dtype,
             const void* grad, float* m, float* v, int64_t n, double lr, double b1,
             double b2, double eps, double bc1, double bc2, float scale, int unscale,
             float ntokens, const int32_t* skip, void* stream);
/* SGD (optim.cpp:26-31): p = float(p - lr*g') with the same g' preprocessing */
int sfk_sgd(int grad_dtype, float* master, void* shadow, int shadow_dtype,
            const void* grad, int64_t n, double lr, float scale, int unscale,
            float ntokens, const int32_t* skip, void* stream);
/* dst = q(dst + src), elementwise: the index-order replica fold of
 * all_reduce (trainer.cpp:75-87) for replicas sharing one GPU */
int sfk_accumulate(int dtype, void* dst, const void* src, int64_t n, void* stream);
/* shadow = q(master) (trainer.cpp:149-156) */
int sfk_cast(const float* src, void* dst, int dst_dtype, int64_t n, void* stream);

/* K/V-cache reorder of the incremental decoder (model.cpp:540-557):
 * dst[m][r] = src[m][idx[r]] for nmat matrices of `rows` rows of row_bytes
 * (mat_bytes apart), moving the first copy_bytes of each row; 16-byte
 * multiples, out of place. */
int sfk_gather_rows(const void* src, void* dst, const int32_t* idx, int rows, int64_t row_bytes,
                    int64_t copy_bytes, int nmat, int64_t mat_bytes, void* stream);

/* Beam candidate selection (generate.cpp:220-262) per logits row (dtype):
 * lse[r], eos_lp[r] = logit[eos] - lse, and the kk best tokens under
 * key = cum[r] + (logit - lse) descending, token ascending on ties
 * (tok/lp: rows x kk, best first). cum == NULL: rank by the raw logit
 * (descending, token ascending) and return raw logits in lp (top-k sampling). */
int sfk_beam_topk(int dtype, const void* logits, int64_t ld, int rows, int vocab, const double* cum, int kk,
                  int eos, float* lse, float* eos_lp, int32_t* tok, float* lp, void* stream);
/* dst = src converted (any dtype pair) */
int sfk_convert(int src_dtype, const void* src, int dst_dtype, void* dst, int64_t n,
                void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SQF_KERNELS_H */
