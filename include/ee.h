/*
 * ee.h — C-ABI of libee.so, the B200 (sm_100a) early-exit hot path.
 *
 * The drop-in boundary for the reference's kernel plugin `eepipe.kernels`
 * (`pkg/src/eepipe/kernels.py:1-41`) and for the raw-array inference math that
 * the reference keeps outside that module (`eepipe/inference.py:118-229`).
 * Granularity is fused hot-path ops rather than the reference's 11 float64
 * micro-kernels; each entry point names the reference function(s) it
 * replaces.
 *
 * Conventions:
 *  - every pointer argument is a DEVICE pointer owned by the caller unless
 *    stated; no allocation happens inside the library; workspaces are
 *    caller-provided and sized by ee_workspace_bytes();
 *  - every call is asynchronous on `stream` (a cudaStream_t passed as void*);
 *  - activations on the residual stream are float32; weights, KV cache and
 *    GEMV inputs use `dtype` (EE_F32 parity mode or EE_BF16 perf mode);
 *  - results are deterministic and ROW-STABLE: the value computed for one row
 *    does not depend on how many rows share the call (the reference's
 *    `dot_rows` contract, `eepipe/_pykernels.py:14-17`, `115-121`), so batched
 *    KV recomputation and pipelined inference agree bitwise;
 *  - return code 0 = OK; otherwise an EE_E* code that the Python host maps to
 *    the reference exception classes (`eepipe/errors.py:4-25`), with a
 *    thread-local message from ee_last_error().
 */
#ifndef EE_H_
#define EE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* return codes -> eepipe.errors */
#define EE_OK 0
#define EE_ESHAPE 1     /* ShapeError */
#define EE_ETOKEN 2     /* TokenError */
#define EE_ENONFINITE 3 /* NonFiniteError */
#define EE_ECONFIG 4    /* ConfigError */
#define EE_ECUDA 5      /* RuntimeError (CUDA launch / runtime failure) */

/* dtypes */
#define EE_F32 0
#define EE_BF16 1
/* bf16 weights in the TILED layout produced by ee_pack_tiled (activations and
 * KV cache stay plain bf16): the TMA-fed GEMV path, K % 512 == 0 */
#define EE_BF16_TILED 2

/* GEMV epilogues */
#define EE_EPI_STORE 0    /* out[r, n] = v            (float32 out)          */
#define EE_EPI_RESIDUAL 1 /* out[r, n] += v           (float32 residual)     */
#define EE_EPI_GELU 2     /* out[r, n] = gelu_erf(v)  (dtype out)            */

/* workspace ops for ee_workspace_bytes */
#define EE_OP_ATTENTION 1
#define EE_OP_EXIT_HEAD 2
#define EE_OP_DECODER 3
#define EE_OP_EXIT_HEAD_TRAIN 4
#define EE_OP_RMSNORM_BWD 5
#define EE_OP_PREFILL 6

const char* ee_last_error(void);
int ee_abi_version(void);
/* number of SMs of the current device (grid sizing), -1 on error */
int ee_device_sms(void);

size_t ee_workspace_bytes(int op, int64_t m, int64_t h, int64_t V, int64_t nh, int64_t s_max);

/* HBM weight layout for the TMA-fed GEMV.  A (N, K) row-major bf16 matrix is
 * re-laid out as [N/16 tiles][K/512 stages][16 rows][512] (zero rows pad N;
 * 16-byte chunk c of row r stored at chunk c ^ (r & 7)), so each pipeline
 * stage is one contiguous 16 KB bulk copy.  ee_tiled_weight_bytes returns 0
 * when the shape is not packable (K % 512 != 0).  One-time, at load.
 * col_scale (K float32, nullable) multiplies column k — how an RMSNorm
 * weight is folded into the matrix that consumes the normed rows. */
size_t ee_tiled_weight_bytes(int64_t N, int64_t K);
int ee_pack_tiled(const void* W, int64_t N, int64_t K, const float* col_scale, void* out,
                  void* stream);

/* Token + position embedding rows: out[r] = tok_emb[tok[r]] + pos_emb[pos[r]]
 * (float32 out).  Replaces `_InferParams.embed` (eepipe/inference.py:187-191)
 * and `embed_tokens` (eepipe/model.py:233-243).  Token ids are validated by
 * the host (TokenError) before the call. */
int ee_embed(const int32_t* tok, const int32_t* pos, int64_t m, const void* tok_emb,
             const void* pos_emb, int64_t h, int dtype, float* out, void* stream);

/* RMSNorm of (optionally gathered) float32 rows into a compact dtype buffer:
 * out[i] = x[rows[i]] * (mean(x^2)+eps)^-1/2 * w  (w == NULL: plain cast).
 * Replaces `rmsnorm_fwd` (eepipe/_pykernels.py:36-41). rows may be NULL. */
int ee_rmsnorm_rows(const float* x, int64_t ldx, const int32_t* rows, int64_t m, int64_t h,
                    const float* w, float eps, void* out, int dtype, void* stream);

/* Row-stable GEMV/GEMM  v[r, n] = sum_k x[r, k] * W[n, k]  with a fused
 * epilogue (EE_EPI_*).  W is (N, K) row-major ("K-major", i.e. the reference
 * matrix transposed once at load).  x is (m, K) in `dtype`.
 * Replaces `dot_rows` (eepipe/_pykernels.py:115-121) and its callers'
 * elementwise tails (`x + dot_rows(..)`, `gelu_fwd(dot_rows(..))`,
 * eepipe/inference.py:227-229). */
int ee_gemv(const void* x, int64_t m, int64_t K, const void* W, int64_t N, int dtype, int epilogue,
            void* out, int64_t ldo, void* stream);

/* Fused Q/K/V projection with the KV-cache write in the epilogue:
 * [q | k | v] = xn @ Wqkv^T,  q -> q_out (float32, m x h),
 * k, v -> kcache/vcache[pos[r]] (dtype, layout (s_max, h)).
 * Replaces the q/k/v `dot_rows` + `KVCache.fill` of `_layer_step`
 * (eepipe/inference.py:219-226). */
int ee_qkv_kvwrite(const void* xn, int64_t m, int64_t h, const void* Wqkv, int dtype, float* q_out,
                   void* kcache, void* vcache, const int32_t* pos, void* stream);

/* Multi-row causal decode attention: row r attends over cache positions
 * 0..pos[r] of one layer (K/V of all rows already written).  Split-KV chunks
 * are keyed by position only and merged in a fixed order (row-stable).
 * q float32 (m, nh*dh); out dtype (m, nh*dh).  max_pos >= max(pos).
 * Replaces `_attend_rows` (eepipe/inference.py:194-213). */
int ee_decode_attention(const float* q, int64_t m, const int32_t* pos, int32_t max_pos,
                        const void* kcache, const void* vcache, int64_t nh, int64_t dh, int dtype,
                        void* out, void* ws, size_t ws_bytes, void* stream);

/* Fused inference exit head: gathers the float32 residual rows x[rows[i]]
 * (rows may be NULL), applies the head's RMSNorm (norm_w; NULL for a
 * minimalistic exit), computes logits = xn @ W^T over the vocabulary WITHOUT
 * writing them (unless logits_dbg != NULL, (m, V) float32), with a split-V
 * (max, sum-exp, argmax) per vocabulary tile and a fixed-order merge, then
 *   token[r] = argmax (lowest index wins ties),
 *   conf[r]  = max softmax probability = 1 / sum exp(l - max),
 *   fire[r]  = threshold < 1 && conf > threshold.
 * *nonfinite is set to 1 if any logit was not finite (host raises
 * NonFiniteError).  m <= 16 per call.  W is (V, h) row-major.
 * Replaces `head_logits` + `exit_decision` (eepipe/inference.py:118-133,
 * 175-185). */
int ee_exit_head_infer(const float* x, int64_t ldx, const int32_t* rows, int64_t m, int64_t h,
                       const float* norm_w, float eps, const void* W, int64_t V, int dtype,
                       float threshold, int32_t* token, float* conf, uint8_t* fire,
                       int32_t* nonfinite, float* logits_dbg, void* ws, size_t ws_bytes,
                       void* stream);

/* ---- decode layer chain (the KV-recompute kernel) -------------------- */

typedef struct {
    const float* attn_norm; /* (h) float32 */
    const void* wqkv;       /* (3h, h) dtype: [wq^T; wk^T; wv^T] */
    const void* wo;         /* (h, h)  dtype: wo^T */
    const float* mlp_norm;  /* (h) float32 */
    const void* w1;         /* (4h, h) dtype: w1^T */
    const void* w2;         /* (h, 4h) dtype: w2^T */
    void* kcache;           /* (s_max, h) dtype */
    void* vcache;           /* (s_max, h) dtype */
} ee_layer_t;

typedef struct {
    int64_t h, nh, s_max, max_rows;
    int dtype;  /* EE_F32, EE_BF16 or EE_BF16_TILED (weights of ee_layer_t) */
    float eps;
    float* x;   /* (max_rows, h) float32 residual rows (the rows of a pass) */
    void* xb;   /* tiled mode: (max_rows, h) bf16 copy of x */
    float* ssq; /* tiled mode: (max_rows, h/16) per-16-column sums of x^2 */
    void* xn;   /* (max_rows, 4h) dtype scratch */
    float* q;   /* (max_rows, h) float32 scratch */
    void* attn; /* (max_rows, h) dtype scratch */
    void* ws;   /* attention workspace (ee_workspace_bytes(EE_OP_ATTENTION, ...)) */
    size_t ws_bytes;
    /* tiled mode, nullable: split-K partials of the multi-row tcgen05 GEMM,
     * >= ee_workspace_bytes(EE_OP_PREFILL, max_rows, h, ...).  Callers set it
     * ONLY for a prompt-prefill pass (every prompt row, computed once in every
     * inference mode) with > 16 rows; with it null every pass takes the
     * row-stable GEMV, so decode rows never depend on the pass width */
    void* pf_ws;
    size_t pf_ws_bytes;
} ee_decoder_t;

/* ee_embed followed, when xb and ssq are non-null (tiled mode), by
 * ee_row_stats of the new rows (out has row stride h): one call per pass. */
int ee_embed_stats(const int32_t* tok, const int32_t* pos, int64_t m, const void* tok_emb,
                   const void* pos_emb, int64_t h, int dtype, float* out, void* xb, float* ssq,
                   void* stream);

/* Asynchronous host -> device copy of `bytes` from PINNED host memory on
 * `stream` (the per-pass control block upload). */
int ee_copy_h2d(void* dst, const void* src, size_t bytes, void* stream);

/* Row statistics for tiled mode: xb = bf16(x), ssq[r][t] = sum_{i<16}
 * x[r][16t+i]^2.  Must be called for rows whose x was written outside the
 * decoder (embedding, rows received from another pipeline stage); the
 * decoder keeps them current for the rows it updates. */
int ee_row_stats(const float* x, int64_t ldx, int64_t m, int64_t h, void* xb, float* ssq,
                 void* stream);

/* One transformer layer for rows [row0, row0+m) of dec->x (float32, updated
 * in place), KV written at pos[i] (the positions of those rows) before any
 * row attends: RMSNorm -> QKV(+KV write) -> attention -> wo + residual ->
 * RMSNorm -> w1 + GELU -> w2 + residual.  In tiled mode the norm weights
 * must have been folded into the Wqkv / W1 columns (ee_pack_tiled with
 * col_scale).  Replaces `_layer_step` (eepipe/inference.py:216-229). */
int ee_decode_layer(const ee_decoder_t* dec, const ee_layer_t* layer, int64_t row0, int64_t m,
                    const int32_t* pos, int32_t max_pos, void* stream);

/* Layers [0, n_layers) of `layers` in order over rows [0, n_rows) of dec->x,
 * which are ordered by entry depth DESCENDING, so the rows a layer must
 * advance (entry < layer) are always a suffix: layer i advances rows
 * [n_rows - m_active[i], n_rows) (m_active[i] == 0 skips the layer); pos
 * holds the positions of rows 0..n_rows-1.  This is the batched back-fill
 * pass of KV recomputation (`run_pass` layer loop,
 * eepipe/inference.py:316-326): one weight read per layer serves every
 * deferred row plus the new one. */
int ee_decode_layers(const ee_decoder_t* dec, const ee_layer_t* layers, int32_t n_layers,
                     int64_t n_rows, const int32_t* m_active, const int32_t* pos, int32_t max_pos,
                     void* stream);

/* ---- the KV-recomputation decode loop, natively ------------------------ */

/* One exit head as the decode loop sees it (heads sorted by (tap, is_final)). */
typedef struct {
    int32_t tap;            /* layer index 0..L the head reads */
    int32_t is_final;
    int32_t kind;           /* 0 minimalistic, 1 norm+embed, 2 mlp+embed */
    const float* norm;      /* nullable: RMSNorm weight before the projection */
    const float* pre_norm;  /* mlp+embed: RMSNorm weight of the MLP prelude */
    const void* w1t;        /* mlp+embed: (4h, h) */
    const void* w2t;        /* mlp+embed: (h, 4h) */
    const void* W;          /* (V, h) output matrix in the `wcode` layout */
    int64_t V;
} ee_head_t;

/* The HBM-resident state of one KV-recomputation engine. */
typedef struct {
    const ee_decoder_t* dec;  /* residual rows + scratch (max_rows >= prompt, max_deferred + 1) */
    const ee_layer_t* layers; /* n_layers entries, layer l at index l - 1 */
    int32_t n_layers;
    const ee_head_t* heads;
    int32_t n_heads;
    int dcode;                /* activation dtype (EE_F32 / EE_BF16) */
    int wcode;                /* head weight layout (EE_F32 / EE_BF16 / EE_BF16_TILED) */
    float eps;
    const void* tok_emb;      /* (V, h) dcode */
    const void* pos_emb;      /* (s_max, h) dcode */
    int32_t* ctrl;            /* device control block (ctrl_cap int32) */
    int32_t* ctrl_host;       /* PINNED host staging, 2 * ctrl_cap int32 */
    int64_t ctrl_cap;
    void* head_ws;            /* ee_workspace_bytes(EE_OP_EXIT_HEAD, 16, h, V_max, ...) */
    size_t head_ws_bytes;
    void* head_x;             /* mlp+embed scratch: (16, h) float32 */
    void* head_xn;            /* (16, h) dcode */
    void* head_mid;           /* (16, 4h) dcode */
    uint8_t* res;             /* result slots the heads write: max_slots x res_stride bytes,
                               * device memory, or res_host itself (host-mapped: the loop
                               * then polls each slot's nonfinite word, armed to -1 at
                               * launch and written last, instead of copy + sync) */
    uint8_t* res_host;        /* PINNED host copy of the result slots */
    int32_t res_stride, max_slots;
    int32_t off_tok, off_conf, off_fire, off_bad;  /* field offsets inside a slot */
    void* stream;
    void* pf_ws;              /* nullable: prefill GEMM workspace, used for the prefill pass only */
    size_t pf_ws_bytes;
} ee_engine_t;

typedef struct {
    const ee_engine_t* engine;
    /* in */
    const int32_t* prompt;    /* host, prompt_len ids (validated by the caller) */
    int32_t prompt_len, max_new, max_deferred, s_max, head_max_rows;
    float threshold;
    int32_t n_heads;          /* == engine->n_heads (conf row width) */
    /* out (host arrays owned by the caller) */
    int32_t* tokens;          /* [max_new] */
    int32_t* exit_layers;     /* [max_new] */
    int32_t* pass_depths;     /* [max_new] depth of the pass that decided each token */
    double* latency_s;        /* [max_new] host seconds between decisions */
    float* conf;              /* [s_max][n_heads] confidences (caller-initialised NaN) */
    uint8_t* kv_mask;         /* nullable [n_layers][s_max] final KV fill mask */
    int32_t n_generated, flushed;
    double total_s;
    int64_t launches, h2d_bytes, d2h_bytes;
} ee_generate_args_t;

/* `generate_kv_recompute` (eepipe/inference.py:256-381) for one prompt in a
 * single call: prefill, the per-token batched back-fill passes with the
 * early-exit decisions, the final flush pass and the KV completeness check.
 * Synchronises `stream` at exit taps / pass ends (the greedy decision is
 * data-dependent) and on return.  Errors: EE_ECONFIG (threshold, prompt,
 * max_deferred, KV discipline), EE_ETOKEN (context overflow),
 * EE_ENONFINITE (non-finite exit logits). */
int ee_generate_kv_recompute(ee_generate_args_t* args);

/* ---- training exit head (fused CE) ---------------------------------- */

/* Weighted cross-entropy of one exit head and its gradients on tcgen05
 * tensor cores, without the (n, V) logits in HBM (four TMA-fed tcgen05
 * GEMMs whose epilogues do the online softmax; see exit_head_train.cu).
 * x (n, h) bf16 (already normed if the head has a norm), W (V, h) bf16
 * (both also read MN-major by the backward GEMMs: no transposed copies),
 * targets int64 (n), validated by the caller.  Writes
 *   *loss  = weight * mean_i CE_i (float32, device scalar),
 *   dx     = d loss / d x  (n, h) float32,
 *   dw_acc += d loss / d W (V, h) float32 (accumulated across microbatches).
 * h, V multiples of 8 (any n).  Workspace: ee_workspace_bytes(EE_OP_EXIT_HEAD_TRAIN,
 * n, h, V, 0, 0).  Replaces `run_head` matmul + `cross_entropy` fwd/bwd + the
 * matmul backward (eepipe/model.py:219-230, eepipe/autodiff.py:158-179,
 * 301-323, eepipe/_ckernels.pyx:130-167). */
int ee_exit_head_train(const void* x, int64_t n, int64_t h, const void* W, int64_t V,
                       const int64_t* targets, float weight, float* loss, float* dx, float* dw_acc,
                       void* ws, size_t ws_bytes, void* stream);

/* The same head split at the autograd boundary (forward / backward):
 *   ee_exit_head_train_fwd: *loss as above; G (n, V) bf16 caller buffer
 *     receives d loss / d logits (kept for the backward);
 *   ee_exit_head_train_bwd: dx = grad * G W (n, h) float32,
 *     dw_acc += grad * G^T x (V, h) float32, where grad points to the
 *     incoming gradient of the loss (device float32 scalar, read by the
 *     epilogues: no host synchronisation; nullptr = 1).
 * Same shapes, workspace and reference boundary as ee_exit_head_train. */
int ee_exit_head_train_fwd(const void* x, int64_t n, int64_t h, const void* W, int64_t V,
                           const int64_t* targets, float weight, float* loss, void* G, void* ws,
                           size_t ws_bytes, void* stream);
int ee_exit_head_train_bwd(const void* x, int64_t n, int64_t h, const void* W, int64_t V,
                           const void* G, const float* grad, float* dx, float* dw_acc, void* ws,
                           size_t ws_bytes, void* stream);

/* dW (in x out, float32) += X^T dY for a bf16 linear layer y = x W, X (T x in)
 * and dY (T x out) bf16 row-major, on the CTA-pair tcgen05 GEMM (operands read
 * MN-major in place).  The training backbone's gradient-accumulation fusion:
 * the weight gradient of every microbatch lands in the float32 accumulator
 * without a bf16 gradient or an accumulation pass (the matmul backward of
 * `eepipe/autodiff.py:170-177` for the layer weights). */
int ee_wgrad_accum(const void* X, const void* dY, int64_t T, int64_t in, int64_t out, float* dW,
                   void* stream);

/* The training MLP block's GEMMs with the GELU fused into the epilogue
 * (CTA-pair tcgen05 GEMM), `gelu_fwd` / `gelu_bwd` of eepipe/_pykernels.py:
 * 27-33 around the w1 / w2 matmuls of eepipe/model.py:214-216:
 *   ee_mlp_up_gelu:  pre = X W1, act = GELU_erf(pre)        (bf16 outputs)
 *   ee_mlp_gelu_bwd: dpre = (dY W2^T) * GELU_erf'(pre)      (bf16 output)
 * X, dY (T x h), pre / act / dpre (T x N) row-major bf16; W1 (h x N) and
 * W2 (N x h) row-major bf16 (the layer's own weights, read in place).  The
 * GEMM result is rounded to bf16 before the element-wise op, as the unfused
 * bf16 path would read it.  h, N multiples of 8. */
int ee_mlp_up_gelu(const void* X, const void* W1, int64_t T, int64_t h, int64_t N, void* pre,
                   void* act, void* stream);
int ee_mlp_gelu_bwd(const void* dY, const void* W2, int64_t T, int64_t h, int64_t N,
                    const void* pre, void* dpre, void* stream);

/* ---- training backbone linears (CTA-pair tcgen05 GEMM) ------------------
 * The forward and input-gradient matmuls of `run_layer` (eepipe/model.py:
 * 207-216; `matmul` fwd / bwd, eepipe/autodiff.py:158-179):
 *   ee_linear_fwd:   Y  = X W   [+ R]   X (T x K), W (K x N), Y / R (T x N)
 *   ee_linear_dgrad: dX = dY W^T [+ R]  dY (T x N), W (K x N), dX / R (T x K)
 * bf16 row-major, float32 accumulation, the optional residual R (nullable)
 * added before the single rounding.  K, N multiples of 8. */
int ee_linear_fwd(const void* X, const void* W, int64_t T, int64_t K, int64_t N, const void* R,
                  void* Y, void* stream);
int ee_linear_dgrad(const void* dY, const void* W, int64_t T, int64_t K, int64_t N, const void* R,
                    void* dX, void* stream);

/* Stacked variants: `parts` same-shape (K x N) weight matrices adjacent in
 * memory (W_j = W + j K N; the q / k / v projections of one block in the
 * flat parameter buffer) as ONE GEMM each way (replaces the three h1 @ wq,
 * h1 @ wk, h1 @ wv matmuls of eepipe/model.py:207-216 and their backward,
 * eepipe/autodiff.py:158-179):
 *   ee_linear_fwd_stacked:   Y (T x parts N) = X [W_0 | ... | W_{p-1}]
 *   ee_linear_dgrad_stacked: dX (T x K) = dY (T x parts N) [W_0 | ...]^T [+ R]
 *   ee_wgrad_accum_stacked:  dW_j (in x out, float32, dW_j = dW + j in out)
 *                            += X^T dY[:, j out : (j + 1) out]
 * N (out, in) multiples of 128, K a multiple of 64. */
int ee_linear_fwd_stacked(const void* X, const void* W, int64_t T, int64_t K, int64_t N,
                          int64_t parts, void* Y, void* stream);
int ee_linear_dgrad_stacked(const void* dY, const void* W, int64_t T, int64_t K, int64_t N,
                            int64_t parts, const void* R, void* dX, void* stream);
int ee_wgrad_accum_stacked(const void* X, const void* dY, int64_t T, int64_t in, int64_t out,
                           int64_t parts, float* dW, void* stream);

/* ---- training backbone causal attention (tcgen05, flash-style) ---------
 * `causal_attention` forward / backward (eepipe/autodiff.py:265-298) and the
 * boundary kernels attention_fwd / attention_bwd (eepipe/_pykernels.py:52-62,
 * eepipe/_ckernels.pyx:170-236) without the (S x S) probabilities in HBM.
 * Q, K, V, O, dO, dQ, dK, dV: (B*S, ld) bf16 row-major, head h in columns
 * [128 h, 128 h + 128) (head_dim 128; the projections' own layout, e.g. the
 * q / k / v column blocks of one fused output); S a multiple of 128.  lse
 * (forward output, backward input) and dsum (backward scratch) are float32
 * [B][H][S].  Deterministic (no atomics); scale 1/sqrt(128). */
int ee_attn_train_fwd(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v,
                      int64_t ldv, int64_t B, int64_t S, int64_t H, void* out, int64_t ldo,
                      float* lse, void* stream);
int ee_attn_train_bwd(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v,
                      int64_t ldv, const void* o, int64_t ldo, const void* dout, int64_t ldd,
                      const float* lse, int64_t B, int64_t S, int64_t H, void* dq, int64_t lddq,
                      void* dk, int64_t lddk, void* dv, int64_t lddv, float* dsum, void* stream);

/* ---- training RMSNorm (bf16 activations, float32 statistics) ---------- */

/* y = x * (mean(x^2) + eps)^-1/2 * w row-wise; x, y (n, h) bf16, w (h) float32,
 * inv_rms (n) float32 saved for the backward.  h % 8 == 0.  Replaces
 * `rmsnorm_fwd` (eepipe/_pykernels.py:36-41, eepipe/_ckernels.pyx:46-65) on the
 * training backbone. */
int ee_rmsnorm_fwd(const void* x, int64_t n, int64_t h, const float* w, float eps, void* y,
                   float* inv_rms, void* stream);

/* gx (n, h) bf16 and gw (h) float32 (overwritten, or accumulated when
 * accumulate_gw != 0) from x, w, inv_rms and gy (n, h) bf16; gw is reduced in
 * a fixed order (deterministic).  gres (n, h) bf16, optional (NULL): a second
 * gradient of x (the residual branch of a pre-norm block) added into gx in the
 * same pass.  Workspace: ee_workspace_bytes(
 * EE_OP_RMSNORM_BWD, n, h, 0, 0, 0).  Replaces `rmsnorm_bwd`
 * (eepipe/_pykernels.py:44-49, eepipe/_ckernels.pyx:68-89). */
int ee_rmsnorm_bwd(const void* x, const float* w, const float* inv_rms, const void* gy,
                   const void* gres, int64_t n, int64_t h, void* gx, float* gw, int accumulate_gw,
                   void* ws, size_t ws_bytes, void* stream);

/* ---- optimizer step (fused, multi-tensor) ----------------------------- */

#define EE_OPT_SGD 0
#define EE_OPT_ADAM 1
#define EE_OPT_ACCUM 2 /* param += grad * grad_scale: float32 gradient accumulation */

/* One parameter tensor of a fused optimizer step; the table itself is a
 * DEVICE array, entries sorted by `start` (prefix element offsets, tensors
 * laid end to end in one index space of `total` elements). */
typedef struct {
    float* param;       /* float32 master weights (n), updated in place      */
    const void* grad;   /* gradient (n), float32 or bf16 (grad_dtype)         */
    float* m;           /* Adam first moment (n), float32; unused for SGD     */
    float* v;           /* Adam second moment (n), float32; unused for SGD    */
    void* param_lp;     /* nullable: bf16 copy of the updated weights (n)     */
    int64_t n;          /* element count                                     */
    int64_t start;      /* offset of element 0 in the virtual index space    */
} ee_opt_tensor_t;

/* One optimizer step over every tensor of `table` in a single launch:
 * SGD p -= lr * g, or Adam m += (1-b1)(g-m), v += (1-b2)(g^2-v),
 * p -= step_size * m / (sqrt(v) + eps), with g = grad * grad_scale and
 * step_size = lr * sqrt(1 - b2^t) / (1 - b1^t) computed by the caller.
 * Replaces `SGD.step` / `Adam.step` (eepipe/training.py:24-53); the caller
 * passes grad_scale = 1 / num_microbatches (eepipe/training.py:108). */
int ee_optimizer_step(const ee_opt_tensor_t* table, int32_t n_tensors, int64_t total, int kind,
                      int grad_dtype, float lr, float beta1, float beta2, float eps,
                      float grad_scale, float step_size, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* EE_H_ */
