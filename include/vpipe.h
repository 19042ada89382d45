/*
 * vpipe — C-ABI of the B200-native Varuna pipeline executor (libvpipe.so).
 *
 * Drop-in boundary. Each entry point names the reference interface it
 * replaces (paths relative to /root/reference; sp/ = pkg/src/spotpipe/).
 * All functions are extern "C", take plain pointers + int64 sizes (+ a
 * cudaStream_t passed as void* for device work) and return int status:
 * VP_OK (0) or a negative VP_ERR_* code, or a positive cudaError_t.
 * PyTorch (or any caller) owns all memory; the library never frees caller
 * memory. There is no CPU fallback for any device entry point.
 */
#ifndef VPIPE_H_
#define VPIPE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
#define VP_OK 0
#define VP_ERR_ARGS (-1)       /* malformed input  -> ConfigError   (sp/core.py:29-30)   */
#define VP_ERR_INFEASIBLE (-2) /* no answer        -> InfeasibleError (sp/core.py:33-34) */
#define VP_ERR_DEADLOCK (-3)   /* event loop stuck -> RuntimeError (sp/engine/_kernel.pyx:544-547) */
#define VP_ERR_NOMEM (-4)      /* -> MemoryError (sp/engine/_kernel.pyx:451-460) */
#define VP_ERR_CAPACITY (-5)   /* caller buffer too small */
#define VP_ERR_UNSUPPORTED (-6)/* shape/layout outside what the kernel supports */
#define VP_ERR_NOTIMPL (-7)

/* Task kind codes; also the within-instant tie-break priority (sp/core.py:22-26). */
#define VP_KIND_BACKWARD 0
#define VP_KIND_RECOMPUTE 1
#define VP_KIND_FORWARD 2

const char* vp_version(void);

/* ======================================================================
 * Control plane (host only)
 * ====================================================================== */

/* Varuna static plan by zero-delay rule simulation.
 * Replaces generate_varuna_schedule -> _simulate_rules
 * (sp/scheduler.py:128-145, 179-284). Times in integer microseconds
 * (the reference rounds seconds with us_from_seconds, sp/core.py:37-38).
 * Outputs: kinds/mbs[capacity] (0-based micro-batches), offsets[P+1]. */
int vp_varuna_schedule(int64_t P, int64_t N, int64_t tf_us, int64_t tb_us, int64_t tr_us,
                       int64_t capacity, int64_t* kinds, int64_t* mbs, int64_t* offsets);

/* GPipe baseline plan. Replaces generate_gpipe_schedule (sp/scheduler.py:148-176). */
int vp_gpipe_schedule(int64_t P, int64_t N, int64_t capacity, int64_t* kinds, int64_t* mbs,
                      int64_t* offsets);

/* Output record of vp_run_replica: caller-allocated arrays, capacity
 * offsets[P] tasks and 2*(P-1)*N messages; per-stage arrays of size P.
 * Mirrors the dict returned by engine.run_replica (sp/engine/py_kernel.py:343-360). */
typedef struct vp_replica_out {
  int64_t *task_stage, *task_kind, *task_mb, *task_start, *task_end;
  int64_t *msg_send, *msg_grant, *msg_arrive, *msg_boundary, *msg_dir, *msg_mb;
  int64_t *last_bwd_end, *peak_stash, *peak_sets, *peak_mem;
  int64_t n_tasks, n_msgs, makespan;
} vp_replica_out;

/* One pipeline replica through the opportunistic Varuna runtime policy.
 * Replaces engine.run_replica (sp/engine/_kernel.pyx:334-351 ≡
 * sp/engine/py_kernel.py:41-360); same 16 arguments, bit-identical results. */
int vp_run_replica(int64_t n_stages, int64_t n_micro, const int64_t* kinds, const int64_t* mbs,
                   const int64_t* offsets, const int64_t* fwd_us, const int64_t* bwd_us,
                   const int64_t* rec_us, const int64_t* act_tx_us, const int64_t* grad_tx_us,
                   const int64_t* exp_grad_tx_us, const int64_t* in_act_bytes,
                   const int64_t* work_bytes, const int64_t* stash_cap, int opportunistic,
                   int serialize_links, vp_replica_out* out);

/* CutPoint -> stage grouping DP. Replaces assign_stages
 * (sp/partitioner.py:269-374); returns boundaries_out[P]. */
int vp_assign_stages(int64_t K, const int64_t* forward_us, const int64_t* acts, int64_t P,
                     double last_stage_weight, int64_t* boundaries_out);

/* CutPoint identification DP. Replaces identify_cutpoints
 * (sp/partitioner.py:124-246); breakable[n-1]; returns boundaries_out[K]. */
int vp_identify_cutpoints(int64_t n, const int64_t* compute_us, const int64_t* acts,
                          const uint8_t* breakable, int64_t K, double tolerance,
                          int64_t* boundaries_out);

/* ======================================================================
 * Device kernels (sm_100a). The reference only prices these
 * (F_i = c_f*params*(m+0.15), B = 2F, R = F: sp/calibration.py:219-221,
 * sp/simulator.py:241-253); see DESIGN.md for each kernel's roofline.
 * Pointers are device pointers; `stream` is a cudaStream_t.
 * ====================================================================== */

/* Device info / runtime. */
int vp_device_sm_count(int* out);

/* GEMM, bf16 operands, fp32 accumulate in TMEM (tcgen05 + TMA).
 *   D[M,N] = epilogue( sum_k A(m,k) * B(n,k) )
 * Operand layouts: a_kmajor=1 -> A stored [M,K] row-major (lda = row stride),
 *                  a_kmajor=0 -> A stored [K,M] row-major (A^T).
 *                  b_kmajor=1 -> B stored [N,K] row-major, b_kmajor=0 -> [K,N].
 * Epilogues (VP_EPI_*), `bias` [N] bf16, `aux` [M,N] bf16 (ldaux):
 *   STORE       D = acc                              (bf16)
 *   BIAS        D = acc + bias                       (bf16)
 *   BIAS_GELU   D = gelu(x), x = bf16(acc + bias); aux (optional) <- gelu'(x)
 *               (bf16: the saving forward keeps the derivative so the backward
 *               DGELU epilogue is a single multiply)
 *   BIAS_RESID  D = aux + acc + bias  (residual add; D may alias aux)
 *   DGELU       D = acc * aux, aux = gelu'(x) from BIAS_GELU (bf16)
 *   ACC_F32     Df32 += acc  (fp32 D, ldd in elements; weight-grad accumulate)
 *   STORE_F32   Df32 = acc   (fp32 D)
 * Replaces the F_i/B_i cost terms of sp/calibration.py:219-221. */
#define VP_EPI_STORE 0
#define VP_EPI_BIAS 1
#define VP_EPI_BIAS_GELU 2
#define VP_EPI_BIAS_RESID 3
#define VP_EPI_DGELU 4
#define VP_EPI_ACC_F32 5
#define VP_EPI_STORE_F32 6
#define VP_EPI_RESID 7   /* D = aux + acc (bias-free residual add) */
int vp_gemm_bf16(int a_kmajor, int b_kmajor, int epilogue, const void* A, int64_t lda,
                 const void* B, int64_t ldb, void* D, int64_t ldd, const void* bias, void* aux,
                 int64_t ldaux, int64_t M, int64_t N, int64_t K, void* stream);
/* Same, with flags: VP_GEMM_DIRECT_STORE writes D with per-thread stores
 * from the epilogue (use when D is an NVLink peer-mapped pointer — the fused
 * "FC2 epilogue -> next stage's ring slot" send). The default path is the
 * 2-CTA (cta_group::2) kernel with TMA-store / TMA-reduce-add epilogues. */
#define VP_GEMM_DIRECT_STORE 1
int vp_gemm_bf16_ex(int a_kmajor, int b_kmajor, int epilogue, const void* A, int64_t lda,
                    const void* B, int64_t ldb, void* D, int64_t ldd, const void* bias, void* aux,
                    int64_t ldaux, int64_t M, int64_t N, int64_t K, int flags, void* stream);
/* As vp_gemm_bf16 (2-CTA path, bf16 output), plus dbias[n] += sum_m D[m, n]
 * (fp32, before the bf16 rounding of D) fused into the epilogue: each warp
 * writes its 32-row partial column sums to `workspace`
 * (vp_gemm_dbias_ws_elems(M, N) floats), reduced in a fixed order afterwards
 * (deterministic). Used for the FC1 bias gradient from the DGELU dgrad. */
int64_t vp_gemm_dbias_ws_elems(int64_t M, int64_t N);
int vp_gemm_bf16_dbias(int a_kmajor, int b_kmajor, int epilogue, const void* A, int64_t lda,
                       const void* B, int64_t ldb, void* D, int64_t ldd, const void* bias,
                       void* aux, int64_t ldaux, int64_t M, int64_t N, int64_t K, float* dbias,
                       float* workspace, void* stream);

/* LayerNorm over rows of x[rows, cols] (bf16 in/out, fp32 stats saved). */
int vp_layernorm_fwd(const void* x, const void* gamma, const void* beta, void* y, float* mean,
                     float* rstd, int64_t rows, int64_t cols, float eps, void* stream);
/* dx (bf16, optionally accumulated into an existing residual grad when
 * accumulate=1: dx += ...), dgamma/dbeta accumulated in fp32. */
int vp_layernorm_bwd(const void* dy, const void* x, const void* gamma, const float* mean,
                     const float* rstd, void* dx, float* dgamma, float* dbeta, int64_t rows,
                     int64_t cols, int accumulate, float* workspace, void* stream);
/* fp32 workspace elements of vp_layernorm_bwd(_ex) for rows of `cols`. */
int64_t vp_layernorm_ws_elems(int64_t cols);
/* As vp_layernorm_bwd, plus (dsum != NULL) dsum[cols] += column sums of the
 * finished dx — the bias gradient of the residual branch feeding dx — in the
 * same pass. Deterministic (fixed-order cross-CTA reduction). */
int vp_layernorm_bwd_ex(const void* dy, const void* x, const void* gamma, const float* mean,
                        const float* rstd, void* dx, float* dgamma, float* dbeta, float* dsum,
                        int64_t rows, int64_t cols, int accumulate, float* workspace,
                        void* stream);
/* The same, also finishing the gradient of the dropped-out residual branch
 * whose output gradient dx is (K7; the reference only prices recompute,
 * sp/calibration.py:219-221): gy = mask(dx)/(1-p) with the site's keep bits
 * (device seed, static salt — the mask its forward GEMM epilogue applied)
 * and dsum += column sums of gy (the branch bias gradient), in one pass.
 * VP_ERR_UNSUPPORTED for row widths without the TMA-ring path; the caller
 * then runs vp_layernorm_bwd_ex + vp_dropout_bwd. */
int vp_layernorm_bwd_dropout(const void* dy, const void* x, const void* gamma, const float* mean,
                             const float* rstd, void* dx, float* dgamma, float* dbeta,
                             float* dsum, void* gy, float p, const uint64_t* seed, uint32_t salt,
                             int64_t rows, int64_t cols, int accumulate, float* workspace,
                             void* stream);

/* Causal/bidirectional fused attention over packed qkv[T, 3h] (T = B*S),
 * heads of size head_dim; o[T, h] bf16; lse[B*heads*S] fp32 saved for bwd. */
int vp_attention_fwd(const void* qkv, void* o, float* lse, int64_t batch, int64_t seq,
                     int64_t heads, int64_t head_dim, int causal, void* stream);
int vp_attention_bwd(const void* qkv, const void* o, const void* dout, const float* lse,
                     void* dqkv, float* delta_ws, int64_t batch, int64_t seq, int64_t heads,
                     int64_t head_dim, int causal, void* stream);
/* As vp_attention_fwd with attention-probability dropout (K7): P[b,h,i,j] is
 * kept iff the mask of element ((b*heads + h)*seq + i)*seq + j (see
 * vp_dropout_dev) under the device-resident seed `*seed` and `salt` is set;
 * the softmax normaliser and lse use the undropped P, kept probabilities are
 * scaled by 1/(1-p). seq even when p > 0. Dropout is not in the reference
 * (its compute is priced, sp/calibration.py:219-221); Varuna recomputes it
 * bit-for-bit in R. */
int vp_attention_fwd_ex(const void* qkv, void* o, float* lse, int64_t batch, int64_t seq,
                        int64_t heads, int64_t head_dim, int causal, float p,
                        const uint64_t* seed, uint32_t salt, const uint32_t* mask_q, void* stream);
/* The keep bits of one attention dropout site, drawn once per (layer,
 * micro-batch) — before the forward, off its softmax critical path — in
 * two layouts of vp_attention_mask_words(batch, seq, heads) uint32 words
 * each (seq % 32 == 0): mask_q word [((b*heads+h)*(seq/32) + key/32)*seq + q]
 * bit key%32 (read by the forward, whose threads own query rows) and mask_k
 * word [((b*heads+h)*(seq/32) + q/32)*seq + key] bit q%32 (read by the
 * backward, whose threads own key rows). Bits = the K7 mask function of
 * (*seed, salt, element ((b*heads+h)*seq + q)*seq + key). Causal: words
 * entirely above the diagonal are not written. */
int64_t vp_attention_mask_words(int64_t batch, int64_t seq, int64_t heads);
int vp_attention_dropout_mask(int64_t batch, int64_t seq, int64_t heads, int causal, float p,
                              const uint64_t* seed, uint32_t salt, uint32_t* mask_q,
                              uint32_t* mask_k, void* stream);
/* Workspace (fp32 elements) of vp_attention_bwd_ex: delta [B*H*S] + the fp32
 * dQ accumulator [B*S*H*D]. */
int64_t vp_attention_bwd_ws_elems(int64_t batch, int64_t seq, int64_t heads, int64_t head_dim);
#define VP_ATTN_DETERMINISTIC 1
/* Backward with one fused tcgen05 kernel per (key block, head) for head_dim
 * 64: S/dP computed once, dK/dV in TMEM, dQ accumulated across key blocks by
 * TMA reduce-add into the fp32 workspace (order-dependent rounding). flags
 * VP_ATTN_DETERMINISTIC (or head_dim != 64) selects the two-kernel
 * deterministic path of vp_attention_bwd. workspace 16-byte aligned. */
int vp_attention_bwd_ex(const void* qkv, const void* o, const void* dout, const float* lse,
                        void* dqkv, float* workspace, int64_t ws_elems, int64_t batch,
                        int64_t seq, int64_t heads, int64_t head_dim, int causal, int flags,
                        float p, const uint64_t* seed, uint32_t salt, const uint32_t* mask_q,
                        const uint32_t* mask_k, float* dbias, void* stream);
/* p > 0: attention-probability dropout of the forward call with the same
 * (seed, salt) — see vp_attention_fwd_ex — differentiated through; mask_q /
 * mask_k (optional): the keep bits vp_attention_dropout_mask drew for that
 * call, read instead of re-hashing every element. */
/* dbias (optional, fused path only, else VP_ERR_UNSUPPORTED): dbias[3*H*D]
 * += column sums of dqkv — the QKV bias gradient — from the dQ post-pass
 * and the dK/dV epilogue partials (fixed-order reductions). */
/* 1 when vp_attention_bwd_ex with these flags (and the VP_ATTN_DETERMINISTIC
 * environment override) takes the fused path, i.e. accepts dbias; callers
 * that get 0 sum the QKV bias gradient themselves. */
int vp_attention_bwd_fuses_bias(int64_t head_dim, int flags);

/* Token + position embedding gather: x[T,h] = wte[ids] + wpe[pos]. */
int vp_embed_fwd(const int64_t* ids, const void* wte, const void* wpe, void* x, int64_t batch,
                 int64_t seq, int64_t hidden, void* stream);
/* dwte[V,h] += scatter(dx), dwpe[S,h] += sum over batch (fp32 accumulators). */
int vp_embed_bwd(const int64_t* ids, const void* dx, float* dwte, float* dwpe, int64_t batch,
                 int64_t seq, int64_t hidden, void* stream);

/* BERT-style embedding with token types: x = wte[ids] + wpe[pos] + tte[types]. */
int vp_embed_typed_fwd(const int64_t* ids, const int64_t* types, const void* wte, const void* wpe,
                       const void* tte, void* x, int64_t batch, int64_t seq, int64_t hidden,
                       void* stream);
/* dwte/dtte scatter-add (fp32), dwpe sum over batch. */
int vp_embed_typed_bwd(const int64_t* ids, const int64_t* types, const void* dx, float* dwte,
                       float* dwpe, float* dtte, int64_t batch, int64_t seq, int64_t hidden,
                       void* stream);
/* dx = dy * gelu'(pre) elementwise (bf16), n elements. */
int vp_gelu_bwd(const void* dy, const void* pre, void* dx, int64_t n, void* stream);

/* Softmax cross-entropy over logits[T,V] (bf16). Writes per-row loss (fp32),
 * adds sum(row_loss)*scale into *loss_sum (optional), and overwrites logits
 * with dlogits = (softmax - onehot) * scale. labels < 0 are ignored. */
int vp_xent_fwd_bwd(void* logits, const int64_t* labels, float* loss_rows, float* loss_sum,
                    int64_t rows, int64_t vocab, float scale, void* stream);
/* As vp_xent_fwd_bwd with the loss scale read from device memory:
 * scale_eff = scale * scale_dev[0] (the dynamic loss scaler's current scale,
 * so captured graphs follow it). */
int vp_xent_fwd_bwd_dev(void* logits, const int64_t* labels, float* loss_rows, float* loss_sum,
                        int64_t rows, int64_t vocab, float scale, const float* scale_dev,
                        void* stream);

/* Column sum of dy[rows, cols] (bf16) accumulated into dbias (fp32), one
 * launch, deterministic. workspace: vp_bias_grad_ws_elems(cols) floats,
 * zero-filled before its first use (arrival counters; left at zero). A
 * workspace sized for C columns may be reused by calls with any cols <= C. */
int64_t vp_bias_grad_ws_elems(int64_t cols);
int vp_bias_grad(const void* dy, float* dbias, int64_t rows, int64_t cols, float* workspace,
                 void* stream);

/* Hash-keyed dropout applied in place: x *= mask(seed, offset, i)/(1-p)
 * (host seed; kept for callers outside the executor). */
int vp_dropout(void* x, int64_t n, float p, uint64_t seed, uint64_t offset, void* stream);

/* K7 dropout-recompute, graph-capturable. The 64-bit seed of the current
 * (step, micro-batch) lives in DEVICE memory — written by vp_set_seed (a
 * one-thread kernel outside any captured graph) before each schedule task —
 * and every dropout site reads it there, keyed with a static per-site
 * `salt`. Mask of element e of a site: b = fmix32(key ^ lo32(e/2)*0x9E3779B1
 * ^ hi32(e/2)*0x85EBCA77), key = fmix32(lo32(seed) ^ fmix32(hi32(seed) ^
 * fmix32(salt))); u = low 16 bits of b for even e, high for odd e; kept iff
 * u >= thr = round(p * 65536), kept values scaled by 65536/(65536 - thr).
 * So R(j) regenerates F(j)'s masks bit for bit (RNG state
 * restored for recompute). */
int vp_set_seed(uint64_t* dst, uint64_t value, void* stream);
/* x[0..n) = value (fp32): the per-step resets of the loss accumulator and
 * the norm / overflow flags. */
int vp_fill_f32(float* x, float value, int64_t n, void* stream);
/* x[n] (bf16, n even) *= mask(e) in place, e = flat index. */
int vp_dropout_dev(void* x, int64_t n, float p, const uint64_t* seed, uint32_t salt,
                   void* stream);
/* Backward of out = resid + dropout(y) for y[rows, cols]: gy = mask(g) (bf16,
 * e = row*cols + col) and dbias[cols] += column sums of gy (fp32, fixed
 * order; workspace as vp_bias_grad's). One pass over g. */
int vp_dropout_bwd(const void* g, void* gy, int64_t rows, int64_t cols, float p,
                   const uint64_t* seed, uint32_t salt, float* dbias, float* workspace,
                   void* stream);
/* D = resid + dropout(A op B^T + bias): the BIAS_RESID epilogue with the K7
 * mask (e = row*N + col, N even) applied to the branch before the residual
 * add; p = 0 is plain BIAS_RESID. flags as vp_gemm_bf16_ex. */
int vp_gemm_bf16_dropout(int a_kmajor, int b_kmajor, const void* A, int64_t lda, const void* B,
                         int64_t ldb, void* D, int64_t ldd, const void* bias, const void* resid,
                         int64_t ldres, int64_t M, int64_t N, int64_t K, float p,
                         const uint64_t* seed, uint32_t salt, int flags, void* stream);

/* Residual add: y = a + b (bf16), n elements. */
int vp_add(const void* a, const void* b, void* y, int64_t n, void* stream);

/* Elementwise product y = a * b (bf16), n elements: the backward of a GELU
 * whose saving forward stored gelu'(pre) (VP_EPI_BIAS_GELU with aux). */
int vp_mul(const void* a, const void* b, void* y, int64_t n, void* stream);

/* Squared-L2 norm and non-finite flag of an fp32 buffer, accumulated into
 * out[0] (sum of squares, fp32) and out[1] (count of non-finite values).
 * Feeds the pipeline-wide overflow/grad-norm agreement. */
int vp_grad_norm_sq(const float* g, int64_t n, float* out, void* stream);

/* Fused unscale + (skip on overflow) + clip + AdamW + fp32 master update +
 * bf16 weight write. `flags` = device [sum_sq, n_nonfinite] after the global
 * reduction; step skipped on device when flags[1] != 0. grad is zeroed.
 * Replaces the 16 B/param optimizer-state model (sp/core.py:17-18). */
int vp_adam_step(float* master, void* weight_bf16, float* grad, float* exp_avg, float* exp_avg_sq,
                 int64_t n, const float* flags, float lr, float beta1, float beta2, float eps,
                 float weight_decay, float inv_loss_scale, float max_grad_norm,
                 float bias_c1, float bias_c2, void* stream);
/* Loss scaling without host round trips (fp16 mixed precision as apex /
 * Megatron run it; the overflow decision is global): the
 * scaler state lives in device memory, float[4] = {loss scale, applied Adam
 * steps, good steps since the last change, scale used by the last step}.
 * vp_adam_step_dev unscales by 1/scaler[0] and takes its bias corrections
 * from step scaler[1]+1 (skipping on overflow as vp_adam_step does);
 * vp_loss_scaler_update then backs the scale off on overflow or grows it
 * after `window` clean steps, and advances the applied-step count only on a
 * clean step. A static scale is growth = backoff = 1. */
int vp_adam_step_dev(float* master, void* weight_bf16, float* grad, float* exp_avg,
                     float* exp_avg_sq, int64_t n, const float* flags, float lr, float beta1,
                     float beta2, float eps, float weight_decay, float max_grad_norm,
                     const float* scaler, void* stream);
int vp_loss_scaler_update(float* scaler, const float* flags, float growth, float backoff,
                          int64_t window, float min_scale, float max_scale, void* stream);

/* Cast fp32 -> bf16 (n elements). */
int vp_cast_f32_bf16(const float* x, void* y, int64_t n, void* stream);
/* DP gradient exchange in bf16 (C1): pack a bucket of the fp32 gradient
 * accumulator to bf16 before the allreduce, unpack the reduced sum back
 * (16-byte aligned buffers). Halves the payload of sp/calibration.py:162-176
 * (2 bytes per parameter, sp/core.py:17-18). */
int vp_grad_pack_bf16(const float* x, void* y, int64_t n, void* stream);
int vp_grad_unpack_bf16(const void* x, float* y, int64_t n, void* stream);

/* ======================================================================
 * Inter-stage P2P over NVLink (device-initiated copies into registered
 * peer buffers). Replaces the modeled transfer + serialized link of
 * send() (sp/engine/py_kernel.py:184-214, sp/calibration.py:95-110).
 * ====================================================================== */
#define VP_IPC_HANDLE_BYTES 64
/* Dedicated device allocation (its own cudaMalloc, so an IPC handle maps
 * exactly this buffer at offset 0) and release. */
int vp_device_alloc(int64_t bytes, void** ptr_out);
int vp_device_free(void* ptr);
/* Export a device allocation / create+export an interprocess event. */
int vp_ipc_get_mem_handle(void* dev_ptr, void* handle_out /*64 bytes*/);
int vp_ipc_open_mem_handle(const void* handle /*64 bytes*/, void** dev_ptr_out);
int vp_ipc_close_mem_handle(void* dev_ptr);
int vp_ipc_event_create(void** event_out, void* handle_out /*64 bytes*/);
int vp_ipc_event_open(const void* handle, void** event_out);
int vp_event_destroy(void* event);
int vp_event_record(void* event, void* stream);
int vp_stream_wait_event(void* stream, void* event);
int vp_event_query(void* event); /* 0 = complete, 1 = pending, else error */
/* SM-driven copy of `bytes` from src into a (peer-mapped) dst, 16B vectors. */
int vp_p2p_put(void* dst, const void* src, int64_t bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* VPIPE_H_ */
