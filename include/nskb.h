/* libnskb — the C ABI behind the B200-native NSK training-step hot path.
 *
 * Every entry point returns an int status (0 = OK); nsk_last_error() gives
 * the message of the last failure on the calling thread. Status codes map
 * back onto the reference's error types in the Python layer
 * (paper_2409_11600_b200/_lib.py):
 *   1 NSK_ERR_OOM    -> NskRuntimeError("out of memory: requested N elements")  (tensor.py:41-44)
 *   2 NSK_ERR_SHAPE  -> NskTypeError                                             (errors.py:43-44)
 *   3 NSK_ERR_CUDA / 4 NSK_ERR_NCCL -> NskRuntimeError
 *   5 NSK_ERR_RANGE  -> NskRuntimeError (index out of range)                     (tensor.py:308-313)
 *   6 NSK_ERR_UNSUPPORTED -> NskRuntimeError
 * Plain pointers and sizes only: device pointers are raw CUDA device
 * addresses, `stream` is a cudaStream_t (NULL = legacy default stream).
 * All kernels fully overwrite their outputs (reference tensor.py:6-8), so
 * NaN-poisoned pooled buffers never leak.
 *
 * Reference interfaces replaced (file:line under /root/reference/pkg/src/nsk):
 *   Buffer / Pool storage ........ tensor.py:29-113   -> nsk_arena_*, nsk_fill_*, nsk_memcpy_*
 *   matmul_t / plain_matmul ...... tensor.py:213-234  -> nsk_gemm, nsk_gemm_simt
 *   elementwise / bias_add ....... tensor.py:247-296  -> nsk_eltwise, nsk_eltwise_bwd, nsk_bias_add, nsk_colsum
 *   onehot ....................... tensor.py:299-317  -> nsk_onehot
 *   GradCache.accumulate/zero .... tensor.py:337-364  -> nsk_axpy, nsk_fill_f32
 *   gradient_rule ................ autodiff.py:253-293 -> nsk_eltwise_bwd, nsk_gemm*, nsk_xent_bwd
 *   rec_cross_entropy / sum_loss . autodiff.py:213-248 -> nsk_xent_fwd, nsk_sum_f32
 *   _accuracy .................... builtins.py:70-80  -> nsk_argmax_correct
 *   sgd_step / adamw_step ........ nn.py:91-119       -> nsk_sgd_multi, nsk_adamw_multi
 *   clip_grad_norm ............... nn.py:122-139      -> nsk_sqnorm_multi, nsk_scale_multi
 *   (absent, restated in oracle/) conv2d, batchnorm, pooling, GRU, embedding, crop/flip
 */
#ifndef NSKB_H
#define NSKB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NSK_ABI_VERSION 1

#define NSK_DTYPE_F32 0
#define NSK_DTYPE_BF16 1

/* ---- runtime, memory, streams, graphs (runtime.cu) ---- */
const char* nsk_last_error(void);
int nsk_abi_version(void);
int nsk_init(int device);
int nsk_device_info(int* sm_count, int* cc_major, int* cc_minor, uint64_t* total_mem);
int nsk_arena_alloc(uint64_t bytes, void* stream, void** out);
int nsk_arena_free(void* ptr, void* stream);
int nsk_arena_stats(uint64_t* out4); /* reserved, in_use, cudaMalloc calls, cache hits */
int nsk_arena_trim(void);
int nsk_pinned_alloc(uint64_t bytes, void** out);
int nsk_pinned_free(void* p);
int nsk_memcpy_h2d(void* dst, const void* src, uint64_t bytes, void* stream);
int nsk_memcpy_d2h(void* dst, const void* src, uint64_t bytes, void* stream);
int nsk_memcpy_d2d(void* dst, const void* src, uint64_t bytes, void* stream);
int nsk_memcpy2d_d2d(void* dst, uint64_t dpitch, const void* src, uint64_t spitch, uint64_t width, uint64_t rows,
                     void* stream);
int nsk_stream_create(void** out);
int nsk_stream_destroy(void* s);
int nsk_stream_sync(void* s);
int nsk_device_sync(void);
int nsk_event_create(int timing, void** out);
int nsk_event_destroy(void* e);
int nsk_event_record(void* e, void* stream);
int nsk_event_wait(void* stream, void* e);
int nsk_event_sync(void* e);
int nsk_event_elapsed_ms(void* start, void* stop, float* ms);
/* event record that becomes an event-record node of a graph under capture (timing inside a replayed step) */
int nsk_event_record_external(void* e, void* stream);
/* measurement utility: occupies `stream` for ns nanoseconds of device time (bench.py enqueues a whole eager step
 * behind it so in-step event brackets contain no host launch gaps) */
int nsk_spin(uint64_t ns, void* stream);
int nsk_graph_begin(void* stream);
int nsk_graph_end(void* stream, void** exec_out, uint64_t* num_nodes);
int nsk_graph_launch(void* exec, void* stream);
int nsk_graph_destroy(void* exec);
int nsk_stream_is_capturing(void* stream, int* out);

/* ---- tcgen05 GEMM / implicit-GEMM conv (umma_gemm.cu) ---- */
/* C[m,n] = sum_k A(m,k) B(n,k) (+ bias[n]) (+ beta*C[m,n]);
 * A(m,k) = A[m*lda+k] (a_mn=0) or A[k*lda+m] (a_mn=1); B likewise with n.
 * dtype NSK_DTYPE_BF16 -> kind::f16, NSK_DTYPE_F32 -> kind::tf32. fp32 accumulate. */
int nsk_gemm(int dtype, int a_mn, int b_mn, int M, int N, int K, const void* A, long long lda, const void* B,
             long long ldb, void* C, long long ldc, int c_f32, const float* bias, float beta, void* stream);

typedef struct NskConvDesc {
  int N, H, W, C; /* input NHWC */
  int K, R, S;    /* filters KRSC */
  int stride, pad;
  int P, Q;       /* output spatial dims */
} NskConvDesc;

int nsk_conv2d_fprop(const NskConvDesc* d, const void* x, const void* w, void* y, int y_f32, void* stream);
/* fprop (bf16 y) that also writes per-CTA channel partials [nparts][2][K] (sum, sum of squares of the stored
 * outputs) for the BatchNorm consuming y; partials must hold 2*SMs x 2 x K floats. */
int nsk_conv2d_fprop_stats(const NskConvDesc* d, const void* x, const void* w, void* y, float* partials,
                           uint64_t partial_floats, int* nparts, void* stream);
int nsk_conv2d_dgrad(const NskConvDesc* d, const void* dy, const void* w, void* dx, void* stream);
/* dx = dgrad + beta * dx (bf16, in place): accumulates a second gradient contribution in the epilogue */
int nsk_conv2d_dgrad_acc(const NskConvDesc* d, const void* dy, const void* w, void* dx, float beta, void* stream);
/* dgrad producing the (complete) gradient of a BatchNorm's output -- the backward of BatchNorm+ReLU fused into
 * the dgrad epilogue: stores dz = relu_mask * (dgrad + beta * dx) (beta 0 or 1; relu_mask may be NULL) and
 * per-CTA partials [nparts][2][C] of sum dz and sum dz * bn_x (bn_x = the BatchNorm's saved bf16 input) for
 * nsk_bn_bwd_partials. Replaces the reduction pass of the reference-restated BatchNorm backward
 * (oracle/restated.py batchnorm_bwd; the reference has no BatchNorm). partials: 2*SMs x 2 x C. */
int nsk_conv2d_dgrad_bnstats(const NskConvDesc* d, const void* dy, const void* w, void* dx, float beta,
                             const void* bn_x, const void* relu_mask, float* partials, uint64_t partial_floats,
                             int* nparts, void* stream);
/* CTAs per weight-gradient launch (0 = default two per SM); see side.py */
int nsk_wgrad_grid_cap(int ctas);
uint64_t nsk_conv2d_wgrad_workspace(const NskConvDesc* d);
int nsk_conv2d_wgrad(const NskConvDesc* d, const void* x, const void* dy, float* dw, float beta, void* ws,
                     uint64_t ws_bytes, void* stream);

/* ---- SIMT GEMM for small / unaligned shapes (fp64 accumulate, like tensor.py:227) ---- */
int nsk_gemm_simt(int a_mn, int b_mn, int M, int N, int K, const float* A, long long lda, const float* B,
                  long long ldb, float* C, long long ldc, const float* bias, float beta, void* stream);

/* ---- elementwise / memory-bound (eltwise.cu) ---- */
#define NSK_EW_ADD 0
#define NSK_EW_SUB 1
#define NSK_EW_HADAMARD 2
#define NSK_EW_SCALAR_ADD 3
#define NSK_EW_SCALAR_MUL 4
#define NSK_EW_RELU 5
#define NSK_EW_SIGMOID 6
#define NSK_EW_TANH 7
#define NSK_EW_NEG 8
#define NSK_EW_COPY 9
int nsk_fill_f32(float* p, uint64_t n, float value, void* stream);
int nsk_fill_bf16(void* p, uint64_t n, float value, void* stream);
int nsk_cast(int src_dtype, const void* src, int dst_dtype, void* dst, uint64_t n, void* stream);
int nsk_eltwise(int kind, int dtype, const void* a, const void* b, float scalar, void* out, uint64_t n, void* stream);
/* gradient of elementwise ops: out = g * f'(saved) for relu (saved=input), sigmoid (saved=output), tanh (saved=output),
 * scalar-mul (out = g*scalar), neg (out = -g), hadamard (out = g*saved) */
int nsk_eltwise_bwd(int kind, int dtype, const void* g, const void* saved, float scalar, void* out, uint64_t n,
                    void* stream);
int nsk_axpy(int dtype, void* y, const void* x, float alpha, uint64_t n, void* stream); /* y += alpha*x */
int nsk_bias_add(int dtype, const void* x, const float* b, void* out, uint64_t rows, uint64_t cols, void* stream);
int nsk_colsum(int dtype, const void* g, float* out, uint64_t rows, uint64_t cols, float beta, void* stream);
int nsk_onehot(const float* idx, uint64_t m, int classes, float* out, int* err_flag, void* stream);
int nsk_check_indices(const float* idx, uint64_t m, int classes, int* err_flag, void* stream);
int nsk_transpose_2d(int dtype, const void* src, void* dst, uint64_t rows, uint64_t cols, void* stream);

/* ---- losses / metrics (xent.cu) ---- */
/* loss_out[0] = mean_i(lse_i - z_{i,t_i}) (f64 math); probs = softmax (f32); err_flag set (1+row) on bad target */
int nsk_xent_fwd(const float* logits, const float* targets, int m, int c, float* probs, float* loss_out,
                 int* err_flag, void* stream);
/* dlogits = (probs - onehot(targets)) * g[0] / m */
int nsk_xent_bwd(const float* probs, const float* targets, const float* g, int m, int c, float* dlogits,
                 void* stream);
int nsk_sum_f32(int dtype, const void* x, uint64_t n, float* out, void* stream); /* f64 accumulate */
int nsk_fill_like_scalar(const float* g, float* out, uint64_t n, void* stream);   /* out[:] = g[0] */
int nsk_argmax_correct(const float* logits, const float* labels, int m, int c, int* count_out, void* stream);

/* ---- optimizers (optim.cu); tensors passed as device arrays of pointers/sizes ---- */
/* hyper-parameters are doubles: the reference optimizers compute in float64 with Python-float constants */
int nsk_sgd_multi(int n_tensors, float* const* w, const float* const* g, float* const* v, void* const* w_bf16,
                  const uint64_t* numel, double lr, double momentum, float grad_scale, void* stream);
int nsk_adamw_multi(int n_tensors, float* const* w, const float* const* g, float* const* m, float* const* v,
                    void* const* w_bf16, const uint64_t* numel, int* step_dev, double lr, double wd, double beta1,
                    double beta2, double eps, const float* grad_scale_dev, void* stream);
/* (step_dev: device int, incremented by the call before use -> bias corrections for t = 1, 2, ...) */
int nsk_sqnorm_multi(int n_tensors, const float* const* g, const uint64_t* numel, double* out, void* stream);
/* (out must hold 1 + 1024 doubles; out[0] = sum of squares in float64) */
/* scale_dev[0] = (norm > max_norm) ? max_norm/norm : 1, norm = sqrt(*sqnorm) ; optional in-place scaling */
int nsk_clip_scale(const double* sqnorm, float max_norm, float* scale_dev, void* stream);
int nsk_scale_multi(int n_tensors, float* const* g, const uint64_t* numel, const float* scale_dev, void* stream);

/* ---- batchnorm / pooling / layout (bn.cu, pool2d.cu) ---- */
/* x [rows, C] (NHWC flattened), bf16; training-mode batch stats (biased var), eps.
 * y = relu?((x-mean)*invstd*gamma + beta + residual?);  ws: nsk_bn_workspace(rows, C) bytes */
uint64_t nsk_bn_workspace(uint64_t rows, int C);
/* running (optional, [2, C]): running mean / unbiased variance updated with `momentum` from this batch */
int nsk_bn_fwd(const void* x, const float* gamma_beta, void* y, float* mean, float* invstd, uint64_t rows, int C,
               float eps, int relu, const void* residual, void* relu_mask, float* running, float momentum, float* ws,
               void* stream);
/* nsk_bn_fwd with the statistics taken from conv partials (nsk_conv2d_fprop_stats) instead of a pass over x */
int nsk_bn_fwd_partials(const float* partials, int nparts, const void* x, const float* gamma_beta, void* y,
                        float* mean, float* invstd, uint64_t rows, int C, float eps, int relu, const void* residual,
                        void* relu_mask, float* running, float momentum, float* ws, void* stream);
/* relu_mask (fwd output, bwd input; NULL without ReLU): one byte per 8 channels, bit j = [y > 0] of channel
 * 8k+j, rows*C/8 bytes. dres (optional) receives the masked gradient flowing to the residual input.
 * dgamma_beta [2, C] (= dgamma_beta*beta_acc + new). */
/* running statistics [2, C] (mean row, unbiased variance row) updated from a training forward's mean/invstd */
int nsk_bn_running_update(const float* mean, const float* invstd, float* running, uint64_t rows, int C,
                          float momentum, float eps, void* stream);
/* inference-mode forward from the running statistics (no batch statistics, nothing saved) */
int nsk_bn_fwd_eval(const void* x, const float* gamma_beta, const float* running, void* y, uint64_t rows, int C,
                    float eps, int relu, const void* residual, float* ws, void* stream);
int nsk_bn_bwd(const void* dy, const void* x, const void* relu_mask, const float* gamma_beta, const float* mean,
               const float* invstd, void* dx, void* dres, float* dgamma_beta, float beta_acc, uint64_t rows, int C,
               float* ws, void* stream);
/* nsk_bn_bwd with dz already ReLU-masked and its statistics taken from dgrad partials (nsk_conv2d_dgrad_bnstats) */
int nsk_bn_bwd_partials(const float* partials, int nparts, const void* dz, const void* x, const float* gamma_beta,
                        const float* mean, const float* invstd, void* dx, void* dres, float* dgamma_beta,
                        float beta_acc, uint64_t rows, int C, float* ws, void* stream);
int nsk_avgpool_fwd(int dtype_in, const void* x, float* y, int N, int HW, int C, void* stream);
int nsk_avgpool_bwd(const float* dy, int dtype_out, void* dx, int N, int HW, int C, void* stream);
/* argmax: one byte per output element (window position r*k+s of the first maximum), written by the forward */
int nsk_maxpool_fwd(const void* x, void* y, void* argmax, int N, int H, int W, int C, int k, int stride, int pad,
                    int P, int Q, void* stream);
int nsk_maxpool_bwd(const void* argmax, const void* dy, void* dx, int N, int H, int W, int C, int k, int stride,
                    int pad, int P, int Q, void* stream);
/* NCHW f32 (host image layout) -> NHWC bf16 with channel padding to Cp (zeros) */
int nsk_nchw_to_nhwc(const float* x, void* y, int N, int C, int H, int W, int Cp, void* stream);
int nsk_nhwc_to_nchw(int dtype_in, const void* x, float* y, int N, int C, int H, int W, int Cp, void* stream);
/* 3x3 (or RxS) im2col for small-channel stems: NHWC bf16 [N,H,W,C] -> [N*P*Q, Kp] bf16 with zero padding */
int nsk_im2col(const void* x, void* out, int N, int H, int W, int C, int R, int S, int stride, int pad, int P, int Q,
               int Kp, void* stream);
/* fused NCHW float32 (host image layout) -> im2col bf16 rows for image stems (Kp % 8 == 0) */
int nsk_im2col_nchw(const float* x, void* out, int N, int C, int H, int W, int R, int S, int stride, int pad, int P,
                    int Q, int Kp, void* stream);
/* adjoint of nsk_im2col: dx[n,h,w,c] (bf16) = sum of the fp32 dcols entries that read x[n,h,w,c] (gather) */
int nsk_col2im(const void* dcols, void* dx, int N, int H, int W, int C, int R, int S, int stride, int pad, int P, int Q,
               int Kp, void* stream);
/* augmentation (K18): uint8 NHWC images, per-image crop offsets (dy,dx in [0,2*pad]) and flip bits
 * drawn on the host; zero-padded crop, flip, normalise -> NHWC bf16 padded to Cp channels */
int nsk_augment_crop_flip(const uint8_t* img, const int32_t* offs, void* out, int N, int H, int W, int C, int pad,
                          const float* mean, const float* std, int Cp, void* stream);

/* ---- sequence ops (embed.cu, gru.cu) ---- */
/* rows of `table` [V, E] gathered by float32 token ids (reference data tensors are float32); with seq_T > 0
 * ids are [B][T] and output row t*B+b holds token [b][t] (time-major for the recurrence). err_flag gets the
 * first bad row (non-integer or out of [0, V)). Backward scatter-adds into dtable (fp32 atomics). */
int nsk_embedding_fwd(const float* table, const float* tokens, uint64_t n, int E, int V, int seq_T, int dtype_out,
                      void* out, int* err_flag, void* stream);
int nsk_embedding_bwd(const void* dout, int dtype_in, const float* tokens, uint64_t n, int E, int seq_T, float* dtable,
                      void* stream);
/* fused GRU recurrence (one cooperative persistent launch for all T steps):
 * gx [T, B, 3H] input projections incl. b (gates r, z, n), U [3H, H], c [3H];
 * hs [T+1, B, H] with hs[0] = h0 (caller-filled); gates [T, B, 4H] = (r, z, n, h.U_n^T + c_n) */
int nsk_gru_fwd(const float* gx, const float* U, const float* c, int T, int B, int H, float* hs, float* gates,
                void* stream);
/* BPTT: dhs [T, B, H] external gradients of h_1..h_T; writes dgx [T, B, 3H] (d pre-activations of gx),
 * dgh [T, B, 3H] (d of h.U^T + c: r, z, n-part), dh0 [B, H]. ws: nsk_gru_bwd_workspace bytes. */
uint64_t nsk_gru_bwd_workspace(int T, int B, int H);
int nsk_gru_bwd(const float* dhs, const float* U, const float* hs, const float* gates, int T, int B, int H, float* dgx,
                float* dgh, float* dh0, void* ws, uint64_t ws_bytes, void* stream);

/* tensor-core GRU recurrence (gru_tc.cu): per group of batch rows one thread-block cluster of H/32 CTAs walks all
 * T steps (NSK_GRU_GROUPS, default 4 groups when they divide B and fit), U (Ubf [3H, H] = the bf16 shadow of U)
 * copied once into each CTA's tensor memory, tcgen05.mma per step, fp32 state and gate math; h exchanged by TMA
 * multicast from a ring in `ws`, the backward's pieces by DSMEM bulk copies (or rings in `ws` where those buffers
 * do not fit). Same outputs as nsk_gru_fwd / nsk_gru_bwd (bias-gradient sums in a different fixed order).
 * Shapes: 1 <= B <= 64, H in 128..512 with H % 64 == 0 (nsk_gru_tc_supported). */
int nsk_gru_tc_supported(int B, int H);
/* diagnostics: 16 globaltimer stamps per (CTA, step) of the last forward launched with NSK_GRU_TRACE=1 */
int nsk_gru_trace(long long* out, int steps);
uint64_t nsk_gru_tc_workspace(int B, int H);
int nsk_gru_fwd_tc(const float* gx, const void* Ubf, const float* c, int T, int B, int H, float* hs, void* hsb,
                   float* gates, void* ws, uint64_t ws_bytes, void* stream);
/* hsb [T+1, B, H] bf16 copy of hs; the backward emits dgx / dgh as bf16 (the weight-gradient GEMM operands) and the
 * bias gradients itself: db (+)= sum_{t,b} dgx, dc (+)= sum_{t,b} dgh (fp32, fixed order; beta 0 or 1). */
int nsk_gru_bwd_tc(const float* dhs, const void* Ubf, const float* hs, const float* gates, int T, int B, int H,
                   void* dgx, void* dgh, float* dh0, float* db, float beta_b, float* dc, float beta_c, void* ws,
                   uint64_t ws_bytes, void* stream);

/* ---- communication (comm.cu): NCCL over NVLink / NVSwitch ---- */
int nsk_comm_unique_id(uint8_t* out128);
int nsk_comm_init(int rank, int world, const uint8_t* uid128, void** comm_out);
int nsk_comm_destroy(void* comm);
int nsk_allreduce(void* comm, void* buf, uint64_t count, int dtype, void* stream); /* in-place sum */
int nsk_allreduce_i32(void* comm, int* buf, uint64_t count, void* stream);
int nsk_comm_check(void* comm);

#ifdef __cplusplus
}
#endif
#endif /* NSKB_H */
