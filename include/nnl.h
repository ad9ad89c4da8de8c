/*
 * nnl.h — C ABI of libnnl.so, the B200 (sm_100a) hot path behind the
 * nanonnl operator API (reference: /root/reference/pkg/src/nanonnl).
 *
 * Conventions:
 *   - every entry point returns int32 status; 0 = OK, nonzero codes map 1:1
 *     onto the reference exception classes (src/errors.py:8-122);
 *     nnl_last_error() returns a thread-local message for the last failure;
 *   - all tensors are caller-owned DEVICE pointers; 4-D activations are
 *     NHWC (channels innermost), conv weights are KRSC ([out][kh][kw][in]),
 *     affine weights keep the reference (I,O) row-major layout;
 *   - dtype codes: NNL_F32 = 0, NNL_F16 = 1 (binary16 storage, fp32 math);
 *   - every call is asynchronous on the cudaStream_t passed as `stream`
 *     (void* here so the header needs no CUDA includes);
 *   - `accumulate` flags implement the reference's NdArray.accumulate
 *     (src/tensor.py:115-123): out = q(out + result) instead of q(result);
 *   - `nonfinite` pointers (nullable) receive an OR of "some written value
 *     is inf/NaN" (src/tensor.py:153-157) so the solver needs no extra pass.
 *
 * Each function names the reference interface it replaces.
 */
#ifndef NNL_H_
#define NNL_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (src/errors.py) ------------------------------------- */
#define NNL_OK 0
#define NNL_ERR_SHAPE_MISMATCH 1          /* errors.py:14  ShapeMismatch */
#define NNL_ERR_KERNEL_TOO_LARGE 2        /* errors.py:22  KernelTooLarge */
#define NNL_ERR_LABEL_OUT_OF_RANGE 3      /* errors.py:44  LabelOutOfRange */
#define NNL_ERR_DEGENERATE_BATCH 4        /* errors.py:48  DegenerateBatch */
#define NNL_ERR_NOT_SETUP 5               /* errors.py:64  NotSetup */
#define NNL_ERR_COLLECTIVE_TIMEOUT 6      /* errors.py:78  CollectiveTimeout */
#define NNL_ERR_SHAPE_MISMATCH_RANKS 7    /* errors.py:74  ShapeMismatchAcrossRanks */
#define NNL_ERR_INVALID_RANGE 8           /* errors.py:18  InvalidRange */
#define NNL_ERR_CUDA 20                   /* CUDA runtime/driver failure */
#define NNL_ERR_UNSUPPORTED 21            /* configuration not implemented */
#define NNL_ERR_INVALID_ARGUMENT 22

#define NNL_F32 0
#define NNL_F16 1

const char* nnl_last_error(void);
int nnl_version(void);
/* number of kernels this library launched since load (or since reset) */
int64_t nnl_launch_count(int reset);
/* 1 when the tensor-core (tcgen05) path is enabled for eligible shapes */
int nnl_set_tc_enabled(int enabled);
/* CTA-pair (tcgen05 cta_group::2) tiles: 0 off, 1 cost heuristic (default),
   2 whenever eligible; returns the previous setting, < 0 only queries
   (initial value from env NNL_TC_PAIRS) */
int nnl_set_tc_pairs(int enabled);
/* programmatic dependent launch of every libnnl kernel (default on; NNL_PDL=0) */
int nnl_set_pdl(int enabled);
/* weight-stationary tiles (whole B operand resident in shared memory) for
   single-N-tile GEMMs; returns the previous setting, < 0 only queries
   (default on; env NNL_TC_RESB=0) */
int nnl_set_tc_resident_b(int enabled);
/* stride-2 narrow-channel convolutions (the stem) over the row-concatenated
   64-channel space-to-depth tensor (1) or the 16-channel one (0); returns the
   previous setting, < 0 only queries (default 1; env NNL_S2D4=0) */
int nnl_set_tc_s2d4(int enabled);
/* stride-1 convolutions over spatial pixel-box tiles (one tiled 4D TMA box per
   filter tap) instead of TMA im2col rows: 0 off, 1 fprop + dgrad (default),
   2 also wgrad; returns the previous setting, < 0 only queries (env NNL_TILE4) */
int nnl_set_tc_tile4(int enabled);
/* 3x3 stride-1 convolutions over 64 channels from one shared input halo per
   (8 x 16)-pixel tile (nine descriptor views) instead of one load per tap;
   returns the previous setting, < 0 only queries (default 1; env NNL_HALO=0) */
int nnl_set_tc_halo(int enabled);
/* 8-warp GEMM epilogues of single-N-tile, TMA-stored outputs interleaved by
   tile (warps 4..7 even tiles, 8..11 odd ones, all columns each) instead of
   split by columns; returns the previous setting, < 0 only queries (default 1;
   env NNL_EPI_IL=0) */
int nnl_set_tc_epi_il(int enabled);

/* ---- geometry ----------------------------------------------------------- */
typedef struct nnl_conv_shape {
  int32_t n, h, w, c;          /* input, NHWC */
  int32_t k;                   /* output maps */
  int32_t r, s;                /* kernel (kh, kw) */
  int32_t stride_h, stride_w;
  int32_t pad_h, pad_w;
  int32_t p, q;                /* output extent; functions.py:122-125 */
} nnl_conv_shape;

typedef struct nnl_pool_shape {
  int32_t n, h, w, c;          /* input, NHWC */
  int32_t kh, kw, sh, sw, ph, pw;
  int32_t p, q;                /* output extent (ignore_border already applied) */
} nnl_pool_shape;

/* ---- storage / numerics: src/tensor.py ---------------------------------- */
/* tensor.py:46-59 quantize_f16 applied to an f32 buffer (RNE, overflow->inf) */
int nnl_quantize_f16(int64_t n, const float* x, float* y, void* stream);
/* NdArray.fill (tensor.py:125-131); value is quantized for F16 */
int nnl_fill(int dtype, int64_t n, void* dst, float value, void* stream);
/* fill from a device scalar (double), used for the dynamic loss-scale seed */
int nnl_fill_from_device(int dtype, int64_t n, void* dst, const double* value, void* stream);
/* NdArray.accumulate / write of another device buffer of the same dtype */
int nnl_accumulate(int dtype, int64_t n, const void* src, void* dst, int accumulate, void* stream);
/* has_inf_or_nan over one buffer (tensor.py:153-157); ORs into *flag */
int nnl_nonfinite(int dtype, int64_t n, const void* x, int32_t* flag, void* stream);
/* RngState.next_uniform (tensor.py:241-252): draw i = f(seed, counter+i) */
int nnl_rng_uniform(uint64_t seed, uint64_t counter, int64_t n, double low, double high,
                    int dtype, void* out, void* stream);

/* ---- Affine: functions.py:82-119 ---------------------------------------- */
/* pass: 0 forward, 1 backward-data, 2 backward-weight.  in_c: channel count of an
   NHWC input (weight rows follow its logical NCHW flattening); in_f for 2-D x */
size_t nnl_affine_workspace_size(int dtype, int64_t batch, int64_t in_f, int64_t out_f, int pass);
int nnl_affine_fwd(int dtype, int64_t batch, int64_t in_f, int64_t in_c, int64_t out_f,
                   const void* x, const void* w, const void* b, void* y,
                   void* ws, size_t ws_bytes, void* stream);
int nnl_affine_bwd_data(int dtype, int64_t batch, int64_t in_f, int64_t in_c, int64_t out_f,
                        const void* dy, const void* w, void* dx, int accumulate,
                        void* ws, size_t ws_bytes, void* stream);
int nnl_affine_bwd_weight(int dtype, int64_t batch, int64_t in_f, int64_t in_c, int64_t out_f,
                          const void* x, const void* dy, void* dw, int acc_w,
                          void* db, int acc_b, int32_t* nonfinite,
                          void* ws, size_t ws_bytes, void* stream);

/* ---- Convolution: functions.py:152-214 ---------------------------------- */
size_t nnl_conv2d_workspace_size(const nnl_conv_shape* cs, int dtype, int pass);
/* y = conv(x, w) + b.  stat_partials (nullable, f32 [nnl_conv2d_stat_rows][2][K])
   receives per-CTA sums of (y - K) and (y - K)^2 over the ROUNDED outputs for a
   following BN, K = stat_shift[k] (nullable: 0) -- the BN's centre, so that a
   channel with |mean| >> std keeps its variance (nnl_bn_fwd_train `shift`). */
int nnl_conv2d_fwd(const nnl_conv_shape* cs, int dtype, const void* x, const void* w,
                   const void* b, void* y, float* stat_partials, const float* stat_shift,
                   void* ws, size_t ws_bytes, void* stream);
int nnl_conv2d_bwd_data(const nnl_conv_shape* cs, int dtype, const void* dy, const void* w,
                        void* dx, int accumulate, void* ws, size_t ws_bytes, void* stream);
int nnl_conv2d_bwd_weight(const nnl_conv_shape* cs, int dtype, const void* x, const void* dy,
                          void* dw, int acc_w, void* db, int acc_b, int32_t* nonfinite,
                          void* ws, size_t ws_bytes, void* stream);
/* Thread-local opt-in (returns the previous value, < 0 only queries): the next
   nnl_conv2d_bwd_weight calls may reuse the space-to-depth copy of x that the
   forward of the same convolution built in the SAME workspace, skipping its
   rebuild.  The caller guarantees that workspace was not used in between (the
   engine gives the stem its own workspace) and that x is unchanged. */
int nnl_conv2d_prep_reuse(int enabled);
/* number of stat-partial rows nnl_conv2d_fwd writes (0 if fusion unsupported) */
int32_t nnl_conv2d_stat_rows(const nnl_conv_shape* cs, int dtype);

/* Backward-data of the convolution that consumes a BatchNormalization[+ReLU]
   output, with the BN backward's statistics pass fused into the epilogue
   (extension of functions.py:418-422; replaces the separate reduction pass of
   nnl_bn_bwd).  g = the convolution's input gradient exactly as
   nnl_conv2d_bwd_data writes it (q(prev + .) when accumulate); then
   gy = g * gate with gate = (gate > 0) (residual tail: gate is the ReLU output
   after the Add2) or (q(gamma*xhat + beta) > 0) (relu: fused BN->ReLU), and
   xhat = (x - save_mean) * save_istd.  Writes q(gy) (canonical: q(0 + gy)) to
   out (NULL: dx) and per-CTA column sums (gy, gy*xhat) to partials
   [nnl_conv2d_bwd_data_bn_rows][2][C], which nnl_bn_bwd_apply consumes. */
typedef struct nnl_bn_bwd_fuse {
  const void* x;               /* BN input, NHWC like dx */
  const void* gate;            /* nullable: residual-tail ReLU output */
  const float* gamma;          /* relu: BN gamma / beta */
  const float* beta;
  const float* save_mean;      /* forward batch statistics */
  const float* save_istd;
  int32_t relu;
  int32_t canonical;
  void* out;                   /* nullable: gated gradient destination */
  float* partials;
} nnl_bn_bwd_fuse;
int32_t nnl_conv2d_bwd_data_bn_rows(const nnl_conv_shape* cs, int dtype);
int nnl_conv2d_bwd_data_bn(const nnl_conv_shape* cs, int dtype, const void* dy, const void* w,
                           void* dx, int accumulate, const nnl_bn_bwd_fuse* bf, void* ws,
                           size_t ws_bytes, void* stream);

/* ---- MaxPooling: functions.py:217-291 ----------------------------------- */
int nnl_maxpool_fwd(int dtype, const nnl_pool_shape* ps, const void* x, void* y,
                    uint8_t* argmax, void* stream);
/* BatchNormalization (batch statistics already finalised into save_mean /
   save_istd by nnl_bn_fwd_train with y = NULL) -> ReLU -> max pooling in one
   pass: y = maxpool(relu(q(gamma * ((x - mean) * istd) + beta))), argmax as
   nnl_maxpool_fwd; relu(BN(x)) is never written (engine fusion of
   functions.py:412-416, :307-314 and :217-291; fp16, C % 8 == 0, 3x3 windows
   with stride 2). */
int nnl_bn_relu_maxpool_ok(int dtype, const nnl_pool_shape* ps);
int nnl_bn_relu_maxpool_fwd(int dtype, const nnl_pool_shape* ps, const void* x,
                            const float* gamma, const float* beta, const float* save_mean,
                            const float* save_istd, void* y, uint8_t* argmax, void* stream);
int nnl_maxpool_bwd(int dtype, const nnl_pool_shape* ps, const void* dy,
                    const uint8_t* argmax, void* dx, int accumulate, void* stream);

/* ---- ReLU: functions.py:294-317 ----------------------------------------- */
int nnl_relu_fwd(int dtype, int64_t n, const void* x, void* y, void* stream);
/* gx = gy * (x > 0) as a multiply (inf*0 = NaN); `x` may be the ReLU output */
int nnl_relu_bwd(int dtype, int64_t n, const void* x, const void* dy, void* dx,
                 int accumulate, void* stream);

/* ---- Add2 / GlobalAveragePooling (extensions, oracle/nnl_oracle.py) ----- */
int nnl_add2_fwd(int dtype, int64_t n, const void* a, const void* b, void* y,
                 int fuse_relu, void* stream);
int nnl_gap_fwd(int dtype, int64_t n, int64_t hw, int64_t c, const void* x, void* y,
                void* stream);
int nnl_gap_bwd(int dtype, int64_t n, int64_t hw, int64_t c, const void* dy, void* dx,
                int accumulate, void* stream);

/* ---- SoftmaxCrossEntropy: functions.py:320-360 -------------------------- */
/* labels are stored in `dtype`; loss_out is a rank-0 buffer of `dtype`;
   row_stats (f32 [3*batch]) keeps (max, logsumexp, log p[label]) per row;
   label_err (nullable) is set to 1 on a label outside [0,classes) */
int nnl_sce_fwd(int dtype, int64_t batch, int64_t classes, const void* logits,
                const void* labels, void* loss_out, float* row_stats,
                int32_t* label_err, void* stream);
int nnl_sce_bwd(int dtype, int64_t batch, int64_t classes, const void* logits,
                const void* labels, const float* row_stats, const void* gloss,
                void* glogits, int accumulate, void* stream);

/* ---- BatchNormalization: functions.py:363-441 --------------------------- */
size_t nnl_bn_workspace_size(int64_t rows, int32_t c);
/* rows = N*H*W (channel-innermost).  stat_partials (nullable) are the conv
   epilogue partials, centred on shift[c]; without them the statistics pass
   centres on x's first row.  mean = K + sum(x-K)/n, var = sum((x-K)^2)/n -
   (sum(x-K)/n)^2 in f64 (the reference's two-pass np.var, functions.py:402,
   without its cancellation).  shift (nullable, f32 [c], in/out) receives the
   batch mean: the centre of the next call.  save_mean/save_istd (f32 [c])
   feed backward.
   residual (nullable): the residual tail BN -> Add2 -> [ReLU] in one pass,
   y = [relu](q(q(BN(x)) + residual)) -- each step rounded exactly as the
   separate functions would (functions.py:412-416, then Add2, then ReLU).
   y = NULL: statistics only (running stats, save_mean / save_istd, shift),
   for a consumer that applies them itself (nnl_bn_relu_maxpool_fwd). */
int nnl_bn_fwd_train(int dtype, int64_t rows, int32_t c, const void* x,
                     const float* gamma, const float* beta,
                     float* running_mean, float* running_var, float eps, float momentum,
                     const float* stat_partials, int32_t n_partials, float* shift,
                     float* save_mean, float* save_istd, void* y, const void* residual,
                     int fuse_relu, void* ws, size_t ws_bytes, void* stream);
int nnl_bn_fwd_eval(int dtype, int64_t rows, int32_t c, const void* x,
                    const float* gamma, const float* beta, const float* mean,
                    const float* var, float eps, float* save_mean, float* save_istd,
                    void* y, const void* residual, int fuse_relu, void* stream);
/* fused_relu: dy is the gradient of relu(BN(x)) (fused BN->ReLU); the gate
   relu(q(gamma*xhat+beta)) > 0 is recomputed from x with the forward's exact
   op sequence, so the ReLU output is never read.
   conv_bias_grad (nullable, dtype [c]): also reduce the ROUNDED dx over rows
   into the bias gradient of the convolution that produced x
   (functions.py:211-212), saving that convolution a pass over dx.
   gate (nullable; exclusive with fused_relu): backward of the residual tail
   BN -> Add2 -> ReLU.  dy is the ReLU output's gradient and gate the ReLU
   output: the BN receives dy * (gate > 0), and dres (the Add2's other input's
   gradient) gets q(dres + dy * (gate > 0)) (acc_res) or q(dy * (gate > 0)). */
int nnl_bn_bwd(int dtype, int64_t rows, int32_t c, const void* x, const void* dy,
               int fused_relu, const void* gate, void* dres, int acc_res,
               const float* gamma, const float* beta, const float* save_mean,
               const float* save_istd, int batch_stat,
               void* dx, int acc_x, float* dgamma, int acc_g, float* dbeta, int acc_b,
               void* conv_bias_grad, int acc_cb,
               int32_t* nonfinite, void* ws, size_t ws_bytes, void* stream);
/* nnl_bn_bwd when the statistics pass already ran in the producing dgrad's
   epilogue (nnl_conv2d_bwd_data_bn): gy is the gated gradient, partials its
   [nparts][2][c] column sums (gy, gy*xhat); finalize + apply only. */
int nnl_bn_bwd_apply(int dtype, int64_t rows, int32_t c, const void* x, const void* gy,
                     const float* partials, int32_t nparts, const float* gamma,
                     const float* save_mean, const float* save_istd, int batch_stat,
                     void* dx, int acc_x, float* dgamma, int acc_g, float* dbeta, int acc_b,
                     void* conv_bias_grad, int acc_cb, int32_t* nonfinite, void* ws,
                     size_t ws_bytes, void* stream);

/* ---- Solver: solver.py:67-164 ------------------------------------------- */
typedef struct nnl_param_slot {
  void* data;        /* visible weight (dtype) */
  void* grad;        /* gradient (dtype) */
  float* master;     /* f32 master (solver.py:89-92) */
  float* momentum;   /* f32 velocity (extension; nullable) */
  int64_t n;
  int32_t dtype;
  int32_t pad_;
} nnl_param_slot;

/* multi-tensor work list: chunk i covers slot[slot] elements [start, start+len) */
typedef struct nnl_chunk {
  int32_t slot;
  int32_t len;
  int64_t start;
} nnl_chunk;

/* device-resident DynamicLossScaler (solver.py:49-64) + step outcome */
typedef struct nnl_scaler_state {
  double loss_scale;
  double scaling_factor;
  int64_t interval;
  int64_t counter;
  int32_t nonfinite;   /* OR of the current step's grads (reset by nnl_scaler_finish) */
  int32_t applied;     /* outcome of the last step: 1 Applied, 0 SkippedInfNan */
} nnl_scaler_state;

/* has_inf_or_nan over every slot grad (solver.py:115-117); ORs into *flag */
int nnl_multi_nonfinite(const nnl_param_slot* slots, const nnl_chunk* chunks, int32_t n_chunks,
                        int32_t* flag, void* stream);
/* scale_grad (solver.py:106-109): g <- q(g * f32(factor)) */
int nnl_multi_scale_grad(const nnl_param_slot* slots, const nnl_chunk* chunks, int32_t n_chunks,
                         float factor, void* stream);
/* sum of squares of every grad in f64 (clip_grad_by_norm, solver.py:119-129) */
int nnl_multi_sumsq(const nnl_param_slot* slots, const nnl_chunk* chunks, int32_t n_chunks,
                    double* out, void* stream);
/* one fused HBM pass (solver.py:100-109,132-155):
 *   scaler == NULL: plain update; else skip when scaler->nonfinite, otherwise
 *   unscale g <- q(g*f32(1/S)) first.
 *   update: d = g + wd*master; v = momentum*v + lr*d; master -= v; w = q(master)
 *   which with momentum = wd = 0 is exactly  master -= f32(lr)*g  (reference).
 *   momentum/weight_decay are the unpinned extension (NNabla Momentum/weight decay). */
int nnl_multi_sgd_update(const nnl_param_slot* slots, const nnl_chunk* chunks, int32_t n_chunks,
                         float lr, float momentum, float weight_decay,
                         nnl_scaler_state* scaler, void* stream);
/* scaler bookkeeping after the update (dynamic_step tail, solver.py:142-153) */
int nnl_scaler_finish(nnl_scaler_state* scaler, void* stream);

/* ---- Data-parallel all_reduce: communicator.py:69-105 ------------------- */
/* slots[i].data is unused here; bucket element = slot offset given by the
 * chunk table's running position: chunk i lands at bucket[chunk_pos[i]]   */
int nnl_bucket_pack(const nnl_param_slot* slots, const nnl_chunk* chunks, const int64_t* chunk_pos,
                    int32_t n_chunks, float* bucket, void* stream);
/* grad = q(bucket / f32(world)); ORs non-finite results into *nonfinite */
int nnl_bucket_unpack_mean(const nnl_param_slot* slots, const nnl_chunk* chunks,
                           const int64_t* chunk_pos, int32_t n_chunks, const float* bucket,
                           int32_t world, int32_t* nonfinite, void* stream);

/* ---- Communicator: communicator.py:69-105 ---------------
 * One rank per process/GPU over NCCL (resolved at run time from the process's
 * libnccl).  nnl_comm_allreduce_mean is the whole bucket exchange of
 * Communicator.all_reduce(buffers, division) on the caller's stream: pack the
 * gradients into the f32 bucket, exchange, unpack grad = q(sum / f32(W))
 * (division) or q(sum), OR-ing non-finite results into *nonfinite.
 *   NNL_COMM_NCCL : ncclAllReduce(sum) (NCCL's ring / NVLS summation order)
 *   NNL_COMM_EXACT: the reference's fold acc = ((b0 + b1) + b2) + ... in
 *                   ascending rank order (R9, communicator.py:99-103), bit-exact,
 *                   with the bytes of a ring all-reduce: send/recv of each
 *                   rank's 1/W slice, fold, in-place all-gather.  Its bucket
 *                   holds nnl_comm_bucket_elems(n) elements and it needs
 *                   nnl_comm_workspace_size(n) bytes of workspace.
 * Errors: CollectiveTimeout for NCCL system/remote failures.  Stream-ordered
 * and CUDA-graph capturable. */
#define NNL_COMM_NCCL 0
#define NNL_COMM_EXACT 1
#define NNL_COMM_ID_BYTES 128
typedef struct nnl_comm nnl_comm;
int nnl_comm_unique_id(void* id_out /* NNL_COMM_ID_BYTES */);
int nnl_comm_init(nnl_comm** out, int32_t world, int32_t rank, const void* unique_id,
                  int32_t mode);
int nnl_comm_destroy(nnl_comm* comm);
int64_t nnl_comm_bucket_elems(const nnl_comm* comm, int64_t n);
size_t nnl_comm_workspace_size(const nnl_comm* comm, int64_t n);
int nnl_comm_allreduce_mean(nnl_comm* comm, const nnl_param_slot* slots, const nnl_chunk* chunks,
                            const int64_t* chunk_pos, int32_t n_chunks, float* bucket, int64_t n,
                            int32_t divide, int32_t* nonfinite, void* ws, size_t ws_bytes,
                            void* stream);
/* plain in-place f32 sum over the ranks (e.g. the step's loss) */
int nnl_comm_allreduce_sum_f32(nnl_comm* comm, float* buf, int64_t n, void* stream);

/* ---- API-boundary marshaling (Variable.d get/set, graph.py:137-155) ------
 * import: f32 NCHW (logical, host order) -> dtype NHWC storage, quantizing;
 * export: dtype NHWC storage -> f32 NCHW.  Non-4-D buffers use n=c=1. */
int nnl_import_f32(int dtype, int32_t n, int32_t c, int32_t hw, const float* src, void* dst,
                   void* stream);
int nnl_export_f32(int dtype, int32_t n, int32_t c, int32_t hw, const void* src, float* dst,
                   void* stream);
/* in-process rank-ordered fold (communicator.py:99-103): out = b0 + b1 + ... (f32) */
int nnl_fold_f32(int32_t k, const float* const* bufs_dev, int64_t n, float* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* NNL_H_ */
