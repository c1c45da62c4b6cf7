/*
 * pfb.h -- C ABI of libpfb, the sm_100a kernel library behind the pfor
 * executor.  Plain pointers, sizes and POD descriptors only (no torch types),
 * so any host (Python ctypes, C++, a cgo/JNI shim) can bind it.
 *
 * Boundary replaced (reference /root/reference/pkg/src/pforvec):
 *   interp.py:161-236  Executor._eval_plain  -- the kind -> kernel dispatch;
 *   each entry point below replaces the NumPy kernel cited beside it.
 *
 * Conventions
 *   - Every function enqueues work on `stream` (a cudaStream_t, passed as
 *     void*) and returns immediately; 0 = launched, >0 = PFB_E_* (host-side
 *     validation failed, nothing launched), <0 = -(cudaError_t) on launch.
 *   - Outputs are allocated by the caller (the executor knows every shape on
 *     the host); kernels never allocate, except where a workspace pointer is
 *     an explicit argument.
 *   - Inputs may be strided views (stride 0 = broadcast of a loop-invariant
 *     operand); outputs are dense row-major unless stated.
 *   - Errors only detectable on the device (index out of bounds, scatter
 *     collision / incomplete cover) are OR-ed into `*dev_err` (a device int32)
 *     as PFB_DEV_* bits; the host reads it at its next sync and raises the
 *     reference's exception class (errors.py IndexOutOfBounds etc.).
 *   - Float storage is fp32, integers int64, bool one byte (0/1).
 */
#ifndef PFB_H_
#define PFB_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PFB_MAX_RANK 8

enum pfb_dtype { PFB_F32 = 0, PFB_I64 = 1, PFB_BOOL = 2 };

typedef struct pfb_tensor {
  void* data;                      /* device pointer to element [0,...,0] */
  int32_t dtype;                   /* pfb_dtype */
  int32_t rank;                    /* 0..PFB_MAX_RANK */
  int64_t shape[PFB_MAX_RANK];
  int64_t stride[PFB_MAX_RANK];    /* in elements; 0 broadcasts */
} pfb_tensor;

enum pfb_status {
  PFB_OK = 0,
  PFB_E_DTYPE = 1,      /* -> DTypeMismatch */
  PFB_E_SHAPE = 2,      /* -> IncompatibleShapes */
  PFB_E_RANK = 3,       /* -> RankError */
  PFB_E_ARG = 4,        /* -> ValueError (unknown op code, bad attr) */
  PFB_E_UNSUPPORTED = 5 /* layout the kernel cannot take; caller materialises */
};

enum pfb_dev_err {
  PFB_DEV_OOB = 1,        /* -> IndexOutOfBounds */
  PFB_DEV_COLLISION = 2,  /* -> IndexCollision */
  PFB_DEV_COVER = 4       /* -> IncompleteCover */
};

/* op codes: same order as reference tensor.py:124-126 */
enum pfb_binary_op { PFB_ADD, PFB_SUB, PFB_MUL, PFB_DIV, PFB_MAX, PFB_MIN, PFB_LESS, PFB_EQUAL };
enum pfb_unary_op { PFB_NEG, PFB_EXP, PFB_LOG, PFB_RELU, PFB_TANH, PFB_SIGMOID, PFB_SQUARE,
                    PFB_LOGICAL_NOT };

/* library / device info */
int pfb_version(void);
int pfb_device_sm_count(void);

/* elementwise (reference tensor.py:140-188): numpy broadcasting via strides */
int pfb_binary(int32_t op, const pfb_tensor* a, const pfb_tensor* b, pfb_tensor* out,
               void* stream);
int pfb_unary(int32_t op, const pfb_tensor* x, pfb_tensor* out, void* stream);
int pfb_cast(const pfb_tensor* x, pfb_tensor* out, void* stream);

/* fused elementwise program: up to 8 inputs, a register program of binary /
 * unary / cast steps (encoding: csrc/elementwise.cu, FusedProgram); one launch for
 * a chain the reference runs as separate NumPy calls. */
int pfb_fused_ew(int32_t n_in, const pfb_tensor* ins, int32_t n_steps, const int32_t* program,
                 pfb_tensor* out, void* stream);
/* multi-output form: the registers out_regs[0..n_out) are
 * stored to outs[k] after the program (n_out <= 8); all outputs share one shape and one
 * stride layout (f32 or u8-bool each).  Lets an elementwise group whose
 * interior values have consumers outside it (the LSTM gate activations kept
 * for the backward pass) run as one launch. */
int pfb_fused_ew_multi(int32_t n_in, const pfb_tensor* ins, int32_t n_steps,
                       const int32_t* program, int32_t n_out, const int32_t* out_regs,
                       pfb_tensor* outs, void* stream);
/* pfb_fused_ew_multi whose inputs may be split-K partial sums (pass F15):
 * parts[2k] = S_k, parts[2k+1] = st_k -- input k is the sum of S_k copies at
 * element offsets j*st_k (j = 0..S_k-1), summed left to right as loaded;
 * S_k <= 1 = a plain input.  The partials are those of pfb_matmul_parts.
 * Specialised kernels only: PFB_E_UNSUPPORTED without NVRTC (the caller then
 * reduces the partials itself). */
int pfb_fused_ew_parts(int32_t n_in, const pfb_tensor* ins, const int64_t* parts,
                       int32_t n_steps, const int32_t* program, int32_t n_out,
                       const int32_t* out_regs, pfb_tensor* outs, void* stream);
/* pfb_fused_ew_parts with row-sum feeds (pass F16): rowsum[k] >= 0 makes
 * input k the sum of input rowsum[k] over the row (the innermost dim of the
 * outputs' layout) -- ins[k] then only describes the broadcast shape (its
 * data is not read); rowsum[k] < 0 = a normal input.  rowsum[k] = j | op << 16
 * sums op(input j) instead, op a unary program opcode (16 + PFB_NEG ..
 * PFB_SQUARE; the softmax's exp).  The sums are computed
 * in the kernel (one row per block: a whole number of warps, <= 1024 wide),
 * so a row reduction feeding an elementwise group costs no launch of its own
 * (cfg5's per-step `reduce_sum(z) < 0` branch mask; reference
 * tensor.reduce_sum, tensor.py:279-283).  parts nullable.  PFB_E_UNSUPPORTED
 * when the row does not fit or NVRTC is absent (the caller then computes the
 * sums with pfb_row_sum_parts / pfb_reduce_sum). */
int pfb_fused_ew_rows(int32_t n_in, const pfb_tensor* ins, const int64_t* parts,
                      const int32_t* rowsum, int32_t n_steps, const int32_t* program,
                      int32_t n_out, const int32_t* out_regs, pfb_tensor* outs, void* stream);
/* q <= 8 weighted column sums in one launch (pass F19): outs[k][c] =
 * sum_r xs[k][r, c] * y[r] (xs[k] [R, C_k] any strides, y [R] or [R, 1]) --
 * the clipped per-example bias-gradient sums of several parameter blocks
 * sharing the clip scales (reference reduce_sum of a product, tensor.py:279-283).
 * outs[k] dense [C_k]. */
int pfb_col_dots(int32_t q, const pfb_tensor* xs, const pfb_tensor* y, pfb_tensor* outs,
                 void* stream);
/* out[i] = sum_s sum_k x_s[i, k], x_s = x + s * part_stride (x: [rows, W] view
 * with unit inner stride): the row sums of a GEMM result still held as
 * split-K partials (pass F15; reference tensor.reduce_sum, tensor.py:279-283). */
int pfb_row_sum_parts(const pfb_tensor* x, int32_t parts, int64_t part_stride, pfb_tensor* out,
                      void* stream);
/* 1 when pfb_fused_ew_parts can run in this process now (NVRTC found, the
 * specialiser enabled) */
int pfb_fused_parts_ok(void);

/* fused programs over >= min_elems elements run as kernels specialised to the
 * program (NVRTC, sm_100a; csrc/fused_jit.cu), bit-identical to the
 * interpreter kernel; enable = 0 forces the interpreter.  min_elems < 0 keeps
 * the threshold (default 0: every program; env PFB_JIT_MIN; PFB_NO_JIT=1 disables).
 * Returns 1 when the specialiser is available in this process. */
/* number of kernels this library has launched in the process (a launch
 * recorded into a CUDA graph counts once, at capture) */
int64_t pfb_kernel_launches(void);
int pfb_fused_jit_config(int32_t enable, int64_t min_elems);
/* host-only check, no device: generate the specialised kernel for a program
 * (integer: i64/bool domain; v: 1 or 4 lanes; modes: 2-bit feed mode per
 * operand, operand 0 = output) and compile it with NVRTC for sm_100a.
 * 0 = compiled, 1 = compile error, PFB_E_UNSUPPORTED = no NVRTC. */
int pfb_fused_jit_check(int32_t integer, int32_t v, uint64_t modes, int32_t n_in,
                        const int32_t* in_dtypes, int32_t n_steps, const int32_t* program,
                        int32_t n_out, const int32_t* out_regs, const int32_t* out_dtypes);

/* select(mask, a, b) = mask ? a : b with broadcasting (predicated cond /
 * while bodies; numpy.where semantics); any dtype, mask is bool. */
/* integer-domain fused elementwise program (i64 / bool registers, int32
 * immediates; same encoding as pfb_fused_ew_multi): loop counters, index
 * arithmetic and masks of converted control flow (reference tensor.py:104-188
 * on i64/bool values), bit-exact with numpy int64 wraparound. */
/* (an f32 output stores the register converted to float: the group's final
 * cast i64 / bool -> f64, e.g. one-hot masks) */
int pfb_fused_int(int32_t n_in, const pfb_tensor* ins, int32_t n_steps, const int32_t* program,
                  int32_t n_out, const int32_t* out_regs, pfb_tensor* outs, void* stream);
int pfb_select(const pfb_tensor* mask, const pfb_tensor* a, const pfb_tensor* b, pfb_tensor* out,
               void* stream);

/* reduce_sum over axes given as a bitmask (reference tensor.py:279-283) */
int pfb_reduce_sum(const pfb_tensor* x, uint32_t axes_mask, pfb_tensor* out, void* ws,
                   int64_t ws_bytes, void* stream);

/* sum over axes of x*y, y broadcast to x (fused square / scaled reductions) */
int pfb_reduce_dot(const pfb_tensor* x, const pfb_tensor* y, uint32_t axes_mask, pfb_tensor* out,
                   void* ws, int64_t ws_bytes, void* stream);

/* strided copy: out (any strides) <- x (any strides, same shape).  Backs
 * transpose / concat / stack / tile_leading / slice_leading materialisation
 * (reference tensor.py:286-303, 383-416). */
int pfb_copy(const pfb_tensor* x, pfb_tensor* out, void* stream);
int pfb_fill(pfb_tensor* out, double value, void* stream);
/* pack n dense tensors into one byte buffer at dst + dst_offsets[i] (one
 * launch per 16): the executor's single D2H of a run's outputs and device
 * error words (reference Executor.run returns host values, interp.py:109-125). */
/* n dense copies srcs[k] -> dsts[k] (same dtype and element count) in one
 * launch: a device-resident loop's carried values back into its state */
int pfb_copy_many(int32_t n, const pfb_tensor* srcs, const pfb_tensor* dsts, void* stream);
int pfb_pack(int32_t n, const pfb_tensor* xs, void* dst, const int64_t* dst_offsets, void* stream);
/* concat of n same-dtype inputs (any strides) along `axis` into out, in one
 * launch per 24 inputs (reference tensor.concat, tensor.py:383-393). */
int pfb_concat(int32_t n, const pfb_tensor* xs, int32_t axis, pfb_tensor* out, void* stream);

/* matmul (reference tensor.py:195-206): rank-2 x rank-2 or batched rank-3;
 * operands may be strided views (any layout).  fp32-accurate: tcgen05
 * kind::tf32 with a 3xTF32 split for large shapes (needs a workspace of
 * pfb_matmul_workspace() bytes for the hi/lo operand planes; with less the
 * SIMT path runs), SIMT fp32 for small/odd ones.
 * `alpha_rows` (nullable, fp32, one per output row) scales each output row in
 * the epilogue; `accumulate` adds into `out` instead of overwriting;
 * `force_path` 0 = auto, 1 = SIMT, 2 = tcgen05. */
int64_t pfb_matmul_workspace(const pfb_tensor* a, const pfb_tensor* b, pfb_tensor* out);
int pfb_matmul(const pfb_tensor* a, const pfb_tensor* b, pfb_tensor* out, void* ws,
               int64_t ws_bytes, void* stream);
int pfb_matmul_ex(const pfb_tensor* a, const pfb_tensor* b, pfb_tensor* out,
                  const float* alpha_rows, int32_t accumulate, int32_t force_path, void* ws,
                  int64_t ws_bytes, void* stream);

/* out = act(a1 @ b1 + a2 @ b2 + bias): two operand pairs, one output
 * (passes.fuse_dual_matmuls -- matmul of a K-concat, or a sum of matmuls;
 * reference tensor.py:195-206 + binary add).  tcgen05 path: both K ranges
 * accumulate in one launch.  force_path 0 = auto (timed once per shape),
 * 1 = two launches, 2 = tcgen05 raw feed, 3 = tcgen05 pre-split. */
int64_t pfb_matmul_dual_workspace(const pfb_tensor* a1, const pfb_tensor* b1,
                                  const pfb_tensor* a2, const pfb_tensor* b2, pfb_tensor* out);
int pfb_matmul_dual(const pfb_tensor* a1, const pfb_tensor* b1, const pfb_tensor* a2,
                    const pfb_tensor* b2, pfb_tensor* out, const pfb_tensor* bias, int32_t act,
                    int32_t force_path, void* ws, int64_t ws_bytes, void* stream);

/* n (<= 8) independent row-dots in one launch (passes.fuse_row_dots):
 * outs[j][i] = sum_k xs[j][i,k] * ys[j][i,k], xs/ys rank-2 [rows, inner_j]
 * views with unit inner stride (any row stride), outs rank-1 [rows].  The
 * per-parameter-block squared norms of per-example gradients (reference
 * reduce_sum(square(g), axes) per block, tensor.py:279-283). */
int pfb_row_dots(int32_t n, const pfb_tensor* xs, const pfb_tensor* ys, pfb_tensor* outs,
                 void* stream);

/* matmul with a fused prologue/epilogue (post-vectorization rewrite
 * passes.fuse_matmul_epilogues; SURVEY.md §8a F3 "GEMM epilogues: bias add,
 * activation, broadcast scale"):
 *   out = act(alpha_rows * (a @ diag(kscale) @ b) [+ out] + bias)
 * `kscale` (nullable) is broadcast to [batch, K] and scales b's rows (the
 * per-example clip factors of a clipped-sum contraction); `bias` (nullable) is
 * broadcast to out's shape (right-aligned; stride 0 = broadcast); `act` is a
 * PFB_ACT_* code.  Replaces the reference's matmul -> mul / add / tanh chain
 * (tensor.py:140-206). */
enum pfb_act { PFB_ACT_NONE = 0, PFB_ACT_TANH = 1, PFB_ACT_SIGMOID = 2, PFB_ACT_RELU = 3 };
/* derivative epilogues (autodiff.py tanh/sigmoid VJPs): out *= (1 - y^2) / y (1 - y) */
enum pfb_dop { PFB_DOP_NONE = 0, PFB_DOP_DTANH = 1, PFB_DOP_DSIGMOID = 2 };
int pfb_matmul_fused(const pfb_tensor* a, const pfb_tensor* b, pfb_tensor* out,
                     const pfb_tensor* kscale, const pfb_tensor* bias, int32_t act,
                     const float* alpha_rows, int32_t accumulate, int32_t force_path, void* ws,
                     int64_t ws_bytes, void* stream);
/* pfb_matmul_fused plus a derivative epilogue: out *= (1 - y^2) (dop =
 * PFB_DOP_DTANH) or y (1 - y) (PFB_DOP_DSIGMOID), y broadcast to out -- the
 * cotangent multiply of the tanh / sigmoid VJPs (reference autodiff.py:106-111)
 * applied to the GEMM that produces the cotangent. */
int pfb_matmul_ep(const pfb_tensor* a, const pfb_tensor* b, pfb_tensor* out,
                  const pfb_tensor* kscale, const pfb_tensor* bias, int32_t act,
                  const pfb_tensor* dy, int32_t dop, const float* alpha_rows, int32_t accumulate,
                  int32_t force_path, void* ws, int64_t ws_bytes, void* stream);

/* Pre-split weights: the tf32 hi / lo planes of a loop-invariant B operand
 * ([K, N] or [batch, K, N] view, any strides), made once and reused by every
 * GEMM that reads it (the executor caches them per constant weight -- the
 * LSTM's Wg is read by 127 GEMMs per step).  pfb_gemm_planes_bytes: the
 * buffer size (0: not splittable); pfb_gemm_split_planes writes it.
 * pfb_matmul_ep2 / pfb_matmul_dual2 = pfb_matmul_ep / pfb_matmul_dual with the
 * planes of B (nullable): the tcgen05 path then splits only A (3 products). */
int64_t pfb_gemm_planes_bytes(const pfb_tensor* b);
int pfb_gemm_split_planes(const pfb_tensor* b, void* planes, void* stream);
int pfb_matmul_ep2(const pfb_tensor* a, const pfb_tensor* b, pfb_tensor* out,
                   const pfb_tensor* kscale, const pfb_tensor* bias, int32_t act,
                   const pfb_tensor* dy, int32_t dop, const void* b_planes, int32_t force_path,
                   void* ws, int64_t ws_bytes, void* stream);
/* Split-K partials GEMM (pass F15; the reference's tensor.matmul,
 * tensor.py:195-206, for a skinny-M 2-D product whose consumers are fused
 * elementwise groups -- the LSTM's per-step GEMMs): parts[s] = A[:, K_s] @
 * B[K_s, :] (+ bias in s = 0), s < S, no reduction; the consumer sums the
 * partials (pfb_fused_ew_parts).  pfb_matmul_parts_count: S for this shape
 * (< 2: use pfb_matmul_ep2); parts is [S, M, N] with unit column stride;
 * b_planes as for pfb_matmul_ep2 (nullable: B is split into the workspace,
 * pfb_matmul_parts_workspace bytes). */
int pfb_matmul_parts_count(const pfb_tensor* a, const pfb_tensor* b, const pfb_tensor* out);
int64_t pfb_matmul_parts_workspace(const pfb_tensor* a, const pfb_tensor* b, const pfb_tensor* out);
int pfb_matmul_parts(const pfb_tensor* a, const pfb_tensor* b, pfb_tensor* parts,
                     const pfb_tensor* bias, const void* b_planes, void* ws, int64_t ws_bytes,
                     void* stream);
/* the dual-operand form (a1 @ b1 + a2 @ b2, as pfb_matmul_dual2): the
 * k-splits run over both K ranges back to back */
int pfb_matmul_dual_parts_count(const pfb_tensor* a1, const pfb_tensor* b1, const pfb_tensor* a2,
                                const pfb_tensor* b2, const pfb_tensor* out);
int64_t pfb_matmul_dual_parts_workspace(const pfb_tensor* a1, const pfb_tensor* b1,
                                        const pfb_tensor* a2, const pfb_tensor* b2,
                                        const pfb_tensor* out);
int pfb_matmul_dual_parts(const pfb_tensor* a1, const pfb_tensor* b1, const pfb_tensor* a2,
                          const pfb_tensor* b2, pfb_tensor* parts, const pfb_tensor* bias,
                          const void* b1_planes, const void* b2_planes, void* ws,
                          int64_t ws_bytes, void* stream);
int pfb_matmul_dual2(const pfb_tensor* a1, const pfb_tensor* b1, const pfb_tensor* a2,
                     const pfb_tensor* b2, pfb_tensor* out, const pfb_tensor* bias, int32_t act,
                     const void* b1_planes, const void* b2_planes, int32_t force_path, void* ws,
                     int64_t ws_bytes, void* stream);

/* device-resident while loops (csrc/loop.cu; reference interp.py:133-154 runs
 * the loop on the host): a CUDA graph with a conditional WHILE node.  The
 * caller captures a `head` graph (condition -> pfb_set_condition) and an
 * `iter` graph (body, carried-state update, condition -> pfb_set_condition)
 * using the handle from pfb_loop_create, then pfb_loop_finalize assembles
 * head -> WHILE { iter } and each pfb_loop_launch runs the whole loop. */
int pfb_loop_create(void** loop, uint64_t* handle);
int pfb_set_condition(uint64_t handle, const void* flag, void* counter, void* stream);
/* the predicated while's test any(mask) (vectorize._convert_while_masked's
 * less(0, reduce_sum(cast(active, i64))), reference interp.py:240-355 loop
 * test) straight into the handle: one launch per trip instead of four.
 * mask: n dense u8 bools. */
int pfb_set_condition_any(uint64_t handle, const void* mask, int64_t n, void* counter,
                          void* stream);
/* pfb_copy_many (the loop's carried write-back) that also sets the loop's
 * conditional to any(srcs[any_pair]) (u8 bools, the predicated while's
 * active mask): one launch per trip for both.  scratch: 2 device int32,
 * zero before the first call (the kernel leaves them zero).  n <= 16. */
int pfb_copy_many_cond(int32_t n, const pfb_tensor* srcs, const pfb_tensor* dsts,
                       int32_t any_pair, uint64_t handle, void* counter, void* scratch,
                       void* stream);
int pfb_loop_finalize(void* loop, void* head_graph, void* iter_graph);
int pfb_loop_launch(void* loop, void* stream);
int pfb_loop_destroy(void* loop);

/* conv family (reference tensor.py:209-260), NHWC / HWIO, SAME, stride 1 */
int pfb_im2col(const pfb_tensor* x, int32_t k1, int32_t k2, pfb_tensor* out, void* stream);
int pfb_conv2d(const pfb_tensor* x, const pfb_tensor* f, pfb_tensor* out, void* stream);
int pfb_conv2d_input_grad(const pfb_tensor* gy, const pfb_tensor* f, pfb_tensor* out,
                          void* stream);
/* per-example filter gradient, the conv2d VJP w.r.t. the filter without the
 * im2col buffer (reference autodiff.py conv2d VJP: matmul(im2col(x)^T, gy),
 * tensor.py:209-229; passes.fuse_conv_filter_grads):
 *   out[b, (p*k2+q)*c + ci, o] = sum_{i,j} x[b, i+p-p1, j+q-p2, ci] gy[b, i, j, o]
 * x [b,h,w,c], gy [b,h,w,o] dense, out [b, k1*k2*c, o]; sq_norm (nullable,
 * [b]) receives each example's sum of squares (the per-example norm term).
 * PFB_E_UNSUPPORTED where no tiled kernel exists for (k1*k2*c, o). */
int pfb_conv2d_filter_grad(const pfb_tensor* x, const pfb_tensor* gy, int32_t k1, int32_t k2,
                           pfb_tensor* out, pfb_tensor* sq_norm, void* stream);

/* indexing (reference tensor.py:306-360, interp.py:210-221) */
/* out[j, (q,) ...] = x[j, idx[j, (q)], ...] for x [n, m, ...], idx [n] or [n, q]:
 * pfor's gather with a stacked operand and a stacked index (the reference's
 * per-iteration fallback loop over tensor.gather_rows, tensor.py:306-318, and
 * vectorize.py:271-273) in one launch; an index outside [0, m) sets
 * PFB_DEV_OOB in dev_err. */
int pfb_gather_stacked(const pfb_tensor* x, const pfb_tensor* idx, pfb_tensor* out,
                       int32_t* dev_err, void* stream);
/* q <= 8 pfb_gather_stacked calls on one operand in one launch (pass F17:
 * the per-step x_t gathers of an unrolled loop body): out[g][j, ...] =
 * x[j, idx[g][j], ...], idx[g] [n]; dev_err[g] (nullable array, nullable
 * entries) gets PFB_DEV_OOB for an index of vector g outside [0, m).  fp32
 * with contiguous 16-byte-aligned rows; PFB_E_UNSUPPORTED otherwise (gather
 * one vector at a time with pfb_gather_stacked). */
int pfb_gather_stacked_many(const pfb_tensor* x, int32_t q, const pfb_tensor* idx,
                            pfb_tensor* out, int32_t* const* dev_err, void* stream);
int pfb_gather_rows(const pfb_tensor* x, const pfb_tensor* idx, pfb_tensor* out,
                    int32_t* dev_err, void* stream);
int pfb_scatter_rows(int32_t n_parts, const pfb_tensor* index_sets, const pfb_tensor* parts,
                     int64_t total, pfb_tensor* out, int32_t* ws_count, int32_t* dev_err,
                     void* stream);
int pfb_scatter_add_rows(const pfb_tensor* idx, const pfb_tensor* updates, int64_t total,
                         pfb_tensor* out, int32_t* dev_err, void* stream);
/* where_true: out has room for n indices; *dev_count receives the count */
int pfb_where_true(const pfb_tensor* mask, pfb_tensor* out, int64_t* dev_count, void* ws,
                   int64_t ws_bytes, void* stream);
/* complement: sorted [0,total) \ idx; out has room for total entries */
int pfb_complement(const pfb_tensor* idx, int64_t total, pfb_tensor* out, int64_t* dev_count,
                   void* ws, int64_t ws_bytes, void* stream);
int pfb_iota(pfb_tensor* out, int64_t start, void* stream);

/* counter-based uniform stream (reference interp.py:52-82), splitmix64 */
int pfb_rng_uniform(uint64_t seed, uint64_t counter, pfb_tensor* out, void* stream);

/* fused per-example gradient statistics: for rank-1
 * per-example gradients g_i = a_i (x) b_i of one weight matrix,
 * sq_norm[i] += |a_i|^2 |b_i|^2 without materialising g. */
int pfb_outer_sq_norm(const pfb_tensor* a, const pfb_tensor* b, pfb_tensor* sq_norm,
                      void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PFB_H_ */
