/*
 * sparseprop.h -- C ABI of the B200-native SparseProp hot path.
 *
 * SparseProp (arXiv 2302.04852): forward and backward of linear and 2-D
 * convolution layers whose weights carry a fixed, arbitrary, unstructured
 * sparsity mask, with work linear in nnz.  "P<n>" = PAPER.md line n.
 *
 * Conventions (all entry points):
 *  - Every tensor pointer is a DEVICE pointer (cudaMalloc'd / torch CUDA
 *    storage) to fp32, int32 or uint8 as typed, unless stated otherwise.
 *  - Linear weights are W (R x C) = out x in (PyTorch nn.Linear.weight
 *    order); the paper's O = X W (P141) is our Y = W X with W = W_paper^T.
 *  - Linear activations are [features x B] row-major, batch contiguous:
 *    the paper's transposed layout X^T (P183 §3.2).
 *  - Conv activations are CHWN [C][H][W][B], batch last: the paper's
 *    permuted SparseConv layout (P293 §3.3).  Conv weights are the dense
 *    [OC][IC][KH][KW] tensor flattened to R = OC rows, C = IC*KH*KW columns.
 *  - Outputs are OVERWRITTEN, never accumulated.  Empty rows / columns give
 *    zeros.  Any B >= 1 is accepted (vector fast paths and scalar tails).
 *  - Every compute call only enqueues work on `stream` (a cudaStream_t
 *    passed as void*; NULL = legacy default stream) and never synchronises
 *    the host; asynchronous device faults surface at the caller's next sync.
 *    sp_weight_create / sp_weight_create_conv synchronise `stream` several
 *    times (to read nnz, the per-block row counts and the tile maxima of
 *    the cached schedule); compute calls never do.
 *  - No output is accumulated with atomics: every output element (Y, dX,
 *    dW) is produced by one thread in a fixed order, or, where a stream-K
 *    schedule cuts a block between CTAs, as raw parts summed in CTA order by
 *    the last CTA to arrive.  Integer atomics are used only for those
 *    arrival tickets and for shared-memory buffer release counters.  Results
 *    are bitwise run-to-run reproducible on a given device and SM budget.
 *  - Errors: every call returns sp_status; no C++ exception crosses the
 *    ABI.  Arguments are validated before any launch; launch failures are
 *    reported as SP_ERR_CUDA.  sp_last_error() gives a thread-local message.
 *  - Handles are immutable in structure after creation and may be shared
 *    across streams and host threads; the vals buffer is mutable in place
 *    (the optimizer writes it) and the caller orders such writes.
 */
#ifndef SPARSEPROP_H
#define SPARSEPROP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sp_weight_s *sp_weight_t; /* opaque: index structure + vals */
typedef void *sp_stream_t;               /* a cudaStream_t */

typedef enum {
    SP_OK = 0,
    SP_ERR_NULL = 1,       /* a required pointer was NULL */
    SP_ERR_SHAPE = 2,      /* non-positive or inconsistent sizes */
    SP_ERR_OVERFLOW = 3,   /* nnz, an index or a size does not fit int32 */
    SP_ERR_ALLOC = 4,      /* device allocation failed */
    SP_ERR_CUDA = 5,       /* a CUDA runtime / launch error */
    SP_ERR_BAD_HANDLE = 6  /* handle NULL or destroyed */
} sp_status;

/* Conv geometry, stride 1 (stride > 1 is out of scope).
 * OH = H + 2*pad - KH + 1, OW = W + 2*pad - KW + 1 (P223 generalised by
 * Alg. 2's pad, P317-P320).  C_out/C_in*KH*KW must match the handle. */
typedef struct {
    int32_t B, C_in, H, W, C_out, KH, KW, pad;
} sp_conv_geom;

/* ---------------------------------------------------------------------- */
/* Weight handle: CSR (P153-P154) + CSC/transposed index copy (P183)      */
/* ---------------------------------------------------------------------- */

/* Build the handle from a dense R x C fp32 weight and an R x C uint8 mask
 * (both device, row-major).  The STRUCTURE is the mask (nonzero byte =
 * kept; on-mask zero values are stored, off-mask values ignored).  Builds
 *   row_ptr[R+1], col_idx[nnz] (ascending per row), vals[nnz] (CSR order),
 *   col_ptr[C+1], row_idx[nnz] (ascending per column),
 *   perm[nnz] (CSC slot k -> CSR slot holding the same (r, c)),
 * plus the tiled copies of both orientations the kernels stream (row blocks x
 * column blocks; masks at most 3 % dense or with at most 2^15
 * nonzeros also get the single-column-block gather tilings of the L2-gather
 * kernels), deterministically on the device; it synchronises `stream` (to
 * read nnz, block row counts and tile maxima).
 * R, C >= 1; R, C and nnz must fit int32 (else SP_ERR_OVERFLOW); R*C may
 * exceed it (no R x C scratch is used).
 * The handle owns all its device buffers. */
sp_status sp_weight_create(int64_t R, int64_t C, const float *dense, const uint8_t *mask,
                           sp_stream_t stream, sp_weight_t *out);

/* Same as sp_weight_create for a conv filter [C_out][C_in][KH][KW] (dense and
 * mask on the device in that order; R = C_out, C = C_in*KH*KW), plus the
 * per-tap tilings the conv kernels stream: implicit im2col by taps -- each
 * filter tap (x, y) is an OC x IC sparse matrix applied to the activation
 * shifted by (x - pad, y - pad), out-of-range positions reading zero (Eq. 3,
 * P224; pruned taps skipped, P248).
 * Synchronises `stream`.  Handles from sp_weight_create also work with the
 * conv entry points (through slower direct kernels). */
sp_status sp_weight_create_conv(int32_t C_out, int32_t C_in, int32_t KH, int32_t KW, const float *dense,
                                const uint8_t *mask, sp_stream_t stream, sp_weight_t *out);

/* Frees the handle's buffers after synchronising `stream` and the device (work on
 * other streams may still read it).  The buffers return to the library's
 * stream-ordered pool (sp_weight_create allocates its three arenas there). */
sp_status sp_weight_destroy(sp_weight_t W, sp_stream_t stream);

/* nnz, R, C of a handle (-1 on a bad handle). */
int64_t sp_weight_nnz(sp_weight_t W);
int64_t sp_weight_rows(sp_weight_t W);
int64_t sp_weight_cols(sp_weight_t W);

/* Device pointer to the handle-owned vals[nnz] (CSR order), writable in
 * place (e.g. by sp_sgd).  Lifetime = the handle's. */
sp_status sp_weight_vals(sp_weight_t W, float **vals);

/* Device pointers to the handle-owned index arrays (read-only). */
sp_status sp_weight_indices(sp_weight_t W, const int32_t **row_ptr, const int32_t **col_idx,
                            const int32_t **col_ptr, const int32_t **row_idx,
                            const int32_t **perm);

/* Scatter an nnz-length device buffer (vals or a gradient, CSR order) into a
 * dense R x C device buffer: exact +0.0 off the mask. */
sp_status sp_weight_to_dense(sp_weight_t W, const float *nz, float *dense_out,
                             sp_stream_t stream);

/* Adjoint of sp_weight_to_dense: nz_out[j] = dense[r_j][c_j] for every stored
 * (r_j, c_j) (CSR order).  Restricts a dense R x C gradient to the mask (the
 * dense path of the §4.2 dispatcher, P427). */
sp_status sp_weight_gather(sp_weight_t W, const float *dense, float *nz_out, sp_stream_t stream);

/* ---------------------------------------------------------------------- */
/* Linear layer (P141-P151 §3.2)                                          */
/* ---------------------------------------------------------------------- */

/* Forward SpMM: Y[r][b] = sum_{j in row r} vals[j] * X[col_idx[j]][b].
 * X: [C x B], Y: [R x B].  (P141 "O = XW", transposed per P183.) */
sp_status sp_linear_fwd(sp_weight_t W, const float *X, float *Y, int64_t B, sp_stream_t stream);

/* Input-gradient SpMM, Eq. (1) (P143-P145): dX = W^T dY, gather form driven
 * by the CSC copy, each dX row produced by exactly one warp (no atomics):
 * dX[c][b] = sum_{k in col c} vals[perm[k]] * dY[row_idx[k]][b].
 * dY: [R x B], dX: [C x B]. */
sp_status sp_linear_bwd_input(sp_weight_t W, const float *dY, float *dX, int64_t B,
                              sp_stream_t stream);

/* Weight-gradient SDDMM, Eq. (2) (P146-P148, P151, P173 "nnz
 * dot-products"): dW[j] = sum_b dY[r_j][b] * X[c_j][b] for every nonzero j
 * (CSR order); nothing is computed off the mask.  X: [C x B], dY: [R x B],
 * dW: [nnz].  B % 4 != 0 and B >= 64: computed on zero-padded copies (see
 * sp_linear_bwd). */
sp_status sp_linear_bwd_weight(sp_weight_t W, const float *X, const float *dY, float *dW,
                               int64_t B, sp_stream_t stream);

/* Fused epilogue variants used by the data-parallel MLP step (north star
 * cfg5): identical arithmetic plus an elementwise epilogue in the same
 * kernel.
 *  sp_linear_fwd_relu:        Y = max(W X, 0)              (ReLU)
 *  sp_linear_bwd_input_relu:  dX = (W^T dY) * [H > 0]      (ReLU', with
 *      H the saved post-ReLU activation [C x B]; ReLU'(0) = 0) */
sp_status sp_linear_fwd_relu(sp_weight_t W, const float *X, float *Y, int64_t B,
                             sp_stream_t stream);
sp_status sp_linear_bwd_input_relu(sp_weight_t W, const float *dY, const float *H, float *dX,
                                   int64_t B, sp_stream_t stream);

/* Fused backward (the paper's Alg. 1 "single pass",
 * P173/P187-P220, made atomic-free by driving it from the CSC copy): ONE pass
 * over the nonzeros produces both
 *   dX = W^T dY                       (as sp_linear_bwd_input)
 *   dW = (dY X^T) restricted to mask  (as sp_linear_bwd_weight)
 * reading each staged dY element once for both products.
 * sp_linear_bwd_relu additionally gates dX by [H > 0] (H: [C x B]).
 * X: [C x B], dY: [R x B], dX: [C x B], dW: [nnz].  Stream-K schedule: each
 * SM runs an equal range of (row block, batch slice, column block) tiles; a
 * dX block cut between CTAs is finished by the last CTA to arrive, which adds
 * the raw parts in CTA order, and dW partials are summed in job order, so the
 * result is bitwise reproducible run to run (it may differ from the separate
 * kernels by fp32 rounding of those regrouped sums).  Falls back to the two
 * separate kernels when the problem is tiny (< 32 tiles) or the rows are too
 * long for the tensor-memory dW columns (same results within the fp32
 * tolerance).  B % 4 != 0: below 64 columns the separate kernels' narrow-lane
 * tail paths run; from 64 on (e.g. the paper's B = 902) the pass runs on
 * zero-padded copies of X, dY (and H) with B rounded up to 4 -- the zero
 * columns add +0 terms to dW and only discarded dX columns -- and dX is
 * copied back (sp_linear_bwd_weight pads the same way).  Scratch comes from
 * the stream-ordered pool; no host sync. */
sp_status sp_linear_bwd(sp_weight_t W, const float *X, const float *dY, float *dX, float *dW, int64_t B,
                        sp_stream_t stream);
sp_status sp_linear_bwd_relu(sp_weight_t W, const float *X, const float *dY, const float *H, float *dX,
                             float *dW, int64_t B, sp_stream_t stream);

/* ---------------------------------------------------------------------- */
/* 2-D convolution, stride 1, CHWN (P222-P248 §3.3, Alg. 2 P297-P347)     */
/* ---------------------------------------------------------------------- */

/* Forward, Eq. (3) with padding, implicit im2col that visits only the
 * stored taps (P248): Y[oc][p][q][b] = sum over nonzeros (ic,x,y) of row oc
 * of w * X[ic][p+x-pad][q+y-pad][b] (0 outside).  X: [C_in][H][W][B],
 * Y: [C_out][OH][OW][B]. */
sp_status sp_conv2d_fwd(sp_weight_t W, const sp_conv_geom *g, const float *X, float *Y,
                        sp_stream_t stream);

/* Input gradient, Eq. (4) (P231-P238, bounds clipped per SURVEY C6):
 * dX[ic][m][n][b] = sum_{(x,y)} sum_{oc in CSC column (ic,x,y)}
 *                   w * dY[oc][m+pad-x][n+pad-y][b] over valid outputs.
 * Gather form (no atomics).  dY: [C_out][OH][OW][B], dX: [C_in][H][W][B]. */
sp_status sp_conv2d_bwd_input(sp_weight_t W, const sp_conv_geom *g, const float *dY, float *dX,
                              sp_stream_t stream);

/* Weight gradient, Eq. (5) (P240-P246), only at the nonzeros (P248):
 * dW[j=(oc,ic,x,y)] = sum_{p,q valid, b} dY[oc][p][q][b] *
 *                     X[ic][p+x-pad][q+y-pad][b].  dW: [nnz], CSR order of
 * the flattened filter == the paper's (oc, ic, x, y) storage order. */
sp_status sp_conv2d_bwd_weight(sp_weight_t W, const sp_conv_geom *g, const float *X,
                               const float *dY, float *dW, sp_stream_t stream);

/* Both conv backward products in one pass over the nonzeros: the paper's
 * Algorithm 2 (P297-P347, readings C5) -- per nonzero, one fmadd updates dX
 * (Eq. 4) and one accumulates dW (Eq. 5) from the same dY value -- driven tap
 * by tap from the transposed (CSC) index of each tap matrix, so dX needs no
 * atomics.  Same layouts and results (within rounding) as
 * sp_conv2d_bwd_input + sp_conv2d_bwd_weight, which it falls back to when
 * the handle is not a tap-tiled conv handle or B % 4 != 0.  Outputs
 * overwritten; no host sync. */
sp_status sp_conv2d_bwd(sp_weight_t W, const sp_conv_geom *g, const float *X, const float *dY,
                        float *dX, float *dW, sp_stream_t stream);

/* NCHW entry points: the paper's second conv kernel, SparseConvOverON
 * (P293, P397-P400: the natural B x C x H x W layout, vectorised over the
 * output width, for large spatial inputs).  Same products and readings as the
 * CHWN calls above, with X / dX [B][C_in][H][W] and Y / dY [B][C_out][OH][OW]:
 * the tap tiles are np x nq spatial tiles of one image (lanes along the output
 * rows), read through NCHW tensor maps whose out-of-bounds zero fill is the
 * halo.  A TMA box's innermost start (here: the width) must be 16-byte
 * aligned, so this direct path takes filters whose every column shift
 * (y - pad) is a multiple of 4 -- 1 x 1 convolutions with pad 0 -- with W and
 * OW multiples of 4 and a handle from sp_weight_create_conv; other shapes run
 * the CHWN kernels (whose slices span output columns x batch jointly) on
 * permuted copies (stream-ordered scratch).  dW in the handle's CSR order. */
sp_status sp_conv2d_fwd_nchw(sp_weight_t W, const sp_conv_geom *g, const float *X, float *Y, sp_stream_t stream);
sp_status sp_conv2d_bwd_input_nchw(sp_weight_t W, const sp_conv_geom *g, const float *dY, float *dX,
                                   sp_stream_t stream);
sp_status sp_conv2d_bwd_weight_nchw(sp_weight_t W, const sp_conv_geom *g, const float *X, const float *dY,
                                    float *dW, sp_stream_t stream);
sp_status sp_conv2d_bwd_nchw(sp_weight_t W, const sp_conv_geom *g, const float *X, const float *dY, float *dX,
                             float *dW, sp_stream_t stream);

/* ---------------------------------------------------------------------- */
/* Step helpers for the data-parallel sparse MLP (north star cfg5)        */
/* ---------------------------------------------------------------------- */

/* dY = Y - T and loss_partial = 1/2 sum (Y - T)^2 over n elements (SURVEY
 * C18).  loss_out: ONE device float; the sum is a fixed-order two-level
 * tree (deterministic).  `scratch` must hold sp_mse_scratch_floats(n)
 * device floats. */
int64_t sp_mse_scratch_floats(int64_t n);
sp_status sp_mse_grad(const float *Y, const float *T, float *dY, float *loss_out,
                      float *scratch, int64_t n, sp_stream_t stream);

/* Plain SGD on the kept weights only: vals[j] -= lr * dW[j]. */
sp_status sp_sgd(float *vals, const float *dW, int64_t nnz, float lr, sp_stream_t stream);

/* Managed weights (a launch-count optimisation for training loops; SURVEY
 * C23 "vals is the one mutable copy" still holds).  Every product first
 * copies the current `vals` into the handle's tiled index copies (one small
 * kernel per launch), because the caller may have written `vals` in place.
 * A caller that updates `vals` ONLY through sp_weight_sgd can declare so:
 * sp_weight_set_managed(W, 1); products then skip that copy while the tiled
 * weights are current.  Writing `vals` any other way while managed gives
 * stale results until sp_weight_set_managed is called again (it marks every
 * tiling stale).  Host-side flag only: no device work, no synchronisation. */
sp_status sp_weight_set_managed(sp_weight_t W, int managed);

/* Plain SGD on the kept weights of a handle, vals[j] -= lr * dW[j] (the same
 * rounding as sp_sgd), also writing each new value into the handle's tiled
 * copies that products have read since the previous update (one kernel; the
 * others are refreshed from vals at their next use).  dW: device [nnz] in
 * CSR slot order.  Enqueued on `stream`; the caller keeps dW alive until it
 * completes. */
sp_status sp_weight_sgd(sp_weight_t W, const float *dW, float lr, sp_stream_t stream);

/* sp_weight_sgd for n handles in ONE kernel (a model's optimizer step):
 * Ws[i] updated with dWs[i] (host arrays of n handles / device pointers),
 * 1 <= n <= SP_SGD_BATCH_MAX.  The same results as n sp_weight_sgd calls. */
#define SP_SGD_BATCH_MAX 64
sp_status sp_weights_sgd(const sp_weight_t *Ws, const float *const *dWs, int32_t n, float lr, sp_stream_t stream);

/* Thread-local message for the last non-OK status on this thread. */
const char *sp_last_error(void);

/* Number of kernels this library has launched in the process so far
 * (provenance: bench.py reports the delta over its timed region). */
uint64_t sp_launch_count(void);

/* SMs the one-wave (stream-K) kernels leave free: their grid is sized to
 * multiProcessorCount - n SMs of the current device (at least 1) for every
 * launch that follows, so that a collective running concurrently on another
 * stream (the data-parallel dW all_reduce) does not push part
 * of the wave into a second one.  Default 0.  Process-wide host setting (no
 * device work).  The stream-K kernels' fp32 summation grouping depends on
 * the grid, so results may change by rounding when n changes. */
sp_status sp_set_sm_reserve(int32_t n);

/* Provenance: the kernel families the last compute call (sp_linear_*,
 * sp_conv2d_*) on this thread launched, "+"-separated in launch order (e.g.
 * "spmm_hyb", "bwd_fused_sk_half").  Thread-local; valid until the next
 * compute call on this thread. */
const char *sp_last_path(void);

/* ---------------------------------------------------------------------- */
/* Data-parallel dW all_reduce over peer memory          */
/* ---------------------------------------------------------------------- */
/* The multi-GPU exchange of the DP step is the SUM of every rank's
 * nnz-length dW buffer (the paper runs one CPU, P367).  This
 * communicator does it without NCCL: each rank's dW lives in a "symmetric"
 * buffer (one per rank, the same size, mapped into every peer over
 * NVLink / NVSwitch with CUDA IPC), and ONE kernel per call does a two-shot
 * all_reduce on [offset, offset + count) floats: the range is cut into
 * `world` chunks; rank r reads chunk r from every peer, adds the values in
 * rank order 0..world-1 (fixed order: every rank ends with bitwise the same
 * sums) and stores the sums into every peer's chunk r (in place).  Each CTA
 * synchronises with its peer CTAs through flag words in the peers' signal
 * buffers (system-scope release / acquire, an epoch counter in device
 * memory: graph-capturable) before reading and after storing.
 * Setup (collective: every rank, same world / count):
 *   sp_comm_create  allocates this rank's buffer (count floats, zeroed) and
 *                   signal words, writes SP_COMM_HANDLE_BYTES of IPC handles
 *                   to handle_out (host memory);
 *   exchange the handles (e.g. torch.distributed.all_gather_object);
 *   sp_comm_open    maps the peers' buffers (handles: world records in rank
 *                   order, this rank's own included).
 * world <= SP_COMM_MAX_WORLD; count >= 1.  The buffer is owned by the
 * communicator (freed by sp_comm_destroy, which synchronises the device). */
#define SP_COMM_HANDLE_BYTES 128
#define SP_COMM_MAX_WORLD 8
typedef struct sp_comm_s *sp_comm_t;
sp_status sp_comm_create(int32_t rank, int32_t world, int64_t count, sp_comm_t *out, void *handle_out);
sp_status sp_comm_open(sp_comm_t c, const void *handles);
/* This rank's symmetric buffer (device, count floats). */
float *sp_comm_buffer(sp_comm_t c);
/* In-place SUM over all ranks of buffer[offset, offset + count), enqueued on
 * `stream`; every rank must make the same sequence of calls (SP_ERR_SHAPE if
 * the range leaves the buffer).  The kernel uses sp_comm_ctas() CTAs: leave
 * that many SMs free with sp_set_sm_reserve when it overlaps one-wave kernels. */
sp_status sp_comm_allreduce(sp_comm_t c, int64_t offset, int64_t count, sp_stream_t stream);
int32_t sp_comm_ctas(void);
sp_status sp_comm_destroy(sp_comm_t c);
/* Single-process test hooks: `world` virtual ranks' buffers on this device;
 * sp_comm_allreduce_as runs rank r's share of one call with the flag
 * synchronisation OFF (the caller runs r = 0..world-1 in order on one stream,
 * which reproduces the multi-GPU result: rank r reads and writes only chunk r). */
sp_status sp_comm_create_local(int32_t world, int64_t count, sp_comm_t *out);
float *sp_comm_local_buffer(sp_comm_t c, int32_t rank);
sp_status sp_comm_allreduce_as(sp_comm_t c, int32_t rank, int64_t offset, int64_t count, sp_stream_t stream);

/* ---------------------------------------------------------------------- */
/* NVLS dW all_reduce: NVLink SHARP multicast           */
/* ---------------------------------------------------------------------- */
/* The same exchange as sp_comm_* (SUM over ranks of the nnz-length dW
 * buffer), reduced by the NVSwitch: every rank's buffer is its
 * own physical memory bound to ONE multicast object over the ranks' GPUs;
 * the kernel (sp_nvls_ctas() CTAs) reads each 16-byte vector of this rank's
 * 1/world chunk once through the multicast address (multimem.ld_reduce.add:
 * the sum of all copies) and stores the sum once (multimem.st: into every
 * copy), between two flag barriers raised by multimem.red.release (epoch per
 * call in device memory: graph-capturable).  Every rank ends with the same
 * values; the addition order is the switch's.
 * Setup (collective, every rank the same world / count), in this order:
 *   sp_nvls_create  rank 0 creates the multicast object (world devices) and,
 *                   for world > 1, writes an exported POSIX fd to *fd_out
 *                   (others: -1); every rank allocates its physical memory;
 *   carry rank 0's fd to the other ranks (SCM_RIGHTS over a Unix socket);
 *   sp_nvls_open    ranks > 0 import it (fd); every rank adds its device;
 *   barrier;  sp_nvls_bind (binds and maps; zeroes the buffer);  barrier.
 * SP_ERR_CUDA when the device has no multicast support (sp_nvls_supported()
 * == 0) or a driver call fails; the buffer and mappings are owned by the
 * communicator (sp_nvls_destroy synchronises the device). */
typedef struct sp_nvls_s *sp_nvls_t;
int32_t sp_nvls_supported(void);
sp_status sp_nvls_create(int32_t rank, int32_t world, int64_t count, sp_nvls_t *out, int32_t *fd_out);
sp_status sp_nvls_open(sp_nvls_t c, int32_t fd);
sp_status sp_nvls_bind(sp_nvls_t c);
/* This rank's buffer (device, count floats; NULL before sp_nvls_bind). */
float *sp_nvls_buffer(sp_nvls_t c);
/* In-place SUM over all ranks of buffer[offset, offset + count) on `stream`;
 * every rank must make the same sequence of calls. */
sp_status sp_nvls_allreduce(sp_nvls_t c, int64_t offset, int64_t count, sp_stream_t stream);
int32_t sp_nvls_ctas(void);
sp_status sp_nvls_destroy(sp_nvls_t c);

/* Library build string (arch, version) for provenance in bench records. */
const char *sp_version(void);

#ifdef __cplusplus
}
#endif

#endif /* SPARSEPROP_H */
