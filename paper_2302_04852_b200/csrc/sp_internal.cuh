// sp_internal.cuh -- internals of libsparseprop (B200 / sm_100a).
//
// The handle, error plumbing and the launcher prototypes shared by the
// translation units of the CUDA path.  Nothing here is shared with oracle/.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/sparseprop.h"

#define SP_MAGIC 0x53505731u /* "SPW1" */

constexpr int kMaxTaps = 25;  // conv filters up to 5x5 use the tap-tiled kernels

// Exact output columns of the conv kernels (4-D TMA path).  A
// slice of 128 columns is
//  - CHWN (the paper's batch-last SparseConv layout, P293): nq output columns
//    q x bs batch elements of one output row p (B <= 128: bs = B, nq = 128 / B;
//    B > 128: bs = 128, nq = 1, bpr = B / 128 slices per q); slice sl -> p = sl / spr;
//  - NCHW (the paper's SparseConvOverON, natural layout vectorised over the
//    output width, P293 / P397): an np x nq spatial tile of one image, nq
//    consecutive output columns per row (lanes over q).
// Tap t reads the input at (p + dp[t], q + dq[t]) through a 4-D tensor map
// whose out-of-bounds zero fill is the halo: no padded copy, no virtual columns.
struct ConvCols {
    int32_t nchw;           // 0: CHWN, 1: NCHW
    int32_t bsh;            // CHWN: log2 bs
    int32_t nq, spr, bpr;   // CHWN: q per slice, slices per output row, batch slices per q
    int32_t np, qsh, nqt, npt;  // NCHW: rows per slice, log2 nq, q tiles / p tiles per image
    int32_t Po, Qo;         // output rows / columns of the product
    int64_t B;
    int64_t rowlen;         // floats between consecutive channels (rows) of an output / X tensor
    int64_t imgstride;      // NCHW: floats per image of the output / X tensor
    int64_t nslice;
    int8_t dp[25], dq[25];  // per-tap input offsets (kMaxTaps)
};

// Device view of one tap tiling (conv kernels index these by tap).
struct TapDev {
    const int32_t *seg;
    const int2 *ent;
    const int32_t *vidx;
    int64_t npad;
    const int32_t *split;  // tmsplit of the tap tiling (nullptr: none)
};

// A tiled copy of one orientation's index structure (built once per handle,
// DESIGN.md §5): rows are grouped in row blocks of RB, the inner dimension in
// column blocks of KC.  Entries are ordered (row block, column block, local
// row, column); segment (t = rb*nkb + kb, local row lr) is
// [seg[t*RB + lr], seg[t*RB + lr + 1]).  ent[e] = (column - kb*KC, value bits)
// with the value refreshed from vals[vidx[e]] before use; vidx[e] is the CSR
// slot of the entry.
struct sp_tiling {
    int RB, KC, nrb, nkb;
    int64_t rows, inner;
    int32_t *seg;   // [nrb*nkb*RB + 1]
    int2 *ent;      // [nnz + 8] (padded)
    int32_t *vidx;  // [nnz]
    int32_t max_tile;  // max (padded) entries in one (row block, column block) tile
    int64_t max_warp_groups8;  // the same in groups of 8 entries (half-warp fused backward)
    int64_t max_warp_groups;  // max entry groups (4 entries, a last one may hold 2) of 4 consecutive tiled rows
                              // (variant 0; RB/NW rows otherwise) over all column blocks
    int64_t npad;      // padded entry total (segments padded to kTilPad with weight-0 entries)
    int64_t cap_ent;   // allocated entries
    // nnz-balanced row placement: tiled position -> row (-1 unused) and back;
    // rowmap == nullptr means identity (conv tap tilings)
    int32_t *rowpos;   // [rows]
    int32_t *rowmap;   // [nrb * RB]
    // split-source SpMM (spmm_hyb.cu, big tilings only): tmsplit[s] = the even
    // entry index from which segment s holds only columns >= KC - kHybTC of its
    // column block (those tile rows are mirrored in TMEM), or the segment end
    int32_t *tmsplit;  // [nrb*nkb*RB] (nullptr: not built)
    // managed weights (sp_weight_sgd): inv[slot] = the entry position of a CSR
    // slot in this tiling; `fresh` = the handle version whose values ent holds
    int32_t *inv;      // [nnz]
    mutable uint64_t fresh;
    mutable bool used;  // a product read this tiling's weights since the last sp_weight_sgd
    // CSC tilings (fused backward): per (row block, warp of RPWg rows), the prefix
    // over column blocks of the warp's entry groups, gpre[g][(rb*NWg + w)*(nkb+1) + k]
    // = sum over column blocks < k of ceil(segment length / (4 << g)) -- the TMEM
    // dW column of a tile's first group without walking the earlier tiles
    int32_t *gpre[2];
    int RPWg;
    bool in_arena;  // buffers carved from the handle's tiling arena (freed with it)
    // split rows (forward tilings of skewed masks, e.g. Zipf head rows): a row
    // with many more entries than the mean is dealt, entry by entry in turn, into
    // `k` part rows placed like any other row, so no warp carries a whole dense
    // row through every tile.  split[pos] = the part slot of a part row (-1 for a
    // whole row; rowmap still gives the real row), part rows store raw sums to a
    // scratch [nparts x B] and split_reduce adds each row's parts in slot order
    int32_t *split;  // [nrb * RB] (nullptr: no split rows)
    int32_t nparts, nsplit;
    int32_t *prow;   // [nsplit] real row of each split row
    int32_t *pptr;   // [nsplit + 1] its part slots [pptr[i], pptr[i+1])
    bool psplit_rows() const { return split != nullptr; }
};

// One tiling's entries as seen by the managed SGD kernel.
struct SgdRef {
    int2 *ent;
    const int32_t *inv;
};

struct sp_weight_s {
    uint32_t magic;
    // device arenas (one cudaMalloc each, sp_weight_create's allocation cost):
    // [0] row_ptr + col_ptr, [1] the nnz-sized index arrays + chunk_ptr,
    // [2] every linear tiling + the managed-SGD table
    void *arena[4];  // [3]: the conv tap tilings (build_conv_taps)
    int64_t R, C, nnz;
    // CSR (P153-P154): row_ptr[R+1], col_idx[nnz], vals[nnz]
    int32_t *row_ptr;
    int32_t *col_idx;
    float *vals;
    // CSC index copy (P183): col_ptr[C+1], row_idx[nnz], perm[nnz]
    int32_t *col_ptr;
    int32_t *row_idx;
    int32_t *perm;
    // row of every CSR slot (for the SDDMM chunk walk and to_dense)
    int32_t *row_of;
    int32_t max_row_nnz, max_col_nnz;
    int32_t *chunk_ptr;  // [R+1] exclusive scan of ceil(row nnz / 32) (gather SDDMM work list)
    // tilings: [orientation 0 = CSR rows, 1 = CSC columns][variant 0 = big, 1 = small]
    sp_tiling til[2][2];
    // CSC tilings of the fused backward (KC = 192): [0] 64-row blocks (32 warps x 2
    // rows), [1] 32-row blocks (32 warps x 1 row, long rows), [2] 64-row blocks
    // as 16 warps x 4 rows (half-warp entries when [0]'s dW columns overflow)
    sp_tiling til_f[3];
    // gather tilings of the very sparse regime (gather.cu's bulk-gather kernels):
    // [orientation], one column block spanning the whole inner dimension (ent.x =
    // inner index * kTilRowBytes), 32-position blocks balanced over 8 units of 4
    // positions; built only when kGatherDensity / kGatherNnz admit the gather path
    sp_tiling til_g[2];
    // [orientation] 128-row blocks with 128-column tiles, built for masks denser
    // than kTilKDensity: their 192-column tiles carry more entries than the
    // stream-K SpMM can stage next to two activation tiles (e.g. 4096^2 at
    // 80-90 %, B = 256, whose per-item grid is too short for the tiled kernels)
    sp_tiling til_k[2];
    // conv handles (sp_weight_create_conv): filter taps and, per tap (x, y),
    // tilings of the OC x IC tap matrix W_xy -- [0]: rows oc / inner ic,
    // [1]: rows ic / inner oc -- whose vidx are slots of THIS handle's CSR.
    int conv_kh, conv_kw;
    sp_tiling tap[kMaxTaps][2];
    // [2] of the fused conv backward: rows ic / inner oc in 64-row blocks (the
    // stream-K TMEM kernel with 2 rows per warp); tapf_groups = max entry groups
    // of one warp's 2 rows over all taps and column blocks
    sp_tiling tapf[kMaxTaps];
    int64_t tapf_groups;
    int64_t tapf_groups8;  // the same in groups of 8 (half-warp fused conv backward)
    mutable uint64_t tap_fresh[3];  // handle version whose vals the tap tilings of each orientation hold (0: never)
    struct TapDev *tapdev;  // device copy of the tap tilings' pointers [3][kMaxTaps]: orient 0, 1, fused
    // managed mode (sp_weight_set_managed): vals change only through
    // sp_weight_sgd, which rewrites the tilings' weights too, so products skip
    // the per-launch refresh while a tiling is at the handle's version
    int managed;
    uint64_t version;
    int nsgd;
    SgdRef *sgdtab;  // device [nsgd]: every built (non-tap) tiling
    sp_tiling *sgdtil[16];  // host: the tiling of each sgdtab entry
};

// The gather tilings are built for masks at most this dense, or this small.
constexpr double kGatherDensity = 0.03;
constexpr double kTilKDensity = 0.07;
constexpr int kTilKC_K = 128;
constexpr int64_t kGatherNnz = 1 << 15;
constexpr int kGatherRB = 32, kGatherUnit = 4;  // positions per block / per warp unit

// Tiling variants (RB rows per CTA, KC inner columns per shared-memory tile).
constexpr int kTilRB[2] = {128, 32};
constexpr int kTilKC[2] = {192, 96};
constexpr int kTilNW[2] = {16, 8};  // warps per CTA of the kernels using each variant (RB = NW * RPW)
// Segments are padded to a multiple of kTilPad entries (offset -kTilRowBytes,
// weight 0, vidx -1), so every segment starts at an even entry (16-byte
// aligned entry pairs).  Kernels walk segments in groups of 4 entries; a
// group whose second pair lies past the segment end (segment length = 2 mod 4)
// masks that pair (no load, weight 0).  A padding entry's offset addresses the
// all-zero row kernels keep just before a tile (or is skipped by a predicated
// load).  Entry columns are stored as byte offsets of a 128-float tile row
// (kTilRowBytes); kernels with narrower tiles shift them down.  Conv tap
// tilings are padded the same way (kTapPad).
constexpr int kTilPad = 2;
// tile rows the split-source SpMM mirrors in TMEM (the last kHybTC of a tile)
constexpr int kHybTC = 63;
constexpr int kTapPad = 2;  // (was 4: groups of 4 without tails; even padding wastes fewer slots)
constexpr int kTilRowBytes = 512;

namespace sp {

// ---- programmatic dependent launch (PDL) ---------------------------------------
// A short consumer kernel (a reduction of a previous kernel's parts) is launched
// as a programmatic dependent: its CTAs may be scheduled on SMs the producer
// grid frees once every producer CTA has called pdl_trigger() (early in the
// producer), do their independent prologue, and pdl_wait() for the producer's
// completion (its memory visible) before reading what it wrote.  Kernels that
// are not launched this way ignore both instructions.
__device__ __forceinline__ void pdl_trigger() {
#ifndef SP_NO_PDL
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
__device__ __forceinline__ void pdl_wait() {
#ifndef SP_NO_PDL
    asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
#ifndef SP_NO_PDL
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...) == cudaSuccess) return;
    cudaGetLastError();  // (clear the failed attempt; launch plainly)
#endif
    kern<<<grid, block, smem, st>>>(static_cast<KArgs>(args)...);
}

void set_error(const std::string &msg);

// Count of kernel launches issued by the library (provenance for bench.py).
void count_launches(int n);

// Provenance of the kernel path a public compute call took (sp_last_path):
// begin_path() at the entry point clears it, note_path() appends a kernel
// family name ("+"-separated) at each launch site of a hot-path kernel.
void begin_path();
void note_path(const char *name);

// Launch-error check after an asynchronous launch.
sp_status check_launch(const char *what);

// SMs a one-wave (stream-K) grid is sized to on the current device: the
// device's multiProcessorCount, less the reserve set by sp_set_sm_reserve
// (SMs left free for a concurrent collective), at least 1.
int num_sms();

// Stream-ordered scratch from a library-owned memory pool per device (its
// release threshold is raised so freed blocks stay cached; the caller's
// default pool is left alone).  Same contract as cudaMallocAsync / FreeAsync.
cudaError_t scratch_alloc(void **p, size_t bytes, cudaStream_t st);
cudaError_t scratch_free(void *p, cudaStream_t st);

inline cudaStream_t S(sp_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

// ---- tmap.cu ----
// Tensor map of a row-major fp32 [rows x B] activation (B % 4 == 0) with a
// box of `box_rows` rows x `box_cols` batch columns, no swizzle, zero OOB
// fill.  Returns false if the driver entry point is unavailable.
bool make_tmap_2d(CUtensorMap *map, const float *base, int64_t rows, int64_t B, int box_cols, int box_rows);
// 4-D map of the input of a conv product ([C][Hi][Wi][B] for CHWN, [B][C][Hi][Wi]
// for NCHW) with the box of one tap tile of cc (kc channels x 128 positions)
bool make_tmap_conv(CUtensorMap *map, const float *base, const ConvCols &cc, int64_t C, int64_t Hi, int64_t Wi,
                    int kc);
// ConvCols of a CHWN product with output Po x Qo, batch B and R output
// channels; false if B fits no exact slicing (B % 4 != 0, or neither
// 128 % B == 0 nor B % 128 == 0)
bool conv_cols(int64_t B, int Po, int Qo, int64_t R, ConvCols *cc);
// ConvCols of an NCHW product (SparseConvOverON); false unless Qo % 4 == 0
bool conv_cols_nchw(int64_t B, int Po, int Qo, int64_t R, ConvCols *cc);

// ---- build.cu ----
sp_status build_weight(int64_t R, int64_t C, const float *dense, const uint8_t *mask,
                       cudaStream_t st, sp_weight_s *w);
void launch_to_dense(const sp_weight_s *w, const float *nz, float *dense, cudaStream_t st);
void launch_gather_dense(const sp_weight_s *w, const float *dense, float *nz, cudaStream_t st);
sp_status build_tilings(sp_weight_s *w, cudaStream_t st);
void free_tilings(sp_weight_s *w);
// every device buffer of a handle (arenas, conv tap tilings)
void free_weight(sp_weight_s *w);
// ent[e].y = bits(vals[vidx[e]]) for one tiling (before an SpMM launch)
void launch_refresh(const sp_tiling &t, const float *vals, int64_t nnz, cudaStream_t st);
// the same unless the handle is managed and the tiling already holds its version
void refresh_if_stale(const sp_weight_s *w, const sp_tiling &t, cudaStream_t st);
// zero n ints on `st` (a programmatic-dependent kernel instead of a memset node:
// the launch chain of the kernels that follow keeps its prologue overlap)
void launch_zero_i32(int *p, int64_t n, cudaStream_t st);
void launch_weights_sgd(sp_weight_s *const *ws, const float *const *dWs, int n, float lr, cudaStream_t st);
// managed SGD: vals[j] -= lr dW[j] and the new value written into every tiling
void launch_weight_sgd(sp_weight_s *w, const float *dW, float lr, cudaStream_t st);

// ---- spmm.cu ----
// Epilogue codes for the SpMM kernels.
enum Epi { EPI_NONE = 0, EPI_RELU = 1, EPI_GATE = 2 };
// out[r][b] = epi(sum over row r of the orientation: w * in[col][b]);
// orient 0: forward (CSR, rows = R, inner = C); 1: dX (CSC, rows = C, inner = R).
void launch_spmm(const sp_weight_s *w, int orient, int64_t B, const float *in, float *out,
                 const float *gate, int epi, cudaStream_t st);

// ---- split rows (build.cu): out[prow[i]][b] = epi(sum of the parts of split row i)
void launch_split_rows_reduce(const sp_tiling &t, const float *vpart, int64_t B, float *out, const float *gate,
                              int epi, cudaStream_t st);

// ---- spmm_sk.cu: stream-K SpMM (B % 4 == 0, big tiling); false if it does not apply
bool launch_spmm_sk(const sp_weight_s *w, int orient, int64_t B, const float *in, float *out, const float *gate,
                    int epi, cudaStream_t st, int64_t s_begin = 0, int64_t s_end = -1);
bool launch_conv_spmm_sk(const sp_weight_s *w, int orient, const ConvCols &cc, const float *in, int64_t Hi,
                         int64_t Wi, float *out, int ntap, cudaStream_t st);

// ---- spmm_hyb.cu: the 32-warp SpMM with the tiles' last rows mirrored in TMEM
bool launch_spmm_hyb(const sp_weight_s *w, int orient, int64_t B, const float *in, float *out, const float *gate,
                     int epi, cudaStream_t st, int64_t nslice_limit = -1);

// ---- gather.cu (very sparse / small regime: no shared-memory staging) ----
bool gather_preferred(const sp_weight_s *w, int orient, int64_t B, bool chunked = false);
// position-gather kernels: mode 0 SpMM (orient 0 fwd / 1 dX), 1 fused backward
// (orient 1), 2 dW alone (orient 0); false when they do not apply
bool launch_gather_pos(const sp_weight_s *w, int orient, int mode, int64_t B, const float *gin, const float *rin,
                    const float *gate, int epi, float *out, float *dW, cudaStream_t st);
void launch_spmm_gather(const sp_weight_s *w, int orient, int64_t B, const float *in, float *out,
                        const float *gate, int epi, cudaStream_t st);
void launch_sddmm_gather(const sp_weight_s *w, const float *X, const float *dY, float *dW, int64_t B,
                         cudaStream_t st);

// ---- sddmm.cu ----
// dW[j] = sum_b dY[row(j)][b] * X[col_idx[j]][b]
sp_status launch_sddmm(const sp_weight_s *w, const float *X, const float *dY, float *dW,
                       int64_t B, cudaStream_t st);

// dW[vidx[e]] = sum_s part[s][e] over a tiling's padded entries
void launch_split_reduce(int64_t npad, int nsplit, const float *part, const int32_t *vidx, float *dW,
                         cudaStream_t st);

// ---- fused.cu ----
// One CSC-driven pass for both backward products of a linear layer (the
// paper's Alg. 1 single pass, P173, made atomic-free):
//   dX = (W^T dY) [* (H > 0) if H]   and   dW = SDDMM(dY, X).
// Returns SP_ERR_SHAPE if the fused path does not apply (caller falls back).
sp_status launch_bwd_fused(const sp_weight_s *w, const float *X, const float *dY, const float *H, float *dX,
                           float *dW, int64_t B, cudaStream_t st);
// conv backward by taps through the stream-K TMEM kernel (dX null: dW alone); false if it does not apply
bool launch_conv_bwd_sk(const sp_weight_s *w, const ConvCols &cc, const float *dY, int64_t OH, int64_t OW,
                        const float *X, float *dX, float *dW, int ntap, cudaStream_t st);
// fused conv backward (dX and dW); falls back to the separate products
sp_status launch_conv_bwd(const sp_weight_s *w, const sp_conv_geom &g, const float *X, const float *dY, float *dX,
                          float *dW, cudaStream_t st);
// dW alone through the stream-K TMEM kernel; false if it does not apply
bool launch_sddmm_sk(const sp_weight_s *w, const float *X, const float *dY, float *dW, int64_t B, cudaStream_t st);

bool launch_conv_spmm(const sp_weight_s *w, int orient, int64_t B, const float *in, int64_t Lp, float *out,
                      const int *sh, int ntap, int64_t Wv, int64_t OHv, int64_t OWv, cudaStream_t st);
void launch_refresh_taps(const sp_weight_s *w, int orient, int ntap, cudaStream_t st);
bool launch_conv_sddmm(const sp_weight_s *w, int64_t B, const float *dYv, const float *Xp, int64_t Lv, int64_t Lp,
                       const int *sh, int ntap, float *dW, cudaStream_t st);

// ---- conv_taps.cu ----
// Build the per-tap tilings of a conv handle (host-side, once, after
// build_weight); frees with free_tilings.
sp_status build_conv_taps(sp_weight_s *w, int OC, int IC, int KH, int KW, cudaStream_t st);

// ---- conv.cu ----
void launch_conv_fwd(const sp_weight_s *w, const sp_conv_geom &g, const float *X, float *Y,
                     cudaStream_t st);
void launch_conv_bwd_input(const sp_weight_s *w, const sp_conv_geom &g, const float *dY,
                           float *dX, cudaStream_t st);
sp_status launch_conv_bwd_weight(const sp_weight_s *w, const sp_conv_geom &g, const float *X,
                                 const float *dY, float *dW, cudaStream_t st);
// NCHW products (SparseConvOverON): op 0 fwd (X -> out = Y), 1 dX (dY -> out = dX),
// 2 fused backward (X, dY -> out = dX, dW), 3 dW alone
sp_status launch_conv_nchw(const sp_weight_s *w, const sp_conv_geom &g, int op, const float *X, const float *dY,
                           float *out, float *dW, cudaStream_t st);

// ---- step.cu ----
int64_t mse_scratch_floats(int64_t n);
void launch_mse(const float *Y, const float *T, float *dY, float *loss, float *scratch, int64_t n,
                cudaStream_t st);
void launch_sgd(float *vals, const float *dW, int64_t nnz, float lr, cudaStream_t st);

}  // namespace sp
