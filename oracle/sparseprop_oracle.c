/*
 * sparseprop_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of what SparseProp's
 * hot path computes (arXiv 2302.04852, §3.2-§3.3), in fp64.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header,
 * table or helper with the CUDA path (paper_2302_04852_b200/csrc), and
 * includes no CUDA header.
 *
 * Everything is fp64 (inputs are the fp32 test values widened exactly).
 * Loops are the plain definitions; no blocking, no fusion, no reordering
 * beyond what the cited passage states.  OpenMP (when nthreads > 1) only
 * splits the outermost independent loop, so each output element keeps its
 * single-thread summation order and results are bitwise identical for any
 * thread count.
 *
 * Citations: "P<n>" = PAPER.md line n.
 *
 * Pins (tests/test_oracle.py): CSR/CSC vs brute-force mask scans; fwd vs a
 * numpy masked-dense matmul; adjoint identity <WX,G> = <X,W^T G>; central
 * finite differences for dX and dW; dW exactly 0 off the mask; conv vs
 * torch.nn.functional.conv2d (float64) and its autograd; conv K=1 reduces to
 * linear; the paper's worked conv-format example (P253-P285).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_OK 0
#define OR_ERR_ALLOC 1
#define OR_ERR_SHAPE 2

/* ------------------------------------------------------------------------ */
/* Sparse representation (P153-P154 §3.2 "Sparse Representation", CSR)      */
/* ------------------------------------------------------------------------ */

/* Count the kept entries of an R x C mask. */
int64_t or_mask_nnz(int64_t R, int64_t C, const uint8_t *mask)
{
    int64_t n = 0;
    for (int64_t i = 0; i < R * C; ++i)
        n += mask[i] != 0;
    return n;
}

/* CSR of W from (dense, mask): the structure is the MASK;
 * columns ascending within each row (C11).  W_rows = row_ptr, W_cols =
 * col_idx, W_vals = vals (P154).  Off-mask dense values are ignored. */
void or_csr_build(int64_t R, int64_t C, const uint8_t *mask, const double *dense,
                  int32_t *row_ptr, int32_t *col_idx, double *vals)
{
    int64_t k = 0;
    row_ptr[0] = 0;
    for (int64_t r = 0; r < R; ++r) {
        for (int64_t c = 0; c < C; ++c) {
            if (mask[r * C + c]) {
                col_idx[k] = (int32_t)c;
                vals[k] = dense[r * C + c];
                ++k;
            }
        }
        row_ptr[r + 1] = (int32_t)k;
    }
}

/* CSC "index copy" of the same matrix (P183: "the transpose of a CSR matrix
 * is ... the same matrix in CSC format"): for c ascending, for r ascending
 * where mask[r][c]: row_idx[k] = r and perm[k] = the CSR slot of (r, c)
 * (SURVEY C11, C23). */
int or_csc_build(int64_t R, int64_t C, const uint8_t *mask,
                 int32_t *col_ptr, int32_t *row_idx, int32_t *perm)
{
    /* CSR slot of every kept (r, c), numbered in row-major scan order. */
    int32_t *slot = (int32_t *)malloc((size_t)(R * C) * sizeof(int32_t));
    if (!slot)
        return OR_ERR_ALLOC;
    int32_t s = 0;
    for (int64_t i = 0; i < R * C; ++i)
        slot[i] = mask[i] ? s++ : -1;
    int64_t k = 0;
    col_ptr[0] = 0;
    for (int64_t c = 0; c < C; ++c) {
        for (int64_t r = 0; r < R; ++r) {
            if (mask[r * C + c]) {
                row_idx[k] = (int32_t)r;
                perm[k] = slot[r * C + c];
                ++k;
            }
        }
        col_ptr[c + 1] = (int32_t)k;
    }
    free(slot);
    return OR_OK;
}

/* Densify an nnz-length buffer (values or gradients) over the CSR support:
 * exact +0.0 off the mask (north star "dW exactly zero off the mask"). */
void or_densify(int64_t R, int64_t C, const int32_t *row_ptr, const int32_t *col_idx,
                const double *nz, double *dense_out)
{
    for (int64_t i = 0; i < R * C; ++i)
        dense_out[i] = 0.0;
    for (int64_t r = 0; r < R; ++r)
        for (int32_t j = row_ptr[r]; j < row_ptr[r + 1]; ++j)
            dense_out[r * C + col_idx[j]] = nz[j];
}

/* ------------------------------------------------------------------------ */
/* Linear layer (P141-P151 §3.2).  North-star orientation Y = W X with W    */
/* R x C (out x in) = the paper's W^T; activations are the      */
/* paper's transposed X^T layout (P183): [features x B], batch contiguous.  */
/* ------------------------------------------------------------------------ */

/* Forward: Y[r][b] = sum_{j in row r} vals[j] * X[col_idx[j]][b]
 * (the paper's O = X W, P141, transposed).  j ascending per element. */
void or_linear_fwd(int64_t R, int64_t B, const int32_t *row_ptr, const int32_t *col_idx,
                   const double *vals, const double *X, double *Y, int nthreads)
{
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
    for (int64_t r = 0; r < R; ++r) {
        double *y = Y + r * B;
        for (int64_t b = 0; b < B; ++b)
            y[b] = 0.0;
        for (int32_t j = row_ptr[r]; j < row_ptr[r + 1]; ++j) {
            const double w = vals[j];
            const double *x = X + (int64_t)col_idx[j] * B;
            for (int64_t b = 0; b < B; ++b)
                y[b] += w * x[b];
        }
    }
}

/* Input gradient, Eq. (1) (P143-P145): dL/dX = dL/dO W^T, i.e. in our
 * orientation dX[c][b] = sum_r W[r][c] dY[r][b], driven by the CSC copy:
 * k ascending over column c's list (rows ascending), value vals[perm[k]]. */
void or_linear_bwd_input(int64_t C, int64_t B, const int32_t *col_ptr, const int32_t *row_idx,
                         const int32_t *perm, const double *vals, const double *dY, double *dX,
                         int nthreads)
{
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
    for (int64_t c = 0; c < C; ++c) {
        double *dx = dX + c * B;
        for (int64_t b = 0; b < B; ++b)
            dx[b] = 0.0;
        for (int32_t k = col_ptr[c]; k < col_ptr[c + 1]; ++k) {
            const double w = vals[perm[k]];
            const double *dy = dY + (int64_t)row_idx[k] * B;
            for (int64_t b = 0; b < B; ++b)
                dx[b] += w * dy[b];
        }
    }
}

/* Weight gradient, Eq. (2) (P146-P148) restricted to the mask (SDDMM, P151,
 * P173 "nnz dot-products"): dW[j] = sum_b dY[r_j][b] * X[c_j][b], b
 * ascending, one dot product per nonzero j in CSR order. */
void or_linear_bwd_weight(int64_t R, int64_t B, const int32_t *row_ptr, const int32_t *col_idx,
                          const double *X, const double *dY, double *dW, int nthreads)
{
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
    for (int64_t r = 0; r < R; ++r) {
        const double *dy = dY + r * B;
        for (int32_t j = row_ptr[r]; j < row_ptr[r + 1]; ++j) {
            const double *x = X + (int64_t)col_idx[j] * B;
            double acc = 0.0;
            for (int64_t b = 0; b < B; ++b)
                acc += dy[b] * x[b];
            dW[j] = acc;
        }
    }
}

/* ------------------------------------------------------------------------ */
/* Convolution (P222-P248 §3.3), stride 1, padding pad.       */
/* Canonical NCHW layout of Eq. (3): X [B][IC][M][N], O [B][OC][OM][ON],     */
/* OM = M + 2 pad - KH + 1.  The weight is held in the paper's own 4-array  */
/* format (P251): och[OC+1], ich[OC*(IC+1)] (offsets relative to och[oc]),  */
/* wx[nnz], wy[nnz] (tap row / column), vals[nnz]; order (oc, ic, x, y).     */
/* ------------------------------------------------------------------------ */

/* Build the 4-array format from a dense [OC][IC][KH][KW] tensor and mask.
 * Storage order is lexicographic (oc, ic, x, y), which is what the paper's
 * index arrays encode (worked example P280-P284; value order per SURVEY C8).
 * Returns nnz. */
int64_t or_conv_format(int64_t OC, int64_t IC, int64_t KH, int64_t KW, const uint8_t *mask,
                       const double *dense, int32_t *och, int32_t *ich, int32_t *wx, int32_t *wy,
                       double *vals)
{
    int64_t k = 0;
    och[0] = 0;
    for (int64_t oc = 0; oc < OC; ++oc) {
        int64_t base = k;
        for (int64_t ic = 0; ic < IC; ++ic) {
            ich[oc * (IC + 1) + ic] = (int32_t)(k - base);
            for (int64_t x = 0; x < KH; ++x)
                for (int64_t y = 0; y < KW; ++y) {
                    int64_t i = ((oc * IC + ic) * KH + x) * KW + y;
                    if (mask[i]) {
                        wx[k] = (int32_t)x;
                        wy[k] = (int32_t)y;
                        vals[k] = dense[i];
                        ++k;
                    }
                }
        }
        ich[oc * (IC + 1) + IC] = (int32_t)(k - base);
        och[oc + 1] = (int32_t)k;
    }
    return k;
}

/* Forward, Eq. (3) (P224-P229) with padding, skipping pruned taps (P248):
 * O[b,oc,p,q] = sum over nonzeros (ic,x,y) of W * X[b,ic,p+x-pad,q+y-pad],
 * out-of-range X read as 0. */
void or_conv2d_fwd(int64_t B, int64_t IC, int64_t M, int64_t N, int64_t OC, int64_t KH,
                   int64_t KW, int64_t pad, const int32_t *och, const int32_t *ich,
                   const int32_t *wx, const int32_t *wy, const double *vals, const double *X,
                   double *O, int nthreads)
{
    const int64_t OM = M + 2 * pad - KH + 1, ON = N + 2 * pad - KW + 1;
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
    for (int64_t b = 0; b < B; ++b)
        for (int64_t oc = 0; oc < OC; ++oc)
            for (int64_t p = 0; p < OM; ++p)
                for (int64_t q = 0; q < ON; ++q) {
                    double acc = 0.0;
                    for (int64_t ic = 0; ic < IC; ++ic) {
                        int64_t s = och[oc] + ich[oc * (IC + 1) + ic];
                        int64_t e = och[oc] + ich[oc * (IC + 1) + ic + 1];
                        for (int64_t si = s; si < e; ++si) {
                            int64_t m = p + wx[si] - pad, n = q + wy[si] - pad;
                            if (m < 0 || m >= M || n < 0 || n >= N)
                                continue;
                            acc += vals[si] * X[((b * IC + ic) * M + m) * N + n];
                        }
                    }
                    O[((b * OC + oc) * OM + p) * ON + q] = acc;
                }
}

/* Backward, Algorithm 2 (P297-P347) with the SURVEY C5 readings: ich
 * offset oc*(IC+1); j := si; shifted coordinates (p+x-pad, q+y-pad);
 * half-open loops; one dW reduction per nonzero.  For every nonzero
 * (oc, ic, x, y) and every output (p, q) in the clipped ranges
 *   p in [max(0, pad-x), min(pad-x+M, OM)),  q likewise (P317-P320),
 * dX[b,ic,p+x-pad,q+y-pad] += dO[b,oc,p,q] * w      (Eq. 4, P231-P238)
 * acc += dO[b,oc,p,q] * X[b,ic,p+x-pad,q+y-pad]     (Eq. 5, P240-P246)
 * dW[si] = acc.  dX is accumulated in fp64 (order differs from a gather,
 * which fp64 makes immaterial at the fp32 tolerance). */
void or_conv2d_bwd(int64_t B, int64_t IC, int64_t M, int64_t N, int64_t OC, int64_t KH,
                   int64_t KW, int64_t pad, const int32_t *och, const int32_t *ich,
                   const int32_t *wx, const int32_t *wy, const double *vals, const double *X,
                   const double *dO, double *dX, double *dW)
{
    const int64_t OM = M + 2 * pad - KH + 1, ON = N + 2 * pad - KW + 1;
    (void)KW;
    for (int64_t i = 0; i < B * IC * M * N; ++i)
        dX[i] = 0.0;
    for (int64_t ic = 0; ic < IC; ++ic) {
        for (int64_t oc = 0; oc < OC; ++oc) {
            int64_t s = och[oc] + ich[oc * (IC + 1) + ic];
            int64_t e = och[oc] + ich[oc * (IC + 1) + ic + 1];
            for (int64_t si = s; si < e; ++si) {
                const double v = vals[si];
                double acc = 0.0;
                int64_t ps = pad - wx[si] > 0 ? pad - wx[si] : 0;
                int64_t pe = pad - wx[si] + M < OM ? pad - wx[si] + M : OM;
                int64_t qs = pad - wy[si] > 0 ? pad - wy[si] : 0;
                int64_t qe = pad - wy[si] + N < ON ? pad - wy[si] + N : ON;
                for (int64_t p = ps; p < pe; ++p)
                    for (int64_t q = qs; q < qe; ++q) {
                        int64_t m = p + wx[si] - pad, n = q + wy[si] - pad;
                        for (int64_t b = 0; b < B; ++b) {
                            double d = dO[((b * OC + oc) * OM + p) * ON + q];
                            dX[((b * IC + ic) * M + m) * N + n] += d * v;
                            acc += d * X[((b * IC + ic) * M + m) * N + n];
                        }
                    }
                dW[si] = acc;
            }
        }
    }
}

int or_num_threads_available(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
