// sp_internal.cuh -- internals of libsparseprop (B200 / sm_100a).
//
// The handle, error plumbing and the launcher prototypes shared by the
// translation units of the CUDA path.  Nothing here is shared with oracle/.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/sparseprop.h"

#define SP_MAGIC 0x53505731u /* "SPW1" */

struct sp_weight_s {
    uint32_t magic;
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
};

namespace sp {

void set_error(const std::string &msg);

// Count of kernel launches issued by the library (provenance for bench.py).
void count_launches(int n);

// Launch-error check after an asynchronous launch.
sp_status check_launch(const char *what);

inline cudaStream_t S(sp_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

// ---- build.cu ----
sp_status build_weight(int64_t R, int64_t C, const float *dense, const uint8_t *mask,
                       cudaStream_t st, sp_weight_s *w);
void launch_to_dense(const sp_weight_s *w, const float *nz, float *dense, cudaStream_t st);

// ---- spmm.cu ----
// Epilogue codes for the SpMM kernels.
enum Epi { EPI_NONE = 0, EPI_RELU = 1, EPI_GATE = 2 };
// out[r][b] = epi(sum_k val(k) * in[idx[k]][b]) over k in [ptr[r], ptr[r+1]),
// val(k) = vals[perm ? perm[k] : k].  rows = #out rows, inner = #in rows.
void launch_spmm(int64_t rows, int64_t inner, int64_t B, const int32_t *ptr, const int32_t *idx,
                 const int32_t *perm, const float *vals, const float *in, float *out,
                 const float *gate, int epi, int max_seg, cudaStream_t st);

// ---- sddmm.cu ----
// dW[j] = sum_b dY[row(j)][b] * X[col_idx[j]][b]
sp_status launch_sddmm(const sp_weight_s *w, const float *X, const float *dY, float *dW,
                       int64_t B, cudaStream_t st);

// ---- conv.cu ----
void launch_conv_fwd(const sp_weight_s *w, const sp_conv_geom &g, const float *X, float *Y,
                     cudaStream_t st);
void launch_conv_bwd_input(const sp_weight_s *w, const sp_conv_geom &g, const float *dY,
                           float *dX, cudaStream_t st);
sp_status launch_conv_bwd_weight(const sp_weight_s *w, const sp_conv_geom &g, const float *X,
                                 const float *dY, float *dW, cudaStream_t st);

// ---- step.cu ----
int64_t mse_scratch_floats(int64_t n);
void launch_mse(const float *Y, const float *T, float *dY, float *loss, float *scratch, int64_t n,
                cudaStream_t st);
void launch_sgd(float *vals, const float *dW, int64_t nnz, float lr, cudaStream_t st);

}  // namespace sp
