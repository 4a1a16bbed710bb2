// build.cu -- sp_weight_create on the device.
//
// From a dense R x C fp32 weight and an R x C uint8 mask, build
//   CSR (P153-P154): row_ptr, col_idx (ascending per row), vals, row_of
//   CSC index copy (P183): col_ptr, row_idx (ascending per column), perm
// deterministically (no atomics): counts -> exclusive scans -> stable
// compaction.  The structure is the mask.  Off the timed
// path (masks change "only a few times", P428).
#include <cuda_runtime.h>

#include <vector>

#include "sp_internal.cuh"

namespace sp {
namespace {

constexpr int kScanThreads = 1024;

// Warp per row: popcount of the row's mask bytes.
__global__ void row_count_kernel(int64_t R, int64_t C, const uint8_t *__restrict__ mask,
                                 int32_t *__restrict__ cnt) {
    const int lane = threadIdx.x & 31;
    const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (r >= R) return;
    const uint8_t *m = mask + r * C;
    int n = 0;
    for (int64_t c = lane; c < C; c += 32) n += m[c] != 0;
#pragma unroll
    for (int o = 16; o; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
    if (lane == 0) cnt[r] = n;
}

// Thread per column: count kept entries down the column (coalesced across
// threads: adjacent threads read adjacent bytes of each mask row).
__global__ void col_count_kernel(int64_t R, int64_t C, const uint8_t *__restrict__ mask,
                                 int32_t *__restrict__ cnt) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= C) return;
    int n = 0;
    for (int64_t r = 0; r < R; ++r) n += mask[r * C + c] != 0;
    cnt[c] = n;
}

// Single-block exclusive scan of n int32 counts into out[0..n] (out[n] = total)
// plus the max count.  Each thread owns a contiguous segment; fixed order.
__global__ void __launch_bounds__(kScanThreads) scan_kernel(int64_t n, const int32_t *__restrict__ in,
                                                            int32_t *__restrict__ out,
                                                            int64_t *__restrict__ info) {
    __shared__ int64_t sums[kScanThreads];
    __shared__ int32_t maxs[kScanThreads];
    const int t = threadIdx.x;
    const int64_t seg = (n + kScanThreads - 1) / kScanThreads;
    const int64_t lo = t * seg, hi = lo + seg < n ? lo + seg : n;
    int64_t s = 0;
    int32_t mx = 0;
    for (int64_t i = lo; i < hi; ++i) {
        s += in[i];
        mx = in[i] > mx ? in[i] : mx;
    }
    sums[t] = s;
    maxs[t] = mx;
    __syncthreads();
    if (t == 0) {
        int64_t run = 0;
        int32_t m = 0;
        for (int i = 0; i < kScanThreads; ++i) {
            int64_t v = sums[i];
            sums[i] = run;
            run += v;
            m = maxs[i] > m ? maxs[i] : m;
        }
        info[0] = run;
        info[1] = m;
    }
    __syncthreads();
    int64_t run = sums[t];
    for (int64_t i = lo; i < hi; ++i) {
        out[i] = (int32_t)run;  // total checked < 2^31 on the host before use
        run += in[i];
    }
    if (t == kScanThreads - 1) out[n] = (int32_t)run;
}

// Warp per row: stable compaction with ballots.  Writes col_idx, vals,
// row_of, and the CSR slot of every kept (r, c) into slot[r*C + c].
__global__ void csr_compact_kernel(int64_t R, int64_t C, const uint8_t *__restrict__ mask,
                                   const float *__restrict__ dense,
                                   const int32_t *__restrict__ row_ptr,
                                   int32_t *__restrict__ col_idx, float *__restrict__ vals,
                                   int32_t *__restrict__ row_of, int32_t *__restrict__ slot) {
    const int lane = threadIdx.x & 31;
    const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (r >= R) return;
    const uint8_t *m = mask + r * C;
    int32_t pos = row_ptr[r];
    for (int64_t c0 = 0; c0 < C; c0 += 32) {
        const int64_t c = c0 + lane;
        const bool keep = c < C && m[c] != 0;
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        if (keep) {
            const int32_t j = pos + __popc(bal & ((1u << lane) - 1u));
            col_idx[j] = (int32_t)c;
            vals[j] = dense[r * C + c];
            row_of[j] = (int32_t)r;
            slot[r * C + c] = j;
        }
        pos += __popc(bal);
    }
}

// Thread per column: rows ascending, perm = CSR slot of (r, c).
__global__ void csc_compact_kernel(int64_t R, int64_t C, const uint8_t *__restrict__ mask,
                                   const int32_t *__restrict__ slot,
                                   const int32_t *__restrict__ col_ptr,
                                   int32_t *__restrict__ row_idx, int32_t *__restrict__ perm) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= C) return;
    int32_t k = col_ptr[c];
    for (int64_t r = 0; r < R; ++r) {
        if (mask[r * C + c]) {
            row_idx[k] = (int32_t)r;
            perm[k] = slot[r * C + c];
            ++k;
        }
    }
}

__global__ void to_dense_kernel(int64_t nnz, int64_t C, const int32_t *__restrict__ row_of,
                                const int32_t *__restrict__ col_idx, const float *__restrict__ nz,
                                float *__restrict__ dense) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < nnz) dense[(int64_t)row_of[j] * C + col_idx[j]] = nz[j];
}

template <typename T>
cudaError_t dmalloc(T **p, int64_t n) {
    return cudaMalloc((void **)p, (size_t)(n > 0 ? n : 1) * sizeof(T));
}

}  // namespace

sp_status build_weight(int64_t R, int64_t C, const float *dense, const uint8_t *mask,
                       cudaStream_t st, sp_weight_s *w) {
    w->R = R;
    w->C = C;
    int32_t *rcnt = nullptr, *ccnt = nullptr, *slot = nullptr;
    int64_t *info = nullptr;
    cudaError_t e = cudaSuccess;
#define SP_TRY(x)                                   \
    do {                                            \
        e = (x);                                    \
        if (e != cudaSuccess) goto fail;            \
    } while (0)
    SP_TRY(cudaMallocAsync((void **)&rcnt, (size_t)R * sizeof(int32_t), st));
    SP_TRY(cudaMallocAsync((void **)&ccnt, (size_t)C * sizeof(int32_t), st));
    SP_TRY(cudaMallocAsync((void **)&info, 4 * sizeof(int64_t), st));
    SP_TRY(dmalloc(&w->row_ptr, R + 1));
    SP_TRY(dmalloc(&w->col_ptr, C + 1));
    {
        row_count_kernel<<<(unsigned)((R + 7) / 8), 256, 0, st>>>(R, C, mask, rcnt);
        col_count_kernel<<<(unsigned)((C + 255) / 256), 256, 0, st>>>(R, C, mask, ccnt);
        scan_kernel<<<1, kScanThreads, 0, st>>>(R, rcnt, w->row_ptr, info);
        scan_kernel<<<1, kScanThreads, 0, st>>>(C, ccnt, w->col_ptr, info + 2);
        SP_TRY(cudaGetLastError());
        int64_t h[4];
        SP_TRY(cudaMemcpyAsync(h, info, sizeof(h), cudaMemcpyDeviceToHost, st));
        SP_TRY(cudaStreamSynchronize(st));  // the one host sync of sp_weight_create
        if (h[0] != h[2]) {
            set_error("internal: row and column nnz totals differ");
            e = cudaErrorUnknown;
            goto fail;
        }
        if (h[0] > INT32_MAX - 1) {
            cudaFreeAsync(rcnt, st);
            cudaFreeAsync(ccnt, st);
            cudaFreeAsync(info, st);
            set_error("nnz does not fit int32");
            return SP_ERR_OVERFLOW;
        }
        w->nnz = h[0];
        w->max_row_nnz = (int32_t)h[1];
        w->max_col_nnz = (int32_t)h[3];
    }
    SP_TRY(dmalloc(&w->col_idx, w->nnz));
    SP_TRY(dmalloc(&w->vals, w->nnz));
    SP_TRY(dmalloc(&w->row_of, w->nnz));
    SP_TRY(dmalloc(&w->row_idx, w->nnz));
    SP_TRY(dmalloc(&w->perm, w->nnz));
    SP_TRY(cudaMallocAsync((void **)&slot, (size_t)(R * C) * sizeof(int32_t), st));
    csr_compact_kernel<<<(unsigned)((R + 7) / 8), 256, 0, st>>>(R, C, mask, dense, w->row_ptr,
                                                              w->col_idx, w->vals, w->row_of,
                                                              slot);
    csc_compact_kernel<<<(unsigned)((C + 127) / 128), 128, 0, st>>>(R, C, mask, slot, w->col_ptr,
                                                                   w->row_idx, w->perm);
    SP_TRY(cudaGetLastError());
    // Temporaries are freed in stream order (no second host sync).
    cudaFreeAsync(slot, st);
    cudaFreeAsync(rcnt, st);
    cudaFreeAsync(ccnt, st);
    cudaFreeAsync(info, st);
    return SP_OK;
fail:
    if (slot) cudaFreeAsync(slot, st);
    if (rcnt) cudaFreeAsync(rcnt, st);
    if (ccnt) cudaFreeAsync(ccnt, st);
    if (info) cudaFreeAsync(info, st);
    set_error(std::string("sp_weight_create: ") + cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? SP_ERR_ALLOC : SP_ERR_CUDA;
#undef SP_TRY
}

void launch_to_dense(const sp_weight_s *w, const float *nz, float *dense, cudaStream_t st) {
    count_launches(w->nnz > 0 ? 1 : 0);
    cudaMemsetAsync(dense, 0, (size_t)(w->R * w->C) * sizeof(float), st);
    if (w->nnz > 0)
        to_dense_kernel<<<(unsigned)((w->nnz + 255) / 256), 256, 0, st>>>(w->nnz, w->C, w->row_of,
                                                                          w->col_idx, nz, dense);
}

}  // namespace sp
