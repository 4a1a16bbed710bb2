// build.cu -- sp_weight_create on the device.
//
// From a dense R x C fp32 weight and an R x C uint8 mask, build
//   CSR (P153-P154): row_ptr, col_idx (ascending per row), vals, row_of
//   CSC index copy (P183): col_ptr, row_idx (ascending per column), perm
// deterministically (no atomics): counts -> exclusive scans -> stable
// compaction.  The structure is the mask.  Off the timed
// path (masks change "only a few times", P428).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
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

// Column counts by row blocks: thread (b, c) counts the kept entries of column
// c in rows [b*rbk, (b+1)*rbk) (coalesced: adjacent threads read adjacent bytes
// of each mask row).  blk[b*C + c] = that count.
__global__ void colblk_count_kernel(int64_t R, int64_t C, int64_t nb, int64_t rbk, const uint8_t *__restrict__ mask,
                                    int32_t *__restrict__ blk) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nb * C) return;
    const int64_t b = i / C, c = i - b * C;
    const int64_t r1 = min(R, (b + 1) * rbk);
    int n = 0;
    for (int64_t r = b * rbk; r < r1; ++r) n += mask[r * C + c] != 0;
    blk[i] = n;
}

// Thread per column: blk[.][c] -> exclusive prefix over the row blocks (fixed
// order), cnt[c] = the column's total.
__global__ void colblk_scan_kernel(int64_t C, int64_t nb, int32_t *__restrict__ blk, int32_t *__restrict__ cnt) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= C) return;
    int32_t run = 0;
    for (int64_t b = 0; b < nb; ++b) {
        const int32_t v = blk[b * C + c];
        blk[b * C + c] = run;
        run += v;
    }
    cnt[c] = run;
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

// Warp per row: stable compaction with ballots.  Writes col_idx, vals, row_of.
__global__ void csr_compact_kernel(int64_t R, int64_t C, const uint8_t *__restrict__ mask,
                                   const float *__restrict__ dense,
                                   const int32_t *__restrict__ row_ptr,
                                   int32_t *__restrict__ col_idx, float *__restrict__ vals,
                                   int32_t *__restrict__ row_of) {
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
        }
        pos += __popc(bal);
    }
}

// CSC compaction by row blocks: thread (b, c) writes column c's kept rows of
// block b (ascending) from position col_ptr[c] + blk[b][c]; perm = the CSR slot
// of (r, c), found by binary search of c in row r's (ascending) col_idx.  No
// R x C scratch: works for any R * C.
__global__ void csc_compact_kernel(int64_t R, int64_t C, int64_t nb, int64_t rbk, const uint8_t *__restrict__ mask,
                                   const int32_t *__restrict__ blk, const int32_t *__restrict__ col_ptr,
                                   const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ col_idx,
                                   int32_t *__restrict__ row_idx, int32_t *__restrict__ perm) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nb * C) return;
    const int64_t b = i / C, c = i - b * C;
    const int64_t r1 = min(R, (b + 1) * rbk);
    int32_t k = col_ptr[c] + blk[i];
    for (int64_t r = b * rbk; r < r1; ++r) {
        if (mask[r * C + c]) {
            int32_t lo = row_ptr[r], hi = row_ptr[r + 1] - 1;  // c is in [lo, hi]
            while (lo < hi) {
                const int32_t mid = (lo + hi) >> 1;
                if (col_idx[mid] < (int32_t)c) lo = mid + 1;
                else hi = mid;
            }
            row_idx[k] = (int32_t)r;
            perm[k] = lo;
            ++k;
        }
    }
}

__global__ void gather_dense_kernel(int64_t nnz, int64_t C, const int32_t *__restrict__ row_of,
                                    const int32_t *__restrict__ col_idx, const float *__restrict__ dense,
                                    float *__restrict__ nz) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < nnz) nz[j] = dense[(int64_t)row_of[j] * C + col_idx[j]];
}

__global__ void chunk_count_kernel(int64_t R, const int32_t *__restrict__ row_ptr, int32_t *__restrict__ cnt) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r < R) cnt[r] = (row_ptr[r + 1] - row_ptr[r] + 31) >> 5;
}

__global__ void to_dense_kernel(int64_t nnz, int64_t C, const int32_t *__restrict__ row_of,
                                const int32_t *__restrict__ col_idx, const float *__restrict__ nz,
                                float *__restrict__ dense) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < nnz) dense[(int64_t)row_of[j] * C + col_idx[j]] = nz[j];
}

// ---- tilings ----
__device__ __forceinline__ int lower_bound_i32(const int32_t *a, int lo, int hi, int key) {
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// thread per (row, column block): entries of the row inside the block
__global__ void til_count_kernel(int64_t rows, int nkb, int KC, int RB, const int32_t *__restrict__ ptr,
                                 const int32_t *__restrict__ idx, const int32_t *__restrict__ rowpos,
                                 int32_t *__restrict__ cnt) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (tid >= rows * nkb) return;
    const int64_t r = tid / nkb;
    const int kb = (int)(tid - r * nkb);
    const int lo = lower_bound_i32(idx, ptr[r], ptr[r + 1], kb * KC);
    const int hi = lower_bound_i32(idx, lo, ptr[r + 1], (kb + 1) * KC);
    const int64_t pos = rowpos[r], rb = pos / RB, lr = pos - rb * RB;
    cnt[(rb * nkb + kb) * RB + lr] = (hi - lo + kTilPad - 1) & ~(kTilPad - 1);  // padded segment
}

__global__ void til_fill_kernel(int64_t rows, int nkb, int KC, int RB, const int32_t *__restrict__ ptr,
                                const int32_t *__restrict__ idx, const int32_t *__restrict__ slotmap,
                                const int32_t *__restrict__ rowpos, const int32_t *__restrict__ seg,
                                const float *__restrict__ vals, int2 *__restrict__ ent, int32_t *__restrict__ vidx) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (tid >= rows * nkb) return;
    const int64_t r = tid / nkb;
    const int kb = (int)(tid - r * nkb);
    const int lo = lower_bound_i32(idx, ptr[r], ptr[r + 1], kb * KC);
    const int hi = lower_bound_i32(idx, lo, ptr[r + 1], (kb + 1) * KC);
    const int64_t pos = rowpos[r], rb = pos / RB, lr = pos - rb * RB;
    int e = seg[(rb * nkb + kb) * RB + lr];
    for (int t = lo; t < hi; ++t, ++e) {
        const int slot = slotmap ? slotmap[t] : t;
        ent[e] = make_int2((idx[t] - kb * KC) * kTilRowBytes, __float_as_int(vals[slot]));
        vidx[e] = slot;
    }
    const int pad = ((hi - lo + kTilPad - 1) & ~(kTilPad - 1)) - (hi - lo);
    for (int t = 0; t < pad; ++t, ++e) {  // padding: offset -kTilRowBytes (zero row / no load), weight 0, no slot
        ent[e] = make_int2(-kTilRowBytes, 0);
        vidx[e] = -1;
    }
}

// tmsplit[s] for every segment: the first entry whose column lies in the
// tile's last kHybTC rows, rounded up to an even index (the pair that straddles
// stays in the shared-memory part), else the segment end.  Padding entries
// (offset < 0) come last in a segment and never start the TMEM part.
__global__ void til_split_kernel(int64_t nseg, int KC, const int32_t *__restrict__ seg, const int2 *__restrict__ ent,
                                 int32_t *__restrict__ split) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nseg) return;
    const int s0 = seg[s], s1 = seg[s + 1];
    const int off0 = (KC - kHybTC) * kTilRowBytes;
    int sp = s1;
    for (int e = s0; e < s1; ++e)
        if (ent[e].x >= off0) {
            sp = e;
            break;
        }
    sp = s0 + ((sp - s0 + 1) & ~1);
    split[s] = sp < s1 ? sp : s1;
}

// inv[vidx[e]] = e over a tiling's (padded) entries: slot -> entry position
__global__ void til_inv_kernel(int64_t cap, const int32_t *__restrict__ vidx, int32_t *__restrict__ inv) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < cap) {
        const int32_t v = vidx[e];
        if (v >= 0) inv[v] = (int32_t)e;
    }
}

// managed SGD: thread per CSR slot, new value to vals and to every tiling
__global__ void weight_sgd_kernel(int64_t nnz, float *__restrict__ vals, const float *__restrict__ dW, float lr,
                                  const SgdRef *__restrict__ tab, int ntab) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= nnz) return;
    const float v = fmaf(-lr, dW[j], vals[j]);  // the same rounding as sp_sgd
    vals[j] = v;
    for (int k = 0; k < ntab; ++k) tab[k].ent[tab[k].inv[j]].y = __float_as_int(v);
}

// max over tiles of the tile's entry count (single block, fixed order)
__global__ void til_max_kernel(int64_t ntiles, int RB, const int32_t *__restrict__ seg, int64_t *__restrict__ out) {
    __shared__ int32_t sh[256];
    int32_t m = 0;
    for (int64_t t = threadIdx.x; t < ntiles; t += blockDim.x) m = max(m, seg[(t + 1) * RB] - seg[t * RB]);
    sh[threadIdx.x] = m;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) sh[threadIdx.x] = max(sh[threadIdx.x], sh[threadIdx.x + o]);
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = sh[0];
}

// max over (row block, warp) of the warp's entry groups (segments walked in
// groups of 4 entries, a last group may hold 2) summed over all column blocks
// (rows rb*RB + w*RPW .. +RPW), single block, fixed order.  Bounds the
// per-warp dW sum columns of the TMEM fused backward (8 groups per column).
__global__ void til_warp_max_kernel(int nrb, int nkb, int RB, int RPW, int GL, const int32_t *__restrict__ seg,
                                    int64_t *__restrict__ out) {
    __shared__ int32_t sh[256];
    const int nw = RB / RPW;
    int32_t m = 0;
    for (int i = threadIdx.x; i < nrb * nw; i += blockDim.x) {
        const int rb = i / nw, wi = i - rb * nw;
        int32_t s = 0;
        for (int kb = 0; kb < nkb; ++kb) {
            const int64_t t = ((int64_t)rb * nkb + kb) * RB + (int64_t)wi * RPW;
            for (int r = 0; r < RPW; ++r) s += (seg[t + r + 1] - seg[t + r] + (1 << GL) - 1) >> GL;
        }
        m = max(m, s);
    }
    sh[threadIdx.x] = m;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) sh[threadIdx.x] = max(sh[threadIdx.x], sh[threadIdx.x + o]);
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = sh[0];
}

// gpre (see sp_tiling): thread per (row block, warp); prefix of the warp's
// groups of 2^GL entries over the column blocks.
__global__ void til_gpre_kernel(int nrb, int nkb, int RB, int RPW, int GL, const int32_t *__restrict__ seg,
                                int32_t *__restrict__ out) {
    const int nw = RB / RPW;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nrb * nw) return;
    const int rb = i / nw, wi = i - rb * nw;
    int32_t s = 0;
    int32_t *o = out + (int64_t)i * (nkb + 1);
    for (int kb = 0; kb < nkb; ++kb) {
        o[kb] = s;
        const int64_t t = ((int64_t)rb * nkb + kb) * RB + (int64_t)wi * RPW;
        for (int r = 0; r < RPW; ++r) s += (seg[t + r + 1] - seg[t + r] + (1 << GL) - 1) >> GL;
    }
    o[nkb] = s;
}

__global__ void til_refresh_kernel(int64_t nnz, const int32_t *__restrict__ vidx, const float *__restrict__ vals,
                                   int2 *__restrict__ ent) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < nnz) {
        const int v = __ldg(vidx + e);
        if (v >= 0) ent[e].y = __float_as_int(__ldg(vals + v));
    }
}


// Bump allocator over one device allocation (256-byte aligned pieces).
struct Arena {
    char *base = nullptr;
    size_t off = 0, cap = 0;
    static size_t al(size_t n) { return (n + 255) & ~(size_t)255; }
    template <typename T>
    T *take(int64_t n) {
        T *p = reinterpret_cast<T *>(base + off);
        off += al((size_t)(n > 0 ? n : 1) * sizeof(T));
        return p;
    }
};
template <typename T>
size_t asize(int64_t n) {
    return Arena::al((size_t)(n > 0 ? n : 1) * sizeof(T));
}

}  // namespace

void free_weight(sp_weight_s *w) {
    for (auto &a : w->arena) {
        cudaFree(a);
        a = nullptr;
    }
    w->row_ptr = w->col_ptr = w->col_idx = w->row_of = w->row_idx = w->perm = w->chunk_ptr = nullptr;
    w->vals = nullptr;
    free_tilings(w);
}

sp_status build_weight(int64_t R, int64_t C, const float *dense, const uint8_t *mask,
                       cudaStream_t st, sp_weight_s *w) {
    w->R = R;
    w->C = C;
    int32_t *rcnt = nullptr, *ccnt = nullptr, *blk = nullptr;
    // column counts / CSC compaction by row blocks: about 256k (block, column) threads
    const int64_t nb = std::max<int64_t>(1, std::min<int64_t>(R, (262144 + C - 1) / C));
    const int64_t rbk = (R + nb - 1) / nb;
    int64_t *info = nullptr;
    cudaError_t e = cudaSuccess;
#define SP_TRY(x)                                   \
    do {                                            \
        e = (x);                                    \
        if (e != cudaSuccess) goto fail;            \
    } while (0)
    SP_TRY(scratch_alloc((void **)&rcnt, (size_t)R * sizeof(int32_t), st));
    SP_TRY(scratch_alloc((void **)&ccnt, (size_t)C * sizeof(int32_t), st));
    SP_TRY(scratch_alloc((void **)&info, 4 * sizeof(int64_t), st));
    SP_TRY(scratch_alloc((void **)&blk, (size_t)(nb * C) * sizeof(int32_t), st));
    {
        Arena a;
        SP_TRY(cudaMalloc((void **)&a.base, asize<int32_t>(R + 1) + asize<int32_t>(C + 1)));
        w->arena[0] = a.base;
        w->row_ptr = a.take<int32_t>(R + 1);
        w->col_ptr = a.take<int32_t>(C + 1);
    }
    {
        row_count_kernel<<<(unsigned)((R + 7) / 8), 256, 0, st>>>(R, C, mask, rcnt);
        colblk_count_kernel<<<(unsigned)((nb * C + 255) / 256), 256, 0, st>>>(R, C, nb, rbk, mask, blk);
        colblk_scan_kernel<<<(unsigned)((C + 255) / 256), 256, 0, st>>>(C, nb, blk, ccnt);
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
            scratch_free(rcnt, st);
            scratch_free(ccnt, st);
            scratch_free(info, st);
            scratch_free(blk, st);
            set_error("nnz does not fit int32");
            return SP_ERR_OVERFLOW;
        }
        w->nnz = h[0];
        w->max_row_nnz = (int32_t)h[1];
        w->max_col_nnz = (int32_t)h[3];
    }
    {
        Arena a;
        SP_TRY(cudaMalloc((void **)&a.base, 5 * asize<int32_t>(w->nnz) + asize<int32_t>(R + 1)));
        w->arena[1] = a.base;
        w->col_idx = a.take<int32_t>(w->nnz);
        w->vals = a.take<float>(w->nnz);
        w->row_of = a.take<int32_t>(w->nnz);
        w->row_idx = a.take<int32_t>(w->nnz);
        w->perm = a.take<int32_t>(w->nnz);
        w->chunk_ptr = a.take<int32_t>(R + 1);
    }
    csr_compact_kernel<<<(unsigned)((R + 7) / 8), 256, 0, st>>>(R, C, mask, dense, w->row_ptr,
                                                              w->col_idx, w->vals, w->row_of);
    csc_compact_kernel<<<(unsigned)((nb * C + 255) / 256), 256, 0, st>>>(R, C, nb, rbk, mask, blk, w->col_ptr,
                                                                       w->row_ptr, w->col_idx, w->row_idx,
                                                                       w->perm);
    SP_TRY(cudaGetLastError());
    // gather-SDDMM work list: chunks of <= 32 consecutive nonzeros of one row
    chunk_count_kernel<<<(unsigned)((R + 255) / 256), 256, 0, st>>>(R, w->row_ptr, rcnt);
    scan_kernel<<<1, kScanThreads, 0, st>>>(R, rcnt, w->chunk_ptr, info);
    {
        const sp_status ts = build_tilings(w, st);
        if (ts != SP_OK) {
            set_error("sp_weight_create: tiling build failed");
            scratch_free(blk, st);
            scratch_free(rcnt, st);
            scratch_free(ccnt, st);
            scratch_free(info, st);
            return ts;
        }
    }
    // Temporaries are freed in stream order (no second host sync).
    scratch_free(blk, st);
    scratch_free(rcnt, st);
    scratch_free(ccnt, st);
    scratch_free(info, st);
    return SP_OK;
fail:
    if (blk) scratch_free(blk, st);
    if (rcnt) scratch_free(rcnt, st);
    if (ccnt) scratch_free(ccnt, st);
    if (info) scratch_free(info, st);
    set_error(std::string("sp_weight_create: ") + cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? SP_ERR_ALLOC : SP_ERR_CUDA;
#undef SP_TRY
}

// nnz-balanced placement of rows into tiled positions (SURVEY §7 "nnz-balanced
// scheduling"): rows sorted by length are dealt in snake order over the row
// blocks, and within a block round-robin (snake) over the NW warps, so every
// CTA and every warp gets a similar share of heavy and light rows (Zipf masks).
// rowpos[r] = tiled position, rowmap[pos] = r (or -1 for unused positions).
static void balanced_rows(const std::vector<int32_t> &ptr, int64_t rows, int RB, int NW, std::vector<int32_t> &rowpos,
                          std::vector<int32_t> &rowmap) {
    const int64_t nrb = (rows + RB - 1) / RB;
    const int RPW = RB / NW;
    std::vector<int32_t> order(rows);
    for (int64_t r = 0; r < rows; ++r) order[r] = (int32_t)r;
    std::stable_sort(order.begin(), order.end(),
                     [&](int32_t a, int32_t b) { return ptr[a + 1] - ptr[a] > ptr[b + 1] - ptr[b]; });
    rowpos.assign(rows, 0);
    rowmap.assign(nrb * RB, -1);
    std::vector<int32_t> used(nrb, 0);
    int64_t k = 0;
    for (int64_t round = 0; k < rows; ++round) {
        for (int64_t j = 0; j < nrb && k < rows; ++j) {
            const int64_t blk = (round & 1) ? nrb - 1 - j : j;
            if (used[blk] >= RB) continue;
            const int s = used[blk]++;
            const int wr = s / NW, wi = (wr & 1) ? NW - 1 - (s % NW) : s % NW;  // snake over warps
            const int64_t pos = blk * RB + (int64_t)wi * RPW + wr;
            rowpos[order[k]] = (int32_t)pos;
            rowmap[pos] = order[k];
            ++k;
        }
    }
}

sp_status build_tilings(sp_weight_s *w, cudaStream_t st) {
    // host copies of the row / column pointers for the balanced placement
    std::vector<int32_t> hptr[2];
    hptr[0].resize(w->R + 1);
    hptr[1].resize(w->C + 1);
    cudaStreamSynchronize(st);
    cudaMemcpy(hptr[0].data(), w->row_ptr, (w->R + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost);
    cudaMemcpy(hptr[1].data(), w->col_ptr, (w->C + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost);
    // the tilings: [orientation][variant] plus the CSC tilings of the fused
    // backward's smaller row blocks (64 and 32 rows, 32 warps x 2 / 1 rows)
    struct Spec {
        int o, RB, KC, NWbal, RPWgrp;
        sp_tiling *t;
    };
    const Spec specs[] = {{0, kTilRB[0], kTilKC[0], kTilNW[0], 4, &w->til[0][0]},
                          {0, kTilRB[1], kTilKC[1], kTilNW[1], kTilRB[1] / kTilNW[1], &w->til[0][1]},
                          {1, kTilRB[0], kTilKC[0], kTilNW[0], 4, &w->til[1][0]},
                          {1, kTilRB[1], kTilKC[1], kTilNW[1], kTilRB[1] / kTilNW[1], &w->til[1][1]},
                          {1, 64, kTilKC[0], 32, 2, &w->til_f[0]},
                          {1, 32, kTilKC[0], 32, 1, &w->til_f[1]},
                          {1, 64, kTilKC[0], 16, 4, &w->til_f[2]}};
    constexpr int NS = sizeof(specs) / sizeof(specs[0]);
    // ---- plan: every tiling's geometry and buffer sizes, then ONE device
    // allocation (the tiling arena) and ONE host -> device copy of the host-built
    // row placements and the managed-SGD table
    struct Plan {
        int64_t rows, inner, nseg, cap, nwg;
    } pl[NS];
    size_t bytes = 0, hbytes = 0;  // arena total; the host-filled region
    for (int si = 0; si < NS; ++si) {
        const Spec &sp_ = specs[si];
        sp_tiling &t = *sp_.t;
        const int o = sp_.o;
        Plan &P = pl[si];
        P.rows = o == 0 ? w->R : w->C;
        P.inner = o == 0 ? w->C : w->R;
        t.RB = sp_.RB;
        t.KC = sp_.KC;
        t.rows = P.rows;
        t.inner = P.inner;
        t.nrb = (int)((P.rows + t.RB - 1) / t.RB);
        t.nkb = (int)((P.inner + t.KC - 1) / t.KC);
        P.nseg = (int64_t)t.nrb * t.nkb * t.RB;
        // upper bound on the padded entry count (each segment pads < kTilPad)
        P.cap = w->nnz + (kTilPad - 1) * std::min<int64_t>(P.nseg, w->nnz) + 8;
        P.nwg = t.RB / sp_.RPWgrp;
        hbytes += asize<int32_t>(P.rows) + asize<int32_t>((int64_t)t.nrb * t.RB);
        bytes += asize<int32_t>(P.nseg + 8) + asize<int2>(P.cap) + asize<int32_t>(P.cap);
        if (w->nnz > 0) bytes += asize<int32_t>(w->nnz);
        if (si == 0 || si == 2) bytes += asize<int32_t>(P.nseg + 8);
        if (o == 1) bytes += 2 * asize<int32_t>((int64_t)t.nrb * P.nwg * (t.nkb + 1));
    }
    hbytes += asize<SgdRef>(NS);
    Arena ar;
    if (cudaMalloc((void **)&ar.base, bytes + hbytes) != cudaSuccess) return SP_ERR_ALLOC;
    w->arena[2] = ar.base;
    // host-filled region first (rowpos / rowmap of every tiling, the SGD table)
    std::vector<char> hreg(hbytes, 0);
    for (int si = 0; si < NS; ++si) {
        sp_tiling &t = *specs[si].t;
        t.in_arena = true;
        const size_t o1 = ar.off;
        t.rowpos = ar.take<int32_t>(pl[si].rows);
        const size_t o2 = ar.off;
        t.rowmap = ar.take<int32_t>((int64_t)t.nrb * t.RB);
        std::vector<int32_t> rowpos, rowmap;
        balanced_rows(hptr[specs[si].o], pl[si].rows, t.RB, specs[si].NWbal, rowpos, rowmap);
        memcpy(hreg.data() + o1, rowpos.data(), rowpos.size() * sizeof(int32_t));
        memcpy(hreg.data() + o2, rowmap.data(), rowmap.size() * sizeof(int32_t));
    }
    const size_t otab = ar.off;
    w->sgdtab = ar.take<SgdRef>(NS);
    for (int si = 0; si < NS; ++si) {
        sp_tiling &t = *specs[si].t;
        const Plan &P = pl[si];
        t.seg = ar.take<int32_t>(P.nseg + 8);
        t.ent = ar.take<int2>(P.cap);
        t.vidx = ar.take<int32_t>(P.cap);
        t.cap_ent = P.cap;
        if (w->nnz > 0) t.inv = ar.take<int32_t>(w->nnz);
        if (si == 0 || si == 2) t.tmsplit = ar.take<int32_t>(P.nseg + 8);
        if (specs[si].o == 1)
            for (int g = 0; g < 2; ++g) t.gpre[g] = ar.take<int32_t>((int64_t)t.nrb * P.nwg * (t.nkb + 1));
    }
    {
        std::vector<SgdRef> tab;
        for (int si = 0; si < NS; ++si)
            if (specs[si].t->inv) tab.push_back({specs[si].t->ent, specs[si].t->inv});
        w->nsgd = (int)tab.size();
        memcpy(hreg.data() + otab, tab.data(), tab.size() * sizeof(SgdRef));
    }
    cudaMemcpyAsync(ar.base, hreg.data(), hbytes, cudaMemcpyHostToDevice, st);

    int64_t *info = nullptr, *mx = nullptr;
    if (scratch_alloc((void **)&info, 2 * NS * sizeof(int64_t), st) != cudaSuccess) return SP_ERR_ALLOC;
    if (scratch_alloc((void **)&mx, 3 * NS * sizeof(int64_t), st) != cudaSuccess) return SP_ERR_ALLOC;
    for (int si = 0; si < NS; ++si) {
        const Spec &sp_ = specs[si];
        const int o = sp_.o;
        const int64_t rows = pl[si].rows;
        const int32_t *ptr = o == 0 ? w->row_ptr : w->col_ptr;
        const int32_t *idx = o == 0 ? w->col_idx : w->row_idx;
        const int32_t *slotmap = o == 0 ? nullptr : w->perm;
        sp_tiling &t = *sp_.t;
        const int64_t nseg = pl[si].nseg, cap = pl[si].cap;
        int32_t *cnt = nullptr;
        if (scratch_alloc((void **)&cnt, (size_t)nseg * sizeof(int32_t), st) != cudaSuccess) {
            scratch_free(info, st);
            scratch_free(mx, st);
            return SP_ERR_ALLOC;
        }
        cudaMemsetAsync(cnt, 0, (size_t)nseg * sizeof(int32_t), st);
        cudaMemsetAsync(t.seg + nseg + 1, 0, 7 * sizeof(int32_t), st);  // slack for 16-byte bulk copies of bounds
        cudaMemsetAsync(t.ent, 0, (size_t)cap * sizeof(int2), st);
        cudaMemsetAsync(t.vidx, 0xff, (size_t)cap * sizeof(int32_t), st);  // -1: no slot
        const int64_t nt = rows * t.nkb;
        til_count_kernel<<<(unsigned)((nt + 255) / 256), 256, 0, st>>>(rows, t.nkb, t.KC, t.RB, ptr, idx, t.rowpos,
                                                                      cnt);
        scan_kernel<<<1, kScanThreads, 0, st>>>(nseg, cnt, t.seg, info + 2 * si);
        til_fill_kernel<<<(unsigned)((nt + 255) / 256), 256, 0, st>>>(rows, t.nkb, t.KC, t.RB, ptr, idx, slotmap,
                                                                     t.rowpos, t.seg, w->vals, t.ent, t.vidx);
        til_max_kernel<<<1, 256, 0, st>>>((int64_t)t.nrb * t.nkb, t.RB, t.seg, mx + si);
        if (w->nnz > 0) til_inv_kernel<<<(unsigned)((cap + 255) / 256), 256, 0, st>>>(cap, t.vidx, t.inv);
        t.fresh = 1;  // built from vals: the handle's first version
        if (t.tmsplit)  // the big tilings (RB = 128, KC = 192): split-source SpMM
            til_split_kernel<<<(unsigned)((nseg + 255) / 256), 256, 0, st>>>(nseg, t.KC, t.seg, t.ent, t.tmsplit);
        if (o == 1) {  // group prefix tables of the fused backward (groups of 4 and of 8)
            const int nwg = (int)pl[si].nwg;
            t.RPWg = sp_.RPWgrp;
            for (int g = 0; g < 2; ++g)
                til_gpre_kernel<<<(unsigned)((t.nrb * nwg + 127) / 128), 128, 0, st>>>(t.nrb, t.nkb, t.RB, sp_.RPWgrp,
                                                                                         2 + g, t.seg, t.gpre[g]);
        }
        til_warp_max_kernel<<<1, 256, 0, st>>>(t.nrb, t.nkb, t.RB, sp_.RPWgrp, 2, t.seg, mx + NS + si);
        til_warp_max_kernel<<<1, 256, 0, st>>>(t.nrb, t.nkb, t.RB, sp_.RPWgrp, 3, t.seg, mx + 2 * NS + si);
        scratch_free(cnt, st);
    }
    std::vector<int64_t> h(3 * NS), hi(2 * NS);
    cudaMemcpyAsync(h.data(), mx, h.size() * sizeof(int64_t), cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(hi.data(), info, hi.size() * sizeof(int64_t), cudaMemcpyDeviceToHost, st);
    const cudaError_t e = cudaStreamSynchronize(st);  // last host sync of sp_weight_create
    for (int si = 0; si < NS; ++si) {
        sp_tiling &t = *specs[si].t;
        t.max_tile = (int32_t)h[si];
        t.max_warp_groups = h[NS + si];
        t.max_warp_groups8 = h[2 * NS + si];
        t.npad = hi[2 * si];  // padded entry total
    }
    scratch_free(info, st);
    scratch_free(mx, st);
    w->version = 1;
    return (e == cudaSuccess && cudaGetLastError() == cudaSuccess) ? SP_OK : SP_ERR_CUDA;
}

void free_tilings(sp_weight_s *w) {
    auto fr = [](sp_tiling &t) {
        if (t.in_arena) {  // the buffers belong to the tiling arena (freed by free_weight)
            t = sp_tiling{};
            return;
        }
        cudaFree(t.seg);
        cudaFree(t.ent);
        cudaFree(t.vidx);
        cudaFree(t.rowpos);
        cudaFree(t.rowmap);
        cudaFree(t.tmsplit);
        t.tmsplit = nullptr;
        cudaFree(t.inv);
        t.inv = nullptr;
        for (auto &g : t.gpre) {
            cudaFree(g);
            g = nullptr;
        }
        t.seg = nullptr;
        t.ent = nullptr;
        t.vidx = nullptr;
        t.rowpos = nullptr;
        t.rowmap = nullptr;
    };
    for (auto &o : w->til)
        for (auto &t : o) fr(t);
    for (auto &o : w->tap)
        for (auto &t : o) fr(t);
    for (auto &t : w->tapf) fr(t);
    for (auto &t : w->til_f) fr(t);

    if (w->tapdev) cudaFree(w->tapdev);
    w->tapdev = nullptr;
    w->sgdtab = nullptr;  // lives in the tiling arena
    w->nsgd = 0;
}

void refresh_if_stale(const sp_weight_s *w, const sp_tiling &t, cudaStream_t st) {
    if (w->managed && t.fresh == w->version) return;
    launch_refresh(t, w->vals, w->nnz, st);
    t.fresh = w->version;
}

void launch_weight_sgd(sp_weight_s *w, const float *dW, float lr, cudaStream_t st) {
    if (w->nnz > 0) {
        count_launches(1);
        weight_sgd_kernel<<<(unsigned)((w->nnz + 255) / 256), 256, 0, st>>>(w->nnz, w->vals, dW, lr, w->sgdtab,
                                                                            w->nsgd);
    }
    ++w->version;  // vals changed; the tilings in the table hold the new values
    auto mark = [&](sp_tiling &t) {
        if (t.inv) t.fresh = w->version;
    };
    for (auto &o : w->til)
        for (auto &t : o) mark(t);
    for (auto &t : w->til_f) mark(t);

}

void launch_refresh(const sp_tiling &t, const float *vals, int64_t nnz, cudaStream_t st) {
    if (nnz > 0) {
        count_launches(1);
        til_refresh_kernel<<<(unsigned)((t.npad + 255) / 256), 256, 0, st>>>(t.npad, t.vidx, vals, t.ent);
    }
}

// ent[e].y = vals[vidx[e]] for every tap tiling of one orientation (grid.y = tap)
__global__ void til_refresh_taps_kernel(const TapDev *__restrict__ taps, const float *__restrict__ vals) {
    const TapDev t = taps[blockIdx.y];
    int2 *ent = const_cast<int2 *>(t.ent);
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < t.npad; e += (int64_t)gridDim.x * blockDim.x) {
        const int v = __ldg(t.vidx + e);
        if (v >= 0) ent[e].y = __float_as_int(__ldg(vals + v));
    }
}

void launch_refresh_taps(const sp_weight_s *w, int orient, int ntap, cudaStream_t st) {
    count_launches(1);
    til_refresh_taps_kernel<<<dim3(64, ntap), 256, 0, st>>>(w->tapdev + orient * kMaxTaps, w->vals);
}

void launch_gather_dense(const sp_weight_s *w, const float *dense, float *nz, cudaStream_t st) {
    if (w->nnz > 0) {
        count_launches(1);
        gather_dense_kernel<<<(unsigned)((w->nnz + 255) / 256), 256, 0, st>>>(w->nnz, w->C, w->row_of, w->col_idx,
                                                                              dense, nz);
    }
}

void launch_to_dense(const sp_weight_s *w, const float *nz, float *dense, cudaStream_t st) {
    count_launches(w->nnz > 0 ? 1 : 0);
    cudaMemsetAsync(dense, 0, (size_t)(w->R * w->C) * sizeof(float), st);
    if (w->nnz > 0)
        to_dense_kernel<<<(unsigned)((w->nnz + 255) / 256), 256, 0, st>>>(w->nnz, w->C, w->row_of,
                                                                          w->col_idx, nz, dense);
}

}  // namespace sp
