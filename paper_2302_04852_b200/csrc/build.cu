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

// Exclusive scan of n int32 counts into out[0..n] (out[n] = total) plus the
// total and the max count (info[0], info[1]), in three coalesced passes over
// 4096-element chunks: chunk sums / maxima, a one-block scan of the chunk sums,
// then each chunk's block scan plus its offset.  Fixed order (deterministic).
constexpr int kScanChunk = 4 * kScanThreads;

__device__ __forceinline__ void chunk_load(int64_t n, const int32_t *__restrict__ in, int64_t c0, int32_t (&v)[4]) {
    const int64_t i0 = c0 + 4 * (int64_t)threadIdx.x;
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = i0 + k < n ? in[i0 + k] : 0;
}

__global__ void __launch_bounds__(kScanThreads) scan_chunks_kernel(int64_t n, const int32_t *__restrict__ in,
                                                                   int64_t *__restrict__ csum,
                                                                   int32_t *__restrict__ cmax) {
    __shared__ int64_t ws[32];
    __shared__ int32_t wm[32];
    int32_t v[4];
    chunk_load(n, in, (int64_t)blockIdx.x * kScanChunk, v);
    int64_t sm = (int64_t)v[0] + v[1] + v[2] + v[3];
    int32_t mx = max(max(v[0], v[1]), max(v[2], v[3]));
    for (int o = 16; o; o >>= 1) {
        sm += __shfl_xor_sync(0xffffffffu, sm, o);
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    if (lane == 0) {
        ws[wp] = sm;
        wm[wp] = mx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t t = 0;
        int32_t m = 0;
        for (int i = 0; i < kScanThreads / 32; ++i) {
            t += ws[i];
            m = max(m, wm[i]);
        }
        csum[blockIdx.x] = t;
        cmax[blockIdx.x] = m;
    }
}

__global__ void scan_top_kernel(int64_t nc, int64_t *__restrict__ csum, const int32_t *__restrict__ cmax,
                                int64_t *__restrict__ info) {
    int64_t run = 0;
    int32_t m = 0;
    for (int64_t c = 0; c < nc; ++c) {
        const int64_t v = csum[c];
        csum[c] = run;
        run += v;
        m = max(m, cmax[c]);
    }
    info[0] = run;
    info[1] = m;
}

__global__ void __launch_bounds__(kScanThreads) scan_apply_kernel(int64_t n, const int32_t *__restrict__ in,
                                                                  const int64_t *__restrict__ coff,
                                                                  const int64_t *__restrict__ info,
                                                                  int32_t *__restrict__ out) {
    __shared__ int64_t ws[32];
    int32_t v[4];
    const int64_t c0 = (int64_t)blockIdx.x * kScanChunk;
    chunk_load(n, in, c0, v);
    const int64_t ts = (int64_t)v[0] + v[1] + v[2] + v[3];
    int64_t inc = ts;  // inclusive warp scan of the thread sums
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) ws[wp] = inc;
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t run = 0;
        for (int i = 0; i < kScanThreads / 32; ++i) {
            const int64_t y = ws[i];
            ws[i] = run;
            run += y;
        }
    }
    __syncthreads();
    int64_t run = coff[blockIdx.x] + ws[wp] + inc - ts;  // exclusive prefix of this thread's first element
    const int64_t i0 = c0 + 4 * (int64_t)threadIdx.x;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if (i0 + k < n) out[i0 + k] = (int32_t)run;  // total checked < 2^31 on the host before use
        run += v[k];
    }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) out[n] = (int32_t)info[0];
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
                                  const SgdRef *__restrict__ tab, int ntab, uint32_t mask) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= nnz) return;
    const float v = fmaf(-lr, dW[j], vals[j]);  // the same rounding as sp_sgd
    vals[j] = v;
    for (int k = 0; k < ntab; ++k)
        if ((mask >> k) & 1u) tab[k].ent[tab[k].inv[j]].y = __float_as_int(v);
}

// max over tiles of the tile's entry count (single block, fixed order)
__global__ void til_max_kernel(int64_t ntiles, int RB, const int32_t *__restrict__ seg,
                               unsigned long long *__restrict__ out) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int32_t m = t < ntiles ? seg[(t + 1) * RB] - seg[t * RB] : 0;
    for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m > 0) atomicMax(out, (unsigned long long)m);  // integer max: order-free
}

// per (row block, warp of RPW rows): its entry groups of 4 and of 8 summed
// over all column blocks -- the maxima bound the per-warp TMEM dW columns of
// the fused backward (out[0]: groups of 4, out[1]: groups of 8) -- and, when
// gpre is given, the prefix tables of both (sp_tiling::gpre).  Thread per
// (row block, warp); maxima by integer atomicMax (order-free).
__global__ void til_warp_groups_kernel(int nrb, int nkb, int RB, int RPW, const int32_t *__restrict__ seg,
                                       unsigned long long *__restrict__ mx4, unsigned long long *__restrict__ mx8,
                                       int32_t *__restrict__ gpre4, int32_t *__restrict__ gpre8) {
    const int nw = RB / RPW;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    int32_t s4 = 0, s8 = 0;
    if (i < nrb * nw) {
        const int rb = i / nw, wi = i - rb * nw;
        const int64_t g0 = (int64_t)i * (nkb + 1);
        for (int kb = 0; kb < nkb; ++kb) {
            if (gpre4) {
                gpre4[g0 + kb] = s4;
                gpre8[g0 + kb] = s8;
            }
            const int64_t t = ((int64_t)rb * nkb + kb) * RB + (int64_t)wi * RPW;
            for (int r = 0; r < RPW; ++r) {
                const int32_t len = seg[t + r + 1] - seg[t + r];
                s4 += (len + 3) >> 2;
                s8 += (len + 7) >> 3;
            }
        }
        if (gpre4) {
            gpre4[g0 + nkb] = s4;
            gpre8[g0 + nkb] = s8;
        }
    }
    for (int o = 16; o; o >>= 1) {
        s4 = max(s4, __shfl_xor_sync(0xffffffffu, s4, o));
        s8 = max(s8, __shfl_xor_sync(0xffffffffu, s8, o));
    }
    if ((threadIdx.x & 31) == 0) {
        if (s4 > 0) atomicMax(mx4, (unsigned long long)s4);
        if (s8 > 0) atomicMax(mx8, (unsigned long long)s8);
    }
}

// Virtual CSR of the forward tilings with split rows: CSR slot j = the t-th
// entry of row r goes to part row vbase[r] + t % kp[r], position t / kp[r] of
// it (columns stay ascending in every part row).
__global__ void vcsr_kernel(int64_t nnz, const int32_t *__restrict__ row_of, const int32_t *__restrict__ row_ptr,
                            const int32_t *__restrict__ kp, const int32_t *__restrict__ vbase,
                            const int32_t *__restrict__ vptr, const int32_t *__restrict__ col_idx,
                            int32_t *__restrict__ vcol, int32_t *__restrict__ vslot) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= nnz) return;
    const int r = row_of[j], t = (int)(j - row_ptr[r]), k = kp[r];
    const int pos = vptr[vbase[r] + t % k] + t / k;
    vcol[pos] = col_idx[j];
    vslot[pos] = (int32_t)j;
}

// out[prow[i]][b] = epi(sum over the part slots of split row i, in slot order)
__global__ void split_rows_reduce_kernel(int nsplit, int64_t B, const int32_t *__restrict__ prow,
                                         const int32_t *__restrict__ pptr, const float *__restrict__ vpart,
                                         float *__restrict__ out, const float *__restrict__ gate, int epi) {
    const int i = blockIdx.y;
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nsplit || b >= B) return;
    const int64_t r = prow[i];
    pdl_wait();  // (a programmatic dependent of the part-row SpMM)
    float s = 0.f;
    for (int k = pptr[i]; k < pptr[i + 1]; ++k) s += vpart[(int64_t)k * B + b];
    if (epi == 1) s = fmaxf(s, 0.f);
    if (epi == 2) s = gate[r * B + b] > 0.f ? s : 0.f;
    out[r * B + b] = s;
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

// out[0..n] = exclusive scan of in[0..n) with out[n] = total; info[0] = total,
// info[1] = max (int64).  Stream-ordered scratch.
cudaError_t launch_scan(int64_t n, const int32_t *in, int32_t *out, int64_t *info, cudaStream_t st) {
    const int64_t nc = std::max<int64_t>(1, (n + kScanChunk - 1) / kScanChunk);
    int64_t *csum = nullptr;
    int32_t *cmax = nullptr;
    cudaError_t e = scratch_alloc((void **)&csum, (size_t)nc * sizeof(int64_t), st);
    if (e != cudaSuccess) return e;
    e = scratch_alloc((void **)&cmax, (size_t)nc * sizeof(int32_t), st);
    if (e != cudaSuccess) {
        scratch_free(csum, st);
        return e;
    }
    scan_chunks_kernel<<<(unsigned)nc, kScanThreads, 0, st>>>(n, in, csum, cmax);
    scan_top_kernel<<<1, 1, 0, st>>>(nc, csum, cmax, info);
    scan_apply_kernel<<<(unsigned)nc, kScanThreads, 0, st>>>(n, in, csum, info, out);
    scratch_free(csum, st);
    scratch_free(cmax, st);
    return cudaGetLastError();
}

}  // namespace

void free_weight(sp_weight_s *w) {
    // the arenas come from the library's stream-ordered pool (cheap to create,
    // cached on release); every stream's work is complete here (the callers
    // synchronise the device first), so the legacy stream orders the frees
    for (auto &a : w->arena) {
        if (a) scratch_free(a, 0);
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
    // column counts / CSC compaction by row blocks: about 64k (block, column)
    // threads -- enough to fill the GPU, few enough blocks that the per-column
    // scan over them stays short
    const int64_t nb = std::max<int64_t>(1, std::min<int64_t>(R, (65536 + C - 1) / C));
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
        SP_TRY(scratch_alloc((void **)&a.base, asize<int32_t>(R + 1) + asize<int32_t>(C + 1), st));
        w->arena[0] = a.base;
        w->row_ptr = a.take<int32_t>(R + 1);
        w->col_ptr = a.take<int32_t>(C + 1);
    }
    {
        row_count_kernel<<<(unsigned)((R + 7) / 8), 256, 0, st>>>(R, C, mask, rcnt);
        colblk_count_kernel<<<(unsigned)((nb * C + 255) / 256), 256, 0, st>>>(R, C, nb, rbk, mask, blk);
        colblk_scan_kernel<<<(unsigned)((C + 255) / 256), 256, 0, st>>>(C, nb, blk, ccnt);
        SP_TRY(launch_scan(R, rcnt, w->row_ptr, info, st));
        SP_TRY(launch_scan(C, ccnt, w->col_ptr, info + 2, st));
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
        SP_TRY(scratch_alloc((void **)&a.base, 5 * asize<int32_t>(w->nnz) + asize<int32_t>(R + 1), st));
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
    SP_TRY(launch_scan(R, rcnt, w->chunk_ptr, info, st));
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
// rows by length, longest first (ties by index): shared by every tiling of one row set
static std::vector<int32_t> length_order(const std::vector<int32_t> &ptr, int64_t rows) {
    std::vector<int32_t> order(rows);
    for (int64_t r = 0; r < rows; ++r) order[r] = (int32_t)r;
    std::stable_sort(order.begin(), order.end(),
                     [&](int32_t a, int32_t b) { return ptr[a + 1] - ptr[a] > ptr[b + 1] - ptr[b]; });
    return order;
}

static void balanced_rows(const std::vector<int32_t> &order, int64_t rows, int RB, int NW, std::vector<int32_t> &rowpos,
                          std::vector<int32_t> &rowmap) {
    const int64_t nrb = (rows + RB - 1) / RB;
    rowpos.assign(rows, 0);
    rowmap.assign(nrb * RB, -1);
    if (NW == 0) {  // longest first (the gather tilings: a warp per position, CTAs launched in
                    // position order -- the long rows start first, a CTA's warps have similar lengths)
        for (int64_t k = 0; k < rows; ++k) {
            rowpos[order[k]] = (int32_t)k;
            rowmap[k] = order[k];
        }
        return;
    }
    const int RPW = RB / NW;
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
    std::vector<Spec> specs = {{0, kTilRB[0], kTilKC[0], kTilNW[0], 4, &w->til[0][0]},
                               {0, kTilRB[1], kTilKC[1], kTilNW[1], kTilRB[1] / kTilNW[1], &w->til[0][1]},
                               {1, kTilRB[0], kTilKC[0], kTilNW[0], 4, &w->til[1][0]},
                               {1, kTilRB[1], kTilKC[1], kTilNW[1], kTilRB[1] / kTilNW[1], &w->til[1][1]},
                               {1, 64, kTilKC[0], 32, 2, &w->til_f[0]},
                               {1, 32, kTilKC[0], 32, 1, &w->til_f[1]},
                               {1, 64, kTilKC[0], 16, 4, &w->til_f[2]}};
    // gather tilings (whole inner dimension in one column block; inner indices
    // times kTilRowBytes must fit an int32 entry offset)
    if (w->nnz > 0 && ((double)w->nnz <= kGatherDensity * (double)w->R * (double)w->C || w->nnz <= kGatherNnz) &&
        std::max(w->R, w->C) < (int64_t)(INT32_MAX / kTilRowBytes)) {
#ifndef SP_GATHER_BALANCED
        specs.push_back({0, kGatherRB, (int)w->C, 0, kGatherUnit, &w->til_g[0]});
        specs.push_back({1, kGatherRB, (int)w->R, 0, kGatherUnit, &w->til_g[1]});
#else
        specs.push_back({0, kGatherRB, (int)w->C, kGatherRB / kGatherUnit, kGatherUnit, &w->til_g[0]});
        specs.push_back({1, kGatherRB, (int)w->R, kGatherRB / kGatherUnit, kGatherUnit, &w->til_g[1]});
#endif
    }
#ifndef SP_TILK_DENSITY
#define SP_TILK_DENSITY kTilKDensity
#endif
    if (w->nnz > (int64_t)(SP_TILK_DENSITY * (double)w->R * (double)w->C)) {
        specs.push_back({0, kTilRB[0], kTilKC_K, kTilNW[0], 4, &w->til_k[0]});
        specs.push_back({1, kTilRB[0], kTilKC_K, kTilNW[0], 4, &w->til_k[1]});
    }
    const int NS = (int)specs.size();
    // ---- split rows of the forward (CSR) tilings: a row with more than
    // L = max(32, 2 * mean) entries (Zipf head rows) becomes k = ceil(n / L)
    // part rows taking its entries in turn, so every part spans all column
    // blocks with ~n / k entries and no warp carries a whole dense row
    const int64_t R = w->R;
    std::vector<int32_t> kp(R, 1), vbase(R), vptr_h, real_of, slot_of;  // part rows per row, ...
    int64_t nv = 0, nsplit = 0, nparts = 0;
    {
        const int64_t L = std::max<int64_t>(32, 2 * ((w->nnz + R - 1) / std::max<int64_t>(R, 1)));
        for (int64_t r = 0; r < R; ++r) {
            const int64_t n = hptr[0][r + 1] - hptr[0][r];
            if (n > L) kp[r] = (int32_t)((n + L - 1) / L);
            vbase[r] = (int32_t)nv;
            nv += kp[r];
            if (kp[r] > 1) {
                ++nsplit;
                nparts += kp[r];
            }
        }
    }
#ifdef SP_NO_SPLIT_ROWS
    const bool splitting = false;
#else
    const bool splitting = nsplit > 0;
#endif
    std::vector<int32_t> vlen_ptr;  // pointer array of the virtual rows (for balanced_rows / the tilings)
    std::vector<int32_t> prow_h, pptr_h;
    if (splitting) {
        vlen_ptr.assign(nv + 1, 0);
        real_of.resize(nv);
        slot_of.assign(nv, -1);
        int32_t slot = 0;
        for (int64_t r = 0; r < R; ++r) {
            const int32_t n = hptr[0][r + 1] - hptr[0][r], k = kp[r];
            if (k > 1) {
                prow_h.push_back((int32_t)r);
                pptr_h.push_back(slot);
            }
            for (int32_t q = 0; q < k; ++q) {
                const int64_t v = vbase[r] + q;
                vlen_ptr[v + 1] = vlen_ptr[v] + (n - q + k - 1) / k;
                real_of[v] = (int32_t)r;
                if (k > 1) slot_of[v] = slot++;
            }
        }
        pptr_h.push_back(slot);
    }
    // ---- plan: every tiling's geometry and buffer sizes, then ONE device
    // allocation (the tiling arena) and ONE host -> device copy of the host-built
    // row placements and the managed-SGD table
    struct Plan {
        int64_t rows, inner, nseg, cap, nwg;
    };
    std::vector<Plan> pl(NS);
    size_t bytes = 0, hbytes = 0;  // arena total; the host-filled region
    for (int si = 0; si < NS; ++si) {
        const Spec &sp_ = specs[si];
        sp_tiling &t = *sp_.t;
        const int o = sp_.o;
        Plan &P = pl[si];
        const bool vs = o == 0 && splitting;  // the tiling places part rows
        P.rows = o == 0 ? (vs ? nv : w->R) : w->C;  // placed (possibly part) rows
        P.inner = o == 0 ? w->C : w->R;
        t.RB = sp_.RB;
        t.KC = sp_.KC;
        t.rows = o == 0 ? w->R : w->C;  // output rows (kernel bounds)
        t.inner = P.inner;
        t.nrb = (int)((P.rows + t.RB - 1) / t.RB);
        t.nkb = (int)((P.inner + t.KC - 1) / t.KC);
        P.nseg = (int64_t)t.nrb * t.nkb * t.RB;
        // upper bound on the padded entry count (each segment pads < kTilPad)
        P.cap = w->nnz + (kTilPad - 1) * std::min<int64_t>(P.nseg, w->nnz) + 8;
        P.nwg = t.RB / sp_.RPWgrp;
        hbytes += asize<int32_t>(P.rows) + asize<int32_t>((int64_t)t.nrb * t.RB);
        if (vs) hbytes += asize<int32_t>((int64_t)t.nrb * t.RB) + asize<int32_t>(nsplit) + asize<int32_t>(nsplit + 1);
        bytes += asize<int32_t>(P.nseg + 8) + asize<int2>(P.cap) + asize<int32_t>(P.cap);
        if (w->nnz > 0) bytes += asize<int32_t>(w->nnz);
        if (si == 0 || si == 2) bytes += asize<int32_t>(P.nseg + 8);
        if (o == 1) bytes += 2 * asize<int32_t>((int64_t)t.nrb * P.nwg * (t.nkb + 1));
    }
    hbytes += asize<SgdRef>(NS);
    Arena ar;
    if (scratch_alloc((void **)&ar.base, bytes + hbytes, st) != cudaSuccess) return SP_ERR_ALLOC;
    w->arena[2] = ar.base;
    // host-filled region first (rowpos / rowmap of every tiling, the SGD table)
    std::vector<char> hreg(hbytes, 0);
    std::vector<int32_t> orders[3];  // length orders of the CSR rows, the CSC rows, the CSR part rows
    for (int si = 0; si < NS; ++si) {
        sp_tiling &t = *specs[si].t;
        t.in_arena = true;
        const size_t o1 = ar.off;
        t.rowpos = ar.take<int32_t>(pl[si].rows);
        const size_t o2 = ar.off;
        t.rowmap = ar.take<int32_t>((int64_t)t.nrb * t.RB);
        std::vector<int32_t> rowpos, rowmap;
        const bool vs = specs[si].o == 0 && splitting;
        // the length order of this tiling's row set (computed once per set)
        const int oset = specs[si].o == 1 ? 1 : vs ? 2 : 0;
        if (orders[oset].empty() && pl[si].rows > 0)
            orders[oset] = length_order(oset == 2 ? vlen_ptr : hptr[specs[si].o], pl[si].rows);
        balanced_rows(orders[oset], pl[si].rows, t.RB, specs[si].NWbal, rowpos, rowmap);
        memcpy(hreg.data() + o1, rowpos.data(), rowpos.size() * sizeof(int32_t));
        if (vs) {  // positions hold part rows: rowmap -> the real row, split -> the part slot
            std::vector<int32_t> sm(rowmap.size(), -1);
            for (size_t pos = 0; pos < rowmap.size(); ++pos)
                if (rowmap[pos] >= 0) {
                    sm[pos] = slot_of[rowmap[pos]];
                    rowmap[pos] = real_of[rowmap[pos]];
                }
            const size_t o3 = ar.off;
            t.split = ar.take<int32_t>((int64_t)t.nrb * t.RB);
            memcpy(hreg.data() + o3, sm.data(), sm.size() * sizeof(int32_t));
            const size_t o4 = ar.off;
            t.prow = ar.take<int32_t>(nsplit);
            memcpy(hreg.data() + o4, prow_h.data(), prow_h.size() * sizeof(int32_t));
            const size_t o5 = ar.off;
            t.pptr = ar.take<int32_t>(nsplit + 1);
            memcpy(hreg.data() + o5, pptr_h.data(), pptr_h.size() * sizeof(int32_t));
            t.nsplit = (int32_t)nsplit;
            t.nparts = (int32_t)nparts;
        }
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
            if (specs[si].t->inv && tab.size() < sizeof(w->sgdtil) / sizeof(w->sgdtil[0])) {
                w->sgdtil[tab.size()] = specs[si].t;
                tab.push_back({specs[si].t->ent, specs[si].t->inv});
            }
        w->nsgd = (int)tab.size();
        memcpy(hreg.data() + otab, tab.data(), tab.size() * sizeof(SgdRef));
    }
    cudaMemcpyAsync(ar.base, hreg.data(), hbytes, cudaMemcpyHostToDevice, st);

    // the virtual CSR of the part rows (device scratch, freed after the build)
    int32_t *vptr_d = nullptr, *vcol_d = nullptr, *vslot_d = nullptr, *kp_d = nullptr, *vbase_d = nullptr;
    int64_t *info = nullptr, *mx = nullptr;
    int32_t *cnt = nullptr;
    // error paths release every scratch buffer (the arena itself belongs to the handle)
    auto fail_alloc = [&]() -> sp_status {
        for (void *p : {(void *)vptr_d, (void *)vcol_d, (void *)vslot_d, (void *)kp_d, (void *)vbase_d, (void *)info,
                        (void *)mx, (void *)cnt})
            if (p) scratch_free(p, st);
        return SP_ERR_ALLOC;
    };
    if (splitting) {
        if (scratch_alloc((void **)&vptr_d, (size_t)(nv + 1) * sizeof(int32_t), st) != cudaSuccess ||
            scratch_alloc((void **)&vcol_d, (size_t)std::max<int64_t>(w->nnz, 1) * sizeof(int32_t), st) != cudaSuccess ||
            scratch_alloc((void **)&vslot_d, (size_t)std::max<int64_t>(w->nnz, 1) * sizeof(int32_t), st) != cudaSuccess ||
            scratch_alloc((void **)&kp_d, (size_t)R * sizeof(int32_t), st) != cudaSuccess ||
            scratch_alloc((void **)&vbase_d, (size_t)R * sizeof(int32_t), st) != cudaSuccess)
            return fail_alloc();
        cudaMemcpyAsync(vptr_d, vlen_ptr.data(), (size_t)(nv + 1) * sizeof(int32_t), cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(kp_d, kp.data(), (size_t)R * sizeof(int32_t), cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(vbase_d, vbase.data(), (size_t)R * sizeof(int32_t), cudaMemcpyHostToDevice, st);
        vcsr_kernel<<<(unsigned)((w->nnz + 255) / 256), 256, 0, st>>>(w->nnz, w->row_of, w->row_ptr, kp_d, vbase_d,
                                                                      vptr_d, w->col_idx, vcol_d, vslot_d);
    }
    if (scratch_alloc((void **)&info, 2 * NS * sizeof(int64_t), st) != cudaSuccess) return fail_alloc();
    if (scratch_alloc((void **)&mx, 3 * NS * sizeof(int64_t), st) != cudaSuccess) return fail_alloc();
    cudaMemsetAsync(mx, 0, 3 * NS * sizeof(int64_t), st);  // atomicMax targets
    for (int si = 0; si < NS; ++si) {
        const Spec &sp_ = specs[si];
        const int o = sp_.o;
        const int64_t rows = pl[si].rows;
        const bool vs = o == 0 && splitting;
        const int32_t *ptr = o == 0 ? (vs ? vptr_d : w->row_ptr) : w->col_ptr;
        const int32_t *idx = o == 0 ? (vs ? vcol_d : w->col_idx) : w->row_idx;
        const int32_t *slotmap = o == 0 ? (vs ? vslot_d : nullptr) : w->perm;
        sp_tiling &t = *sp_.t;
        const int64_t nseg = pl[si].nseg, cap = pl[si].cap;
        cnt = nullptr;
        if (scratch_alloc((void **)&cnt, (size_t)nseg * sizeof(int32_t), st) != cudaSuccess) return fail_alloc();
        cudaMemsetAsync(cnt, 0, (size_t)nseg * sizeof(int32_t), st);
        cudaMemsetAsync(t.seg + nseg + 1, 0, 7 * sizeof(int32_t), st);  // slack for 16-byte bulk copies of bounds
        cudaMemsetAsync(t.ent, 0, (size_t)cap * sizeof(int2), st);
        cudaMemsetAsync(t.vidx, 0xff, (size_t)cap * sizeof(int32_t), st);  // -1: no slot
        const int64_t nt = rows * t.nkb;
        til_count_kernel<<<(unsigned)((nt + 255) / 256), 256, 0, st>>>(rows, t.nkb, t.KC, t.RB, ptr, idx, t.rowpos,
                                                                      cnt);
        if (launch_scan(nseg, cnt, t.seg, info + 2 * si, st) != cudaSuccess) return fail_alloc();
        til_fill_kernel<<<(unsigned)((nt + 255) / 256), 256, 0, st>>>(rows, t.nkb, t.KC, t.RB, ptr, idx, slotmap,
                                                                     t.rowpos, t.seg, w->vals, t.ent, t.vidx);
        const int64_t ntl = (int64_t)t.nrb * t.nkb;
        til_max_kernel<<<(unsigned)((ntl + 255) / 256), 256, 0, st>>>(ntl, t.RB, t.seg,
                                                                     (unsigned long long *)(mx + si));
        if (w->nnz > 0) til_inv_kernel<<<(unsigned)((cap + 255) / 256), 256, 0, st>>>(cap, t.vidx, t.inv);
        t.fresh = 1;  // built from vals: the handle's first version
        if (t.tmsplit)  // the big tilings (RB = 128, KC = 192): split-source SpMM
            til_split_kernel<<<(unsigned)((nseg + 255) / 256), 256, 0, st>>>(nseg, t.KC, t.seg, t.ent, t.tmsplit);
        // per-warp group maxima (and, for the fused backward's CSC tilings, the
        // group prefix tables of groups of 4 and of 8)
        {
            const int nwg = (int)pl[si].nwg;
            if (o == 1) t.RPWg = sp_.RPWgrp;
            til_warp_groups_kernel<<<(unsigned)((t.nrb * nwg + 127) / 128), 128, 0, st>>>(
                t.nrb, t.nkb, t.RB, sp_.RPWgrp, t.seg, (unsigned long long *)(mx + NS + si),
                (unsigned long long *)(mx + 2 * NS + si), o == 1 ? t.gpre[0] : nullptr, o == 1 ? t.gpre[1] : nullptr);
        }
        scratch_free(cnt, st);
        cnt = nullptr;
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
    for (int32_t *p : {vptr_d, vcol_d, vslot_d, kp_d, vbase_d})
        if (p) scratch_free(p, st);
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
    for (auto &t : w->til_g) fr(t);
    for (auto &t : w->til_k) fr(t);

    w->tapdev = nullptr;  // lives in the tap arena (arena[3], freed by free_weight)
    w->sgdtab = nullptr;  // lives in the tiling arena
    w->nsgd = 0;
}

__global__ void zero_i32_kernel(int *p, int64_t n) {
    pdl_wait();  // (the buffer may have been another kernel's scratch a moment ago)
    pdl_trigger();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = 0;
}

void launch_zero_i32(int *p, int64_t n, cudaStream_t st) {
#ifdef SP_ZERO_MEMSET
    cudaMemsetAsync(p, 0, (size_t)n * sizeof(int), st);
#else
    if (n <= 0) return;
    count_launches(1);
    launch_pdl(zero_i32_kernel, dim3((unsigned)std::min<int64_t>(148, (n + 255) / 256)), dim3(256), 0, st, p, n);
#endif
}

void refresh_if_stale(const sp_weight_s *w, const sp_tiling &t, cudaStream_t st) {
    t.used = true;
    if (w->managed && t.fresh == w->version) return;
    launch_refresh(t, w->vals, w->nnz, st);
    t.fresh = w->version;
}

// the tilings of sgdtab that get the new values (those read since the last update)
static uint32_t sgd_mask(const sp_weight_s *w) {
    uint32_t mask = 0;
    for (int k = 0; k < w->nsgd && k < 32; ++k) {
#ifndef SP_SGD_ALL
        if (w->sgdtil[k]->used && w->sgdtil[k]->fresh == w->version) mask |= 1u << k;
#else
        mask |= 1u << k;
#endif
    }
    return mask;
}
static void sgd_mark(sp_weight_s *w, uint32_t mask) {
    ++w->version;  // vals changed; the updated tilings hold the new values
    for (int k = 0; k < w->nsgd && k < 32; ++k) {
        if ((mask >> k) & 1u) w->sgdtil[k]->fresh = w->version;
        w->sgdtil[k]->used = false;
    }
}

// one kernel for many handles: grid over the concatenated slots
struct SgdBatch {
    int n;
    float lr;
    int64_t off[SP_SGD_BATCH_MAX + 1];
    float *vals[SP_SGD_BATCH_MAX];
    const float *dW[SP_SGD_BATCH_MAX];
    const SgdRef *tab[SP_SGD_BATCH_MAX];
    int ntab[SP_SGD_BATCH_MAX];
    uint32_t mask[SP_SGD_BATCH_MAX];
};
__global__ void weights_sgd_kernel(const __grid_constant__ SgdBatch b) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= b.off[b.n]) return;
    int lo = 0, hi = b.n;  // handle i with off[i] <= g < off[i+1]
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (b.off[mid] <= g) lo = mid;
        else hi = mid;
    }
    const int64_t j = g - b.off[lo];
    const float v = fmaf(-b.lr, b.dW[lo][j], b.vals[lo][j]);  // the same rounding as sp_sgd
    b.vals[lo][j] = v;
    const SgdRef *tab = b.tab[lo];
    for (int k = 0; k < b.ntab[lo]; ++k)
        if ((b.mask[lo] >> k) & 1u) tab[k].ent[tab[k].inv[j]].y = __float_as_int(v);
}

void launch_weights_sgd(sp_weight_s *const *ws, const float *const *dWs, int n, float lr, cudaStream_t st) {
    SgdBatch b{};
    b.n = n;
    b.lr = lr;
    for (int i = 0; i < n; ++i) {
        b.off[i + 1] = b.off[i] + ws[i]->nnz;
        b.vals[i] = ws[i]->vals;
        b.dW[i] = dWs[i];
        b.tab[i] = ws[i]->sgdtab;
        b.ntab[i] = ws[i]->nsgd;
        b.mask[i] = sgd_mask(ws[i]);
    }
    if (b.off[n] > 0) {
        count_launches(1);
        weights_sgd_kernel<<<(unsigned)((b.off[n] + 255) / 256), 256, 0, st>>>(b);
    }
    for (int i = 0; i < n; ++i) sgd_mark(ws[i], b.mask[i]);
}

void launch_weight_sgd(sp_weight_s *w, const float *dW, float lr, cudaStream_t st) {
    // the new values go to vals and to the tilings the products have read since the
    // last update (a training step uses 2 of the 7-9); the others fall behind and are
    // refreshed from vals at their next use (refresh_if_stale)
    const uint32_t mask = sgd_mask(w);
    if (w->nnz > 0) {
        count_launches(1);
        weight_sgd_kernel<<<(unsigned)((w->nnz + 255) / 256), 256, 0, st>>>(w->nnz, w->vals, dW, lr, w->sgdtab,
                                                                            w->nsgd, mask);
    }
    sgd_mark(w, mask);
}

void launch_split_rows_reduce(const sp_tiling &t, const float *vpart, int64_t B, float *out, const float *gate,
                              int epi, cudaStream_t st) {
    count_launches(1);
    note_path("split_rows_reduce");
    launch_pdl(split_rows_reduce_kernel, dim3((unsigned)((B + 255) / 256), (unsigned)t.nsplit), dim3(256), 0, st,
               t.nsplit, B, t.prow, t.pptr, vpart, out, gate, epi);
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
    // a managed handle's vals change only through sp_weight_sgd (which bumps the
    // version): the tap tilings refresh once per version, like the linear tilings
    if (w->managed && w->tap_fresh[orient] == w->version) return;
    count_launches(1);
    til_refresh_taps_kernel<<<dim3(64, ntap), 256, 0, st>>>(w->tapdev + orient * kMaxTaps, w->vals);
    w->tap_fresh[orient] = w->version;
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
