// spmm_hyb.cu -- forward SpMM (K2) and CSC-driven dX SpMM (K3) with the gathers
// split between shared memory and TENSOR MEMORY.  SURVEY §8(a) rows a-2, a-3.
//
//   out[r][b] = epi( sum over the entries (c, w) of row r of w * in[c][b] )
//
// The kernel is spmm_tiled_kernel's 32-warp layout (spmm.cu: RB = 128 rows of
// 4 per warp, 128 batch columns per CTA, [KC = 192 x 128] activation tiles by
// 2-D TMA into two shared-memory buffers, entries staged alongside) plus a
// second gather source.  Every gathered activation row costs 4 shared-memory
// wavefronts, and the shared-memory data path is what bounds the LDS kernel
// (DESIGN.md §5); a tcgen05.ld of the same 16 bytes per lane from TMEM runs on
// a separate path at about twice the rate (tools/micro/tmgather.cu).  So the
// last TC = 63 rows of every tile are also copied into a 256-column TMEM
// buffer (tcgen05.cp.32x128b.warpx4: each 512-byte row lands in the same 4
// columns of all four lane quarters), and a group of 4 entries whose columns
// all fall in those rows (entries are column-sorted within a segment, so these
// are the segment's last groups) is gathered from TMEM -- but only once the
// copy is known complete (a non-blocking mbarrier test); until then, and for
// every other group, from shared memory, which still holds the whole tile.
// Both sources hold the same values, so the result does not depend on which
// one served a group: every output element is produced by one lane with its
// entries in ascending order (no atomics, bitwise reproducible, independent
// of B, identical to spmm_tiled_kernel's result).
//
// Copies: the first 8 warps to start tile q each issue 8 of its 63 row copies
// and commit them to tfull[q & 1]; whoever refills shared-memory buffer q & 1
// with tile q + 2 first waits for that commit (the copies read the buffer).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "sp_internal.cuh"
#include "tile.cuh"

namespace sp {
namespace {

// Unpredicated gathers of all but a segment's last slot rely on even padding.
static_assert(kTilPad == 2 && kTapPad == 2, "only a segment's last slot may be padding");

constexpr int HY_NW = 32, HY_RPW = 4, HY_RB = HY_NW * HY_RPW, HY_BT = 128;
constexpr int HY_TC = kHybTC;  // tile rows mirrored in TMEM (the last TC of the KC)
constexpr int HY_ISSUE = 8;    // warps issuing a tile's copies

struct HybArgs {
    int64_t rows, B;
    int KC, nkb, cap;
    const int32_t *seg;
    const int32_t *split;
    const int2 *ent;
    float *out;
    const float *gate;
    const int32_t *rowmap;
    const int32_t *psplit;  // tiled position -> part slot of a split row (-1 whole; nullptr: none)
    float *vpart;          // [nparts x B] raw sums of the part rows
    unsigned long long *stats;  // SP_SPMM_HYB_STATS=1: [groups from TMEM, all groups] (measurement only)
};

__device__ __forceinline__ void hy_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void hy_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// non-blocking: has the phase with this parity completed?
__device__ __forceinline__ bool mbar_test(uint64_t *bar, unsigned parity) {
    unsigned ok;
    asm volatile(
        "{\n.reg .pred P;\n"
        "mbarrier.test_wait.parity.shared::cta.b64 P, [%1], %2;\n"
        "selp.u32 %0, 1, 0, P;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

// descriptor of one 512-byte tile row as 32 rows x 16 bytes (SBO = 128, no swizzle)
__device__ __forceinline__ uint64_t hy_desc(const void *p) {
    return (uint64_t)((smem_u32(p) >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 32) | ((uint64_t)1 << 46);
}

__device__ __forceinline__ void hy_gather4(uint32_t t0, uint32_t t1, uint32_t t2, uint32_t t3, float (&x)[4][4]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%16];\n"
        "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%4, %5, %6, %7}, [%17];\n"
        "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%8, %9, %10, %11}, [%18];\n"
        "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%12, %13, %14, %15}, [%19];\n"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(t0), "r"(t1), "r"(t2), "r"(t3)
        : "memory");
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) x[u][v] = __uint_as_float(r[4 * u + v]);
}
__device__ __forceinline__ void hy_gather2(uint32_t t0, uint32_t t1, float (&x)[4][4]) {
    uint32_t r[8];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%8];\n"
        "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%4, %5, %6, %7}, [%9];\n"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
        : "r"(t0), "r"(t1)
        : "memory");
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) x[u][v] = __uint_as_float(r[4 * u + v]);
}

template <int EPI, bool STATS>
__global__ void __launch_bounds__(HY_NW * 32, 1) spmm_hyb_kernel(const HybArgs a, const __grid_constant__ CUtensorMap tmap) {
    extern __shared__ __align__(128) float smem[];  // [2][KC + 1][BT] floats (a zero row before each tile), [2][cap+2] int2
    __shared__ uint64_t full[2], tfull[2];
    __shared__ int released[2], ticket[2];
    __shared__ uint32_t tmem_base;
    int2 *ents = reinterpret_cast<int2 *>(smem + (size_t)2 * (a.KC + 1) * HY_BT);

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int rb = blockIdx.x;
    const int64_t b0 = (int64_t)blockIdx.y * HY_BT;
    const size_t tile_sz = (size_t)a.KC * HY_BT;
    const size_t buf_sz = tile_sz + HY_BT;
    const int ebuf = a.cap + 2;
    const int ntile = a.nkb;
    const int c0 = a.KC - HY_TC;  // first mirrored tile row

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (threadIdx.x == 32) {
        for (int b = 0; b < 2; ++b) {
            mbar_init(&full[b], 1);
            mbar_init(&tfull[b], HY_ISSUE);
            released[b] = 0;
            ticket[b] = 0;
        }
        fence_mbar_init();
    }
    for (int i = threadIdx.x; i < HY_BT; i += HY_NW * 32) {  // the zero rows in front of the two tiles
        smem[i] = 0.f;
        smem[buf_sz + i] = 0.f;
    }
    hy_before();
    __syncthreads();
    hy_after();
    const uint32_t tq = tmem_base + ((uint32_t)(32 * (warp & 3)) << 16);
    if (warp < 4) {  // zero columns in front of each TMEM buffer (padding entries read them)
        asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %1, %1, %1};" ::"r"(tq), "r"(0u) : "memory");
        asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %1, %1, %1};" ::"r"(tq + 256), "r"(0u)
                     : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    hy_before();
    __syncthreads();
    hy_after();

    auto entry_range = [&](int kb, int &e0, int &e1) {
        const int64_t tb = ((int64_t)rb * a.nkb + kb) * HY_RB;
        e0 = __ldg(a.seg + tb) & ~1;
        e1 = __ldg(a.seg + tb + HY_RB);
    };
    auto issue = [&](int q, int buf) {  // one thread: TMA of tile q into buffer buf
        int e0, e1;
        entry_range(q, e0, e1);
        const unsigned eb = (unsigned)(((e1 - e0) * 8 + 15) & ~15);
        mbar_arrive_expect_tx(&full[buf], (unsigned)(tile_sz * sizeof(float)) + eb);
        tma_load_2d(smem + buf * buf_sz + HY_BT, &tmap, (int)b0, q * a.KC, &full[buf]);
        if (eb) tma_load_1d(ents + buf * ebuf, a.ent + e0, eb, &full[buf]);
    };
    pdl_wait();  // (launched as a programmatic dependent: the prologue above overlapped the previous kernel)
    if (threadIdx.x == 0) {
        issue(0, 0);
        if (ntile > 1) issue(1, 1);
    }
    pdl_trigger();
    // lane l <= RPW: the l-th segment bound of this warp's rows in tile q;
    // lanes 8 + i: row i's TMEM split (tmsplit)
    auto seg_bounds = [&](int q) -> int {
        const int64_t sb = ((int64_t)rb * a.nkb + q) * HY_RB + warp * HY_RPW;
        if (lane <= HY_RPW) return __ldg(a.seg + sb + lane);
        if (lane >= 8 && lane < 8 + HY_RPW) return __ldg(a.split + sb + lane - 8);
        return 0;
    };
    int sg = seg_bounds(0);

    float acc[HY_RPW][4];
#pragma unroll
    for (int i = 0; i < HY_RPW; ++i)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[i][v] = 0.f;

    for (int q = 0; q < ntile; ++q) {
        const int buf = q & 1;
        const unsigned par = (unsigned)(q >> 1) & 1u;
        const int sgn = q + 1 < ntile ? seg_bounds(q + 1) : 0;
        mbar_wait(&full[buf], par);
        // the first HY_ISSUE warps to start this tile copy its last TC rows into TMEM
        if (lane == 0) {
            const int t = atomicAdd(&ticket[buf], 1);
            if (t == HY_NW - 1) ticket[buf] = 0;  // every warp has drawn: reset for tile q + 2
            if (t < HY_ISSUE) {
                hy_after();
                const uint32_t dst = tmem_base + (uint32_t)(buf * 256 + 4);
                const char *src = reinterpret_cast<const char *>(smem + buf * buf_sz + HY_BT) + (size_t)c0 * 512;
                for (int c = t; c < HY_TC; c += HY_ISSUE)
                    asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(dst + 4 * c),
                                 "l"(hy_desc(src + c * 512))
                                 : "memory");
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 smem_u32(&tfull[buf]))
                             : "memory");
            }
        }
        __syncwarp();
        int ea, e1;
        entry_range(q, ea, e1);
        const char *tb = reinterpret_cast<const char *>(smem + buf * buf_sz + HY_BT + lane * 4);
        const int2 *es = ents + buf * ebuf - ea;
        // TMEM column of an entry in the mirrored rows (padding -> the zero columns)
        const uint32_t tcol = tq + (uint32_t)(buf * 256);
        bool tm_ok = false;
        unsigned n_tm = 0, n_all = 0;
        // groups of 4 entries (a last lone pair) of [e0, e1) from shared memory / TMEM
        auto lds_part = [&](float (&ac)[4], int e0, int e1) {
            for (int e = e0; e < e1; e += 4) {
                const int4 p01 = ld_entry_pair(es + e, true);
                float x[4][4];
                if (e + 2 < e1) {
                    const int4 p23 = ld_entry_pair(es + e + 2, true);
                    lds_vec<4>(reinterpret_cast<const float *>(tb + p01.x), x[0]);
                    lds_vec<4>(reinterpret_cast<const float *>(tb + p01.z), x[1]);
                    lds_vec<4>(reinterpret_cast<const float *>(tb + p23.x), x[2]);
                    lds_vec<4>(reinterpret_cast<const float *>(tb + p23.z), x[3]);
                    fma_bcast<4>(ac, __int_as_float(p01.y), x[0]);
                    fma_bcast<4>(ac, __int_as_float(p01.w), x[1]);
                    fma_bcast<4>(ac, __int_as_float(p23.y), x[2]);
                    fma_bcast<4>(ac, __int_as_float(p23.w), x[3]);
                } else {
                    lds_vec<4>(reinterpret_cast<const float *>(tb + p01.x), x[0]);
                    lds_vec<4>(reinterpret_cast<const float *>(tb + p01.z), x[1]);
                    fma_bcast<4>(ac, __int_as_float(p01.y), x[0]);
                    fma_bcast<4>(ac, __int_as_float(p01.w), x[1]);
                }
            }
        };
        // column = tb0 + (off >> 7) for mirrored rows; a segment's padding entry
        // (offset < 0) can only be its last slot, which selects the zero columns
        const uint32_t tb0 = pin_u32(tcol + (uint32_t)(4 - 4 * c0));
        auto tm_part = [&](float (&ac)[4], int e0, int e1) {
            for (int e = e0; e < e1; e += 4) {
                const int4 p01 = ld_entry_pair(es + e, true);
                float x[4][4];
                if (e + 2 < e1) {
                    const int4 p23 = ld_entry_pair(es + e + 2, true);
                    hy_gather4(tb0 + (uint32_t)(p01.x >> 7), tb0 + (uint32_t)(p01.z >> 7), tb0 + (uint32_t)(p23.x >> 7),
                               p23.z >= 0 ? tb0 + (uint32_t)(p23.z >> 7) : tcol, x);
                    fma_bcast<4>(ac, __int_as_float(p01.y), x[0]);
                    fma_bcast<4>(ac, __int_as_float(p01.w), x[1]);
                    fma_bcast<4>(ac, __int_as_float(p23.y), x[2]);
                    fma_bcast<4>(ac, __int_as_float(p23.w), x[3]);
                } else {
                    hy_gather2(tb0 + (uint32_t)(p01.x >> 7), p01.z >= 0 ? tb0 + (uint32_t)(p01.z >> 7) : tcol, x);
                    fma_bcast<4>(ac, __int_as_float(p01.y), x[0]);
                    fma_bcast<4>(ac, __int_as_float(p01.w), x[1]);
                }
            }
        };
#pragma unroll
        for (int i = 0; i < HY_RPW; ++i) {
            const int s0 = __shfl_sync(kFull, sg, i), s1 = __shfl_sync(kFull, sg, i + 1);
            const int sp = __shfl_sync(kFull, sg, 8 + i);  // [s0, sp): shared memory; [sp, s1): mirrored rows
            lds_part(acc[i], s0, sp);
            if (sp < s1 && !tm_ok) {  // is the TMEM copy of this tile complete yet? (non-blocking)
                tm_ok = __shfl_sync(kFull, (int)mbar_test(&tfull[buf], par), 0) != 0;
                if (tm_ok) hy_after();
            }
            if (tm_ok)
                tm_part(acc[i], sp, s1);
            else
                lds_part(acc[i], sp, s1);
            if constexpr (STATS) {
                n_tm += tm_ok ? (unsigned)(s1 - sp) : 0u;
                n_all += (unsigned)(s1 - s0);
            }
        }
        if (STATS && lane == 0) {
            atomicAdd(a.stats, (unsigned long long)n_tm);
            atomicAdd(a.stats + 1, (unsigned long long)n_all);
        }
        // release the buffer; the last warp done with tile q refills it with tile q+2
        // once the TMEM copies of tile q (which read it) are complete
        hy_before();
        __syncwarp();
        if (lane == 0) {
            __threadfence_block();
            if (atomicAdd(&released[buf], 1) == HY_NW - 1) {
                released[buf] = 0;
                __threadfence_block();
                if (q + 2 < ntile) {
                    mbar_wait(&tfull[buf], par);
                    hy_after();
                    issue(q + 2, buf);
                }
            }
        }
        __syncwarp();
        sg = sgn;
    }
    // the copies of the last tiles complete before TMEM is released
    if (lane == 0 && warp == 0) {
        for (int q = std::max(0, ntile - 2); q < ntile; ++q) mbar_wait(&tfull[q & 1], (unsigned)(q >> 1) & 1u);
    }

    const int64_t bl = b0 + lane * 4;
    // Epilogue: ReLU / ReLU' gate fused; each element written once.
    if (bl < a.B) {
#pragma unroll
        for (int i = 0; i < HY_RPW; ++i) {
            const int64_t tpos = (int64_t)rb * HY_RB + warp * HY_RPW + i;
            const int64_t r = a.rowmap ? (int64_t)__ldg(a.rowmap + tpos) : tpos;
            if (r < 0 || r >= a.rows) continue;
            if (a.psplit) {  // a part row: raw sums to its slot (split_reduce applies the epilogue)
                const int sv = __ldg(a.psplit + tpos);
                if (sv >= 0) {
                    *reinterpret_cast<float4 *>(a.vpart + (int64_t)sv * a.B + bl) =
                        make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
                    continue;
                }
            }
            float o[4];
            if (EPI == EPI_GATE) {
                const float4 g = __ldg(reinterpret_cast<const float4 *>(a.gate + r * a.B + bl));
                o[0] = g.x > 0.f ? acc[i][0] : 0.f;
                o[1] = g.y > 0.f ? acc[i][1] : 0.f;
                o[2] = g.z > 0.f ? acc[i][2] : 0.f;
                o[3] = g.w > 0.f ? acc[i][3] : 0.f;
            } else {
#pragma unroll
                for (int v = 0; v < 4; ++v) o[v] = EPI == EPI_RELU ? fmaxf(acc[i][v], 0.f) : acc[i][v];
            }
            *reinterpret_cast<float4 *>(a.out + r * a.B + bl) = make_float4(o[0], o[1], o[2], o[3]);
        }
    }
    hy_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
}

constexpr int kSmemHyb = 226 * 1024;

}  // namespace

// The 32-warp big-tiling SpMM with the TMEM mirror; false when it does not
// apply (ragged B, a tiling other than RB = 128 / KC = 192, staged entries
// that do not fit).
bool launch_spmm_hyb(const sp_weight_s *w, int orient, int64_t B, const float *in, float *out, const float *gate,
                     int epi, cudaStream_t st, int64_t nslice_limit) {
    const sp_tiling &t = w->til[orient][0];
    if ((B & 3) != 0 || t.seg == nullptr || t.tmsplit == nullptr || t.RB != HY_RB || t.KC <= HY_TC || t.nkb == 0)
        return false;
    const size_t tiles = (size_t)2 * (t.KC + 1) * HY_BT * sizeof(float);
    const int cap = (t.max_tile + 2 + 3) & ~3;
    const size_t smem = tiles + (size_t)2 * (cap + 2) * sizeof(int2);
    if (smem > (size_t)kSmemHyb) return false;
    CUtensorMap tmap{};
    if (!make_tmap_2d(&tmap, in, t.inner, B, HY_BT, t.KC)) return false;
    refresh_if_stale(w, t, st);
    unsigned long long *stats = nullptr;  // entry counters of a measurement build (none in the product)
    float *vpart = nullptr;
    if (t.split && scratch_alloc((void **)&vpart, (size_t)t.nparts * B * sizeof(float), st) != cudaSuccess)
        return false;
    HybArgs a{t.rows, B, t.KC, t.nkb, cap, t.seg, t.tmsplit, t.ent, out, gate, t.rowmap, t.split, vpart, stats};
    int64_t nsl = (B + HY_BT - 1) / HY_BT;
    if (nslice_limit >= 0) {  // only the first nslice_limit slices (the rest run elsewhere: launch_spmm)
        if (t.split || nslice_limit < 1 || nslice_limit > nsl) return false;
        nsl = nslice_limit;
    }
    dim3 grid((unsigned)t.nrb, (unsigned)nsl);
    auto launch = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        count_launches(1);
        note_path("spmm_hyb");
        launch_pdl(kern, grid, dim3(HY_NW * 32), smem, st, a, tmap);
        if (vpart) {
            launch_split_rows_reduce(t, vpart, B, out, gate, epi, st);
            scratch_free(vpart, st);
        }
    };
    if (epi == EPI_RELU)
        launch(spmm_hyb_kernel<EPI_RELU, false>);
    else if (epi == EPI_GATE)
        launch(spmm_hyb_kernel<EPI_GATE, false>);
    else
        launch(spmm_hyb_kernel<EPI_NONE, false>);
    return true;
}

}  // namespace sp
