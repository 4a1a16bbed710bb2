// spmm_tm.cu -- forward SpMM (K2, sp_linear_fwd) and CSC-driven dX SpMM (K3,
// sp_linear_bwd_input) with the activation tile gathered from TENSOR MEMORY.
// SURVEY §8(a) rows a-2, a-3.
//
//   out[r][b] = epi( sum over the entries (c, w) of row r of w * in[c][b] )
//
// Why tensor memory: every FMA of an unstructured SpMM consumes
// one activation value fetched at a data-dependent (warp-uniform) row.  From
// shared memory that fetch (one LDS.128 per 4 FMAs per lane) caps the loop at
// ~20 % of the FP32 pipe; a tcgen05.ld.32x32b.x4 at a warp-uniform TMEM column
// delivers the same 16 bytes per lane at about twice the rate (loop ceiling
// ~40 %, tools/micro/tmgather.cu).  TMEM is not a TMA destination, so a tile
// goes global -> shared memory (2-D TMA box [KC x 128]) -> TMEM
// (tcgen05.cp.32x128b.warpx4: one 512-byte tile row is copied into the same
// 4 columns of all four 32-lane quarters, so every warp sees the whole tile in
// its own lanes; lane t of any quarter holds in[c][b0 + 4t .. 4t+3] in
// columns 4c..4c+3 of the buffer).
//
// Geometry: a CTA is 32 warps x 4 rows (RB = 128 rows, tiled by the
// nnz-balanced placement) x 128 batch columns; the inner dimension runs in
// column blocks of KC = 63 (a TMEM buffer = 4 zero columns, which padding
// entries address, + 63 x 4 tile columns = 256; two buffers fill the 512
// columns).  The CTA is persistent: it walks its items (row block, batch
// slice) = blockIdx.x, +gridDim.x, ... as one sequence of tiles, so the
// pipeline runs across item boundaries.  Three shared-memory stages hold the
// TMA'd tiles and their entries; two TMEM buffers hold the copies.  Whoever
// (last warp) releases TMEM buffer q&1 after tile q issues the copy of tile
// q+2 into it and the TMA of tile q+3 into tile q's (now free) stage.
//
// Every output element is produced by exactly one lane, entries ascending:
// no atomics, bitwise reproducible, the same per-element order at any B.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "sp_internal.cuh"
#include "tile.cuh"

namespace sp {
namespace {

constexpr int TM_BT = 128, TM_SMAX = 6;
constexpr int TM_KC = kTmKC;                          // 63 inner columns per tile
constexpr int TM_TILE_BYTES = TM_KC * TM_BT * 4;      // 32256
constexpr int TM_BUF = 256;                           // TMEM columns per buffer

struct TmArgs {
    int64_t rows, B;
    int nrb, nkb, nsl, nitems;
    int stage_bytes, nstage;
    int dbg;  // timing experiments only (SP_SPMM_TM_DBG): bit 0 skips the copies, bit 1 the entry loop
    const int32_t *seg;
    const int2 *ent;
    float *out;
    const float *gate;
    const int32_t *rowmap;
    long long *trace;  // dbg bit 2: per-tile clock64 stamps of CTA 0 (timing experiments only)
};

__device__ __forceinline__ void tmf_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmf_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// mbarrier wait that suspends the warp (time-limit hint) instead of spinning:
// waiting warps then take no issue slots from the computing ones
__device__ __forceinline__ void mbar_sleep_wait(uint64_t *bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred P;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1, %2;\n"
        "@!P bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(1000000u)
        : "memory");
}

// shared-memory descriptor of one 512-byte tile row seen as 32 rows x 16 bytes
// (no swizzle: 8-row core matrices 128 bytes apart = SBO; version 1)
__device__ __forceinline__ uint64_t row_desc(const void *p) {
    return (uint64_t)((smem_u32(p) >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 32) | ((uint64_t)1 << 46);
}

// 4 / 2 gathers of 16 bytes per lane from TMEM columns t[u], then one wait
__device__ __forceinline__ void tm_gather4(const uint32_t (&t)[4], float (&x)[4][4]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%16];\n"
        "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%4, %5, %6, %7}, [%17];\n"
        "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%8, %9, %10, %11}, [%18];\n"
        "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%12, %13, %14, %15}, [%19];\n"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(t[0]), "r"(t[1]), "r"(t[2]), "r"(t[3])
        : "memory");
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) x[u][v] = __uint_as_float(r[4 * u + v]);
}
__device__ __forceinline__ void tm_gather8(const uint32_t (&t)[8], float (&x)[8][4]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%32];\n"
        "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%4, %5, %6, %7}, [%33];\n"
        "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%8, %9, %10, %11}, [%34];\n"
        "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%12, %13, %14, %15}, [%35];\n"
        "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%16, %17, %18, %19}, [%36];\n"
        "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%20, %21, %22, %23}, [%37];\n"
        "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%24, %25, %26, %27}, [%38];\n"
        "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%28, %29, %30, %31}, [%39];\n"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(t[0]), "r"(t[1]), "r"(t[2]), "r"(t[3]), "r"(t[4]), "r"(t[5]), "r"(t[6]), "r"(t[7])
        : "memory");
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) x[u][v] = __uint_as_float(r[4 * u + v]);
}
__device__ __forceinline__ void tm_gather2(uint32_t t0, uint32_t t1, float (&x)[4][4]) {
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

template <int EPI, int NC, int NP, int TM_RPW>
__global__ void __launch_bounds__((NC + NP) * 32, 1)
    spmm_tm_kernel(const TmArgs a, const __grid_constant__ CUtensorMap tmap) {
    constexpr int RB = NC * TM_RPW;
    const int TM_S = a.nstage;
    extern __shared__ __align__(1024) unsigned char smraw[];
    __shared__ uint64_t sfull[TM_SMAX], tfull[2], tempty[2];
    __shared__ uint32_t tmem_base;

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nkb = a.nkb;
    const int my_items = (a.nitems - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
    const int ntile = my_items * nkb;

    // tile q of this CTA -> item (row block rb, batch slice sl), column block kb
    auto decode = [&](int q, int &rb, int &sl, int &kb) {
        const int k = q / nkb;
        kb = q - k * nkb;
        const int item = (int)blockIdx.x + k * (int)gridDim.x;
        sl = item / a.nrb;
        rb = item - sl * a.nrb;
    };
    auto stage = [&](int s) { return smraw + (size_t)s * a.stage_bytes; };
    // TMA of tile q (activation box + its entries) into stage q % S (one thread)
    auto issue_tma = [&](int q) {
        int rb, sl, kb;
        decode(q, rb, sl, kb);
        const int s = q % TM_S;
        const int64_t tb = ((int64_t)rb * nkb + kb) * RB;
        const int e0 = __ldg(a.seg + tb) & ~1, e1 = __ldg(a.seg + tb + RB);
        const unsigned eb = (unsigned)(((e1 - e0) * 8 + 15) & ~15);
        constexpr unsigned sb = (RB + 4) * 4;  // the tile's RB + 1 segment bounds (16-byte multiple)
        mbar_arrive_expect_tx(&sfull[s], (unsigned)TM_TILE_BYTES + sb + eb);
        tma_load_2d(stage(s), &tmap, sl * TM_BT, kb * TM_KC, &sfull[s]);
        tma_load_1d(stage(s) + TM_TILE_BYTES, a.seg + tb, sb, &sfull[s]);
        if (eb) tma_load_1d(stage(s) + TM_TILE_BYTES + sb, a.ent + e0, eb, &sfull[s]);
    };

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (threadIdx.x == 32) {
        for (int s = 0; s < TM_S; ++s) mbar_init(&sfull[s], 1);
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], NP);   // one commit per producer warp
            mbar_init(&tempty[b], NC);  // one arrive per compute warp
        }
        fence_mbar_init();
    }
    tmf_before();
    __syncthreads();
    tmf_after();
    const uint32_t tq = tmem_base + ((uint32_t)(32 * (warp & 3)) << 16);
    if (warp < 4) {  // the zero columns in front of each buffer (padding entries read them)
        asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %1, %1, %1};" ::"r"(tq), "r"(0u) : "memory");
        asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %1, %1, %1};" ::"r"(tq + TM_BUF), "r"(0u)
                     : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    tmf_before();
    __syncthreads();
    tmf_after();

    if (warp >= NC) {
        // ---- producer warps: lane 0 of each copies its share (rows p, p+NP, ...)
        // of every tile from shared memory into TMEM; producer 0 also issues
        // the TMA loads, S tiles ahead of the copies
        const int p = warp - NC;
        if (lane == 0) {
            if (p == 0)
                for (int q = 0; q < TM_S && q < ntile; ++q) issue_tma(q);
            for (int q = 0; q < ntile; ++q) {
                const int b = q & 1, s = q % TM_S;
                if (q >= 2) {
                    mbar_sleep_wait(&tempty[b], (unsigned)((q - 2) >> 1) & 1u);  // tile q-2 released buffer b
                    if ((a.dbg & 4) && blockIdx.x == 0 && p == 0 && q < 64) a.trace[q * 40 + 32] = clock64();
                    if (p == 0 && q - 2 + TM_S < ntile) issue_tma(q - 2 + TM_S);  // and its stage
                }
                mbar_sleep_wait(&sfull[s], (unsigned)(q / TM_S) & 1u);
                tmf_after();
                if ((a.dbg & 4) && blockIdx.x == 0 && p == 0 && q < 64) a.trace[q * 40 + 33] = clock64();
                const uint32_t dst = tmem_base + (uint32_t)(b * TM_BUF + 4);
                const unsigned char *src = stage(s);
                if (!(a.dbg & 1))
                for (int c = p; c < TM_KC; c += NP)
                    asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(dst + 4 * c),
                                 "l"(row_desc(src + c * 512))
                                 : "memory");
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 smem_u32(&tfull[b]))
                             : "memory");
            }
        }
    } else {
        // ---- compute warps: 4 rows each, gathers from TMEM
        float acc[TM_RPW][4];
        int kb = 0, item = (int)blockIdx.x;
        int sl = item / a.nrb, rb = item - sl * a.nrb;
        for (int q = 0; q < ntile; ++q) {
            const int b = q & 1, s = q % TM_S;
            if (kb == 0) {
#pragma unroll
                for (int i = 0; i < TM_RPW; ++i)
#pragma unroll
                    for (int v = 0; v < 4; ++v) acc[i][v] = 0.f;
            }
            mbar_sleep_wait(&tfull[b], (unsigned)(q >> 1) & 1u);
            mbar_sleep_wait(&sfull[s], (unsigned)(q / TM_S) & 1u);  // bounds + entries of tile q (TMA -> smem)
            tmf_after();
            if ((a.dbg & 4) && blockIdx.x == 0 && lane == 0 && q < 64) a.trace[q * 40 + warp] = clock64();
            const int32_t *sb = reinterpret_cast<const int32_t *>(stage(s) + TM_TILE_BYTES);
            const int ea = sb[0] & ~1;
            const int sg = lane <= TM_RPW ? sb[warp * TM_RPW + lane] : 0;
            const int2 *es = reinterpret_cast<const int2 *>(stage(s) + TM_TILE_BYTES + (RB + 4) * 4) - ea;
            const uint32_t tcol = tq + (uint32_t)(b * TM_BUF + 4);
#pragma unroll
            // rows in pairs: the first 4 slots of both rows' segments are fetched
            // together (8 gathers in flight, no branches: slots past a segment's
            // end read the zero columns with weight 0); longer segments finish in
            // groups of 4 and a last lone pair (segments have even lengths)
            auto rest = [&](float (&ac)[4], int s0, int s1) {
                for (int e = s0 + 4; e < s1; e += 4) {
                    const int4 p01 = *reinterpret_cast<const int4 *>(es + e);
                    float x[4][4];
                    if (e + 2 < s1) {
                        const int4 p23 = *reinterpret_cast<const int4 *>(es + e + 2);
                        const uint32_t t[4] = {tcol + (uint32_t)(p01.x >> 7), tcol + (uint32_t)(p01.z >> 7),
                                               tcol + (uint32_t)(p23.x >> 7), tcol + (uint32_t)(p23.z >> 7)};
                        tm_gather4(t, x);
                        fma_bcast<4>(ac, __int_as_float(p01.y), x[0]);
                        fma_bcast<4>(ac, __int_as_float(p01.w), x[1]);
                        fma_bcast<4>(ac, __int_as_float(p23.y), x[2]);
                        fma_bcast<4>(ac, __int_as_float(p23.w), x[3]);
                    } else {
                        tm_gather2(tcol + (uint32_t)(p01.x >> 7), tcol + (uint32_t)(p01.z >> 7), x);
                        fma_bcast<4>(ac, __int_as_float(p01.y), x[0]);
                        fma_bcast<4>(ac, __int_as_float(p01.w), x[1]);
                    }
                }
            };
#pragma unroll
            for (int i = 0; i < TM_RPW; i += 2) {
                if (a.dbg & 2) break;
                const int s0 = __shfl_sync(kFull, sg, i), s1 = __shfl_sync(kFull, sg, i + 1),
                          s2 = __shfl_sync(kFull, sg, i + 2);
                const int n0 = s1 - s0, n1 = s2 - s1;
                const int4 a01 = *reinterpret_cast<const int4 *>(es + s0);
                const int4 a23 = *reinterpret_cast<const int4 *>(es + s0 + 2);
                const int4 b01 = *reinterpret_cast<const int4 *>(es + s1);
                const int4 b23 = *reinterpret_cast<const int4 *>(es + s1 + 2);
                const uint32_t t[8] = {tcol + (uint32_t)((n0 > 0 ? a01.x : -512) >> 7),
                                       tcol + (uint32_t)((n0 > 1 ? a01.z : -512) >> 7),
                                       tcol + (uint32_t)((n0 > 2 ? a23.x : -512) >> 7),
                                       tcol + (uint32_t)((n0 > 3 ? a23.z : -512) >> 7),
                                       tcol + (uint32_t)((n1 > 0 ? b01.x : -512) >> 7),
                                       tcol + (uint32_t)((n1 > 1 ? b01.z : -512) >> 7),
                                       tcol + (uint32_t)((n1 > 2 ? b23.x : -512) >> 7),
                                       tcol + (uint32_t)((n1 > 3 ? b23.z : -512) >> 7)};
                float x[8][4];
                tm_gather8(t, x);
                fma_bcast<4>(acc[i], __int_as_float(n0 > 0 ? a01.y : 0), x[0]);
                fma_bcast<4>(acc[i], __int_as_float(n0 > 1 ? a01.w : 0), x[1]);
                fma_bcast<4>(acc[i], __int_as_float(n0 > 2 ? a23.y : 0), x[2]);
                fma_bcast<4>(acc[i], __int_as_float(n0 > 3 ? a23.w : 0), x[3]);
                fma_bcast<4>(acc[i + 1], __int_as_float(n1 > 0 ? b01.y : 0), x[4]);
                fma_bcast<4>(acc[i + 1], __int_as_float(n1 > 1 ? b01.w : 0), x[5]);
                fma_bcast<4>(acc[i + 1], __int_as_float(n1 > 2 ? b23.y : 0), x[6]);
                fma_bcast<4>(acc[i + 1], __int_as_float(n1 > 3 ? b23.w : 0), x[7]);
                rest(acc[i], s0, s1);
                rest(acc[i + 1], s1, s2);
            }
            // release TMEM buffer b and tile q's stage
            tmf_before();
            __syncwarp();
            if ((a.dbg & 4) && blockIdx.x == 0 && lane == 0 && q < 64) a.trace[q * 40 + 16 + warp] = clock64();
            if (lane == 0) mbar_arrive(&tempty[b]);

            if (kb == nkb - 1) {  // item done: ReLU / ReLU' gate fused, each element written once
                const int64_t bl = (int64_t)sl * TM_BT + lane * 4;
                if (bl < a.B) {
#pragma unroll
                    for (int i = 0; i < TM_RPW; ++i) {
                        const int64_t tpos = (int64_t)rb * RB + warp * TM_RPW + i;
                        const int64_t r = a.rowmap ? (int64_t)__ldg(a.rowmap + tpos) : tpos;
                        if (r < 0 || r >= a.rows) continue;
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
            }
            if (++kb == nkb) {  // next item
                kb = 0;
                item += (int)gridDim.x;
                sl = item / a.nrb;
                rb = item - sl * a.nrb;
            }
        }
    }

    tmf_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
}

constexpr int kSmemOptin = 227 * 1024;

}  // namespace

// SP_SPMM_TM=1 forces the TMEM-gather SpMM, =0 disables it; default: on.
int spmm_tm_mode() {
    static const int v = [] {
        const char *e = getenv("SP_SPMM_TM");
        return e ? (e[0] == '1' ? 1 : 0) : -1;
    }();
    return v;
}

// variant 0: 28 compute warps x 4 rows (RB = 112) + 4 copy warps; 1: 24 x 4
// (RB = 96) + 8; 2: 16 x 8 (RB = 128) + 8.  SP_SPMM_TM_VAR picks (default 0).
static int spmm_tm_var() {
    static const int v = [] {
        const char *e = getenv("SP_SPMM_TM_VAR");
        return e ? atoi(e) : 0;
    }();
    return v;
}

bool launch_spmm_tm(const sp_weight_s *w, int orient, int64_t B, const float *in, float *out, const float *gate,
                    int epi, cudaStream_t st) {
    const int var = std::min(std::max(spmm_tm_var(), 0), 3);
    const sp_tiling &t = w->til_t[orient][var];
    if ((B & 3) != 0 || t.seg == nullptr || t.nrb == 0 || t.nkb == 0) return false;
    const int cap = (t.max_tile + 8 + 3) & ~3;  // + the 4 masked slots a last row's first group reads
    const int stage_bytes = (TM_TILE_BYTES + (256 + 4) * 4 + cap * 8 + 127) & ~127;  // tile, bounds, entries
    const int nstage = std::min<int>(TM_SMAX, (kSmemOptin - 1024) / stage_bytes);
    if (nstage < 3) return false;
    const size_t smem = (size_t)nstage * stage_bytes;
    const int64_t nsl = (B + TM_BT - 1) / TM_BT;
    const int64_t nitems = (int64_t)t.nrb * nsl;
    if (nitems > INT32_MAX / 2 || nitems * t.nkb > INT32_MAX / 2) return false;
    CUtensorMap tmap{};
    if (!make_tmap_2d(&tmap, in, t.inner, B, TM_BT, TM_KC)) return false;
    refresh_if_stale(w, t, st);
    static const int dbg = [] {
        const char *e = getenv("SP_SPMM_TM_DBG");
        return e ? atoi(e) : 0;
    }();
    static long long *trace = nullptr;
    if ((dbg & 4) && !trace) {
        cudaMalloc(&trace, 64 * 40 * sizeof(long long));
        cudaMemset(trace, 0, 64 * 40 * sizeof(long long));
    }
    TmArgs a{t.rows, B, t.nrb, t.nkb, (int)nsl, (int)nitems, stage_bytes, nstage, dbg, t.seg, t.ent, out, gate,
             t.rowmap, trace};
    int nsm = 148;
    {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    }
    const unsigned grid = (unsigned)std::min<int64_t>(nitems, nsm);
    auto launch = [&](auto kern, int nthr) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        count_launches(1);
        note_path("spmm_tm");
        kern<<<grid, nthr, smem, st>>>(a, tmap);
    };
#define SP_TM_LAUNCH(NC, NP, RPW)                                                       \
    do {                                                                                \
        if (epi == EPI_RELU) launch(spmm_tm_kernel<EPI_RELU, NC, NP, RPW>, (NC + NP) * 32); \
        else if (epi == EPI_GATE) launch(spmm_tm_kernel<EPI_GATE, NC, NP, RPW>, (NC + NP) * 32); \
        else launch(spmm_tm_kernel<EPI_NONE, NC, NP, RPW>, (NC + NP) * 32);             \
    } while (0)
    if (var == 0) SP_TM_LAUNCH(28, 4, 4);
    else if (var == 1) SP_TM_LAUNCH(24, 8, 4);
    else if (var == 2) SP_TM_LAUNCH(16, 4, 8);
    else SP_TM_LAUNCH(16, 4, 16);
#undef SP_TM_LAUNCH
    if (dbg & 4) {  // print CTA 0's per-tile stamps (cycles relative to tile 0's first wait-done)
        long long h[64 * 40];
        cudaStreamSynchronize(st);
        cudaMemcpy(h, trace, sizeof(h), cudaMemcpyDeviceToHost);
        const long long t0 = h[0];
        for (int q = 0; q < 64; ++q) {
            long long wmin = h[q * 40], wmax = h[q * 40], dmin = h[q * 40 + 16], dmax = h[q * 40 + 16];
            for (int k = 1; k < 16; ++k) {
                wmin = std::min(wmin, h[q * 40 + k]);
                wmax = std::max(wmax, h[q * 40 + k]);
                dmin = std::min(dmin, h[q * 40 + 16 + k]);
                dmax = std::max(dmax, h[q * 40 + 16 + k]);
            }
            fprintf(stderr, "tile %2d: start %7lld..%7lld done %7lld..%7lld | prod tempty %7lld sfull %7lld\n", q,
                    wmin - t0, wmax - t0, dmin - t0, dmax - t0, h[q * 40 + 32] ? h[q * 40 + 32] - t0 : 0,
                    h[q * 40 + 33] - t0);
        }
    }
    return true;
}

}  // namespace sp
