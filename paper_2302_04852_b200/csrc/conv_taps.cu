// conv_taps.cu -- per-tap tilings of a sparse conv filter (host-side build,
// once per handle; off the timed path like sp_weight_create itself).
//
// Implicit im2col by taps: for a stride-1 conv with filter W[oc][ic][x][y],
// Eq. (3) (P224) is a sum over the KH*KW taps of sparse OC x IC matrices
// W_xy applied to a SHIFTED view of the spatially padded activation, so each
// tap is an ordinary SpMM / SDDMM on a column-shifted operand and pruned taps
// cost nothing (P248).  Each tap matrix gets the same row-block x column-block
// tiling as a linear layer, with its entries' vidx pointing at
// the conv handle's own CSR slots, so the weights are read from (and dW is
// written to) the handle's vals / dW in the paper's (oc, ic, x, y) order.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <thread>
#include <vector>

#include "sp_internal.cuh"

namespace sp {
namespace {

// Host build of one tiling from a row-compressed structure (rows ascending,
// idx ascending within a row) whose entries carry the CSR slot `slot`.
// Column block of a tap tiling: the inner dimension (a channel count) split into
// equal blocks of at most kTilKC[0] (256 -> 2 x 128 rather than 192 + 64, so no
// tile is mostly zero fill), a multiple of 8 rows.
static int even_kc(int64_t inner) {
    const int64_t nk = (inner + kTilKC[0] - 1) / kTilKC[0];
    const int64_t kc = (inner + nk - 1) / nk;
    return (int)std::max<int64_t>(8, (kc + 7) & ~7);
}

// one tiling built on the host: its arrays, then placed in the handle's tap arena
struct HostTiling {
    std::vector<int32_t> seg, vid, split;
    std::vector<int2> ent;
};

void tiling_from_host(int64_t rows, int64_t inner, int RB, int KC, const std::vector<int32_t> &ptr,
                      const std::vector<int32_t> &idx, const std::vector<int32_t> &slot, sp_tiling &t,
                      HostTiling &h) {
    t.RB = RB;
    t.KC = KC;
    t.rows = rows;
    t.inner = inner;
    t.nrb = (int)((rows + RB - 1) / RB);
    t.nkb = (int)((inner + KC - 1) / KC);
    const int64_t nseg = (int64_t)t.nrb * t.nkb * RB;
    std::vector<int32_t> cnt(nseg, 0);
    for (int64_t r = 0; r < rows; ++r) {
        const int64_t rb = r / RB, lr = r % RB;
        for (int32_t k = ptr[r]; k < ptr[r + 1]; ++k) {
            const int kb = idx[k] / KC;
            cnt[(rb * t.nkb + kb) * RB + lr]++;
        }
    }
    std::vector<int32_t> &seg = h.seg;
    seg.assign(nseg + 1, 0);
    for (int64_t i = 0; i < nseg; ++i) seg[i + 1] = seg[i] + ((cnt[i] + kTapPad - 1) & ~(kTapPad - 1));
    const int64_t npad = seg[nseg];
    h.ent.assign(npad + 8, make_int2(-kTilRowBytes, 0));
    h.vid.assign(npad + 8, -1);
    std::vector<int32_t> fill(nseg, 0);
    for (int64_t r = 0; r < rows; ++r) {
        const int64_t rb = r / RB, lr = r % RB;
        for (int32_t k = ptr[r]; k < ptr[r + 1]; ++k) {
            const int kb = idx[k] / KC;
            const int64_t sgi = (rb * t.nkb + kb) * RB + lr;
            const int64_t e = seg[sgi] + fill[sgi]++;
            h.ent[e] = make_int2((idx[k] - kb * KC) * kTilRowBytes, 0);
            h.vid[e] = slot[k];
        }
    }
    // tmsplit (TMEM-mirrored SpMM, spmm_sk.cu): the even entry index from which a
    // segment holds only columns >= KC - kHybTC of its block (padding comes last)
    h.split.clear();
    if (KC > kHybTC) {
        h.split.assign(nseg + 8, 0);
        const int off0 = (KC - kHybTC) * kTilRowBytes;
        for (int64_t i = 0; i < nseg; ++i) {
            int32_t sp = seg[i + 1];
            for (int32_t e = seg[i]; e < seg[i + 1]; ++e)
                if (h.ent[e].x >= off0) {
                    sp = e;
                    break;
                }
            sp = seg[i] + ((sp - seg[i] + 1) & ~1);
            h.split[i] = std::min(sp, seg[i + 1]);
        }
    }
    int32_t mx = 0;
    for (int64_t ti = 0; ti < (int64_t)t.nrb * t.nkb; ++ti) mx = std::max(mx, seg[(ti + 1) * RB] - seg[ti * RB]);
    t.max_tile = mx;
    t.npad = npad;
    t.cap_ent = npad + 8;
}

size_t al256(size_t n) { return (n + 255) & ~(size_t)255; }

}  // namespace

sp_status build_conv_taps(sp_weight_s *w, int OC, int IC, int KH, int KW, cudaStream_t st) {
    const int KK = KH * KW;
    w->conv_kh = KH;
    w->conv_kw = KW;
    if (KK > kMaxTaps) return SP_OK;  // larger filters use the direct conv kernels
    cudaStreamSynchronize(st);
    std::vector<int32_t> rp(OC + 1), ci(w->nnz);
    cudaMemcpy(rp.data(), w->row_ptr, (OC + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost);
    if (w->nnz) cudaMemcpy(ci.data(), w->col_idx, w->nnz * sizeof(int32_t), cudaMemcpyDeviceToHost);
    std::vector<TapDev> td(3 * kMaxTaps);
    std::vector<HostTiling> host(3 * (size_t)KK);
    constexpr int kFusedRB = 64, kFusedRPW = 2;  // fused conv backward: 32 warps x 2 rows
    std::vector<int64_t> wgroups((IC + kFusedRB - 1) / kFusedRB * (kFusedRB / kFusedRPW), 0);
    std::vector<int64_t> wgroups8(wgroups.size(), 0);
    // the taps' host builds are independent: one thread per tap
    std::vector<std::vector<int64_t>> wg_tap(KK, std::vector<int64_t>(wgroups.size(), 0)), wg8_tap = wg_tap;
    auto build_tap = [&](int tp) {
        std::vector<int64_t> &wgroups = wg_tap[tp], &wgroups8 = wg8_tap[tp];
        // rows oc, inner ic  (entries in (oc, ic) order: col_idx ascending)
        std::vector<int32_t> p0(OC + 1, 0), i0, s0;
        // rows ic, inner oc
        std::vector<std::vector<std::pair<int32_t, int32_t>>> cols(IC);
        for (int oc = 0; oc < OC; ++oc) {
            for (int32_t j = rp[oc]; j < rp[oc + 1]; ++j) {
                if (ci[j] % KK != tp) continue;
                const int ic = ci[j] / KK;
                i0.push_back(ic);
                s0.push_back(j);
                cols[ic].push_back({oc, j});
            }
            p0[oc + 1] = (int32_t)i0.size();
        }
        std::vector<int32_t> p1(IC + 1, 0), i1, s1;
        for (int ic = 0; ic < IC; ++ic) {
            for (auto &e : cols[ic]) {
                i1.push_back(e.first);
                s1.push_back(e.second);
            }
            p1[ic + 1] = (int32_t)i1.size();
        }
        tiling_from_host(OC, IC, kTilRB[0], even_kc(IC), p0, i0, s0, w->tap[tp][0], host[3 * tp + 0]);
        tiling_from_host(IC, OC, kTilRB[0], even_kc(OC), p1, i1, s1, w->tap[tp][1], host[3 * tp + 1]);
        tiling_from_host(IC, OC, kFusedRB, even_kc(OC), p1, i1, s1, w->tapf[tp], host[3 * tp + 2]);
        const sp_tiling &tf = w->tapf[tp];
        // entry groups per warp of 2 rows, summed over taps: groups of 4 (whole-warp
        // entries; segments have even length, so a last group may hold 2) and of 8
        // (half-warp entries)
        const int KCf = tf.KC;
        for (int ic = 0; ic < IC; ++ic) {
            std::vector<int32_t> cnt(tf.nkb, 0);
            for (int32_t k = p1[ic]; k < p1[ic + 1]; ++k) cnt[i1[k] / KCf]++;
            for (int kb = 0; kb < tf.nkb; ++kb)
            {
                const int64_t wi = (ic / kFusedRB) * (kFusedRB / kFusedRPW) + (ic % kFusedRB) / kFusedRPW;
                const int32_t n = (cnt[kb] + kTapPad - 1) & ~(kTapPad - 1);
                wgroups[wi] += (n + 3) / 4;
                wgroups8[wi] += (n + 7) / 8;  // half-warp fused backward: groups of 8
            }
        }
    };
    {
        std::vector<std::thread> th;
        for (int tp = 0; tp < KK; ++tp) th.emplace_back(build_tap, tp);
        for (auto &t : th) t.join();
    }
    for (int tp = 0; tp < KK; ++tp)
        for (size_t i = 0; i < wgroups.size(); ++i) {
            wgroups[i] += wg_tap[tp][i];
            wgroups8[i] += wg8_tap[tp][i];
        }
    w->tapf_groups = wgroups.empty() ? 0 : *std::max_element(wgroups.begin(), wgroups.end());
    w->tapf_groups8 = wgroups8.empty() ? 0 : *std::max_element(wgroups8.begin(), wgroups8.end());
    // every tap tiling and the TapDev table in ONE arena filled by ONE copy (it had
    // been 3-4 allocations and copies per tiling: 27 tilings for a 3 x 3 filter)
    auto tiling_of = [&](int k) -> sp_tiling & { return k % 3 == 2 ? w->tapf[k / 3] : w->tap[k / 3][k % 3]; };
    size_t bytes = al256(td.size() * sizeof(TapDev));
    for (int k = 0; k < 3 * KK; ++k) {
        const HostTiling &h = host[k];
        bytes += al256(h.seg.size() * 4) + al256(h.ent.size() * sizeof(int2)) + al256(h.vid.size() * 4) +
                 al256(h.split.size() * 4);
    }
    char *base = nullptr;
    if (scratch_alloc((void **)&base, bytes, st) != cudaSuccess) return SP_ERR_ALLOC;
    w->arena[3] = base;
    std::vector<char> hbuf(bytes, 0);
    size_t off = al256(td.size() * sizeof(TapDev));
    auto put = [&](const void *src, size_t n) -> char * {
        memcpy(hbuf.data() + off, src, n);
        char *d = base + off;
        off += al256(n);
        return d;
    };
    for (int k = 0; k < 3 * KK; ++k) {
        const HostTiling &h = host[k];
        sp_tiling &t = tiling_of(k);
        t.in_arena = true;
        t.seg = reinterpret_cast<int32_t *>(put(h.seg.data(), h.seg.size() * 4));
        t.ent = reinterpret_cast<int2 *>(put(h.ent.data(), h.ent.size() * sizeof(int2)));
        t.vidx = reinterpret_cast<int32_t *>(put(h.vid.data(), h.vid.size() * 4));
        t.tmsplit = h.split.empty() ? nullptr : reinterpret_cast<int32_t *>(put(h.split.data(), h.split.size() * 4));
        const int tp = k / 3, o = k % 3;
        td[o * kMaxTaps + tp] = TapDev{t.seg, t.ent, t.vidx, t.npad, t.tmsplit};
    }
    memcpy(hbuf.data(), td.data(), td.size() * sizeof(TapDev));
    w->tapdev = reinterpret_cast<TapDev *>(base);
    cudaMemcpyAsync(base, hbuf.data(), bytes, cudaMemcpyHostToDevice, st);
    return cudaStreamSynchronize(st) == cudaSuccess ? SP_OK : SP_ERR_CUDA;  // (hbuf lives until the copy is done)
}

}  // namespace sp
