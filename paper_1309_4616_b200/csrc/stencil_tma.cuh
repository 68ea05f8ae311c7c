// TMA-pipelined stencil pass (v2): the hot path on sm_100a.
//
// One producer warp streams the slab through a ring of shared-memory stages
// with cp.async.bulk.tensor (TMA) and mbarrier transaction counts; eight
// consumer warps compute from shared memory only.  A stage j holds
//   W(j): the w_{k-1} plane (3D) / row (2D) j of this CTA's tile with a
//         one-point halo (x from x0-2 so the centre columns stay 16-byte
//         aligned), out-of-bounds parts zero-filled by TMA (= homogeneous
//         Dirichlet ghosts);
//   P(j), G(j): p_{k-1} and the Rosenbrock diagonal of the tile's points.
// The march-axis ghosts (plane/row -1 and L) are produced by re-targeting
// the TMA coordinate (periodic wrap, Neumann clamp) or left to the zero fill;
// in-plane Neumann / periodic ghosts are patched by the consumer.  Data in
// flight is bounded by the ring depth, not by registers, which is what the
// register-queue v1 kernel ran out of (25% warps active, latency bound).
//
// 3D tile: 64 x 8 points (thread (q, r) owns x = x0 + 2q, 2q+1 of row r);
// 2D tile: 512 x 1 (warps own 64-wide segments), marching y.
#pragma once

#include <cuda.h>

#include "series.cuh"

namespace es {

template <bool DIM3>
struct TShape;
template <>
struct TShape<true> {
    static constexpr int TX = 64, TY = 8, WR = TY + 2, WROW = TX + 4, PR = TY;
};
template <>
struct TShape<false> {
    static constexpr int TX = 512, TY = 1, WR = 1, WROW = TX + 4, PR = 1;
};

constexpr int TMA_CONSUMER_WARPS = 8;
// device-internal coefficient kind: the sampled D array (ES_COEFF_ARRAY)
// streamed by TMA through the second slot of the PG ring (the g' slot; only
// without a g' diagonal) instead of per-thread loads
constexpr int ES_COEFF_STAGED = 3;
constexpr int TMA_THREADS = 32 * (TMA_CONSUMER_WARPS + 1);

// tensor maps of one pass; for 2D, W needs two maps (256-wide and 4-wide
// boxes: TMA boxes are at most 256 elements per dimension)
// MAP_HLO_1 / MAP_HHI_1: the second parity of the peer-memory slab series'
// double-buffered halo planes (node k reads parity k & 1)
enum {
    MAP_WA_V = 0, MAP_WB_V, MAP_WA_0, MAP_WB_0, MAP_WA_1, MAP_WB_1, MAP_P_0, MAP_P_1, MAP_G, MAP_HLO, MAP_HHI,
    MAP_HLO_1, MAP_HHI_1,
    // two-node pass (stencil_tb.cuh): w tiles with a two-point halo, g' tiles with a one-point halo
    MAP_T_V, MAP_T_0, MAP_T_1, MAP_T_G, MAP_T_PV,
    // two-node pass on a peer-memory slab: two-plane w halos by parity, g' boundary planes
    MAP_T_HLO0, MAP_T_HLO1, MAP_T_HHI0, MAP_T_HHI1, MAP_T_GLO, MAP_T_GHI, MAP_T_P0, MAP_T_P1,
    // two-node 2D pass (stencil_tb2d.cuh): 8-wide tails of the w rows, the 4-wide tail of the staged D
    MAP_T2_W8_V, MAP_T2_W8_0, MAP_T2_W8_1, MAP_T2_G4,
    // two-node pass (TB_GP): g' interior tiles riding in the P stages
    MAP_T_GP,
    // two-node 2D pass, R8 row view (8, nx/8, ny): w windows (v, wbuf[0], wbuf[1]), D window,
    // p rows (v, pbuf[0], pbuf[1]), D row interior
    MAP_T2R_W_V, MAP_T2R_W_0, MAP_T2R_W_1, MAP_T2R_G, MAP_T2R_P_V, MAP_T2R_P_0, MAP_T2R_P_1, MAP_T2R_D,
    // ... with R-row stages (stencil_tb2r.cuh): the same arrays, boxes of T3_R rows
    MAP_T3_W_V, MAP_T3_W_0, MAP_T3_W_1, MAP_T3_G, MAP_T3_P_V, MAP_T3_P_0, MAP_T3_P_1, MAP_T3_D, MAP_COUNT
};

struct alignas(64) TmaMaps {
    CUtensorMap m[MAP_COUNT];
};

// Two rings: W (the w_{k-1} stencil tiles; a plane stays resident while it is
// the zm / c / zp of three consecutive outputs) and PG (p_{k-1} and g' tiles,
// one output each).  Depths are chosen so three CTAs fit an SM and each ring
// keeps ~3 stages of prefetch in flight.
template <bool DIM3, bool PG, bool GD>
struct TLayout {
    using T = TShape<DIM3>;
    static constexpr int SW = DIM3 ? 6 : 8;
    static constexpr int SP = PG ? (GD ? 4 : 6) : 0;
    static constexpr int W_BYTES = T::WR * T::WROW * 8;
    static constexpr int W_STAGE = (W_BYTES + 127) & ~127;
    static constexpr int P_BYTES = T::PR * T::TX * 8;
    static constexpr int PG_STAGE = (GD ? 2 : 1) * P_BYTES;
    static constexpr int W_RING = SW * W_STAGE;
    static constexpr int PG_RING = SP * PG_STAGE;
    static constexpr int BAR_OFF = W_RING + PG_RING;
    static constexpr int ITEMQ_OFF = BAR_OFF + 2 * (SW + SP) * 8;  // int per W stage
    static constexpr int RED_OFF = ITEMQ_OFF + ((SW * 4 + 15) & ~15);
};

// ----- PTX helpers ----------------------------------------------------------

ES_DEV uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

ES_DEV void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(count) : "memory");
}
ES_DEV void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
ES_DEV void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(bar)) : "memory");
}
#ifndef ES_MBAR_HINT
#define ES_MBAR_HINT 0  // try_wait suspend-time hint in ns (0: the system limit)
#endif
ES_DEV void mbar_wait(uint64_t *bar, uint32_t parity) {
    const uint32_t a = su32(bar);
    uint32_t ok = 0;
    do {
        if constexpr (ES_MBAR_HINT > 0) {
            asm volatile(
                "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0, 1, 0, p; }"
                : "=r"(ok)
                : "r"(a), "r"(parity), "n"(ES_MBAR_HINT)
                : "memory");
        } else {
            asm volatile(
                "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                : "=r"(ok)
                : "r"(a), "r"(parity)
                : "memory");
        }
    } while (!ok);
}
// mbar_wait for warps off the critical path (a ring's producer, the marching
// kernels' edge warps): try_wait with a suspend-time hint, so a waiting warp
// sleeps until the phase completes instead of re-issuing the probe (the spin
// took ~14-26 % of the issue slots of the marching passes)
#ifndef ES_MBAR_SLEEP_NS
#define ES_MBAR_SLEEP_NS 20000
#endif
ES_DEV void mbar_wait_sleep(uint64_t *bar, uint32_t parity) {
    const uint32_t a = su32(bar);
    uint32_t ok = 0;
    do {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0, 1, 0, p; }"
            : "=r"(ok)
            : "r"(a), "r"(parity), "n"(ES_MBAR_SLEEP_NS)
            : "memory");
    } while (!ok);
}
ES_DEV void tma_acquire(const CUtensorMap *m) {
    asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(m) : "memory");
}
ES_DEV void tma_load(void *dst, const CUtensorMap *m, uint64_t *bar, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            su32(dst)),
        "l"(m), "r"(su32(bar)), "r"(x), "r"(y)
        : "memory");
}
ES_DEV void tma_load(void *dst, const CUtensorMap *m, uint64_t *bar, int x, int y, int z) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
        "[%2];" ::"r"(su32(dst)),
        "l"(m), "r"(su32(bar)), "r"(x), "r"(y), "r"(z)
        : "memory");
}

// march-axis source index of stage j (ghost handling; -1 / L are left to
// the TMA zero fill unless the mode says otherwise)
template <bool DIM3>
ES_DEV int march_src(const Geom &g, int j, int L) {
    if (j >= 0 && j < L) return j;
    if (g.mode == ES_MODE_PERIODIC) return j < 0 ? L - 1 : 0;
    if (g.mode == ES_MODE_NEUMANN) {
        const bool at = DIM3 ? (j < 0 ? g.at_lo : g.at_hi) : true;
        if (at) return j < 0 ? 0 : L - 1;
    }
    return j;
}

// Maps used by one pass (pointers into param or global memory).
struct PassMaps {
    const CUtensorMap *wa, *wb, *p, *g;
    const CUtensorMap *hlo = nullptr, *hhi = nullptr;  // slab halo planes (3D, multi-GPU)
};

// Work items: (chunk, tile), chunk-major so all CTAs sweep the planes
// together (neighbour tiles' halo rows stay L2 resident); CTAs are
// persistent and take items round-robin, and their rings run continuously
// across items (no pipeline refill per item).
struct Items {
    int tiles_x, ntiles, nchunks, chunk_len, L;
};

template <bool DIM3>
ES_DEV Items items_of(const Geom &g, int chunk_len) {
    using T = TShape<DIM3>;
    Items it;
    it.tiles_x = (int)((g.nx + T::TX - 1) / T::TX);
    it.ntiles = DIM3 ? it.tiles_x * (int)((g.ny + T::TY - 1) / T::TY) : it.tiles_x;
    it.L = DIM3 ? (int)g.lz : (int)g.ny;
    it.chunk_len = chunk_len;
    it.nchunks = (it.L + chunk_len - 1) / chunk_len;
    return it;
}

struct Item {
    int chunk, tile, x0, y0, mb, me;
};

template <bool DIM3>
ES_DEV Item item_at(const Items &its, int i) {
    using T = TShape<DIM3>;
    Item r;
    r.chunk = i / its.ntiles;
    r.tile = i % its.ntiles;
    r.x0 = (r.tile % its.tiles_x) * T::TX;
    r.y0 = DIM3 ? (r.tile / its.tiles_x) * T::TY : 0;
    r.mb = r.chunk * its.chunk_len;
    r.me = min(its.L, r.mb + its.chunk_len);
    return r;
}

// Producer (one lane of warp 8).  Items are claimed from a global counter
// (work != nullptr: the concurrently processed items form one contiguous
// index window, so neighbour tiles' halo rows are still in L2) or taken
// round-robin; the item index travels to the consumers in a per-stage slot
// published by the stage's mbarrier.  A -1 slot ends the consumers' loop.
template <bool DIM3, bool PG, bool GD>
ES_DEV void tma_produce(const Geom &g, const Items &its, const PassMaps &mp, char *smem, bool load_p,
                        unsigned *work) {
    using Lt = TLayout<DIM3, PG, GD>;
    uint64_t *wfull = reinterpret_cast<uint64_t *>(smem + Lt::BAR_OFF);
    uint64_t *wempty = wfull + Lt::SW;
    uint64_t *pfull = wempty + Lt::SW;
    uint64_t *pempty = pfull + Lt::SP;
    volatile int *itemq = reinterpret_cast<volatile int *>(smem + Lt::ITEMQ_OFF);
    const bool use_pg = PG && (load_p || GD);
    uint32_t uw = 0, up = 0;
    const int total = its.ntiles * its.nchunks;
    int i = work ? (int)atomicAdd(work, 1u) : (int)blockIdx.x;
    while (i < total) {
        const Item it = item_at<DIM3>(its, i);
        int inext = -1;
        for (int j = it.mb - 1; j <= it.me; ++j, ++uw) {
            // claim the next item a few planes before this one ends: the
            // atomic's latency hides behind the ring, and a CTA never holds
            // more than the item it is about to start
            if (j == max(it.mb - 1, it.me - 3)) inext = work ? (int)atomicAdd(work, 1u) : i + (int)gridDim.x;
            const uint32_t s = uw % Lt::SW;
            if (uw >= (uint32_t)Lt::SW) mbar_wait(&wempty[s], ((uw / Lt::SW) - 1) & 1);
            char *st = smem + s * Lt::W_STAGE;
            itemq[s] = i;
            mbar_expect_tx(&wfull[s], Lt::W_BYTES);
            const int js = march_src<DIM3>(g, j, its.L);
            if constexpr (DIM3) {
                if (j < 0 && g.halo_lo)  // neighbour slab's last plane
                    tma_load(st, mp.hlo, &wfull[s], it.x0 - 2, it.y0 - 1);
                else if (j >= its.L && g.halo_hi)
                    tma_load(st, mp.hhi, &wfull[s], it.x0 - 2, it.y0 - 1);
                else
                    tma_load(st, mp.wa, &wfull[s], it.x0 - 2, it.y0 - 1, js);
            } else {
                tma_load(st, mp.wa, &wfull[s], it.x0 - 2, js);
                tma_load(st + 2048, mp.wa, &wfull[s], it.x0 + 254, js);
                tma_load(st + 4096, mp.wb, &wfull[s], it.x0 + 510, js);
            }
            // P/G of plane j-1 follow one W plane behind (the consumer needs
            // them together with W(j), its zp)
            const int jp = j - 1;
            if constexpr (PG) {
                if (use_pg && jp >= it.mb && jp < it.me) {
                    const uint32_t sp = up % Lt::SP;
                    if (up >= (uint32_t)Lt::SP) mbar_wait(&pempty[sp], ((up / Lt::SP) - 1) & 1);
                    char *pst = smem + Lt::W_RING + sp * Lt::PG_STAGE;
                    mbar_expect_tx(&pfull[sp], (load_p ? Lt::P_BYTES : 0) + (GD ? Lt::P_BYTES : 0));
                    if constexpr (DIM3) {
                        if (load_p) tma_load(pst, mp.p, &pfull[sp], it.x0, it.y0, jp);
                        if (GD) tma_load(pst + Lt::P_BYTES, mp.g, &pfull[sp], it.x0, it.y0, jp);
                    } else {
                        if (load_p) {
                            tma_load(pst, mp.p, &pfull[sp], it.x0, jp);
                            tma_load(pst + 2048, mp.p, &pfull[sp], it.x0 + 256, jp);
                        }
                        if (GD) {
                            tma_load(pst + Lt::P_BYTES, mp.g, &pfull[sp], it.x0, jp);
                            tma_load(pst + Lt::P_BYTES + 2048, mp.g, &pfull[sp], it.x0 + 256, jp);
                        }
                    }
                    ++up;
                }
            }
        }
        i = inext;
    }
    // end-of-work marker in the next W slot
    const uint32_t s = uw % Lt::SW;
    if (uw >= (uint32_t)Lt::SW) mbar_wait(&wempty[s], ((uw / Lt::SW) - 1) & 1);
    itemq[s] = -1;
    mbar_arrive(&wfull[s]);
}

// Consumers (warps 0..7): one point pair per thread per plane.  After each
// item they write its per-plane partial sums (LEJA) and run the reduction
// tickets among themselves (named barrier 1).
// Epilogues of a plain (non-Leja) pass.
enum { EPI_AXPY = 0, EPI_ROSPRO = 1 };

template <bool DIM3, int COEFF, bool GD, bool LEJA, bool PG, int EPI = EPI_AXPY>
ES_DEV void tma_consume(const Geom &g, const Pass &ps, const Items &its, char *smem,
                        const SeriesParams *P, int k) {
    using T = TShape<DIM3>;
    using Lt = TLayout<DIM3, PG, GD>;
    uint64_t *wfull = reinterpret_cast<uint64_t *>(smem + Lt::BAR_OFF);
    uint64_t *wempty = wfull + Lt::SW;
    uint64_t *pfull = wempty + Lt::SW;
    uint64_t *pempty = pfull + Lt::SP;
    const int t = threadIdx.x;
    const int lane = t & 31, warp = t >> 5;
    const int q = t % (T::TX / 2), r = t / (T::TX / 2);
    const int64_t plane = g.nx * g.ny;
    const int wcol = (DIM3 ? r + 1 : 0) * T::WROW + 2 + 2 * q;
    const int pidx = r * T::TX + 2 * q;
    const bool use_pg = PG && (ps.p_src != nullptr || GD);
    const volatile int *itemq = reinterpret_cast<const volatile int *>(smem + Lt::ITEMQ_OFF);
    uint32_t uw = 0, up = 0;
    unsigned long long gp_lo = ~0ull, gp_hi = 0ull, bad = ~0ull;  // EPI_ROSPRO

    auto wst = [&](uint32_t u) { return reinterpret_cast<const double *>(smem + (u % Lt::SW) * Lt::W_STAGE); };
    auto wwait = [&](uint32_t u) { mbar_wait(&wfull[u % Lt::SW], (u / Lt::SW) & 1); };
    auto wrelease = [&](uint32_t u) {  // one elected arrival per consumer warp
        __syncwarp();
        if (lane == 0) mbar_arrive(&wempty[u % Lt::SW]);
    };

    for (;;) {
        wwait(uw);
        const int i = itemq[uw % Lt::SW];
        if (i < 0) break;
        const Item it = item_at<DIM3>(its, i);
        const int64_t ix = it.x0 + 2 * q;
        const int64_t iy = DIM3 ? (int64_t)it.y0 + r : 0;
        const bool act = ix < g.nx && iy < g.ny;
        double ox2[2] = {1.0, 1.0}, dco[2] = {1.0, 1.0};
        if constexpr (COEFF == ES_COEFF_RADIAL) {
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const double x = axis_coord(ix + j, g.nx);
                ox2[j] = add(1.0, mul(x, x));
            }
            if (DIM3 && act) {
                const double y = axis_coord(iy, g.ny);
                dco[0] = radial_from_sq(ox2[0], y);
                dco[1] = radial_from_sq(ox2[1], y);
            }
        }
        const uint32_t u0 = uw;  // W counter of plane mb-1
        double acc_w = 0.0, acc_p = 0.0;  // this thread's sums over the item's planes
        wwait(u0 + 1);
        for (int m = it.mb; m < it.me; ++m) {
            const uint32_t um = u0 + (uint32_t)(m - it.mb);  // plane m-1
            wwait(um + 2);
            const double *Wm = wst(um), *Wc = wst(um + 1), *Wp = wst(um + 2);
            const double *Pc = nullptr;
            if constexpr (PG) {
                if (use_pg) {
                    mbar_wait(&pfull[up % Lt::SP], (up / Lt::SP) & 1);
                    Pc = reinterpret_cast<const double *>(smem + Lt::W_RING + (up % Lt::SP) * Lt::PG_STAGE);
                }
            }
            if (act) {
                const double2 c = *reinterpret_cast<const double2 *>(Wc + wcol);
                double xm0 = Wc[wcol - 1], xp1 = Wc[wcol + 2];
                double2 ym, yp, zm, zp;
                if constexpr (DIM3) {
                    ym = *reinterpret_cast<const double2 *>(Wc + wcol - T::WROW);
                    yp = *reinterpret_cast<const double2 *>(Wc + wcol + T::WROW);
                    zm = *reinterpret_cast<const double2 *>(Wm + wcol);
                    zp = *reinterpret_cast<const double2 *>(Wp + wcol);
                } else {
                    ym = *reinterpret_cast<const double2 *>(Wm + wcol);
                    yp = *reinterpret_cast<const double2 *>(Wp + wcol);
                    zm = make_double2(0.0, 0.0);
                    zp = zm;
                }
                const int64_t row_base = DIM3 ? ((int64_t)m * plane + iy * g.nx) : (int64_t)m * g.nx;
                if (g.mode != ES_MODE_ZERO) {  // in-plane ghosts the zero fill got wrong
                    const bool neu = g.mode == ES_MODE_NEUMANN;
                    if (ix == 0) xm0 = neu ? c.x : __ldg(ps.src + row_base + g.nx - 1);
                    if (ix + 2 == g.nx) xp1 = neu ? c.y : __ldg(ps.src + row_base);
                    if constexpr (DIM3) {
                        if (iy == 0)
                            ym = neu ? c : *reinterpret_cast<const double2 *>(ps.src + m * plane + (g.ny - 1) * g.nx + ix);
                        if (iy == g.ny - 1) yp = neu ? c : *reinterpret_cast<const double2 *>(ps.src + m * plane + ix);
                    } else {
                        zm = c;  // single-plane grid: z ghosts are the point itself
                        zp = c;
                    }
                }
                const double cc[2] = {c.x, c.y};
                const double xm[2] = {xm0, c.x}, xp[2] = {c.y, xp1};
                const double ymv[2] = {ym.x, ym.y}, ypv[2] = {yp.x, yp.y};
                const double zmv[2] = {zm.x, zm.y}, zpv[2] = {zp.x, zp.y};
                double yy = 0.0;
                if constexpr (COEFF == ES_COEFF_RADIAL && !DIM3) yy = axis_coord(m, g.ny);
                double2 pv = make_double2(0.0, 0.0), gv = make_double2(0.0, 0.0);
                if constexpr (LEJA) {
                    if (ps.p_src) pv = *reinterpret_cast<const double2 *>(Pc + pidx);
                }
                if constexpr (GD) gv = *reinterpret_cast<const double2 *>(Pc + Lt::P_BYTES / 8 + pidx);  // g' or D
                const double pvv[2] = {pv.x, pv.y}, gvv[2] = {gv.x, gv.y};
                double wn[2], pn[2];
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    double lap = lap7(cc[j], xm[j], xp[j], ymv[j], ypv[j], zmv[j], zpv[j], g.wx, g.wy, g.wz);
                    if constexpr (COEFF == ES_COEFF_RADIAL) lap = mul(DIM3 ? dco[j] : radial_from_sq(ox2[j], yy), lap);
                    if constexpr (COEFF == ES_COEFF_ARRAY) lap = mul(__ldg(g.coeff + row_base + ix + j), lap);
                    if constexpr (COEFF == ES_COEFF_STAGED) lap = mul(gvv[j], lap);
                    if constexpr (GD && COEFF != ES_COEFF_STAGED) lap = sub(lap, mul(gvv[j], cc[j]));
                    wn[j] = add(mul(ps.alpha, lap), mul(ps.beta, cc[j]));
                    if constexpr (LEJA) {
                        const double pold = ps.p_src ? pvv[j] : mul(ps.d0, cc[j]);
                        pn[j] = add(pold, mul(ps.dk, wn[j]));
                    }
                }
                const int64_t o = row_base + ix;
                if constexpr (EPI == EPI_ROSPRO) {
                    // F = g(u) - A u and g'(u) in the same pass (build-defined
                    // Rosenbrock prologue; same expressions as k_combustion,
                    // k_combustion_jac and the alpha=1, beta=0 apply)
                    double fv[2], gpv[2];
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        const double x = cc[j];
                        const double rr = __drcp_rn(x);  // = div(1.0, x), correctly rounded either way
                        const double e = exp(mul(20.0, sub(1.0, rr)));
                        const double gval = mul(mul(0.25, sub(2.0, x)), e);
                        const double q = mul(mul(5.0, sub(2.0, x)), mul(rr, rr));
                        gpv[j] = mul(e, sub(q, 0.25));
                        fv[j] = sub(gval, wn[j]);
                        const unsigned long long od = ord(gpv[j]);
                        gp_lo = od < gp_lo ? od : gp_lo;
                        gp_hi = od > gp_hi ? od : gp_hi;
                        if (x <= 0.0 && (unsigned long long)(o + j) < bad) bad = (unsigned long long)(o + j);
                    }
                    *reinterpret_cast<double2 *>(ps.dst + o) = make_double2(fv[0], fv[1]);
                    *reinterpret_cast<double2 *>(ps.p_dst + o) = make_double2(gpv[0], gpv[1]);
                } else {
                    *reinterpret_cast<double2 *>(ps.dst + o) = make_double2(wn[0], wn[1]);
                }
                if constexpr (LEJA) {
                    *reinterpret_cast<double2 *>(ps.p_dst + o) = make_double2(pn[0], pn[1]);
                    acc_w = add(acc_w, add(mul(wn[0], wn[0]), mul(wn[1], wn[1])));
                    acc_p = add(acc_p, add(mul(pn[0], pn[0]), mul(pn[1], pn[1])));
                }
            }
            wrelease(um);
            if constexpr (PG) {
                if (use_pg) {
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&pempty[up % Lt::SP]);
                    ++up;
                }
            }
        }
        const uint32_t L = (uint32_t)(it.me - it.mb);
        wrelease(u0 + L);      // planes me-1 and me
        wrelease(u0 + L + 1);
        uw = u0 + L + 2;
        if constexpr (LEJA) {
            // (chunk, tile, warp) partial: lane-sequential over the item's
            // planes, then the warp's xor tree; reduced by k_slice_reduce
            acc_w = warp_sum(acc_w);
            acc_p = warp_sum(acc_p);
            if (lane == 0) {
                double *dst = P->part + (((int64_t)it.chunk * its.ntiles + it.tile) * TMA_CONSUMER_WARPS + warp) * 2;
                dst[0] = acc_w;
                dst[1] = acc_p;
            }
        }
    }
    if constexpr (EPI == EPI_ROSPRO) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long a = __shfl_xor_sync(0xffffffffu, gp_lo, o);
            const unsigned long long b = __shfl_xor_sync(0xffffffffu, gp_hi, o);
            const unsigned long long c = __shfl_xor_sync(0xffffffffu, bad, o);
            gp_lo = a < gp_lo ? a : gp_lo;
            gp_hi = b > gp_hi ? b : gp_hi;
            bad = c < bad ? c : bad;
        }
        if (lane == 0) {
            atomicMin(ps.aux, gp_lo);
            atomicMax(ps.aux + 1, gp_hi);
            atomicMin(ps.aux + 2, bad);
        }
    }
}

// Shared-memory footprint of one CTA.
template <bool DIM3, bool PG, bool GD>
constexpr size_t tma_smem_bytes(int) {
    return (size_t)TLayout<DIM3, PG, GD>::RED_OFF;
}

// Whole pass for one persistent CTA: barrier set-up, warp-specialised streaming.
template <bool DIM3, int COEFF, bool GD, bool LEJA, int EPI = EPI_AXPY>
ES_DEV void tma_pass(const Geom &g, const Pass &ps, const PassMaps &mp, int chunk_len, bool acquire_maps,
                     char *smem, const SeriesParams *P, int k, unsigned *work) {
    constexpr bool PG = LEJA || GD;
    using Lt = TLayout<DIM3, PG, GD>;
    const Items its = items_of<DIM3>(g, chunk_len);
    if (threadIdx.x == 0) {
        uint64_t *bars = reinterpret_cast<uint64_t *>(smem + Lt::BAR_OFF);
        for (int s = 0; s < Lt::SW; ++s) {
            mbar_init(&bars[s], 1);
            mbar_init(&bars[Lt::SW + s], TMA_CONSUMER_WARPS);
        }
        for (int s = 0; s < Lt::SP; ++s) {
            mbar_init(&bars[2 * Lt::SW + s], 1);
            mbar_init(&bars[2 * Lt::SW + Lt::SP + s], TMA_CONSUMER_WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5;
    if (warp == TMA_CONSUMER_WARPS) {
        if ((threadIdx.x & 31) == 0) {
            if (acquire_maps) {
                if (g.halo_lo) tma_acquire(mp.hlo);
                if (g.halo_hi) tma_acquire(mp.hhi);
                tma_acquire(mp.wa);
                if (!DIM3) tma_acquire(mp.wb);
                if (LEJA && ps.p_src) tma_acquire(mp.p);
                if (GD) tma_acquire(mp.g);
            }
            tma_produce<DIM3, PG, GD>(g, its, mp, smem, LEJA && ps.p_src != nullptr, work);
        }
    } else {
        tma_consume<DIM3, COEFF, GD, LEJA, PG, EPI>(g, ps, its, smem, P, k);
    }
}

}  // namespace es
