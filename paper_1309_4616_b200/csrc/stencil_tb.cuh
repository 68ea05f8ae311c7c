// Two Newton-Leja nodes per pass over HBM (temporal blocking), 3D slabs.
//
// A node reads w_{k-1}, p_{k-1} (+ g') and writes w_k, p_k: 32 (40) B/point.
// Nodes k and k+1 fused into one pass read w_{k-1}, p_{k-1} (+ g') once and
// write p_k, w_{k+1}, p_{k+1}: 40 (48) B/point for TWO nodes.  w_k never
// leaves the SM: each 64x8 tile computes it on its tile plus a one-point
// ring (66x10, from w_{k-1} tiles with a two-point halo, 72x12) into a
// 4-plane shared-memory window, and node k+1 reads its stencil neighbours
// from there one plane later.  The ring is recomputed by neighbouring tiles
// with identical inputs and expression trees, so every value -- and every
// per-(chunk, tile, warp) norm partial, accumulated by the same thread in
// the same plane order as the one-node kernel -- is bitwise the one-node
// kernel's; the stopping test runs twice per pass (k, then k+1).
//
// Scope: homogeneous Dirichlet (TMA zero fill) and Neumann (mirrored ghosts)
// on one domain (periodic wrap and slab halos use the one-node kernel).
//
// Ring buffers (producer = warp 8, one lane):
//   W: w_{k-1} tiles of planes mb-2 .. me+1 (72x12, from x0-4, y0-2);
//   G: g' tiles of planes mb-1 .. me (68x10, from x0-2, y0-1; GD only);
//   P: p_{k-1} tiles of planes mb .. me-1 (64x8; v on the first pass);
//   V: w_k windows (68x10), written by warp group A, read by group C.
// Group A (warps 0-3), plane j = mb-1 .. me: w_k of plane j on the window.
// Group C (warps 4-7), plane j: p_k of plane j's interior, then w_{k+1},
// p_{k+1} of plane j-1's interior.
#pragma once

#include "stencil_tma.cuh"

namespace es {

// tile: 64 x TB_TY points; warp group A (TB_AW warps), C (TB_CW warps, two
// rows per thread), one producer warp.  64 x 8 with 4 + 4 warps runs two
// CTAs per SM; 64 x 16 with 7 + 8 runs one CTA of 16 warps (128 registers).
#ifndef TB_TY
#define TB_TY 16
#endif
#if TB_TY == 8
#define TB_AW_DEF 4
#define TB_CW_DEF 4
#define TB_MINB 2
#else
#define TB_AW_DEF 7
#define TB_CW_DEF 8
#define TB_MINB 1
#endif
constexpr int TB_AW = TB_AW_DEF, TB_CW = TB_CW_DEF;
static_assert(TB_TY == 2 * TB_CW, "group C threads own two rows each");
constexpr int TB_NA = 32 * TB_AW, TB_NC = 32 * TB_CW;
constexpr int TB_THREADS = 32 * (TB_AW + TB_CW + 1);
constexpr int TB_WX = 72, TB_WY = TB_TY + 4;  // w_{k-1}: x0-4 .. x0+67, y0-2 .. y0+TY+1
constexpr int TB_EX = 68, TB_EY = TB_TY + 2;  // w_k window: x0-2 .. x0+65 (even start: pair loads), y0-1 .. y0+TY
constexpr int TB_PAIRS = TB_EX / 2 * TB_EY;  // point pairs per window plane
constexpr int TB_APT = (TB_PAIRS + TB_NA - 1) / TB_NA;  // window pairs per group-A thread
static_assert(TB_APT == 3, "group A loop is written for three pairs per thread");
constexpr int TB_GX = 68, TB_GY = TB_TY + 2;  // g': x0-2 .. x0+65, y0-1 .. y0+TY
#ifndef TB_SV
#define TB_SV 5  // w_k window planes in flight between the warp groups (>= 4: j-2 .. j+1)
#endif
// TB_GP: group C's g' (interior of its output plane) rides in the P stage of
// that plane instead of the shared G ring, so G slots are released by group
// A alone and the ring no longer couples A to C's lag (A's top stall was the
// G-full wait); the G ring shrinks to pay for the larger P stages
#ifndef TB_GP
#define TB_GP 0  // measured slower (573 vs 556 us per 512^3 node; shallower G / P rings), kept as an option
#endif
#ifndef TB_SG
#define TB_SG (TB_GP ? 3 : 6)
#endif
#ifndef TB_SP
#define TB_SP 5
#endif
#ifndef TB_SW_GD
#if TB_TY == 8
#define TB_SW_GD 6
#else
#define TB_SW_GD 7
#endif
#endif
#ifndef TB_SW_NG
#define TB_SW_NG 9
#endif

template <bool GD>
struct TbLayout {
    // ring depths: two CTAs per SM (<= 113 KiB each) at 64 x 8; one CTA per
    // SM (<= 226 KiB) at 64 x 16
    static constexpr int SW = GD ? TB_SW_GD : TB_SW_NG, SG = GD ? TB_SG : 0, SP = TB_SP;
    static constexpr int W_STAGE = (TB_WX * TB_WY * 8 + 127) & ~127;
    static constexpr int G_STAGE = (TB_GX * TB_GY * 8 + 127) & ~127;
    static constexpr int P_PLANE = 64 * TB_TY * 8;                     // p_{k-1} tile
    static constexpr int P_STAGE = (GD && TB_GP ? 2 : 1) * P_PLANE;  // + g' tile of the same plane (TB_GP)
    static constexpr int V_SLOT = TB_EX * TB_EY * 8;
    static constexpr int W_OFF = 0;
    static constexpr int G_OFF = W_OFF + SW * W_STAGE;
    static constexpr int P_OFF = G_OFF + SG * G_STAGE;
    static constexpr int V_OFF = P_OFF + SP * P_STAGE;
    static constexpr int BAR_OFF = (V_OFF + TB_SV * V_SLOT + 7) & ~7;
    static constexpr int NBAR = 2 * (SW + SG + SP + TB_SV);
    static constexpr int ITEMQ_OFF = BAR_OFF + NBAR * 8;
    static constexpr int VITEM_OFF = ITEMQ_OFF + ((SW * 4 + 15) & ~15);
    static constexpr int BYTES = VITEM_OFF + ((TB_SV * 4 + 15) & ~15);  // one item slot per V slot
};

// Work items of the two-node pass: (z chunk, 64 x TB_TY tile), chunk-major.
// Norm partials keep the one-node kernel's (chunk, 64 x 8 tile, row) layout.
struct TbItems {
    int tiles_x, ntiles8, ntiles, nchunks, chunk_len, L;
    int edges_first;  // slab of a peer-memory series: both boundary chunks first (their halo pushes overlap the rest)
};

ES_DEV TbItems tb_items_of(const Geom &g, int chunk_len) {
    TbItems it;
    it.tiles_x = (int)((g.nx + 63) / 64);
    it.ntiles8 = it.tiles_x * (int)((g.ny + 7) / 8);
    it.ntiles = it.tiles_x * (int)((g.ny + TB_TY - 1) / TB_TY);
    it.L = (int)g.lz;
    it.chunk_len = chunk_len;
    it.nchunks = (it.L + chunk_len - 1) / chunk_len;
    it.edges_first = (g.halo_lo != nullptr || g.halo_hi != nullptr) && it.nchunks > 2;
    return it;
}

struct TbItem {
    int chunk, x0, y0, mb, me, tile8;  // tile8: one-node index of the 64 x 8 tile at row y0
};

ES_DEV TbItem tb_item_at(const TbItems &its, int i) {
    TbItem r;
    r.chunk = i / its.ntiles;
    if (its.edges_first) r.chunk = r.chunk == 0 ? 0 : r.chunk == 1 ? its.nchunks - 1 : r.chunk - 1;
    const int t = i % its.ntiles, tx = t % its.tiles_x, ty = t / its.tiles_x;
    r.x0 = tx * 64;
    r.y0 = ty * TB_TY;
    r.mb = r.chunk * its.chunk_len;
    r.me = min(its.L, r.mb + its.chunk_len);
    r.tile8 = (r.y0 / 8) * its.tiles_x + tx;
    return r;
}

struct TbMaps {
    const CUtensorMap *w, *g, *p;
    const CUtensorMap *gp = nullptr;  // g' interior tiles (64 x TB_TY) riding in the P stages (TB_GP)
    // peer-memory slabs: the neighbours' two w planes (this pass's parity) and g' planes, or null
    const CUtensorMap *hlo = nullptr, *hhi = nullptr, *glo = nullptr, *ghi = nullptr;
};

template <bool GD>
ES_DEV void tb_produce(const Geom &g, const TbItems &its, const TbMaps &mp, char *smem, bool load_p,
                       unsigned *work) {
    using Lt = TbLayout<GD>;
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + Lt::BAR_OFF);
    uint64_t *wfull = bar, *wempty = wfull + Lt::SW, *gfull = wempty + Lt::SW, *gempty = gfull + Lt::SG,
             *pfull = gempty + Lt::SG, *pempty = pfull + Lt::SP;
    volatile int *itemq = reinterpret_cast<volatile int *>(smem + Lt::ITEMQ_OFF);
    uint32_t uw = 0, ug = 0, up = 0;
    const int total = its.ntiles * its.nchunks;
    int i = work ? (int)atomicAdd(work, 1u) : (int)blockIdx.x;
    while (i < total) {
        const TbItem it = tb_item_at(its, i);
        int inext = -1;
        for (int t = it.mb - 2; t <= it.me + 1; ++t) {
            if (t == max(it.mb - 2, it.me - 3)) inext = work ? (int)atomicAdd(work, 1u) : i + (int)gridDim.x;
            {  // W(t)
                const uint32_t s = uw % Lt::SW;
                if (uw >= (uint32_t)Lt::SW) mbar_wait(&wempty[s], ((uw / Lt::SW) - 1) & 1);
                itemq[s] = i;
                mbar_expect_tx(&wfull[s], TB_WX * TB_WY * 8);
                char *dst = smem + Lt::W_OFF + s * Lt::W_STAGE;
                if (t < 0 && mp.hlo)  // planes -2, -1 from the lower neighbour
                    tma_load(dst, mp.hlo, &wfull[s], it.x0 - 4, it.y0 - 2, t + 2);
                else if (t >= its.L && mp.hhi)  // planes L, L+1 from the upper neighbour
                    tma_load(dst, mp.hhi, &wfull[s], it.x0 - 4, it.y0 - 2, t - its.L);
                else
                    tma_load(dst, mp.w, &wfull[s], it.x0 - 4, it.y0 - 2, march_src<true>(g, t, its.L));
                ++uw;
            }
            const int tg = t - 1;  // G(t-1), P(t-1): what consumer iteration t-1 needs besides W(t)
            if constexpr (GD) {
                if (tg >= it.mb - 1 && tg <= it.me) {
                    const uint32_t s = ug % Lt::SG;
                    if (ug >= (uint32_t)Lt::SG) mbar_wait(&gempty[s], ((ug / Lt::SG) - 1) & 1);
                    mbar_expect_tx(&gfull[s], TB_GX * TB_GY * 8);
                    char *dst = smem + Lt::G_OFF + s * Lt::G_STAGE;
                    if (tg < 0 && mp.glo)
                        tma_load(dst, mp.glo, &gfull[s], it.x0 - 2, it.y0 - 1);
                    else if (tg >= its.L && mp.ghi)
                        tma_load(dst, mp.ghi, &gfull[s], it.x0 - 2, it.y0 - 1);
                    else
                        tma_load(dst, mp.g, &gfull[s], it.x0 - 2, it.y0 - 1, tg);
                    ++ug;
                }
            }
            if (load_p && tg >= it.mb && tg < it.me) {
                const uint32_t s = up % Lt::SP;
                if (up >= (uint32_t)Lt::SP) mbar_wait(&pempty[s], ((up / Lt::SP) - 1) & 1);
                mbar_expect_tx(&pfull[s], Lt::P_STAGE);
                tma_load(smem + Lt::P_OFF + s * Lt::P_STAGE, mp.p, &pfull[s], it.x0, it.y0, tg);
                if constexpr (GD && TB_GP)
                    tma_load(smem + Lt::P_OFF + s * Lt::P_STAGE + Lt::P_PLANE, mp.gp, &pfull[s], it.x0, it.y0, tg);
                ++up;
            }
        }
        i = inext;
    }
    const uint32_t s = uw % Lt::SW;  // end-of-work marker
    if (uw >= (uint32_t)Lt::SW) mbar_wait(&wempty[s], ((uw / Lt::SW) - 1) & 1);
    itemq[s] = -1;
    mbar_arrive(&wfull[s]);
}

template <int COEFF>
ES_DEV double tb_coeff(const Geom &g, int64_t x, int64_t y, int64_t z) {
    if constexpr (COEFF == ES_COEFF_RADIAL) {
        const double xc = axis_coord(x, g.nx);
        return radial_from_sq(add(1.0, mul(xc, xc)), axis_coord(y, g.ny));
    } else if constexpr (COEFF == ES_COEFF_ARRAY) {
        return __ldg(g.coeff + (z * g.ny + y) * g.nx + x);
    }
    return 1.0;
}

// w_k at one window point (x, y) of plane z (scalar path: window edges at the
// domain boundary, where Dirichlet ghosts are 0 and Neumann ghosts mirror).
template <int COEFF, bool GD>
ES_DEV double tb_point_scalar(const Geom &g, const double *Wm, const double *Wc, const double *Wp, const double *Gj,
                              int64_t x0, int64_t y0, int64_t x, int64_t y, int z, double alpha, double beta) {
    const bool neu = g.mode == ES_MODE_NEUMANN;
    if (!(x >= 0 && x < g.nx && y >= 0 && y < g.ny) && !neu) return 0.0;
    x = min(max(x, (int64_t)0), g.nx - 1);  // Neumann ghost of w_k = w_k at the mirrored point
    y = min(max(y, (int64_t)0), g.ny - 1);
    const int o = (int)(y - (y0 - 2)) * TB_WX + (int)(x - (x0 - 4));
    const double c = Wc[o];
    double xm = Wc[o - 1], xp = Wc[o + 1], ym = Wc[o - TB_WX], yp = Wc[o + TB_WX];
    if (neu) {  // the TMA zero fill is the Dirichlet ghost of w_{k-1}; Neumann mirrors
        if (x == 0) xm = c;
        if (x == g.nx - 1) xp = c;
        if (y == 0) ym = c;
        if (y == g.ny - 1) yp = c;
    }
    double lap = lap7(c, xm, xp, ym, yp, Wm[o], Wp[o], g.wx, g.wy, g.wz);
    if constexpr (COEFF != ES_COEFF_NONE) lap = mul(tb_coeff<COEFF>(g, x, y, z), lap);
    if constexpr (GD) lap = sub(lap, mul(Gj[(int)(y - (y0 - 1)) * TB_GX + (int)(x - (x0 - 2))], c));
    return add(mul(alpha, lap), mul(beta, c));
}

// ---- consumers: two warp groups joined by the V ring -------------------------
// A (warps 0-3) computes w_k on the window of plane j into V(j); C (warps 4-7)
// forms p_k of plane j from V(j) and P(j), then w_{k+1}, p_{k+1} of plane j-1
// from V(j-2..j).  The groups hand planes over through per-slot mbarriers, so
// neither waits for the other at every plane (A runs up to two planes ahead).

struct TbBars {
    uint64_t *wfull, *wempty, *gfull, *gempty, *pfull, *pempty, *vfull, *vempty;
};

template <bool GD>
ES_DEV TbBars tb_bars(char *smem) {
    using Lt = TbLayout<GD>;
    uint64_t *b = reinterpret_cast<uint64_t *>(smem + Lt::BAR_OFF);
    TbBars r;
    r.wfull = b;
    r.wempty = r.wfull + Lt::SW;
    r.gfull = r.wempty + Lt::SW;
    r.gempty = r.gfull + Lt::SG;
    r.pfull = r.gempty + Lt::SG;
    r.pempty = r.pfull + Lt::SP;
    r.vfull = r.pempty + Lt::SP;
    r.vempty = r.vfull + TB_SV;
    return r;
}

ES_DEV void warp_arrive(uint64_t *b) {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(b);
}

ES_DEV void a_group_sync() { asm volatile("bar.sync 2, %0;" ::"n"(TB_NA) : "memory"); }

// slot / phase of a ring position
template <int S>
struct Ring {
    uint32_t slot = 0, phase = 0;
    ES_DEV void next() {
        if (++slot == (uint32_t)S) {
            slot = 0;
            phase ^= 1u;
        }
    }
};

// w_k at a window pair whose stencils need no ghost handling
// (Dirichlet: also at window points outside the domain, which the caller
// masks to the zero ghost -- a sampled coefficient is then read at the
// clamped point, the value is discarded)
template <int COEFF, bool GD>
ES_DEV double2 tb_fast_pair(const Geom &g, const double *Wm, const double *Wc, const double *Wp, const double *Gj,
                            int ey, int ex, int64_t x, int64_t y, int j, double alpha, double beta) {
    const int o = (ey + 1) * TB_WX + ex + 2;
    const double2 c = *reinterpret_cast<const double2 *>(Wc + o);
    const double2 ym = *reinterpret_cast<const double2 *>(Wc + o - TB_WX);
    const double2 yp = *reinterpret_cast<const double2 *>(Wc + o + TB_WX);
    const double2 zm = *reinterpret_cast<const double2 *>(Wm + o);
    const double2 zp = *reinterpret_cast<const double2 *>(Wp + o);
    double l0 = lap7(c.x, Wc[o - 1], c.y, ym.x, yp.x, zm.x, zp.x, g.wx, g.wy, g.wz);
    double l1 = lap7(c.y, c.x, Wc[o + 2], ym.y, yp.y, zm.y, zp.y, g.wx, g.wy, g.wz);
    if constexpr (COEFF == ES_COEFF_ARRAY) {
        const int64_t xc = min(max(x, (int64_t)0), g.nx - 2), yc = min(max(y, (int64_t)0), g.ny - 1);
        l0 = mul(tb_coeff<COEFF>(g, xc, yc, j), l0);
        l1 = mul(tb_coeff<COEFF>(g, xc + 1, yc, j), l1);
    } else if constexpr (COEFF != ES_COEFF_NONE) {
        l0 = mul(tb_coeff<COEFF>(g, x, y, j), l0);
        l1 = mul(tb_coeff<COEFF>(g, x + 1, y, j), l1);
    }
    if constexpr (GD) {
        const double2 gv = *reinterpret_cast<const double2 *>(Gj + ey * TB_GX + ex);
        l0 = sub(l0, mul(gv.x, c.x));
        l1 = sub(l1, mul(gv.y, c.y));
    }
    return make_double2(add(mul(alpha, l0), mul(beta, c.x)), add(mul(alpha, l1), mul(beta, c.y)));
}

template <int COEFF, bool GD>
ES_DEV void tb_group_a(const Geom &g, const SeriesParams *P, int k, const TbItems &its, char *smem) {
    using Lt = TbLayout<GD>;
    const TbBars B = tb_bars<GD>(smem);
    const volatile int *itemq = reinterpret_cast<const volatile int *>(smem + Lt::ITEMQ_OFF);
    volatile int *vitem = reinterpret_cast<volatile int *>(smem + Lt::VITEM_OFF);
    double *vwin = reinterpret_cast<double *>(smem + Lt::V_OFF);
    const int a = threadIdx.x;  // 0 .. TB_NA-1
    const bool neu = g.mode == ES_MODE_NEUMANN;
    const bool has_lo = g.halo_lo != nullptr, has_hi = g.halo_hi != nullptr;  // peer slabs below / above
    const double alpha = P->alpha, beta_k = sub(-P->shift, P->xi[k - 1]);
    int pey[3], pex[3];
#pragma unroll
    for (int h = 0; h < 3; ++h) {
        const int pr = a + TB_NA * h;
        pey[h] = pr < TB_PAIRS ? pr / (TB_EX / 2) : -1;
        pex[h] = 2 * (pr % (TB_EX / 2));
    }
    Ring<Lt::SW> wr;  // W ring position of the next plane to wait for
    Ring<Lt::SG> gr;
    Ring<TB_SV> vr;
    uint32_t vuses = 0;  // V slots handed out so far
    auto wst = [&](uint32_t s) { return reinterpret_cast<const double *>(smem + Lt::W_OFF + s * Lt::W_STAGE); };
    auto vslot = [&](uint32_t s) { return vwin + s * (TB_EX * TB_EY); };
    auto take_v = [&]() {  // wait until C released the slot's previous plane
        if (vuses >= (uint32_t)TB_SV) mbar_wait(&B.vempty[vr.slot], vr.phase ^ 1u);
        ++vuses;
    };
    for (;;) {
        mbar_wait(&B.wfull[wr.slot], wr.phase);
        const int i = itemq[wr.slot];
        if (i < 0) {  // end of work: tell C through the next V slot
            take_v();
            if (a == 0) vitem[vr.slot] = -1;
            warp_arrive(&B.vfull[vr.slot]);
            break;
        }
        const TbItem it = tb_item_at(its, i);
        bool fast[3], in0[3], in1[3];
#pragma unroll
        for (int h = 0; h < 3; ++h) {
            const int64_t x = it.x0 - 2 + pex[h], y = it.y0 - 1 + pey[h];
            const int64_t lo = neu ? 1 : 0, xhi = neu ? g.nx - 2 : g.nx - 1, yhi = neu ? g.ny - 2 : g.ny - 1;
            fast[h] = x >= lo && x + 1 <= xhi && y >= lo && y <= yhi;
            const bool yin = y >= 0 && y < g.ny;
            in0[h] = yin && x >= 0 && x < g.nx;
            in1[h] = yin && x + 1 >= 0 && x + 1 < g.nx;
        }
        // W slots of planes j-1, j, j+1 (plane mb-2 is at wr)
        Ring<Lt::SW> rm = wr, rc = wr;
        rc.next();
        Ring<Lt::SW> rp = rc;
        rp.next();
        mbar_wait(&B.wfull[rc.slot], rc.phase);
        uint32_t v_prev = 0;  // slot of V(j-1)
#pragma unroll 2
        for (int j = it.mb - 1; j <= it.me; ++j) {
            mbar_wait(&B.wfull[rp.slot], rp.phase);
            const double *Wm = wst(rm.slot), *Wc = wst(rc.slot), *Wp = wst(rp.slot);
            const double *Gj = nullptr;
            if constexpr (GD) {
                mbar_wait(&B.gfull[gr.slot], gr.phase);
                Gj = reinterpret_cast<const double *>(smem + Lt::G_OFF + gr.slot * Lt::G_STAGE);
            }
            take_v();
            double *Vj = vslot(vr.slot);
            if (j == it.mb - 1 && a == 0) vitem[vr.slot] = i;
            const bool zin = (j >= 0 || has_lo) && (j < its.L || has_hi);
            bool arrive_prev = false;
            if (zin && !neu) {
                // Dirichlet: every pair by the ghost-free formula (TMA's zero
                // fill is the ghost of w_{k-1}), points outside the domain
                // masked to w_k's zero ghost.  Straight-line code, so the
                // three pairs' loads and fp64 chains interleave.  A thread
                // without a third pair computes one at a valid window spot
                // and does not store it.
                double2 wk[3];
#pragma unroll
                for (int h = 0; h < 3; ++h) {
                    if (h == 2 && a >= (TB_PAIRS - 2 * TB_NA + 31) / 32 * 32) break;  // no third pair in this warp
                    const int ey = pey[h] < 0 ? 0 : pey[h], ex = pex[h];
                    const int64_t x = it.x0 - 2 + ex, y = it.y0 - 1 + ey;
                    wk[h] = tb_fast_pair<COEFF, GD>(g, Wm, Wc, Wp, Gj, ey, ex, x, y, j, alpha, beta_k);
                }
#pragma unroll
                for (int h = 0; h < 3; ++h) {
                    if (pey[h] < 0) continue;
                    const double2 w = make_double2(in0[h] ? wk[h].x : 0.0, in1[h] ? wk[h].y : 0.0);
                    *reinterpret_cast<double2 *>(Vj + pey[h] * TB_EX + pex[h]) = w;
                }
            } else if (zin) {
#pragma unroll
                for (int h = 0; h < 3; ++h) {
                    const int ey = pey[h], ex = pex[h];
                    if (ey < 0) break;
                    const int64_t x = it.x0 - 2 + ex, y = it.y0 - 1 + ey;
                    const double2 wk =
                        fast[h] ? tb_fast_pair<COEFF, GD>(g, Wm, Wc, Wp, Gj, ey, ex, x, y, j, alpha, beta_k)
                                : make_double2(
                                      tb_point_scalar<COEFF, GD>(g, Wm, Wc, Wp, Gj, it.x0, it.y0, x, y, j, alpha, beta_k),
                                      tb_point_scalar<COEFF, GD>(g, Wm, Wc, Wp, Gj, it.x0, it.y0, x + 1, y, j, alpha,
                                                                 beta_k));
                    *reinterpret_cast<double2 *>(Vj + ey * TB_EX + ex) = wk;
                }
                if (neu && j == 0 && !has_lo) {  // the mirrored plane below the domain = w_k of plane 0
                    a_group_sync();
                    double *Vb = vslot(v_prev);
                    for (int e = a; e < TB_EX * TB_EY; e += TB_NA) Vb[e] = Vj[e];
                    arrive_prev = true;
                }
            } else if (j >= 0) {  // plane L: zeros (Dirichlet) or the mirrored plane L-1 (Neumann)
                if (neu) a_group_sync();
                const double *Vs = vslot(v_prev);
                for (int e = a; e < TB_EX * TB_EY; e += TB_NA) Vj[e] = neu ? Vs[e] : 0.0;
            } else if (!neu) {  // plane -1, Dirichlet
                for (int e = a; e < TB_EX * TB_EY; e += TB_NA) Vj[e] = 0.0;
            }
            warp_arrive(&B.wempty[rm.slot]);  // W(j-1): last read by A of plane j
            if constexpr (GD) {
                warp_arrive(&B.gempty[gr.slot]);
                gr.next();
            }
            if (arrive_prev) warp_arrive(&B.vfull[v_prev]);
            if (!(neu && j < 0 && !has_lo)) warp_arrive(&B.vfull[vr.slot]);  // Neumann plane -1 arrives with plane 0
            v_prev = vr.slot;
            vr.next();
            rm = rc;
            rc = rp;
            rp.next();
        }
        warp_arrive(&B.wempty[rm.slot]);  // W(me), W(me+1)
        warp_arrive(&B.wempty[rc.slot]);
        wr = rp;
    }
}

template <int COEFF, bool GD, bool PEER>
ES_DEV void tb_group_c(const Geom &g, const SeriesParams *P, int k, bool two, const TbItems &its, char *smem) {
    using Lt = TbLayout<GD>;
    const TbBars B = tb_bars<GD>(smem);
    const volatile int *vitem = reinterpret_cast<const volatile int *>(smem + Lt::VITEM_OFF);
    const double *vwin = reinterpret_cast<const double *>(smem + Lt::V_OFF);
    const int c = threadIdx.x - TB_NA, cw = c >> 5, q = c & 31;  // rows cw and cw + TB_CW, pair x0 + 2q
    const int64_t nx = g.nx, plane = g.nx * g.ny;
    const double wx = g.wx, wy = g.wy, wz = g.wz;
    const int pass = P->state->pass;
    double *w1_dst = P->wbuf[pass & 1];  // w_{k+1}, or w_k on a one-node pass
    double *pk_dst = P->pbuf[k & 1], *pk1_dst = P->pbuf[(k + 1) & 1];
    const bool store_pk = tb_store_pk(*P, two);
    const double alpha = P->alpha, dk = P->dd[k];
    const double dk1 = two ? P->dd[k + 1] : 0.0, beta_k1 = two ? sub(-P->shift, P->xi[k]) : 0.0;
    const double pscale = k == 1 ? P->dd[0] : 1.0;  // first pass: P tiles hold v, p_0 = dd_0 v
    // PEER (x2): when an item of a boundary chunk is done, its group-C threads
    // copy what they just wrote of planes 0, 1 / L-2, L-1 (the w this pass
    // writes: w_{k+1}, or w_k on a one-node pass) into the neighbours'
    // two-plane halo buffers of the next pass's parity -- boundary chunks are
    // swept first, so the NVLink stores overlap the rest of the sweep; the
    // inner loop is untouched and k_slice_p2p2 only fences
    double *peer_lo = nullptr, *peer_hi = nullptr;
    if constexpr (PEER) {
        const int par = (pass + 1) & 1;
        peer_lo = P->peer_lo[par];
        peer_hi = P->peer_hi[par];
    }
    Ring<Lt::SG> gr;
    Ring<Lt::SP> pr;
    Ring<TB_SV> vr;
    auto vslot = [&](uint32_t s) { return vwin + s * (TB_EX * TB_EY); };
    for (;;) {
        mbar_wait(&B.vfull[vr.slot], vr.phase);
        const int i = vitem[vr.slot];
        if (i < 0) break;
        const TbItem it = tb_item_at(its, i);
        const int64_t xa = it.x0 + 2 * q;
        bool act[2];
        int64_t ya[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            ya[h] = it.y0 + cw + TB_CW * h;
            act[h] = xa < g.nx && ya[h] < g.ny;
        }
        double acc_w0[2] = {0.0, 0.0}, acc_p0[2] = {0.0, 0.0}, acc_w1[2] = {0.0, 0.0}, acc_p1[2] = {0.0, 0.0};
        double pk_prev[4] = {0.0, 0.0, 0.0, 0.0};
        // element offsets of this thread's two rows in plane j (advanced by a plane per iteration)
        int64_t off0 = (int64_t)(it.mb - 1) * plane + ya[0] * nx + xa;
        const int64_t drow = (int64_t)TB_CW * nx;  // row h = 1 is TB_CW rows below row 0
        // w_k at this thread's pairs of planes j-2, j-1 (centre values kept in
        // registers across planes: the zm / c of the next plane's stencil)
        double2 vm1[2] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0)}, vc1[2] = {vm1[0], vm1[1]};
        uint32_t s1 = 0;      // V slot of plane j-1
        uint32_t p_prev = 0;  // P slot of plane j-1 (TB_GP: held for its g')
#pragma unroll 2
        for (int j = it.mb - 1; j <= it.me; ++j) {
            if (j > it.mb - 1) mbar_wait(&B.vfull[vr.slot], vr.phase);
            const uint32_t s0 = vr.slot;
            const double *Vj = vslot(s0);
            double2 vcur[2];
#pragma unroll
            for (int h = 0; h < 2; ++h)
                vcur[h] = *reinterpret_cast<const double2 *>(Vj + (cw + TB_CW * h + 1) * TB_EX + 2 * q + 2);
            // ---- B: p_k of plane j (+ node k norms)
            double pk_cur[4] = {0.0, 0.0, 0.0, 0.0};
            const uint32_t p_held = p_prev;  // P stage of plane j-1 (its g' serves part C below, TB_GP)
            if (j >= it.mb && j < it.me) {
                mbar_wait(&B.pfull[pr.slot], pr.phase);
                const double *Pc = reinterpret_cast<const double *>(smem + Lt::P_OFF + pr.slot * Lt::P_STAGE);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int r = cw + TB_CW * h;
                    const double2 vk = vcur[h];
                    const double2 po = *reinterpret_cast<const double2 *>(Pc + r * 64 + 2 * q);
                    // pscale is 1.0 after the first pass, and 1.0 * x == x bit for bit
                    const double p0 = mul(pscale, po.x), p1 = mul(pscale, po.y);
                    pk_cur[2 * h] = add(p0, mul(dk, vk.x));
                    pk_cur[2 * h + 1] = add(p1, mul(dk, vk.y));
                    if (act[h]) {
                        const int64_t off = off0 + h * drow;
                        if (store_pk)
                            *reinterpret_cast<double2 *>(pk_dst + off) = make_double2(pk_cur[2 * h], pk_cur[2 * h + 1]);
                        if (!two) *reinterpret_cast<double2 *>(w1_dst + off) = vk;  // the next pass starts from w_k
                        acc_w0[h] = add(acc_w0[h], add(mul(vk.x, vk.x), mul(vk.y, vk.y)));
                        acc_p0[h] = add(acc_p0[h], add(mul(pk_cur[2 * h], pk_cur[2 * h]),
                                                       mul(pk_cur[2 * h + 1], pk_cur[2 * h + 1])));
                    }
                }
                if constexpr (GD && TB_GP) {
                    p_prev = pr.slot;  // kept until part C of plane j (next iteration) read its g'
                } else {
                    warp_arrive(&B.pempty[pr.slot]);
                }
                pr.next();
            }
            // ---- C: w_{k+1}, p_{k+1} of plane j-1 (+ node k+1 norms); both rows side by side
            const int jc = j - 1;
            if (two && jc >= it.mb && jc < it.me) {
                const double *Vc = vslot(s1);
                const double *Gc = nullptr;
                if constexpr (GD && TB_GP) {  // g' tile of plane j-1 in its (held) P stage, 64-wide rows
                    Gc = reinterpret_cast<const double *>(smem + Lt::P_OFF + p_held * Lt::P_STAGE + Lt::P_PLANE);
                } else if constexpr (GD) {
                    mbar_wait(&B.gfull[gr.slot], gr.phase);  // complete already; orders the TMA bytes for C
                    Gc = reinterpret_cast<const double *>(smem + Lt::G_OFF + gr.slot * Lt::G_STAGE);
                }
                double wn[4], pn[4];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int r = cw + TB_CW * h;
                    const int o = (r + 1) * TB_EX + 2 * q + 2;
                    const double2 cc = vc1[h], zm = vm1[h], zp = vcur[h];
                    const double2 ym = *reinterpret_cast<const double2 *>(Vc + o - TB_EX);
                    const double2 yp = *reinterpret_cast<const double2 *>(Vc + o + TB_EX);
                    double l0 = lap7(cc.x, Vc[o - 1], cc.y, ym.x, yp.x, zm.x, zp.x, wx, wy, wz);
                    double l1 = lap7(cc.y, cc.x, Vc[o + 2], ym.y, yp.y, zm.y, zp.y, wx, wy, wz);
                    if constexpr (COEFF != ES_COEFF_NONE) {
                        l0 = mul(tb_coeff<COEFF>(g, xa, ya[h], jc), l0);
                        l1 = mul(tb_coeff<COEFF>(g, xa + 1, ya[h], jc), l1);
                    }
                    if constexpr (GD) {
                        const double2 gv = TB_GP ? *reinterpret_cast<const double2 *>(Gc + r * 64 + 2 * q)
                                                 : *reinterpret_cast<const double2 *>(Gc + (r + 1) * TB_GX + 2 * q + 2);
                        l0 = sub(l0, mul(gv.x, cc.x));
                        l1 = sub(l1, mul(gv.y, cc.y));
                    }
                    wn[2 * h] = add(mul(alpha, l0), mul(beta_k1, cc.x));
                    wn[2 * h + 1] = add(mul(alpha, l1), mul(beta_k1, cc.y));
                    pn[2 * h] = add(pk_prev[2 * h], mul(dk1, wn[2 * h]));
                    pn[2 * h + 1] = add(pk_prev[2 * h + 1], mul(dk1, wn[2 * h + 1]));
                }
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    if (!act[h]) continue;
                    const int64_t off = off0 - plane + h * drow;  // plane jc = j - 1
                    *reinterpret_cast<double2 *>(w1_dst + off) = make_double2(wn[2 * h], wn[2 * h + 1]);
                    *reinterpret_cast<double2 *>(pk1_dst + off) = make_double2(pn[2 * h], pn[2 * h + 1]);
                    acc_w1[h] = add(acc_w1[h], add(mul(wn[2 * h], wn[2 * h]), mul(wn[2 * h + 1], wn[2 * h + 1])));
                    acc_p1[h] = add(acc_p1[h], add(mul(pn[2 * h], pn[2 * h]), mul(pn[2 * h + 1], pn[2 * h + 1])));
                }
            }
            if constexpr (GD && TB_GP) {
                if (jc >= it.mb && jc < it.me) warp_arrive(&B.pempty[p_held]);  // P(j-1): p and g' both read
            } else if constexpr (GD) {
                if (jc >= it.mb - 1) {  // G(j-1): C's share of the release
                    warp_arrive(&B.gempty[gr.slot]);
                    gr.next();
                }
            }
            if (j - 1 >= it.mb - 1) warp_arrive(&B.vempty[s1]);  // V(j-1): its neighbours were last read above
#pragma unroll
            for (int e = 0; e < 4; ++e) pk_prev[e] = pk_cur[e];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                vm1[h] = vc1[h];
                vc1[h] = vcur[h];
            }
            s1 = s0;
            vr.next();
            off0 += plane;
        }
        warp_arrive(&B.vempty[s1]);  // V(me)
        if constexpr (GD && !TB_GP) {  // G(me)
            warp_arrive(&B.gempty[gr.slot]);
            gr.next();
        }
        if constexpr (PEER) {  // this thread's own stores of the boundary planes, read back and pushed
            if ((peer_lo && it.mb < 2) || (peer_hi && it.me > its.L - 2)) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    if (!act[h]) continue;
                    const int64_t in_plane = ya[h] * nx + xa;
                    for (int z = it.mb; z < it.me; ++z) {
                        const bool lo = peer_lo && z < 2, hi = peer_hi && z >= its.L - 2;
                        if (!lo && !hi) continue;
                        const double2 val = *reinterpret_cast<const double2 *>(w1_dst + z * plane + in_plane);
                        if (lo) *reinterpret_cast<double2 *>(peer_lo + z * plane + in_plane) = val;
                        if (hi) *reinterpret_cast<double2 *>(peer_hi + (z - (its.L - 2)) * plane + in_plane) = val;
                    }
                }
            }
        }
        // (chunk, tile, row-warp) partials of both nodes, one-node kernel layout
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const double w0 = warp_sum(acc_w0[h]), p0 = warp_sum(acc_p0[h]);
            const double w1 = warp_sum(acc_w1[h]), p1 = warp_sum(acc_p1[h]);
            const int r = cw + TB_CW * h;
            if (q == 0 && it.y0 + (r & ~7) < g.ny) {  // the 64 x 8 tile of row r exists
                const int64_t e =
                    ((int64_t)it.chunk * its.ntiles8 + it.tile8 + (r >> 3) * its.tiles_x) * TMA_CONSUMER_WARPS + (r & 7);
                double *d0p = P->part + e * 2;
                d0p[0] = w0;
                d0p[1] = p0;
                double *d1p = P->part + ((int64_t)P->nslices * P->ntiles + e) * 2;
                d1p[0] = w1;
                d1p[1] = p1;
            }
        }
    }
    if constexpr (PEER) __threadfence_system();  // the halo pushes, before the slice kernel's arrival
}

template <int COEFF, bool GD, bool PEER = false>
ES_DEV void tb_pass(const SeriesParams *P, int k, bool two, char *smem) {
    using Lt = TbLayout<GD>;
    // a private copy: the ring waits' memory clobbers would otherwise make
    // every use of a weight / extent a reload from the parameter block
    const Geom g = P->g;
    const TbItems its = tb_items_of(g, P->chunk_len);
    const TmaMaps &M = *static_cast<const TmaMaps *>(P->maps);
    const int pass = P->state->pass;
    // W: w_{k-1} (v on the first pass; pass p writes wbuf[p & 1]); P: p_{k-1}
    // (pbuf[(k - 1) & 1]), or v on the first pass (p_0 = dd_0 v)
    TbMaps mp{&M.m[pass == 0 ? MAP_T_V : (pass & 1) ? MAP_T_0 : MAP_T_1], &M.m[MAP_T_G],
              &M.m[k == 1 ? MAP_T_PV : ((k - 1) & 1) ? MAP_T_P1 : MAP_T_P0]};
    if (g.halo_lo) mp.hlo = &M.m[(pass & 1) ? MAP_T_HLO1 : MAP_T_HLO0];  // pass p reads halo parity p & 1
    if (g.halo_hi) mp.hhi = &M.m[(pass & 1) ? MAP_T_HHI1 : MAP_T_HHI0];
    if (GD && TB_GP) mp.gp = &M.m[MAP_T_GP];
    if (GD && g.halo_lo) mp.glo = &M.m[MAP_T_GLO];
    if (GD && g.halo_hi) mp.ghi = &M.m[MAP_T_GHI];
    if (threadIdx.x == 0) {
        const TbBars B = tb_bars<GD>(smem);
        for (int s = 0; s < Lt::SW; ++s) {
            mbar_init(&B.wfull[s], 1);
            mbar_init(&B.wempty[s], TB_AW);  // A group
        }
        for (int s = 0; s < Lt::SG; ++s) {
            mbar_init(&B.gfull[s], 1);
            mbar_init(&B.gempty[s], TB_GP ? TB_AW : TB_AW + TB_CW);  // A (and C unless TB_GP)
        }
        for (int s = 0; s < Lt::SP; ++s) {
            mbar_init(&B.pfull[s], 1);
            mbar_init(&B.pempty[s], TB_CW);  // C group
        }
        for (int s = 0; s < TB_SV; ++s) {
            mbar_init(&B.vfull[s], TB_AW);
            mbar_init(&B.vempty[s], TB_CW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int warp = threadIdx.x / 32;
    if (warp == TB_AW + TB_CW) {
        if ((threadIdx.x & 31) == 0) {
            tma_acquire(mp.w);
            if (GD) tma_acquire(mp.g);
            tma_acquire(mp.p);
            for (const CUtensorMap *h : {mp.hlo, mp.hhi, mp.glo, mp.ghi, mp.gp})
                if (h) tma_acquire(h);
            tb_produce<GD>(g, its, mp, smem, true, P->work);
        }
    } else if (warp < TB_AW) {
        tb_group_a<COEFF, GD>(g, P, k, its, smem);
    } else {
        tb_group_c<COEFF, GD, PEER>(g, P, k, two, its, smem);
    }
}

}  // namespace es
