// Two Newton-Leja nodes per HBM pass on single-plane (2D) grids (C2).
//
// The 2D form of stencil_tb.cuh: rows play the role of planes.  A pass takes
// w_{k-1} and computes w_k = A w_{k-1} and w_{k+1} = A w_k row by row; w_k
// lives only in a shared-memory row window (the 256-wide tile plus one
// point each side) and is never written.  Per point the pass reads w_{k-1},
// p_{k-1} and the sampled coefficient D once, and writes p_k, w_{k+1} and
// p_{k+1}: 48 B for two nodes instead of 80 (2 x 40 with the streamed D).
//
// Tiles are 512 points wide (x0 = 512 t, the one-node 2D tile), row chunks
// 4x the one-node 2D plan's; the norm partials keep the one-node kernel's
// (row chunk, tile, 64-column warp) layout -- a group-C thread owns the x
// pairs of one-node consumer threads c and c + 128, accumulates each one's
// rows in order and flushes at every one-node chunk end -- so
// k_slice_reduce2 sums exactly what the one-node series sums, in the same
// order (test_two_node_2d_bitwise).
//
// Rings (producer = the last warp, one lane):
//   W: w_{k-1} rows mb-2 .. me+1, x0-4 .. x0+515 (520; boxes 256 + 256 + 8);
//   G: D rows mb-1 .. me, x0-2 .. x0+513 (516; boxes 256 + 256 + 4) -- staged D only;
//   P: p_{k-1} rows mb .. me-1, x0 .. x0+511 (v on the first pass);
//   V: w_k row windows x0-2 .. x0+513, written by group A, read by group C.
// Group A (5 warps, 258 pairs): w_k of row j on the window.  Group C
// (4 warps, 256 pairs): p_k of row j, then w_{k+1}, p_{k+1} of row j-1.
//
// Scope: homogeneous Dirichlet (TMA zero fill) and Neumann (mirrored ghosts),
// coefficient none or the staged sampled D, no g' diagonal.
#pragma once

#include "stencil_tb.cuh"

namespace es {

// interior tile width: 256 (two CTAs of 10 warps per SM, one pair per
// thread) measured faster than 512 (one CTA, two pairs per thread: 121 vs
// 110 us per 4096^2 node; 512 at two CTAs/SM spills)
#ifndef T2_TX
#define T2_TX 256
#endif
constexpr int T2_WX = T2_TX + 8;            // w_{k-1}: x0-4 .. x0+T2_TX+3
constexpr int T2_EX = T2_TX + 4;            // w_k window / D: x0-2 .. x0+T2_TX+1
// R8 (nx % 8 == 0): the row viewed as 8-element chunks -- a 3D tensor map
// (8, nx/8, ny) whose box (8, TX/8 + 2, 1) covers x0-8 .. x0+TX+7 contiguously
// -- so a w or D row window is ONE TMA (two on the plain row maps: boxes are
// at most 256 wide); the producer's issue rate was the pass's limit
constexpr int T2_RX = T2_TX + 16;           // R8 row window: x0-8 .. x0+T2_TX+7
constexpr int T2_PAIRS = T2_EX / 2;         // window pairs
#ifndef T2_AWARPS
#define T2_AWARPS 5  // group A warps
#endif
#ifndef T2_CWARPS
#define T2_CWARPS 4  // group C warps
#endif
constexpr int T2_AW = T2_AWARPS, T2_CW = T2_CWARPS;
constexpr int T2_NA = 32 * T2_AW, T2_NC = 32 * T2_CW;
constexpr int T2_THREADS = 32 * (T2_AW + T2_CW + 1);
#ifndef T2_MINB
#define T2_MINB (T2_TX == 256 ? 2 : 1)  // CTAs per SM the register allocation is sized for
#endif
constexpr int T2_APT = (T2_PAIRS + T2_NA - 1) / T2_NA;  // window pairs per A thread (a, a + 160)
constexpr int T2_CPT = T2_TX / (2 * T2_NC);             // pairs per C thread (c, c + 128)
static_assert(T2_NC * 2 * T2_CPT == T2_TX && T2_APT <= 2 && (T2_TX == 256 || T2_TX == 512), "tile geometry");

#ifndef T2_SW
#define T2_SW 8
#endif
#ifndef T2_SG
#define T2_SG 6
#endif
#ifndef T2_SP
#define T2_SP 6
#endif
#ifndef T2_SV
#define T2_SV 6
#endif
// T2_DP: group C's D (interior of its output row) rides in the P stage of
// that row, so G stages are released by group A alone (no A-C coupling
// through the G ring; shared memory is plentiful in 2D)
#ifndef T2_DP
#define T2_DP 1
#endif

template <bool STAGED>
struct Tb2Layout {
    static constexpr int SW = T2_SW, SG = STAGED ? T2_SG : 0, SP = T2_SP, SV = T2_SV;
    static constexpr int W_STAGE = (T2_RX * 8 + 127) & ~127;  // holds either window
    static constexpr int G_STAGE = (T2_RX * 8 + 127) & ~127;
    static constexpr int P_ROW = T2_TX * 8;
    static constexpr int P_STAGE = (STAGED && T2_DP ? 2 : 1) * P_ROW;  // p_{k-1} row (+ D row interior, T2_DP)
    static constexpr int V_SLOT = T2_EX * 8;
    static constexpr int W_OFF = 0;
    static constexpr int G_OFF = W_OFF + SW * W_STAGE;
    static constexpr int P_OFF = G_OFF + SG * G_STAGE;
    static constexpr int V_OFF = P_OFF + SP * P_STAGE;
    static constexpr int BAR_OFF = (V_OFF + SV * V_SLOT + 7) & ~7;
    static constexpr int NBAR = 2 * (SW + SG + SP + SV);
    static constexpr int ITEMQ_OFF = BAR_OFF + NBAR * 8;
    static constexpr int VITEM_OFF = ITEMQ_OFF + ((SW * 4 + 15) & ~15);
    static constexpr int BYTES = VITEM_OFF + ((SV * 4 + 15) & ~15);
};

struct Tb2Items {
    int tiles, nchunks, chunk_len, ny;
};

ES_DEV Tb2Items tb2_items_of(const Geom &g, int chunk_len) {
    Tb2Items it;
    it.tiles = (int)((g.nx + T2_TX - 1) / T2_TX);
    it.ny = (int)g.ny;
    it.chunk_len = chunk_len;
    it.nchunks = (it.ny + chunk_len - 1) / chunk_len;
    return it;
}

struct Tb2Item {
    int chunk, tile, x0, mb, me;
};

ES_DEV Tb2Item tb2_item_at(const Tb2Items &its, int i) {
    Tb2Item r;
    r.chunk = i / its.tiles;
    r.tile = i % its.tiles;
    r.x0 = r.tile * T2_TX;
    r.mb = r.chunk * its.chunk_len;
    r.me = min(its.ny, r.mb + its.chunk_len);
    return r;
}

struct Tb2Maps {
    const CUtensorMap *wa, *wb8;  // w_{k-1}: 256- and 8-wide row boxes
    const CUtensorMap *ga, *gb4;  // staged D: 256- and 4-wide row boxes
    const CUtensorMap *p;         // p_{k-1} (or v): 256-wide row box
    const CUtensorMap *dp;        // staged D: 256-wide row box at x0 (T2_DP)
};

template <bool STAGED>
struct Tb2Bars {
    uint64_t *wfull, *wempty, *gfull, *gempty, *pfull, *pempty, *vfull, *vempty;
    ES_DEV explicit Tb2Bars(char *smem) {
        using Lt = Tb2Layout<STAGED>;
        uint64_t *b = reinterpret_cast<uint64_t *>(smem + Lt::BAR_OFF);
        wfull = b;
        wempty = wfull + Lt::SW;
        gfull = wempty + Lt::SW;
        gempty = gfull + Lt::SG;
        pfull = gempty + Lt::SG;
        pempty = pfull + Lt::SP;
        vfull = pempty + Lt::SP;
        vempty = vfull + Lt::SV;
    }
};

// source row of W / G stage t: rows -1 / ny are the zero fill (Dirichlet,
// out-of-bounds TMA coordinate) or the mirrored boundary row (Neumann)
ES_DEV int tb2_row(const Geom &g, int t) {
    if (t >= 0 && t < g.ny) return t;
    if (g.mode == ES_MODE_NEUMANN) return t < 0 ? 0 : (int)g.ny - 1;
    return t;
}

template <bool STAGED, bool R8>
ES_DEV void tb2_produce(const Geom &g, const Tb2Items &its, const Tb2Maps &mp, char *smem, unsigned *work) {
    using Lt = Tb2Layout<STAGED>;
    const Tb2Bars<STAGED> B(smem);
    volatile int *itemq = reinterpret_cast<volatile int *>(smem + Lt::ITEMQ_OFF);
    uint32_t uw = 0, ug = 0, up = 0;
    const int total = its.tiles * its.nchunks;
    int i = work ? (int)atomicAdd(work, 1u) : (int)blockIdx.x;
    while (i < total) {
        const Tb2Item it = tb2_item_at(its, i);
        int inext = -1;
        for (int t = it.mb - 2; t <= it.me + 1; ++t) {
            if (t == max(it.mb - 2, it.me - 3)) inext = work ? (int)atomicAdd(work, 1u) : i + (int)gridDim.x;
            {  // W(t)
                const uint32_t s = uw % Lt::SW;
                if (uw >= (uint32_t)Lt::SW) mbar_wait(&B.wempty[s], ((uw / Lt::SW) - 1) & 1);
                itemq[s] = i;
                mbar_expect_tx(&B.wfull[s], (R8 ? T2_RX : T2_WX) * 8);
                char *dst = smem + Lt::W_OFF + s * Lt::W_STAGE;
                const int r = tb2_row(g, t);
                if constexpr (R8) {
                    tma_load(dst, mp.wa, &B.wfull[s], 0, (it.x0 - 8) / 8, r);
                } else {
#pragma unroll
                    for (int b = 0; b < T2_TX / 256; ++b)
                        tma_load(dst + 256 * 8 * b, mp.wa, &B.wfull[s], it.x0 - 4 + 256 * b, r);
                    tma_load(dst + T2_TX * 8, mp.wb8, &B.wfull[s], it.x0 + T2_TX - 4, r);
                }
                ++uw;
            }
            const int tg = t - 1;  // G(t-1), P(t-1): what consumer row t-1 needs besides W(t)
            if constexpr (STAGED) {
                if (tg >= it.mb - 1 && tg <= it.me) {
                    const uint32_t s = ug % Lt::SG;
                    if (ug >= (uint32_t)Lt::SG) mbar_wait(&B.gempty[s], ((ug / Lt::SG) - 1) & 1);
                    mbar_expect_tx(&B.gfull[s], (R8 ? T2_RX : T2_EX) * 8);
                    char *dst = smem + Lt::G_OFF + s * Lt::G_STAGE;
                    const int r = tb2_row(g, tg);
                    if constexpr (R8) {
                        tma_load(dst, mp.ga, &B.gfull[s], 0, (it.x0 - 8) / 8, r);
                    } else {
#pragma unroll
                        for (int b = 0; b < T2_TX / 256; ++b)
                            tma_load(dst + 256 * 8 * b, mp.ga, &B.gfull[s], it.x0 - 2 + 256 * b, r);
                        tma_load(dst + T2_TX * 8, mp.gb4, &B.gfull[s], it.x0 + T2_TX - 2, r);
                    }
                    ++ug;
                }
            }
            if (tg >= it.mb && tg < it.me) {
                const uint32_t s = up % Lt::SP;
                if (up >= (uint32_t)Lt::SP) mbar_wait(&B.pempty[s], ((up / Lt::SP) - 1) & 1);
                mbar_expect_tx(&B.pfull[s], Lt::P_STAGE);
                char *dst = smem + Lt::P_OFF + s * Lt::P_STAGE;
                if constexpr (R8) {
                    tma_load(dst, mp.p, &B.pfull[s], 0, it.x0 / 8, tg);
                    if constexpr (STAGED && T2_DP) tma_load(dst + Lt::P_ROW, mp.dp, &B.pfull[s], 0, it.x0 / 8, tg);
                } else {
#pragma unroll
                    for (int b = 0; b < T2_TX / 256; ++b)
                        tma_load(dst + 256 * 8 * b, mp.p, &B.pfull[s], it.x0 + 256 * b, tg);
                    if constexpr (STAGED && T2_DP) {
#pragma unroll
                        for (int b = 0; b < T2_TX / 256; ++b)
                            tma_load(dst + Lt::P_ROW + 256 * 8 * b, mp.dp, &B.pfull[s], it.x0 + 256 * b, tg);
                    }
                }
                ++up;
            }
        }
        i = inext;
    }
    const uint32_t s = uw % Lt::SW;  // end-of-work marker
    if (uw >= (uint32_t)Lt::SW) mbar_wait(&B.wempty[s], ((uw / Lt::SW) - 1) & 1);
    itemq[s] = -1;
    mbar_arrive(&B.wfull[s]);
}

ES_DEV void a2_group_sync() { asm volatile("bar.sync 2, %0;" ::"n"(T2_NA) : "memory"); }

// w_k at window pair e of row j (x = x0 - 2 + 2e).  Dirichlet: the
// ghost-free formula everywhere (TMA's zero fill is the ghost of w_{k-1}),
// points outside the domain masked to the zero ghost.  Neumann: window
// points outside the domain take w_k of the mirrored point, and stencils at
// the domain edge use the point itself as the ghost.
template <bool STAGED, bool R8>
ES_DEV double2 tb2_pair(const Geom &g, const double *Wm, const double *Wc, const double *Wp, const double *Gj,
                        int x0, int e, double alpha, double beta, bool neu, double wx, double wy, double wz) {
    constexpr int WO = R8 ? 8 : 4, GO = R8 ? 8 : 2;  // window origins x0 - WO (w_{k-1}), x0 - GO (D)
    const int64_t nx = g.nx;
    const int64_t xa = x0 - 2 + 2 * e;
    double out[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        int64_t x = xa + h;
        const bool in = x >= 0 && x < nx;
        if (neu) x = min(max(x, (int64_t)0), nx - 1);
        const int o = (int)(x - (x0 - WO));  // W index
        const double c = Wc[o];
        double xm = Wc[o - 1], xp = Wc[o + 1];
        if (neu) {
            if (x == 0) xm = c;
            if (x == nx - 1) xp = c;
        }
        const double z = neu ? c : 0.0;
        double lap = lap7(c, xm, xp, Wm[o], Wp[o], z, z, wx, wy, wz);
        if constexpr (STAGED) lap = mul(Gj[x - (x0 - GO)], lap);
        const double w = add(mul(alpha, lap), mul(beta, c));
        out[h] = (neu || in) ? w : 0.0;
    }
    return make_double2(out[0], out[1]);
}

// tb2_pair where neither point needs a ghost rule: x0-2+2e .. +1 inside
// [1, nx-2] (Neumann) / the domain (Dirichlet: TMA's zero fill is the
// ghost of w_{k-1}; points outside are masked by the caller).  Pair loads.
template <bool STAGED, bool R8>
ES_DEV double2 tb2_pair_fast(const double *Wm, const double *Wc, const double *Wp, const double *Gj, int e,
                             double alpha, double beta, bool neu, double wx, double wy, double wz) {
    constexpr int WO = R8 ? 8 : 4, GO = R8 ? 8 : 2;
    const int o = WO - 2 + 2 * e;  // W index of x = x0 - 2 + 2e
    const double2 c = *reinterpret_cast<const double2 *>(Wc + o);
    const double2 ym = *reinterpret_cast<const double2 *>(Wm + o);
    const double2 yp = *reinterpret_cast<const double2 *>(Wp + o);
    const double z0 = neu ? c.x : 0.0, z1 = neu ? c.y : 0.0;
    double l0 = lap7(c.x, Wc[o - 1], c.y, ym.x, yp.x, z0, z0, wx, wy, wz);
    double l1 = lap7(c.y, c.x, Wc[o + 2], ym.y, yp.y, z1, z1, wx, wy, wz);
    if constexpr (STAGED) {
        const double2 d = *reinterpret_cast<const double2 *>(Gj + GO - 2 + 2 * e);
        l0 = mul(d.x, l0);
        l1 = mul(d.y, l1);
    }
    return make_double2(add(mul(alpha, l0), mul(beta, c.x)), add(mul(alpha, l1), mul(beta, c.y)));
}

template <bool STAGED, bool R8>
ES_DEV void tb2_group_a(const Geom &g, const SeriesParams *P, int k, const Tb2Items &its, char *smem) {
    using Lt = Tb2Layout<STAGED>;
    const Tb2Bars<STAGED> B(smem);
    const volatile int *itemq = reinterpret_cast<const volatile int *>(smem + Lt::ITEMQ_OFF);
    volatile int *vitem = reinterpret_cast<volatile int *>(smem + Lt::VITEM_OFF);
    double *vwin = reinterpret_cast<double *>(smem + Lt::V_OFF);
    const int a = threadIdx.x;  // 0 .. T2_NA-1: window pairs a, a + T2_NA
    const bool neu = g.mode == ES_MODE_NEUMANN;
    const double wx = g.wx, wy = g.wy, wz = g.wz;
    const double alpha = P->alpha, beta_k = sub(-P->shift, P->xi[k - 1]);
    bool valid[T2_APT];  // window pair a + T2_NA h exists (warp-uniform except in one warp)
#pragma unroll
    for (int h = 0; h < T2_APT; ++h) valid[h] = a + T2_NA * h < T2_PAIRS;
    Ring<Lt::SW> wr;
    Ring<(Lt::SG > 0 ? Lt::SG : 1)> gr;
    Ring<Lt::SV> vr;
    uint32_t vuses = 0;
    auto wst = [&](uint32_t s) { return reinterpret_cast<const double *>(smem + Lt::W_OFF + s * Lt::W_STAGE); };
    auto vslot = [&](uint32_t s) { return vwin + s * T2_EX; };
    auto take_v = [&]() {
        if (vuses >= (uint32_t)Lt::SV) mbar_wait(&B.vempty[vr.slot], vr.phase ^ 1u);
        ++vuses;
    };
    for (;;) {
        mbar_wait(&B.wfull[wr.slot], wr.phase);
        const int i = itemq[wr.slot];
        if (i < 0) {
            take_v();
            if (a == 0) vitem[vr.slot] = -1;
            warp_arrive(&B.vfull[vr.slot]);
            break;
        }
        const Tb2Item it = tb2_item_at(its, i);
        // this thread's window pairs: ghost-free (fast) or at the domain edge
        bool fast[T2_APT], in0[T2_APT], in1[T2_APT];
#pragma unroll
        for (int h = 0; h < T2_APT; ++h) {
            const int64_t xe = it.x0 - 2 + 2 * (a + T2_NA * h);
            fast[h] = !neu || !valid[h] || (xe >= 1 && xe + 1 <= g.nx - 2);  // Dirichlet: every pair (masked)
            in0[h] = xe >= 0 && xe < g.nx;
            in1[h] = xe + 1 >= 0 && xe + 1 < g.nx;
        }
        bool all_fast = true;
#pragma unroll
        for (int h = 0; h < T2_APT; ++h) all_fast = all_fast && fast[h];
        Ring<Lt::SW> rm = wr, rc = wr;
        rc.next();
        Ring<Lt::SW> rp = rc;
        rp.next();
        mbar_wait(&B.wfull[rc.slot], rc.phase);
        uint32_t v_prev = 0;
#pragma unroll 2
        for (int j = it.mb - 1; j <= it.me; ++j) {
            mbar_wait(&B.wfull[rp.slot], rp.phase);
            const double *Wm = wst(rm.slot), *Wc = wst(rc.slot), *Wp = wst(rp.slot);
            const double *Gj = nullptr;
            if constexpr (STAGED) {
                mbar_wait(&B.gfull[gr.slot], gr.phase);
                Gj = reinterpret_cast<const double *>(smem + Lt::G_OFF + gr.slot * Lt::G_STAGE);
            }
            take_v();
            double *Vj = vslot(vr.slot);
            if (j == it.mb - 1 && a == 0) vitem[vr.slot] = i;
            const bool rin = j >= 0 && j < its.ny;
            bool arrive_prev = false;
            if (rin) {
                if (all_fast) {  // straight-line: the pairs' loads and fp64 chains interleave
                    double2 wk[T2_APT];
#pragma unroll
                    for (int h = 0; h < T2_APT; ++h) {
                        const int e = valid[h] ? a + T2_NA * h : 0;  // a spare lane computes pair 0, stores nothing
                        wk[h] = tb2_pair_fast<STAGED, R8>(Wm, Wc, Wp, Gj, e, alpha, beta_k, neu, wx, wy, wz);
                        if (!neu) wk[h] = make_double2(in0[h] ? wk[h].x : 0.0, in1[h] ? wk[h].y : 0.0);
                    }
#pragma unroll
                    for (int h = 0; h < T2_APT; ++h)
                        if (valid[h]) *reinterpret_cast<double2 *>(Vj + 2 * (a + T2_NA * h)) = wk[h];
                } else {
#pragma unroll
                    for (int h = 0; h < T2_APT; ++h) {
                        if (!valid[h]) continue;
                        const int e = a + T2_NA * h;
                        *reinterpret_cast<double2 *>(Vj + 2 * e) =
                            fast[h] ? tb2_pair_fast<STAGED, R8>(Wm, Wc, Wp, Gj, e, alpha, beta_k, neu, wx, wy, wz)
                                    : tb2_pair<STAGED, R8>(g, Wm, Wc, Wp, Gj, it.x0, e, alpha, beta_k, neu, wx, wy, wz);
                    }
                }
                if (neu && j == 0) {  // the mirrored row below the domain = w_k of row 0
                    a2_group_sync();
                    double *Vb = vslot(v_prev);
                    for (int e = a; e < T2_EX; e += T2_NA) Vb[e] = Vj[e];
                    arrive_prev = true;
                }
            } else if (j >= 0) {  // row ny: zeros (Dirichlet) or the mirrored row ny-1 (Neumann)
                if (neu) a2_group_sync();
                const double *Vs = vslot(v_prev);
                for (int e = a; e < T2_EX; e += T2_NA) Vj[e] = neu ? Vs[e] : 0.0;
            } else if (!neu) {  // row -1, Dirichlet
                for (int e = a; e < T2_EX; e += T2_NA) Vj[e] = 0.0;
            }
            warp_arrive(&B.wempty[rm.slot]);  // W(j-1): last read by A of row j
            if constexpr (STAGED) {
                warp_arrive(&B.gempty[gr.slot]);
                gr.next();
            }
            if (arrive_prev) warp_arrive(&B.vfull[v_prev]);
            if (!(neu && j < 0)) warp_arrive(&B.vfull[vr.slot]);  // Neumann row -1 arrives with row 0
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

template <bool STAGED>
ES_DEV void tb2_group_c(const Geom &g, const SeriesParams *P, int k, bool two, const Tb2Items &its, char *smem) {
    using Lt = Tb2Layout<STAGED>;
    const Tb2Bars<STAGED> B(smem);
    const volatile int *vitem = reinterpret_cast<const volatile int *>(smem + Lt::VITEM_OFF);
    const double *vwin = reinterpret_cast<const double *>(smem + Lt::V_OFF);
    // pairs x0 + 2c + 256 h (h = 0, 1): the one-node consumer threads c and c + 128
    const int c = threadIdx.x - T2_NA, cw = c >> 5, lane = c & 31;
    const int64_t nx = g.nx;
    const bool neu = g.mode == ES_MODE_NEUMANN;
    const double wx = g.wx, wy = g.wy, wz = g.wz;
    const int pass = P->state->pass;
    double *w1_dst = P->wbuf[pass & 1];  // w_{k+1}, or w_k on a one-node pass
    double *pk_dst = P->pbuf[k & 1], *pk1_dst = P->pbuf[(k + 1) & 1];
    const bool store_pk = tb_store_pk(*P, two);
    const double alpha = P->alpha, dk = P->dd[k];
    const double dk1 = two ? P->dd[k + 1] : 0.0, beta_k1 = two ? sub(-P->shift, P->xi[k]) : 0.0;
    const double pscale = k == 1 ? P->dd[0] : 1.0;  // first pass: P rows hold v, p_0 = dd_0 v
    const int tiles = (int)((nx + 511) / 512);       // the one-node plan's 512-wide tiles
    const int CL = P->norm_chunk;
    const int64_t half = (int64_t)P->nslices * P->ntiles * 2;
    Ring<(Lt::SG > 0 ? Lt::SG : 1)> gr;
    Ring<Lt::SP> pr;
    Ring<Lt::SV> vr;
    auto vslot = [&](uint32_t s) { return vwin + s * T2_EX; };
    for (;;) {
        mbar_wait(&B.vfull[vr.slot], vr.phase);
        const int i = vitem[vr.slot];
        if (i < 0) break;
        const Tb2Item it = tb2_item_at(its, i);
        bool act[T2_CPT];
#pragma unroll
        for (int h = 0; h < T2_CPT; ++h) act[h] = it.x0 + 2 * c + 256 * h < nx;
        // one-node norm layout: (row chunk, tile, 64-column warp cw + 4 h) entries
        const int64_t ent_base = (int64_t)(it.x0 / 512) * TMA_CONSUMER_WARPS + (it.x0 % 512) / 64 + cw;
        // a 512-wide one-node tile whose right half lies outside the domain
        // (256-wide tiles): its warps 4-7 hold only inactive lanes (zero partials)
        const bool pad_half = T2_TX == 256 && it.x0 % 512 == 0 && it.x0 + 256 >= nx;
        double acc_w0[T2_CPT], acc_p0[T2_CPT], acc_w1[T2_CPT], acc_p1[T2_CPT];
        double2 pk_prev[T2_CPT], vm1[T2_CPT], vc1[T2_CPT];  // p_k of row j-1, w_k centres of rows j-2, j-1
#pragma unroll
        for (int h = 0; h < T2_CPT; ++h) {
            acc_w0[h] = acc_p0[h] = acc_w1[h] = acc_p1[h] = 0.0;
            pk_prev[h] = vm1[h] = vc1[h] = make_double2(0.0, 0.0);
        }
        uint32_t s1 = 0;
        uint32_t p_prev = 0;  // P slot of row j-1 (T2_DP: held for its D)
        int64_t off0 = (int64_t)(it.mb - 1) * nx + it.x0 + 2 * c;  // element offset of pair h = 0 in row j
        auto flush = [&](double (&aw)[T2_CPT], double (&ap)[T2_CPT], int row, int64_t node_half) {
#pragma unroll
            for (int h = 0; h < T2_CPT; ++h) {
                const double w = warp_sum(aw[h]), p = warp_sum(ap[h]);
                if (lane == 0) {
                    double *d = P->part + node_half +
                                (((int64_t)(row / CL) * tiles) * TMA_CONSUMER_WARPS + ent_base + 4 * h) * 2;
                    d[0] = w;
                    d[1] = p;
                    if (pad_half) {
                        d[8] = 0.0;
                        d[9] = 0.0;
                    }
                }
                aw[h] = 0.0;
                ap[h] = 0.0;
            }
        };
#pragma unroll 2
        for (int j = it.mb - 1; j <= it.me; ++j) {
            if (j > it.mb - 1) mbar_wait(&B.vfull[vr.slot], vr.phase);
            const uint32_t s0 = vr.slot;
            const double *Vj = vslot(s0);
            double2 vcur[T2_CPT];
#pragma unroll
            for (int h = 0; h < T2_CPT; ++h) vcur[h] = *reinterpret_cast<const double2 *>(Vj + 2 * c + 256 * h + 2);
            // ---- p_k of row j (+ node k norms)
            double2 pk_cur[T2_CPT];
#pragma unroll
            for (int h = 0; h < T2_CPT; ++h) pk_cur[h] = make_double2(0.0, 0.0);
            const uint32_t p_held = p_prev;  // P stage of row j-1 (its D serves part C below, T2_DP)
            if (j >= it.mb && j < it.me) {
                mbar_wait(&B.pfull[pr.slot], pr.phase);
                const double *Pc = reinterpret_cast<const double *>(smem + Lt::P_OFF + pr.slot * Lt::P_STAGE);
#pragma unroll
                for (int h = 0; h < T2_CPT; ++h) {
                    const double2 po = *reinterpret_cast<const double2 *>(Pc + 2 * c + 256 * h);
                    pk_cur[h] = make_double2(add(mul(pscale, po.x), mul(dk, vcur[h].x)),
                                             add(mul(pscale, po.y), mul(dk, vcur[h].y)));
                }
#pragma unroll
                for (int h = 0; h < T2_CPT; ++h) {
                    if (!act[h]) continue;
                    if (store_pk) *reinterpret_cast<double2 *>(pk_dst + off0 + 256 * h) = pk_cur[h];
                    if (!two) *reinterpret_cast<double2 *>(w1_dst + off0 + 256 * h) = vcur[h];  // next pass starts from w_k
                    acc_w0[h] = add(acc_w0[h], add(mul(vcur[h].x, vcur[h].x), mul(vcur[h].y, vcur[h].y)));
                    acc_p0[h] = add(acc_p0[h], add(mul(pk_cur[h].x, pk_cur[h].x), mul(pk_cur[h].y, pk_cur[h].y)));
                }
                if constexpr (STAGED && T2_DP)
                    p_prev = pr.slot;  // kept until part C of row j (next iteration) read its D
                else
                    warp_arrive(&B.pempty[pr.slot]);
                pr.next();
                if ((j + 1) % CL == 0 || j + 1 == it.me) flush(acc_w0, acc_p0, j, 0);
            }
            // ---- w_{k+1}, p_{k+1} of row j-1 (+ node k+1 norms)
            const int jc = j - 1;
            if (two && jc >= it.mb && jc < it.me) {
                const double *Vc = vslot(s1);
                const double *Gc = nullptr;  // D of row j-1, indexed from x0 - 2
                if constexpr (STAGED && T2_DP) {
                    Gc = reinterpret_cast<const double *>(smem + Lt::P_OFF + p_held * Lt::P_STAGE + Lt::P_ROW) - 2;
                } else if constexpr (STAGED) {
                    mbar_wait(&B.gfull[gr.slot], gr.phase);  // complete already; orders the TMA bytes for C
                    Gc = reinterpret_cast<const double *>(smem + Lt::G_OFF + gr.slot * Lt::G_STAGE);
                }
                double2 wn[T2_CPT], pn[T2_CPT];
#pragma unroll
                for (int h = 0; h < T2_CPT; ++h) {
                    const int o = 2 * c + 256 * h + 2;
                    const double2 cc = vc1[h];
                    const double xm0 = Vc[o - 1], xp1 = Vc[o + 2];
                    const double z0 = neu ? cc.x : 0.0, z1 = neu ? cc.y : 0.0;
                    double l0 = lap7(cc.x, xm0, cc.y, vm1[h].x, vcur[h].x, z0, z0, wx, wy, wz);
                    double l1 = lap7(cc.y, cc.x, xp1, vm1[h].y, vcur[h].y, z1, z1, wx, wy, wz);
                    if constexpr (STAGED) {
                        const double2 d = *reinterpret_cast<const double2 *>(Gc + o);
                        l0 = mul(d.x, l0);
                        l1 = mul(d.y, l1);
                    }
                    wn[h] = make_double2(add(mul(alpha, l0), mul(beta_k1, cc.x)), add(mul(alpha, l1), mul(beta_k1, cc.y)));
                    pn[h] = make_double2(add(pk_prev[h].x, mul(dk1, wn[h].x)), add(pk_prev[h].y, mul(dk1, wn[h].y)));
                }
#pragma unroll
                for (int h = 0; h < T2_CPT; ++h) {
                    if (!act[h]) continue;
                    *reinterpret_cast<double2 *>(w1_dst + off0 - nx + 256 * h) = wn[h];
                    *reinterpret_cast<double2 *>(pk1_dst + off0 - nx + 256 * h) = pn[h];
                    acc_w1[h] = add(acc_w1[h], add(mul(wn[h].x, wn[h].x), mul(wn[h].y, wn[h].y)));
                    acc_p1[h] = add(acc_p1[h], add(mul(pn[h].x, pn[h].x), mul(pn[h].y, pn[h].y)));
                }
                if ((jc + 1) % CL == 0 || jc + 1 == it.me) flush(acc_w1, acc_p1, jc, half);
            }
            if constexpr (STAGED && T2_DP) {
                if (jc >= it.mb && jc < it.me) warp_arrive(&B.pempty[p_held]);  // P(j-1): p and D both read
            } else if constexpr (STAGED) {
                if (jc >= it.mb - 1) {  // G(j-1): C's share of the release
                    warp_arrive(&B.gempty[gr.slot]);
                    gr.next();
                }
            }
            if (j - 1 >= it.mb - 1) warp_arrive(&B.vempty[s1]);  // V(j-1): its neighbours were last read above
#pragma unroll
            for (int h = 0; h < T2_CPT; ++h) {
                pk_prev[h] = pk_cur[h];
                vm1[h] = vc1[h];
                vc1[h] = vcur[h];
            }
            s1 = s0;
            vr.next();
            off0 += nx;
        }
        warp_arrive(&B.vempty[s1]);  // V(me)
        if constexpr (STAGED && !T2_DP) {  // G(me)
            warp_arrive(&B.gempty[gr.slot]);
            gr.next();
        }
    }
}

template <bool STAGED, bool R8>
ES_DEV void tb2_pass(const SeriesParams *P, int k, bool two, char *smem) {
    using Lt = Tb2Layout<STAGED>;
    const Geom g = P->g;
    const Tb2Items its = tb2_items_of(g, P->chunk_len);
    const TmaMaps &M = *static_cast<const TmaMaps *>(P->maps);
    const int pass = P->state->pass;
    // W: w_{k-1} (v on the first pass; pass p writes wbuf[p & 1]); P: p_{k-1} (v on the first pass)
    const int wi = pass == 0 ? 0 : (pass & 1) ? 1 : 2;  // v, wbuf[0], wbuf[1]
    const int pi = k == 1 ? 0 : ((k - 1) & 1) ? 2 : 1;  // p_{k-1}: v, pbuf[0], pbuf[1]
    const Tb2Maps mp = R8 ? Tb2Maps{&M.m[MAP_T2R_W_V + wi], nullptr, &M.m[MAP_T2R_G], nullptr, &M.m[MAP_T2R_P_V + pi],
                                    &M.m[MAP_T2R_D]}
                          : Tb2Maps{&M.m[wi == 0 ? MAP_WA_V : wi == 1 ? MAP_WA_0 : MAP_WA_1],
                                    &M.m[wi == 0 ? MAP_T2_W8_V : wi == 1 ? MAP_T2_W8_0 : MAP_T2_W8_1], &M.m[MAP_G],
                                    &M.m[MAP_T2_G4], &M.m[k == 1 ? MAP_WA_V : ((k - 1) & 1) ? MAP_P_1 : MAP_P_0],
                                    &M.m[MAP_G]};
    if (threadIdx.x == 0) {
        const Tb2Bars<STAGED> B(smem);
        for (int s = 0; s < Lt::SW; ++s) {
            mbar_init(&B.wfull[s], 1);
            mbar_init(&B.wempty[s], T2_AW);
        }
        for (int s = 0; s < Lt::SG; ++s) {
            mbar_init(&B.gfull[s], 1);
            mbar_init(&B.gempty[s], STAGED && T2_DP ? T2_AW : T2_AW + T2_CW);
        }
        for (int s = 0; s < Lt::SP; ++s) {
            mbar_init(&B.pfull[s], 1);
            mbar_init(&B.pempty[s], T2_CW);
        }
        for (int s = 0; s < Lt::SV; ++s) {
            mbar_init(&B.vfull[s], T2_AW);
            mbar_init(&B.vempty[s], T2_CW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int warp = threadIdx.x / 32;
    if (warp == T2_AW + T2_CW) {
        if ((threadIdx.x & 31) == 0) {
            for (const CUtensorMap *m : {mp.wa, mp.wb8, mp.p})
                if (m) tma_acquire(m);
            if (STAGED)
                for (const CUtensorMap *m : {mp.ga, mp.gb4, mp.dp})
                    if (m) tma_acquire(m);
            tb2_produce<STAGED, R8>(g, its, mp, smem, P->work);
        }
    } else if (warp < T2_AW) {
        tb2_group_a<STAGED, R8>(g, P, k, its, smem);
    } else {
        tb2_group_c<STAGED>(g, P, k, two, its, smem);
    }
}

}  // namespace es
