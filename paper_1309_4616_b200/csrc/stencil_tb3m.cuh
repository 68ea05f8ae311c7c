// Two Newton-Leja nodes per HBM pass on 3D slabs, plane-marching form (C3/C4).
//
// The pass of stencil_tb.cuh (w_k = A w_{k-1} and w_{k+1} = A w_k, the
// partial sums p_k, p_{k+1}; 40 B/point for two nodes with g') without its
// producer/consumer split between the two nodes -- the structure that took
// the 2D pass from 207 to 158 us (stencil_tb2m.cuh).  Each of the eight
// compute warps owns rows 2w and 2w + 1 of the 64 x 16 tile (T3M_ADJ; else w
// and w + 8, group C's rows; lane q: the pair x0 + 2q, so the norm partials land in the same
// (chunk, 64 x 8 tile, row) entries in the same order) and marches down the
// item's z chunk; w_{k-1} of planes j-1, j and w_k of planes j-2, j-1, j and
// p_k of the current plane stay in registers whose roles rotate over a
// three-way unrolled step:
//
//   step j:  w_k(j)        from w_{k-1}(j-1), w_{k-1}(j) (registers),
//                          w_{k-1}(j+1) (stage j+1), x/y neighbours (stage j)
//            p_k(j)        = p_{k-1}(j) + d_k w_k(j)
//            w_{k+1}(j-1)  from w_k(j-2), w_k(j-1), w_k(j) (registers) and the
//                          x/y neighbours of w_k(j-1) (the shared plane V(j-1))
//            p_{k+1}(j-1)  = p_k(j-1) + d_{k+1} w_{k+1}(j-1)
//
// w_k on the tile's one-point ring (rows y0-1, y0+16; columns x0-1, x0+64)
// comes from two edge warps, point by point with tb_point_scalar's
// expression (the neighbour tiles compute the same values the same way).
// Stage j (one per plane, producer = the last warp, one lane) holds
// W (w_{k-1}, 72 x 20 from x0-4, y0-2), G (g', 68 x 18 from x0-2, y0-1) and
// P (p_{k-1}, 64 x 16) -- the two-node kernel's own tensor maps; it is
// released one step late so the C part re-reads g'(j-1) instead of
// carrying it.
//
// Scope: one domain (no slab halos, no peer pushes), coefficient none,
// homogeneous Dirichlet or Neumann, with or without g'.
#pragma once

#include <type_traits>

#include "stencil_tb2m.cuh"  // tm_v_ready; stencil_tb.cuh

namespace es {

#ifndef T3M_S
#define T3M_S 6  // stages (planes) in flight
#endif
#ifndef T3M_PKR
#define T3M_PKR 0  // 1: re-derive p_k(j-1) from its (still held) P stage instead of carrying it
#endif
#ifndef T3M_LAG
// planes between a step's w_k (A part) and its w_{k+1} (C part): 1 or 2.  2
// makes the two fp64 chains of a step independent but holds four stages
// (two planes of prefetch at 6 stages): measured 1.12 vs 1.00 ms per 512^3 pass
#define T3M_LAG 1
#endif
// T3M_EARLY (LAG 1): publish w_k(j) before the C part, three V slots -- the
// other warps' wait for plane j then ends when every warp's A part is done
// (bitwise; measured equal, 945 vs 944 us per 512^3 pass)
#ifndef T3M_EARLY
#define T3M_EARLY 0
#endif
constexpr int T3M_NV = (T3M_LAG == 2 || T3M_EARLY) ? 3 : 2;  // shared w_k plane slots
#ifndef T3M_NW
#define T3M_NW 8  // compute warps: rows w + T3M_NW h of the 16-row tile
#endif
constexpr int T3M_RPW = 16 / T3M_NW;               // rows per compute warp
// T3M_ADJ: a warp owns adjacent rows (R w + h) instead of rows w + T3M_NW h,
// so one y neighbour of each row is the other row's register (LAG 1 only;
// 4 of 16 128-bit shared loads per step saved: 512^3 pass 912 -> 893 us)
#ifndef T3M_ADJ
#define T3M_ADJ 1
#endif
#define T3M_ROW(w, h) (T3M_ADJ ? T3M_RPW * (w) + (h) : (w) + T3M_NW * (h))
constexpr int T3M_THREADS = 32 * (T3M_NW + 3);     // + two edge warps + producer
static_assert(TB_TY == 16, "the plane-marching pass tiles 64 x 16");

template <bool GD>
struct T3mLayout {
    static constexpr int W_BYTES = (TB_WX * TB_WY * 8 + 127) & ~127;
    static constexpr int G_BYTES = GD ? (TB_GX * TB_GY * 8 + 127) & ~127 : 0;
    static constexpr int P_BYTES = 64 * TB_TY * 8;
    static constexpr int STAGE = W_BYTES + G_BYTES + P_BYTES;
    static constexpr int G_OFF = W_BYTES, P_OFF = W_BYTES + G_BYTES;
    static constexpr int V_SLOT = TB_EX * TB_EY;  // w_k of a plane with its ring, 68 x 18 from x0-2, y0-1
    static constexpr int V_OFF = T3M_S * STAGE;
    static constexpr int BAR_OFF = V_OFF + T3M_NV * V_SLOT * 8;
    static constexpr int NBAR = 2 * T3M_S + T3M_NV;
    static constexpr int ITEMQ_OFF = BAR_OFF + NBAR * 8;
    static constexpr int BYTES = ITEMQ_OFF + ((T3M_S * 4 + 15) & ~15);
};

template <bool GD>
struct T3mBars {
    uint64_t *full, *empty, *vfull;
    ES_DEV explicit T3mBars(char *smem) {
        full = reinterpret_cast<uint64_t *>(smem + T3mLayout<GD>::BAR_OFF);
        empty = full + T3M_S;
        vfull = empty + T3M_S;
    }
};

template <bool GD>
ES_DEV void t3m_produce(const Geom &g, const TbItems &its, const TbMaps &mp, char *smem, unsigned *work) {
    using Lt = T3mLayout<GD>;
    const T3mBars<GD> B(smem);
    volatile int *itemq = reinterpret_cast<volatile int *>(smem + Lt::ITEMQ_OFF);
    uint32_t q = 0;
    const int total = its.ntiles * its.nchunks;
    int i = work ? (int)atomicAdd(work, 1u) : (int)blockIdx.x;
    while (i < total) {
        const TbItem it = tb_item_at(its, i);
        int inext = -1;
        for (int t = it.mb - 2; t <= it.me + 1; ++t, ++q) {
            if (t == max(it.mb - 2, it.me - 3)) inext = work ? (int)atomicAdd(work, 1u) : i + (int)gridDim.x;
            const uint32_t s = q % T3M_S;
            if (q >= (uint32_t)T3M_S) mbar_wait_sleep(&B.empty[s], ((q / T3M_S) - 1) & 1);
            itemq[s] = i;
            const bool gplane = GD && t >= it.mb - 1 && t <= it.me;
            const bool pplane = t >= it.mb && t < it.me;
            mbar_expect_tx(&B.full[s], TB_WX * TB_WY * 8 + (gplane ? TB_GX * TB_GY * 8 : 0) + (pplane ? Lt::P_BYTES : 0));
            char *st = smem + s * Lt::STAGE;
            tma_load(st, mp.w, &B.full[s], it.x0 - 4, it.y0 - 2, march_src<true>(g, t, its.L));
            if (gplane) tma_load(st + Lt::G_OFF, mp.g, &B.full[s], it.x0 - 2, it.y0 - 1, t);
            if (pplane) tma_load(st + Lt::P_OFF, mp.p, &B.full[s], it.x0, it.y0, t);
        }
        i = inext;
    }
    const uint32_t s = q % T3M_S;  // end-of-work marker
    if (q >= (uint32_t)T3M_S) mbar_wait_sleep(&B.empty[s], ((q / T3M_S) - 1) & 1);
    itemq[s] = -1;
    mbar_arrive(&B.full[s]);
}

// one step's V slot (u % T3M_NV): wait until every warp has finished step u - 1
ES_DEV void t3m_v_ready(uint64_t *vfull, uint32_t u, bool sleep = false) {
    if (u == 0) return;
    if (sleep)
        mbar_wait_sleep(&vfull[(u - 1) % T3M_NV], ((u - 1) / T3M_NV) & 1);
    else
        mbar_wait(&vfull[(u - 1) % T3M_NV], ((u - 1) / T3M_NV) & 1);
}

// w_k at one ring point (x, y) of plane j: tb_point_scalar's expression with
// the z neighbours from registers; 0 outside the domain (the Dirichlet ghost;
// Neumann stencils at the domain edge use their own centre instead)
template <bool GD, bool NEU>
ES_DEV double t3m_ring_point(const Geom &g, const char *st, int64_t x0, int64_t y0, int64_t x, int64_t y, double zm,
                             double zp, double alpha, double beta) {
    if (!(x >= 0 && x < g.nx && y >= 0 && y < g.ny)) return 0.0;
    const double *Wc = reinterpret_cast<const double *>(st);
    const int o = (int)(y - (y0 - 2)) * TB_WX + (int)(x - (x0 - 4));
    const double c = Wc[o];
    double xm = Wc[o - 1], xp = Wc[o + 1], ym = Wc[o - TB_WX], yp = Wc[o + TB_WX];
    if constexpr (NEU) {
        if (x == 0) xm = c;
        if (x == g.nx - 1) xp = c;
        if (y == 0) ym = c;
        if (y == g.ny - 1) yp = c;
    }
    double lap = lap7(c, xm, xp, ym, yp, zm, zp, g.wx, g.wy, g.wz);
    if constexpr (GD) {
        const double *Gj = reinterpret_cast<const double *>(st + T3mLayout<GD>::G_OFF);
        lap = sub(lap, mul(Gj[(int)(y - (y0 - 1)) * TB_GX + (int)(x - (x0 - 2))], c));
    }
    return add(mul(alpha, lap), mul(beta, c));
}

// The edge warps: warp e (0, 1) owns ring row y0-1 / y0+16 (lane q: the
// points x0+2q, x0+2q+1) and, in lanes 0-15, ring column x0-1 / x0+64 at
// row y0+q.
template <bool GD, bool NEU>
ES_DEV void t3m_edge(const Geom &g, const SeriesParams *P, int k, const TbItems &its, char *smem, int e) {
    using Lt = T3mLayout<GD>;
    const T3mBars<GD> B(smem);
    const volatile int *itemq = reinterpret_cast<const volatile int *>(smem + Lt::ITEMQ_OFF);
    double *vrow = reinterpret_cast<double *>(smem + Lt::V_OFF);
    const int q = threadIdx.x & 31;
    const double alpha = P->alpha, beta_k = sub(-P->shift, P->xi[k - 1]);
    auto stage = [&](uint32_t s) { return smem + (s % T3M_S) * Lt::STAGE; };
    uint32_t s = 0, u = 0;
    for (;;) {
        mbar_wait_sleep(&B.full[s % T3M_S], (s / T3M_S) & 1);
        const int i = itemq[s % T3M_S];
        if (i < 0) break;
        const TbItem it = tb_item_at(its, i);
        int64_t px[3], py[3];
        px[0] = it.x0 + 2 * q;
        px[1] = px[0] + 1;
        py[0] = py[1] = e == 0 ? it.y0 - 1 : it.y0 + TB_TY;
        px[2] = e == 0 ? it.x0 - 1 : it.x0 + 64;
        py[2] = it.y0 + (q & 15);
        const bool col = q < 16;
        int wo[3], vo[3];
#pragma unroll
        for (int h = 0; h < 3; ++h) {
            wo[h] = (int)(py[h] - (it.y0 - 2)) * TB_WX + (int)(px[h] - (it.x0 - 4));
            vo[h] = (int)(py[h] - (it.y0 - 1)) * TB_EX + (int)(px[h] - (it.x0 - 2));
        }
        double em[3], ec[3];
        {
            const double *W0 = reinterpret_cast<const double *>(stage(s));
            mbar_wait_sleep(&B.full[(s + 1) % T3M_S], ((s + 1) / T3M_S) & 1);
            const double *W1 = reinterpret_cast<const double *>(stage(s + 1));
#pragma unroll
            for (int h = 0; h < 3; ++h) {
                em[h] = W0[wo[h]];
                ec[h] = W1[wo[h]];
            }
            warp_arrive(&B.empty[s % T3M_S]);
            ++s;  // s: stage of plane j
        }
        for (int j = it.mb - 1; j <= it.me + T3M_LAG - 1; ++j, ++u) {
            double wv[3] = {0.0, 0.0, 0.0};
            if (j <= it.me) {  // (LAG 2: the compute warps' extra C-only step has no plane)
                mbar_wait_sleep(&B.full[(s + 1) % T3M_S], ((s + 1) / T3M_S) & 1);
                const char *st = stage(s);
                const double *Wn = reinterpret_cast<const double *>(stage(s + 1));
                double ep[3];
#pragma unroll
                for (int h = 0; h < 3; ++h) ep[h] = Wn[wo[h]];
                if (j >= 0 && j < its.L) {
#pragma unroll
                    for (int h = 0; h < 3; ++h)
                        if (h < 2 || col)
                            wv[h] = t3m_ring_point<GD, NEU>(g, st, it.x0, it.y0, px[h], py[h], em[h], ep[h], alpha, beta_k);
                }
#pragma unroll
                for (int h = 0; h < 3; ++h) {
                    em[h] = ec[h];
                    ec[h] = ep[h];
                }
            }
            t3m_v_ready(B.vfull, u, true);
            double *V = vrow + (u % T3M_NV) * Lt::V_SLOT;
            V[vo[0]] = wv[0];
            V[vo[1]] = wv[1];
            if (col) V[vo[2]] = wv[2];
            warp_arrive(&B.vfull[u % T3M_NV]);
            if (j <= it.me) {
                warp_arrive(&B.empty[s % T3M_S]);
                ++s;
            }
        }
        warp_arrive(&B.empty[s % T3M_S]);  // plane me + 1
        ++s;
    }
}

template <bool GD, bool NEU>
ES_DEV void t3m_compute(const Geom &g, const SeriesParams *P, int k, bool two, const TbItems &its, char *smem) {
    using Lt = T3mLayout<GD>;
    const T3mBars<GD> B(smem);
    const volatile int *itemq = reinterpret_cast<const volatile int *>(smem + Lt::ITEMQ_OFF);
    double *vrow = reinterpret_cast<double *>(smem + Lt::V_OFF);
    const int w = threadIdx.x >> 5, q = threadIdx.x & 31;  // rows w + T3M_NW h; pair x0 + 2q
    const int64_t nx = g.nx, plane = g.nx * g.ny;
    const double wx = g.wx, wy = g.wy, wz = g.wz;
    const int pass = P->state->pass;
    double *const w1_dst = P->wbuf[pass & 1];  // w_{k+1}, or w_k on a one-node pass
    double *const pk_dst = P->pbuf[k & 1], *const pk1_dst = P->pbuf[(k + 1) & 1];
    double *const part = P->part;
    const bool store_pk = tb_store_pk(*P, two);
    const double alpha = P->alpha, beta_k = sub(-P->shift, P->xi[k - 1]), dk = P->dd[k];
    const double dk1 = two ? P->dd[k + 1] : 0.0, beta_k1 = two ? sub(-P->shift, P->xi[k]) : 0.0;
    const double pscale = k == 1 ? P->dd[0] : 1.0;  // first pass: P tiles hold v, p_0 = dd_0 v
    const int64_t half = (int64_t)P->nslices * P->ntiles * 2;
    // shared-memory offsets (doubles) of this lane's pair in row h of a W / G / P / V plane
    constexpr int R = T3M_RPW;
    int ow[R], og[R], op[R], ov[R];
#pragma unroll
    for (int h = 0; h < R; ++h) {
        const int r = T3M_ROW(w, h);
        ow[h] = (r + 2) * TB_WX + 2 * q + 4;
        og[h] = (r + 1) * TB_GX + 2 * q + 2;
        op[h] = r * 64 + 2 * q;
        ov[h] = (r + 1) * TB_EX + 2 * q + 2;
    }
    uint32_t s = 0, u = 0;
    // register roles rotate over three steps (no copies): w_{k-1} of planes
    // j-1, j, j+1; w_k of planes j-2, j-1, j; p_k of planes j-1, j
    double2 W0[R], W1[R], W2[R], U0[R], U1[R], U2[R], K0[R], K1[R], K2[R];
    for (;;) {
        mbar_wait(&B.full[s % T3M_S], (s / T3M_S) & 1);
        const int i = itemq[s % T3M_S];
        if (i < 0) break;
        const TbItem it = tb_item_at(its, i);
        const int64_t xa = it.x0 + 2 * q;
        int64_t ya[R];
        bool in0[R], in1[R];
#pragma unroll
        for (int h = 0; h < R; ++h) {
            ya[h] = it.y0 + T3M_ROW(w, h);
            in0[h] = xa < nx && ya[h] < g.ny;
            in1[h] = xa + 1 < nx && ya[h] < g.ny;
        }
        // warp-uniform: does this warp hold a domain-edge column / row (Neumann
        // ghost rules) or points outside the domain (Dirichlet masks)?
        const bool xedge = it.x0 == 0 || it.x0 + 64 >= nx;
        const int ylast = it.y0 + T3M_ROW(w, R - 1);  // this warp's last row
        const bool yedge = it.y0 + T3M_ROW(w, 0) == 0 || ylast >= g.ny - 1;
        const bool special = NEU ? (xedge || yedge) : (it.x0 + 64 > nx || ylast >= g.ny);
        double acc_w0[R], acc_p0[R], acc_w1[R], acc_p1[R];
#pragma unroll
        for (int h = 0; h < R; ++h) acc_w0[h] = acc_p0[h] = acc_w1[h] = acc_p1[h] = 0.0;
        {
            const double *S0 = reinterpret_cast<const double *>(smem + (s % T3M_S) * Lt::STAGE);
            mbar_wait(&B.full[(s + 1) % T3M_S], ((s + 1) / T3M_S) & 1);
            const double *S1 = reinterpret_cast<const double *>(smem + ((s + 1) % T3M_S) * Lt::STAGE);
#pragma unroll
            for (int h = 0; h < R; ++h) {
                W0[h] = *reinterpret_cast<const double2 *>(S0 + ow[h]);
                W1[h] = *reinterpret_cast<const double2 *>(S1 + ow[h]);
                U0[h] = U1[h] = K0[h] = make_double2(0.0, 0.0);
            }
            ++s;  // s: stage of plane j (plane mb - 2 is released by the first step)
        }
        const int64_t off0 = (int64_t)(it.mb - 1) * plane + it.y0 * nx + xa + (int64_t)T3M_ROW(w, 0) * nx;  // row h = 0, plane j
        const int64_t drow = (int64_t)(T3M_ROW(w, 1) - T3M_ROW(w, 0)) * nx;
        double *pk_row = pk_dst + off0, *wk_row = w1_dst + off0;
        double *wn_row = w1_dst + off0 - plane, *pn_row = pk1_dst + off0 - plane;
        int j = it.mb - 1;
        // FULL (a compile-time tag): every lane of this warp holds domain points -- no per-lane guards
        auto step = [&](auto full, auto steady, double2 (&vm)[R], double2 (&vc)[R], double2 (&vp)[R], double2 (&um)[R], double2 (&uc)[R],
                        double2 (&wk)[R], double2 (&pk_prev)[R], double2 (&pk)[R]) -> bool {
            const char *st = smem + (s % T3M_S) * Lt::STAGE;  // plane j
            const double *Wn = reinterpret_cast<const double *>(smem + ((s + 1) % T3M_S) * Lt::STAGE);
            mbar_wait(&B.full[(s + 1) % T3M_S], ((s + 1) / T3M_S) & 1);
#pragma unroll
            for (int h = 0; h < R; ++h) vp[h] = *reinterpret_cast<const double2 *>(Wn + ow[h]);
            // ---- w_k(j)
            if (decltype(steady)::value || (j >= 0 && j < its.L)) {  // steady: an interior plane / row
                const double *Wc = reinterpret_cast<const double *>(st);
                const double *Gc = reinterpret_cast<const double *>(st + Lt::G_OFF);
#pragma unroll
                for (int h = 0; h < R; ++h) {
                    // T3M_ADJ: the warp's other row is a y neighbour held in registers
                    const double2 ym = T3M_ADJ && h > 0 ? vc[h > 0 ? h - 1 : 0]
                                                        : *reinterpret_cast<const double2 *>(Wc + ow[h] - TB_WX);
                    const double2 yp = T3M_ADJ && h < R - 1 ? vc[h < R - 1 ? h + 1 : 0]
                                                            : *reinterpret_cast<const double2 *>(Wc + ow[h] + TB_WX);
                    double xm = Wc[ow[h] - 1], xp = Wc[ow[h] + 2];
                    double ym0 = ym.x, ym1 = ym.y, yp0 = yp.x, yp1 = yp.y;
                    if (NEU && special) {  // the point itself is the ghost at the domain edge
                        if (xa == 0) xm = vc[h].x;
                        if (xa + 1 == nx - 1) xp = vc[h].y;
                        if (ya[h] == 0) {
                            ym0 = vc[h].x;
                            ym1 = vc[h].y;
                        }
                        if (ya[h] == g.ny - 1) {
                            yp0 = vc[h].x;
                            yp1 = vc[h].y;
                        }
                    }
                    double l0 = lap7(vc[h].x, xm, vc[h].y, ym0, yp0, vm[h].x, vp[h].x, wx, wy, wz);
                    double l1 = lap7(vc[h].y, vc[h].x, xp, ym1, yp1, vm[h].y, vp[h].y, wx, wy, wz);
                    if constexpr (GD) {
                        const double2 gv = *reinterpret_cast<const double2 *>(Gc + og[h]);
                        l0 = sub(l0, mul(gv.x, vc[h].x));
                        l1 = sub(l1, mul(gv.y, vc[h].y));
                    }
                    wk[h] = make_double2(add(mul(alpha, l0), mul(beta_k, vc[h].x)),
                                         add(mul(alpha, l1), mul(beta_k, vc[h].y)));
                    if (!NEU && special) wk[h] = make_double2(in0[h] ? wk[h].x : 0.0, in1[h] ? wk[h].y : 0.0);
                }
            } else {
#pragma unroll
                for (int h = 0; h < R; ++h) wk[h] = NEU && j == its.L ? uc[h] : make_double2(0.0, 0.0);  // plane L mirrors L - 1
            }
            // ---- p_k(j) (+ node k norms)
            if (decltype(steady)::value || (j >= it.mb && j < it.me)) {
                const double *Pc = reinterpret_cast<const double *>(st + Lt::P_OFF);
#pragma unroll
                for (int h = 0; h < R; ++h) {
                    const double2 po = *reinterpret_cast<const double2 *>(Pc + op[h]);
                    // pscale is 1.0 after the first pass, and 1.0 * x == x bit for bit
                    pk[h] = make_double2(add(mul(pscale, po.x), mul(dk, wk[h].x)),
                                         add(mul(pscale, po.y), mul(dk, wk[h].y)));
                    if (decltype(full)::value || in0[h]) {
                        if (store_pk) *reinterpret_cast<double2 *>(pk_row + h * drow) = pk[h];
                        if (!two) *reinterpret_cast<double2 *>(wk_row + h * drow) = wk[h];  // the next pass starts from w_k
                        acc_w0[h] = add(acc_w0[h], add(mul(wk[h].x, wk[h].x), mul(wk[h].y, wk[h].y)));
                        acc_p0[h] = add(acc_p0[h], add(mul(pk[h].x, pk[h].x), mul(pk[h].y, pk[h].y)));
                    }
                }
            }
            // ---- w_{k+1}(j-1), p_{k+1}(j-1) (+ node k+1 norms)
            t3m_v_ready(B.vfull, u);
            if constexpr (T3M_EARLY) {  // publish w_k(j) now (slot u % 3 held V(u-3), read at step u-2)
                double *Vn = vrow + (u % T3M_NV) * Lt::V_SLOT;
#pragma unroll
                for (int h = 0; h < R; ++h) *reinterpret_cast<double2 *>(Vn + ov[h]) = wk[h];
                warp_arrive(&B.vfull[u % T3M_NV]);
            }
            const int jc = j - 1;
            if (two && (decltype(steady)::value || (jc >= it.mb && jc < it.me))) {
                const double *Vc = vrow + ((u - 1) % T3M_NV) * Lt::V_SLOT;  // w_k(j-1) with its ring
                const double *Gp = reinterpret_cast<const double *>(smem + ((s - 1) % T3M_S) * Lt::STAGE + Lt::G_OFF);
                double2 pkp[R];  // p_k(j-1)
#pragma unroll
                for (int h = 0; h < R; ++h) {
                    if constexpr (T3M_PKR) {  // the same expression on the same operands: bitwise the carried value
                        const double2 po = *reinterpret_cast<const double2 *>(
                            smem + ((s - 1) % T3M_S) * Lt::STAGE + Lt::P_OFF + 8 * op[h]);
                        pkp[h] = make_double2(add(mul(pscale, po.x), mul(dk, uc[h].x)),
                                              add(mul(pscale, po.y), mul(dk, uc[h].y)));
                    } else {
                        pkp[h] = pk_prev[h];
                    }
                }
#pragma unroll
                for (int h = 0; h < R; ++h) {
                    const double2 cc = uc[h];
                    const double2 ym = T3M_ADJ && h > 0 ? uc[h > 0 ? h - 1 : 0]
                                                        : *reinterpret_cast<const double2 *>(Vc + ov[h] - TB_EX);
                    const double2 yp = T3M_ADJ && h < R - 1 ? uc[h < R - 1 ? h + 1 : 0]
                                                            : *reinterpret_cast<const double2 *>(Vc + ov[h] + TB_EX);
                    double xm = Vc[ov[h] - 1], xp = Vc[ov[h] + 2];
                    double ym0 = ym.x, ym1 = ym.y, yp0 = yp.x, yp1 = yp.y;
                    double2 zm = um[h], zp = wk[h];
                    if (NEU) {
                        if (special) {
                            if (xa == 0) xm = cc.x;
                            if (xa + 1 == nx - 1) xp = cc.y;
                            if (ya[h] == 0) {
                                ym0 = cc.x;
                                ym1 = cc.y;
                            }
                            if (ya[h] == g.ny - 1) {
                                yp0 = cc.x;
                                yp1 = cc.y;
                            }
                        }
                        if (jc == 0) zm = cc;  // plane -1 mirrors plane 0
                    }
                    double l0 = lap7(cc.x, xm, cc.y, ym0, yp0, zm.x, zp.x, wx, wy, wz);
                    double l1 = lap7(cc.y, cc.x, xp, ym1, yp1, zm.y, zp.y, wx, wy, wz);
                    if constexpr (GD) {
                        const double2 gv = *reinterpret_cast<const double2 *>(Gp + og[h]);
                        l0 = sub(l0, mul(gv.x, cc.x));
                        l1 = sub(l1, mul(gv.y, cc.y));
                    }
                    const double2 wn = make_double2(add(mul(alpha, l0), mul(beta_k1, cc.x)),
                                                    add(mul(alpha, l1), mul(beta_k1, cc.y)));
                    const double2 pn =
                        make_double2(add(pkp[h].x, mul(dk1, wn.x)), add(pkp[h].y, mul(dk1, wn.y)));
                    if (decltype(full)::value || in0[h]) {
                        *reinterpret_cast<double2 *>(wn_row + h * drow) = wn;
                        *reinterpret_cast<double2 *>(pn_row + h * drow) = pn;
                        acc_w1[h] = add(acc_w1[h], add(mul(wn.x, wn.x), mul(wn.y, wn.y)));
                        acc_p1[h] = add(acc_p1[h], add(mul(pn.x, pn.x), mul(pn.y, pn.y)));
                    }
                }
            }
            // ---- publish w_k(j): the x/y neighbours of the next step's C part
            if constexpr (!T3M_EARLY) {
                double *Vn = vrow + (u % T3M_NV) * Lt::V_SLOT;
#pragma unroll
                for (int h = 0; h < R; ++h) *reinterpret_cast<double2 *>(Vn + ov[h]) = wk[h];
                warp_arrive(&B.vfull[u % T3M_NV]);
            }
            warp_arrive(&B.empty[(s - 1) % T3M_S]);  // plane j - 1: its g' was last read above
            ++j;
            ++s;
            ++u;
            pk_row += plane;
            wk_row += plane;
            wn_row += plane;
            pn_row += plane;
            return j <= it.me;
        };
        auto march = [&](auto full) {
            for (;;) {
                // three steady steps (interior planes: every part active, no range checks)
                if constexpr (decltype(full)::value) {
                    if (j >= it.mb + 1 && j + 2 <= it.me - 1) {
                        step(full, std::true_type{}, W0, W1, W2, U0, U1, U2, K0, K1);
                        step(full, std::true_type{}, W1, W2, W0, U1, U2, U0, K1, K2);
                        step(full, std::true_type{}, W2, W0, W1, U2, U0, U1, K2, K0);
                        continue;
                    }
                }
                if (!step(full, std::false_type{}, W0, W1, W2, U0, U1, U2, K0, K1)) break;
                if (!step(full, std::false_type{}, W1, W2, W0, U1, U2, U0, K1, K2)) break;
                if (!step(full, std::false_type{}, W2, W0, W1, U2, U0, U1, K2, K0)) break;
            }
        };
        if (it.x0 + 64 <= nx && ylast < g.ny)
            march(std::true_type{});
        else
            march(std::false_type{});
        warp_arrive(&B.empty[(s - 1) % T3M_S]);  // planes me, me + 1
        warp_arrive(&B.empty[s % T3M_S]);
        ++s;
        // (chunk, 64 x 8 tile, row) partials of both nodes, one-node kernel layout
#pragma unroll
        for (int h = 0; h < R; ++h) {
            const double w0 = warp_sum(acc_w0[h]), p0 = warp_sum(acc_p0[h]);
            const double w1 = warp_sum(acc_w1[h]), p1 = warp_sum(acc_p1[h]);
            const int r = T3M_ROW(w, h);
            if (q == 0 && it.y0 + (r & ~7) < g.ny) {  // the 64 x 8 tile of row r exists
                const int64_t e =
                    ((int64_t)it.chunk * its.ntiles8 + it.tile8 + (r >> 3) * its.tiles_x) * TMA_CONSUMER_WARPS + (r & 7);
                double *d0p = part + e * 2;
                d0p[0] = w0;
                d0p[1] = p0;
                double *d1p = part + half + e * 2;
                d1p[0] = w1;
                d1p[1] = p1;
            }
        }
    }
}

// T3M_LAG == 2: the C part of step j works on plane j - 2, so it depends on
// nothing the step's A part computes -- the two fp64 chains of a step are
// independent and interleave.  w_k of planes j-3 .. j (four register roles),
// p_k(j-2) re-derived from its P stage, g'(j-2) and P(j-2) held until step j,
// three V slots.
template <bool GD, bool NEU>
ES_DEV void t3m_compute2(const Geom &g, const SeriesParams *P, int k, bool two, const TbItems &its, char *smem) {
    using Lt = T3mLayout<GD>;
    constexpr int R = T3M_RPW;
    const T3mBars<GD> B(smem);
    const volatile int *itemq = reinterpret_cast<const volatile int *>(smem + Lt::ITEMQ_OFF);
    double *vrow = reinterpret_cast<double *>(smem + Lt::V_OFF);
    const int w = threadIdx.x >> 5, q = threadIdx.x & 31;  // rows w + T3M_NW h; pair x0 + 2q
    const int64_t nx = g.nx, plane = g.nx * g.ny;
    const double wx = g.wx, wy = g.wy, wz = g.wz;
    const int pass = P->state->pass;
    double *const w1_dst = P->wbuf[pass & 1];
    double *const pk_dst = P->pbuf[k & 1], *const pk1_dst = P->pbuf[(k + 1) & 1];
    double *const part = P->part;
    const bool store_pk = tb_store_pk(*P, two);
    const double alpha = P->alpha, beta_k = sub(-P->shift, P->xi[k - 1]), dk = P->dd[k];
    const double dk1 = two ? P->dd[k + 1] : 0.0, beta_k1 = two ? sub(-P->shift, P->xi[k]) : 0.0;
    const double pscale = k == 1 ? P->dd[0] : 1.0;
    const int64_t half = (int64_t)P->nslices * P->ntiles * 2;
    int ow[R], og[R], op[R], ov[R];
#pragma unroll
    for (int h = 0; h < R; ++h) {
        const int r = w + T3M_NW * h;
        ow[h] = (r + 2) * TB_WX + 2 * q + 4;
        og[h] = (r + 1) * TB_GX + 2 * q + 2;
        op[h] = r * 64 + 2 * q;
        ov[h] = (r + 1) * TB_EX + 2 * q + 2;
    }
    uint32_t s = 0, u = 0;
    double2 W0[R], W1[R], W2[R], W3[R], U0[R], U1[R], U2[R], U3[R];
    for (;;) {
        mbar_wait(&B.full[s % T3M_S], (s / T3M_S) & 1);
        const int i = itemq[s % T3M_S];
        if (i < 0) break;
        const TbItem it = tb_item_at(its, i);
        const int64_t xa = it.x0 + 2 * q;
        int64_t ya[R];
        bool in0[R], in1[R];
#pragma unroll
        for (int h = 0; h < R; ++h) {
            ya[h] = it.y0 + w + T3M_NW * h;
            in0[h] = xa < nx && ya[h] < g.ny;
            in1[h] = xa + 1 < nx && ya[h] < g.ny;
        }
        const int ylast = it.y0 + w + T3M_NW * (R - 1);
        const bool xedge = it.x0 == 0 || it.x0 + 64 >= nx;
        const bool yedge = it.y0 + w == 0 || ylast >= g.ny - 1;
        const bool special = NEU ? (xedge || yedge) : (it.x0 + 64 > nx || ylast >= g.ny);
        double acc_w0[R], acc_p0[R], acc_w1[R], acc_p1[R];
#pragma unroll
        for (int h = 0; h < R; ++h) acc_w0[h] = acc_p0[h] = acc_w1[h] = acc_p1[h] = 0.0;
        {
            const double *S0 = reinterpret_cast<const double *>(smem + (s % T3M_S) * Lt::STAGE);
            mbar_wait(&B.full[(s + 1) % T3M_S], ((s + 1) / T3M_S) & 1);
            const double *S1 = reinterpret_cast<const double *>(smem + ((s + 1) % T3M_S) * Lt::STAGE);
#pragma unroll
            for (int h = 0; h < R; ++h) {
                W0[h] = *reinterpret_cast<const double2 *>(S0 + ow[h]);
                W1[h] = *reinterpret_cast<const double2 *>(S1 + ow[h]);
                U0[h] = U1[h] = U2[h] = make_double2(0.0, 0.0);
            }
            ++s;  // s: stage of plane j
        }
        const int64_t off0 = (int64_t)(it.mb - 1) * plane + it.y0 * nx + xa + (int64_t)w * nx;  // row 0, plane j
        const int64_t drow = (int64_t)T3M_NW * nx;
        double *pk_row = pk_dst + off0, *wk_row = w1_dst + off0;
        double *wn_row = w1_dst + off0 - 2 * plane, *pn_row = pk1_dst + off0 - 2 * plane;
        int j = it.mb - 1;
        // roles: vm, vc, vp = w_{k-1}(j-1, j, j+1); um, uc, up, wk = w_k(j-3, j-2, j-1, j)
        auto step = [&](double2 (&vm)[R], double2 (&vc)[R], double2 (&vp)[R], double2 (&um)[R], double2 (&uc)[R],
                        double2 (&up)[R], double2 (&wk)[R]) -> bool {
            const bool a_part = j <= it.me;  // the last step (plane me + 1) is C only
            if (a_part) mbar_wait(&B.full[(s + 1) % T3M_S], ((s + 1) / T3M_S) & 1);
            t3m_v_ready(B.vfull, u);  // every warp finished step u - 1 (V(u-2) complete, slot u % 3 free)
            // ---- C part: w_{k+1}(j-2), p_{k+1}(j-2) -- independent of this step's A part
            const int jc = j - 2;
            if (two && jc >= it.mb && jc < it.me) {
                const double *Vc = vrow + ((u - 2) % T3M_NV) * Lt::V_SLOT;  // w_k(j-2) with its ring
                const char *sc = smem + ((s - 2) % T3M_S) * Lt::STAGE;      // g', P of plane j-2
                const double *Gp = reinterpret_cast<const double *>(sc + Lt::G_OFF);
                const double *Pp = reinterpret_cast<const double *>(sc + Lt::P_OFF);
#pragma unroll
                for (int h = 0; h < R; ++h) {
                    const double2 cc = uc[h];
                    const double2 ym = *reinterpret_cast<const double2 *>(Vc + ov[h] - TB_EX);
                    const double2 yp = *reinterpret_cast<const double2 *>(Vc + ov[h] + TB_EX);
                    double xm = Vc[ov[h] - 1], xp = Vc[ov[h] + 2];
                    double ym0 = ym.x, ym1 = ym.y, yp0 = yp.x, yp1 = yp.y;
                    double2 zm = um[h], zp = up[h];
                    if (NEU) {
                        if (special) {
                            if (xa == 0) xm = cc.x;
                            if (xa + 1 == nx - 1) xp = cc.y;
                            if (ya[h] == 0) {
                                ym0 = cc.x;
                                ym1 = cc.y;
                            }
                            if (ya[h] == g.ny - 1) {
                                yp0 = cc.x;
                                yp1 = cc.y;
                            }
                        }
                        if (jc == 0) zm = cc;              // plane -1 mirrors plane 0
                        if (jc == its.L - 1) zp = cc;      // plane L mirrors plane L - 1
                    }
                    double l0 = lap7(cc.x, xm, cc.y, ym0, yp0, zm.x, zp.x, wx, wy, wz);
                    double l1 = lap7(cc.y, cc.x, xp, ym1, yp1, zm.y, zp.y, wx, wy, wz);
                    if constexpr (GD) {
                        const double2 gv = *reinterpret_cast<const double2 *>(Gp + og[h]);
                        l0 = sub(l0, mul(gv.x, cc.x));
                        l1 = sub(l1, mul(gv.y, cc.y));
                    }
                    const double2 po = *reinterpret_cast<const double2 *>(Pp + op[h]);
                    // p_k(j-2): the A part's expression on the same operands (bitwise)
                    const double2 pkc = make_double2(add(mul(pscale, po.x), mul(dk, cc.x)),
                                                     add(mul(pscale, po.y), mul(dk, cc.y)));
                    const double2 wn = make_double2(add(mul(alpha, l0), mul(beta_k1, cc.x)),
                                                    add(mul(alpha, l1), mul(beta_k1, cc.y)));
                    const double2 pn = make_double2(add(pkc.x, mul(dk1, wn.x)), add(pkc.y, mul(dk1, wn.y)));
                    if (in0[h]) {
                        *reinterpret_cast<double2 *>(wn_row + h * drow) = wn;
                        *reinterpret_cast<double2 *>(pn_row + h * drow) = pn;
                        acc_w1[h] = add(acc_w1[h], add(mul(wn.x, wn.x), mul(wn.y, wn.y)));
                        acc_p1[h] = add(acc_p1[h], add(mul(pn.x, pn.x), mul(pn.y, pn.y)));
                    }
                }
            }
            // ---- A part: w_k(j), p_k(j)
            if (a_part) {
                const char *st = smem + (s % T3M_S) * Lt::STAGE;
                const double *Wn = reinterpret_cast<const double *>(smem + ((s + 1) % T3M_S) * Lt::STAGE);
#pragma unroll
                for (int h = 0; h < R; ++h) vp[h] = *reinterpret_cast<const double2 *>(Wn + ow[h]);
                if (j >= 0 && j < its.L) {
                    const double *Wc = reinterpret_cast<const double *>(st);
                    const double *Gc = reinterpret_cast<const double *>(st + Lt::G_OFF);
#pragma unroll
                    for (int h = 0; h < R; ++h) {
                        const double2 ym = *reinterpret_cast<const double2 *>(Wc + ow[h] - TB_WX);
                        const double2 yp = *reinterpret_cast<const double2 *>(Wc + ow[h] + TB_WX);
                        double xm = Wc[ow[h] - 1], xp = Wc[ow[h] + 2];
                        double ym0 = ym.x, ym1 = ym.y, yp0 = yp.x, yp1 = yp.y;
                        if (NEU && special) {
                            if (xa == 0) xm = vc[h].x;
                            if (xa + 1 == nx - 1) xp = vc[h].y;
                            if (ya[h] == 0) {
                                ym0 = vc[h].x;
                                ym1 = vc[h].y;
                            }
                            if (ya[h] == g.ny - 1) {
                                yp0 = vc[h].x;
                                yp1 = vc[h].y;
                            }
                        }
                        double l0 = lap7(vc[h].x, xm, vc[h].y, ym0, yp0, vm[h].x, vp[h].x, wx, wy, wz);
                        double l1 = lap7(vc[h].y, vc[h].x, xp, ym1, yp1, vm[h].y, vp[h].y, wx, wy, wz);
                        if constexpr (GD) {
                            const double2 gv = *reinterpret_cast<const double2 *>(Gc + og[h]);
                            l0 = sub(l0, mul(gv.x, vc[h].x));
                            l1 = sub(l1, mul(gv.y, vc[h].y));
                        }
                        wk[h] = make_double2(add(mul(alpha, l0), mul(beta_k, vc[h].x)),
                                             add(mul(alpha, l1), mul(beta_k, vc[h].y)));
                        if (!NEU && special) wk[h] = make_double2(in0[h] ? wk[h].x : 0.0, in1[h] ? wk[h].y : 0.0);
                    }
                } else {
#pragma unroll
                    for (int h = 0; h < R; ++h) wk[h] = make_double2(0.0, 0.0);
                }
                if (j >= it.mb && j < it.me) {
                    const double *Pc = reinterpret_cast<const double *>(st + Lt::P_OFF);
#pragma unroll
                    for (int h = 0; h < R; ++h) {
                        const double2 po = *reinterpret_cast<const double2 *>(Pc + op[h]);
                        const double2 pk = make_double2(add(mul(pscale, po.x), mul(dk, wk[h].x)),
                                                        add(mul(pscale, po.y), mul(dk, wk[h].y)));
                        if (in0[h]) {
                            if (store_pk) *reinterpret_cast<double2 *>(pk_row + h * drow) = pk;
                            if (!two) *reinterpret_cast<double2 *>(wk_row + h * drow) = wk[h];
                            acc_w0[h] = add(acc_w0[h], add(mul(wk[h].x, wk[h].x), mul(wk[h].y, wk[h].y)));
                            acc_p0[h] = add(acc_p0[h], add(mul(pk.x, pk.x), mul(pk.y, pk.y)));
                        }
                    }
                }
            }
            // ---- publish w_k(j) (x/y neighbours of the C part two steps on)
            double *Vn = vrow + (u % T3M_NV) * Lt::V_SLOT;
#pragma unroll
            for (int h = 0; h < R; ++h) *reinterpret_cast<double2 *>(Vn + ov[h]) = wk[h];
            warp_arrive(&B.vfull[u % T3M_NV]);
            if (j >= it.mb) warp_arrive(&B.empty[(s - 2) % T3M_S]);  // plane j - 2: g', P last read above
            ++j;
            ++u;
            if (a_part) ++s;
            pk_row += plane;
            wk_row += plane;
            wn_row += plane;
            pn_row += plane;
            return j <= it.me + 1;
        };
        for (;;) {
            if (!step(W0, W1, W2, U0, U1, U2, U3)) break;
            if (!step(W1, W2, W3, U1, U2, U3, U0)) break;
            if (!step(W2, W3, W0, U2, U3, U0, U1)) break;
            if (!step(W3, W0, W1, U3, U0, U1, U2)) break;
        }
        // s: stage of plane me + 1 (the C-only last step did not advance it); planes me, me + 1 still held
        warp_arrive(&B.empty[(s - 1) % T3M_S]);
        warp_arrive(&B.empty[s % T3M_S]);
        ++s;
#pragma unroll
        for (int h = 0; h < R; ++h) {
            const double w0 = warp_sum(acc_w0[h]), p0 = warp_sum(acc_p0[h]);
            const double w1 = warp_sum(acc_w1[h]), p1 = warp_sum(acc_p1[h]);
            const int r = w + T3M_NW * h;
            if (q == 0 && it.y0 + (r & ~7) < g.ny) {
                const int64_t e =
                    ((int64_t)it.chunk * its.ntiles8 + it.tile8 + (r >> 3) * its.tiles_x) * TMA_CONSUMER_WARPS + (r & 7);
                double *d0p = part + e * 2;
                d0p[0] = w0;
                d0p[1] = p0;
                double *d1p = part + half + e * 2;
                d1p[0] = w1;
                d1p[1] = p1;
            }
        }
    }
}

template <bool GD, bool NEU>
ES_DEV void t3m_pass(const SeriesParams *P, int k, bool two, char *smem) {
    using Lt = T3mLayout<GD>;
    const Geom g = P->g;
    const TbItems its = tb_items_of(g, P->chunk_len);
    const TmaMaps &M = *static_cast<const TmaMaps *>(P->maps);
    const int pass = P->state->pass;
    const TbMaps mp{&M.m[pass == 0 ? MAP_T_V : (pass & 1) ? MAP_T_0 : MAP_T_1], &M.m[MAP_T_G],
                    &M.m[k == 1 ? MAP_T_PV : ((k - 1) & 1) ? MAP_T_P1 : MAP_T_P0]};
    if (threadIdx.x == 0) {
        const T3mBars<GD> B(smem);
        for (int s = 0; s < T3M_S; ++s) {
            mbar_init(&B.full[s], 1);
            mbar_init(&B.empty[s], T3M_NW + 2);
        }
        for (int s = 0; s < T3M_NV; ++s) mbar_init(&B.vfull[s], T3M_NW + 2);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int warp = threadIdx.x / 32;
    if (warp == T3M_NW + 2) {
        if ((threadIdx.x & 31) == 0) {
            tma_acquire(mp.w);
            tma_acquire(mp.p);
            if (GD) tma_acquire(mp.g);
            t3m_produce<GD>(g, its, mp, smem, P->work);
        }
    } else if (warp >= T3M_NW) {
        t3m_edge<GD, NEU>(g, P, k, its, smem, warp - T3M_NW);
    } else {
        if constexpr (T3M_LAG == 2)
            t3m_compute2<GD, NEU>(g, P, k, two, its, smem);
        else
            t3m_compute<GD, NEU>(g, P, k, two, its, smem);
    }
}

}  // namespace es
