// Two Newton-Leja nodes per HBM pass on single-plane (2D) grids, row-marching
// form (C2).
//
// Same pass as stencil_tb2d.cuh -- w_k = A w_{k-1} and w_{k+1} = A w_k, the
// partial sums p_k, p_{k+1}, 48 B per point for two nodes -- but without the
// producer/consumer split between the two nodes.  Each compute warp owns
// TM_PP groups of 64 columns (lane l: the pairs x0 + 64 (TM_PP w + h) + 2 l)
// and marches down the rows of its item; the rows of w_{k-1} and w_k it
// needs in y stay in registers:
//
//   step t:  w_k(t)        from w_{k-1}(t-1), w_{k-1}(t) (registers),
//                          w_{k-1}(t+1) (stage t+1), x-neighbours (stage t)
//            p_k(t)        = p_{k-1}(t) + d_k w_k(t)
//            w_{k+1}(t-1)  from w_k(t-2), w_k(t-1), w_k(t) (registers) and the
//                          x-neighbours of w_k(t-1) (the shared row V(t-1))
//            p_{k+1}(t-1)  = p_k(t-1) + d_{k+1} w_{k+1}(t-1)
//
// so per row a warp waits once for its stage and once for the previous
// row's V (published by every warp one step earlier: no lock-step).  The
// x-neighbours of w_k just outside the tile (x0 - 1, x0 + TX) come from a
// small edge warp that evaluates those two points per row the way their
// owning tile does.  Norm partials keep the one-node kernel's (row chunk,
// 512-wide tile, 64-column warp) layout with the one-node lane order, so
// k_slice_reduce2 sums exactly what the one-node series sums
// (test_two_node_2d_bitwise).
//
// Stage t (one per row, producer = the last warp, one lane):
//   W: w_{k-1} row t, x0-4 .. x0+TX+3 (rows mb-2 .. me+1; v on the first pass);
//   D: staged coefficient row t, x0-2 .. x0+TX+1 (rows mb-1 .. me);
//   P: p_{k-1} row t, x0 .. x0+TX-1 (rows mb .. me-1; v on the first pass).
// A stage is read at steps t-1 (the fresh row) and t, then released.
//
// Scope as stencil_tb2d.cuh: homogeneous Dirichlet (TMA zero fill) and
// Neumann (mirrored ghosts), no coefficient or the staged sampled D, no g'.
#pragma once

#include <type_traits>

#include "stencil_tb2d.cuh"

namespace es {

#ifndef TM_NW
#define TM_NW 4  // compute warps
#endif
#ifndef TM_PP
#define TM_PP 2  // pairs per lane: a warp owns 64 TM_PP columns (TM_PP one-node norm warps)
#endif
#ifndef TM_S
#define TM_S 8  // stages (rows) in flight
#endif
constexpr int TM_TX = 64 * TM_PP * TM_NW;
constexpr int TM_THREADS = 32 * (TM_NW + 2);  // + edge warp + producer warp
#ifndef TM_MINB
#define TM_MINB (TM_TX == 512 ? 2 : 4)
#endif
static_assert(TM_TX == 256 || TM_TX == 512, "tile width: one-node tiles are 512 wide");

template <bool STAGED>
struct TmLayout {
    static constexpr int W_BYTES = ((TM_TX + 8) * 8 + 127) & ~127;
    static constexpr int D_BYTES = STAGED ? ((TM_TX + 4) * 8 + 127) & ~127 : 0;
    static constexpr int P_BYTES = TM_TX * 8;
    static constexpr int STAGE = W_BYTES + D_BYTES + P_BYTES;
    static constexpr int D_OFF = W_BYTES, P_OFF = W_BYTES + D_BYTES;
    static constexpr int V_SLOT = TM_TX + 4;  // w_k of a row, x0-2 .. x0+TX+1
    static constexpr int V_OFF = TM_S * STAGE;
    static constexpr int BAR_OFF = V_OFF + 2 * V_SLOT * 8;
    static constexpr int NBAR = 2 * TM_S + 2;
    static constexpr int ITEMQ_OFF = BAR_OFF + NBAR * 8;
    static constexpr int BYTES = ITEMQ_OFF + ((TM_S * 4 + 15) & ~15);
};

template <bool STAGED>
struct TmBars {
    uint64_t *full, *empty, *vfull;
    ES_DEV explicit TmBars(char *smem) {
        full = reinterpret_cast<uint64_t *>(smem + TmLayout<STAGED>::BAR_OFF);
        empty = full + TM_S;
        vfull = empty + TM_S;
    }
};

ES_DEV Tb2Item tm_item_at(const Tb2Items &its, int i) {
    Tb2Item r;
    r.chunk = i / its.tiles;
    r.tile = i % its.tiles;
    r.x0 = r.tile * TM_TX;
    r.mb = r.chunk * its.chunk_len;
    r.me = min(its.ny, r.mb + its.chunk_len);
    return r;
}

template <bool STAGED>
ES_DEV void tm_produce(const Geom &g, const Tb2Items &its, const Tb2Maps &mp, char *smem, unsigned *work) {
    using Lt = TmLayout<STAGED>;
    const TmBars<STAGED> B(smem);
    volatile int *itemq = reinterpret_cast<volatile int *>(smem + Lt::ITEMQ_OFF);
    uint32_t q = 0;
    const int total = its.tiles * its.nchunks;
    int i = work ? (int)atomicAdd(work, 1u) : (int)blockIdx.x;
    while (i < total) {
        const Tb2Item it = tm_item_at(its, i);
        int inext = -1;
        for (int t = it.mb - 2; t <= it.me + 1; ++t, ++q) {
            if (t == max(it.mb - 2, it.me - 3)) inext = work ? (int)atomicAdd(work, 1u) : i + (int)gridDim.x;
            const uint32_t s = q % TM_S;
            if (q >= (uint32_t)TM_S) mbar_wait_sleep(&B.empty[s], ((q / TM_S) - 1) & 1);
            itemq[s] = i;
            const bool drow = STAGED && t >= it.mb - 1 && t <= it.me;
            const bool prow = t >= it.mb && t < it.me;
            mbar_expect_tx(&B.full[s], (TM_TX + 8) * 8 + (drow ? (TM_TX + 4) * 8 : 0) + (prow ? TM_TX * 8 : 0));
            char *st = smem + s * Lt::STAGE;
            const int r = tb2_row(g, t);
#pragma unroll
            for (int b = 0; b < TM_TX / 256; ++b) tma_load(st + 256 * 8 * b, mp.wa, &B.full[s], it.x0 - 4 + 256 * b, r);
            tma_load(st + TM_TX * 8, mp.wb8, &B.full[s], it.x0 + TM_TX - 4, r);
            if (drow) {
                const int rd = tb2_row(g, t);
#pragma unroll
                for (int b = 0; b < TM_TX / 256; ++b)
                    tma_load(st + Lt::D_OFF + 256 * 8 * b, mp.ga, &B.full[s], it.x0 - 2 + 256 * b, rd);
                tma_load(st + Lt::D_OFF + TM_TX * 8, mp.gb4, &B.full[s], it.x0 + TM_TX - 2, rd);
            }
            if (prow) {
#pragma unroll
                for (int b = 0; b < TM_TX / 256; ++b)
                    tma_load(st + Lt::P_OFF + 256 * 8 * b, mp.p, &B.full[s], it.x0 + 256 * b, t);
            }
        }
        i = inext;
    }
    const uint32_t s = q % TM_S;  // end-of-work marker
    if (q >= (uint32_t)TM_S) mbar_wait_sleep(&B.empty[s], ((q / TM_S) - 1) & 1);
    itemq[s] = -1;
    mbar_arrive(&B.full[s]);
}

// one row step's V slot: wait until every warp has finished the previous
// step (its C part read V(t-2), which this step overwrites)
ES_DEV void tm_v_ready(uint64_t *vfull, uint32_t u, bool sleep = false) {
    if (u == 0) return;
    if (sleep)
        mbar_wait_sleep(&vfull[(u - 1) & 1], ((u - 1) >> 1) & 1);
    else
        mbar_wait(&vfull[(u - 1) & 1], ((u - 1) >> 1) & 1);
}

// The edge warp: w_k at x0 - 1 (lane 0) and x0 + TX (lane 1) of every row,
// by tb2_pair's formula (neither point is at a Neumann domain edge: x0 and
// TX are even; outside the domain the value is the Dirichlet zero ghost, and
// Neumann stencils at the domain edge never read it).
template <bool STAGED>
ES_DEV void tm_edge(const Geom &g, const SeriesParams *P, int k, const Tb2Items &its, char *smem) {
    using Lt = TmLayout<STAGED>;
    const TmBars<STAGED> B(smem);
    const volatile int *itemq = reinterpret_cast<const volatile int *>(smem + Lt::ITEMQ_OFF);
    double *vrow = reinterpret_cast<double *>(smem + Lt::V_OFF);
    const int lane = threadIdx.x & 31;
    const bool neu = g.mode == ES_MODE_NEUMANN;
    const double wx = g.wx, wy = g.wy, wz = g.wz;
    const double alpha = P->alpha, beta_k = sub(-P->shift, P->xi[k - 1]);
    auto stage = [&](uint32_t q) { return smem + (q % TM_S) * Lt::STAGE; };
    uint32_t q = 0, u = 0;
    for (;;) {
        mbar_wait_sleep(&B.full[q % TM_S], (q / TM_S) & 1);
        const int i = itemq[q % TM_S];
        if (i < 0) break;
        const Tb2Item it = tm_item_at(its, i);
        const int64_t x = lane == 0 ? (int64_t)it.x0 - 1 : (int64_t)it.x0 + TM_TX;
        const bool in = x >= 0 && x < g.nx;
        const int wo = lane == 0 ? 3 : TM_TX + 4;  // W index of x
        const int go = lane == 0 ? 1 : TM_TX + 2;  // D / V index of x
        double em = 0.0, ec = 0.0;
        if (lane < 2) em = reinterpret_cast<const double *>(stage(q))[wo];
        mbar_wait_sleep(&B.full[(q + 1) % TM_S], ((q + 1) / TM_S) & 1);
        if (lane < 2) ec = reinterpret_cast<const double *>(stage(q + 1))[wo];
        warp_arrive(&B.empty[q % TM_S]);
        ++q;  // q: stage of row t
        for (int t = it.mb - 1; t <= it.me; ++t, ++q, ++u) {
            mbar_wait_sleep(&B.full[(q + 1) % TM_S], ((q + 1) / TM_S) & 1);
            double w = 0.0, ep = 0.0;
            if (lane < 2) {
                const double *Wc = reinterpret_cast<const double *>(stage(q));
                ep = reinterpret_cast<const double *>(stage(q + 1))[wo];
                if (in && t >= 0 && t < its.ny) {
                    const double z = neu ? ec : 0.0;
                    double lap = lap7(ec, Wc[wo - 1], Wc[wo + 1], em, ep, z, z, wx, wy, wz);
                    if constexpr (STAGED) lap = mul(reinterpret_cast<const double *>(stage(q) + Lt::D_OFF)[go], lap);
                    w = add(mul(alpha, lap), mul(beta_k, ec));
                }
            }
            tm_v_ready(B.vfull, u, true);
            if (lane < 2) vrow[(u & 1) * Lt::V_SLOT + go] = w;
            warp_arrive(&B.vfull[u & 1]);
            warp_arrive(&B.empty[q % TM_S]);
            em = ec;
            ec = ep;
        }
        warp_arrive(&B.empty[q % TM_S]);  // row me + 1
        ++q;
    }
}

template <bool STAGED, bool NEU>
ES_DEV void tm_compute(const Geom &g, const SeriesParams *P, int k, bool two, const Tb2Items &its, char *smem) {
    using Lt = TmLayout<STAGED>;
    constexpr int PP = TM_PP;
    const TmBars<STAGED> B(smem);
    const volatile int *itemq = reinterpret_cast<const volatile int *>(smem + Lt::ITEMQ_OFF);
    double *vrow = reinterpret_cast<double *>(smem + Lt::V_OFF);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int e0 = 64 * PP * w + 2 * lane;  // pair h of this lane: tile offset e0 + 64 h
    const int64_t nx = g.nx;
    const double wx = g.wx, wy = g.wy, wz = g.wz;
    const int pass = P->state->pass;
    double *const w1_dst = P->wbuf[pass & 1];  // w_{k+1}, or w_k on a one-node pass
    double *const pk_dst = P->pbuf[k & 1], *const pk1_dst = P->pbuf[(k + 1) & 1];
    const bool store_pk = tb_store_pk(*P, two);
    double *const part = P->part;
    const double alpha = P->alpha, beta_k = sub(-P->shift, P->xi[k - 1]), dk = P->dd[k];
    const double dk1 = two ? P->dd[k + 1] : 0.0, beta_k1 = two ? sub(-P->shift, P->xi[k]) : 0.0;
    const double pscale = k == 1 ? P->dd[0] : 1.0;  // first pass: P rows hold v, p_0 = dd_0 v
    const int tiles = (int)((nx + 511) / 512);       // the one-node plan's 512-wide tiles
    const int CL = P->norm_chunk;                    // item starts are multiples of CL
    const int64_t slice_stride = (int64_t)tiles * TMA_CONSUMER_WARPS * 2;
    const int64_t half = (int64_t)P->nslices * P->ntiles * 2;
    uint32_t q = 0, u = 0;
    // register roles rotate over three steps (no copies): w_{k-1} rows t-1, t,
    // t+1; w_k rows t-2, t-1, t; p_k of rows t-1, t.  D of row t-1 is re-read
    // from its stage, released one step late.
    double2 W0[PP], W1[PP], W2[PP], U0[PP], U1[PP], U2[PP], K0[PP], K1[PP], K2[PP];
    for (;;) {
        mbar_wait(&B.full[q % TM_S], (q / TM_S) & 1);
        const int i = itemq[q % TM_S];
        if (i < 0) break;
        const Tb2Item it = tm_item_at(its, i);
        const int64_t xw = it.x0 + 64 * PP * w;  // this warp's first column
        const bool lo_edge = NEU && xw == 0;                                      // lane 0, pair 0: x = 0
        const bool hi_edge = NEU && nx - 1 >= xw && nx - 1 < xw + 64 * PP;       // holds x = nx - 1
        const bool partial = !NEU && xw + 64 * PP > nx;                           // Dirichlet: lanes outside
        bool in0[PP], in1[PP], xlo[PP], xhi[PP];
#pragma unroll
        for (int h = 0; h < PP; ++h) {
            const int64_t x = xw + 64 * h + 2 * lane;
            in0[h] = x < nx;
            in1[h] = x + 1 < nx;
            xlo[h] = x == 0;
            xhi[h] = x + 1 == nx - 1;
        }
        // norm partials: (row chunk, 512-wide tile, 64-column warp) entries of the one-node layout
        const int64_t ent = (int64_t)(it.x0 / 512) * TMA_CONSUMER_WARPS + (it.x0 % 512) / 64 + PP * w;
        const bool pad_half = TM_TX == 256 && it.x0 % 512 == 0 && it.x0 + 256 >= nx;
        double *part0 = part + (int64_t)(it.mb / CL) * slice_stride + ent * 2;  // node k
        double *part1 = part0 + half;                                          // node k + 1
        int rows0 = 0, rows1 = 0;  // rows accumulated since the last flush
        double acc_w0[PP], acc_p0[PP], acc_w1[PP], acc_p1[PP];
#pragma unroll
        for (int h = 0; h < PP; ++h) acc_w0[h] = acc_p0[h] = acc_w1[h] = acc_p1[h] = 0.0;
        auto flush = [&](double (&aw)[PP], double (&ap)[PP], double *&dst) {
#pragma unroll
            for (int h = 0; h < PP; ++h) {
                const double sw = warp_sum(aw[h]), sp = warp_sum(ap[h]);
                if (lane == 0) {
                    dst[2 * h] = sw;
                    dst[2 * h + 1] = sp;
                    if (pad_half) {
                        dst[2 * h + 8] = 0.0;
                        dst[2 * h + 9] = 0.0;
                    }
                }
                aw[h] = 0.0;
                ap[h] = 0.0;
            }
            dst += slice_stride;
        };
        {
            const char *s0 = smem + (q % TM_S) * Lt::STAGE + 8 * (4 + e0);
            mbar_wait(&B.full[(q + 1) % TM_S], ((q + 1) / TM_S) & 1);
            const char *s1 = smem + ((q + 1) % TM_S) * Lt::STAGE + 8 * (4 + e0);
#pragma unroll
            for (int h = 0; h < PP; ++h) {
                W0[h] = *reinterpret_cast<const double2 *>(s0 + 512 * h);
                W1[h] = *reinterpret_cast<const double2 *>(s1 + 512 * h);
                U0[h] = U1[h] = K0[h] = make_double2(0.0, 0.0);
            }
            ++q;  // q: stage of row t (row mb - 2 is released by the first step)
        }
        // global row pointers of this lane's pair 0: row t (p_k, w_k) and row t - 1 (w_{k+1}, p_{k+1})
        const int64_t off0 = (int64_t)(it.mb - 1) * nx + it.x0 + e0;
        double *pk_row = pk_dst + off0, *wk_row = w1_dst + off0;
        double *wn_row = w1_dst + off0 - nx, *pn_row = pk1_dst + off0 - nx;
        int t = it.mb - 1;
        // full (a compile-time tag): every lane of this warp holds domain columns -- no per-lane guards
        auto step = [&](auto full, double2 (&vm)[PP], double2 (&vc)[PP], double2 (&vp)[PP], double2 (&um)[PP],
                        double2 (&uc)[PP], double2 (&wk)[PP], double2 (&pk_prev)[PP], double2 (&pk)[PP]) -> bool {
            const char *st = smem + (q % TM_S) * Lt::STAGE;  // row t
            const char *sn = smem + ((q + 1) % TM_S) * Lt::STAGE + 8 * (4 + e0);  // row t + 1, this lane's pair 0
            mbar_wait(&B.full[(q + 1) % TM_S], ((q + 1) / TM_S) & 1);
#pragma unroll
            for (int h = 0; h < PP; ++h) vp[h] = *reinterpret_cast<const double2 *>(sn + 512 * h);
            // ---- w_k(t)
            if (t >= 0 && t < its.ny) {
                const double *Wc = reinterpret_cast<const double *>(st) + e0;
#pragma unroll
                for (int h = 0; h < PP; ++h) {
                    double xm = Wc[3 + 64 * h], xp = Wc[6 + 64 * h];
                    if (lo_edge || hi_edge) {  // Neumann domain edges: the point itself is the ghost
                        if (xlo[h]) xm = vc[h].x;
                        if (xhi[h]) xp = vc[h].y;
                    }
                    const double z0 = NEU ? vc[h].x : 0.0, z1 = NEU ? vc[h].y : 0.0;
                    double l0 = lap7(vc[h].x, xm, vc[h].y, vm[h].x, vp[h].x, z0, z0, wx, wy, wz);
                    double l1 = lap7(vc[h].y, vc[h].x, xp, vm[h].y, vp[h].y, z1, z1, wx, wy, wz);
                    if constexpr (STAGED) {
                        const double2 d = *reinterpret_cast<const double2 *>(st + Lt::D_OFF + 8 * (2 + e0 + 64 * h));
                        l0 = mul(d.x, l0);
                        l1 = mul(d.y, l1);
                    }
                    wk[h] = make_double2(add(mul(alpha, l0), mul(beta_k, vc[h].x)),
                                         add(mul(alpha, l1), mul(beta_k, vc[h].y)));
                    if (partial) wk[h] = make_double2(in0[h] ? wk[h].x : 0.0, in1[h] ? wk[h].y : 0.0);
                }
            } else {
#pragma unroll
                for (int h = 0; h < PP; ++h) wk[h] = NEU && t == its.ny ? uc[h] : make_double2(0.0, 0.0);  // row ny mirrors ny - 1
            }
            // ---- p_k(t) (+ node k norms)
            if (t >= it.mb && t < it.me) {
                const double *Pc = reinterpret_cast<const double *>(st + Lt::P_OFF) + e0;
#pragma unroll
                for (int h = 0; h < PP; ++h) {
                    const double2 po = *reinterpret_cast<const double2 *>(Pc + 64 * h);
                    pk[h] = make_double2(add(mul(pscale, po.x), mul(dk, wk[h].x)),
                                         add(mul(pscale, po.y), mul(dk, wk[h].y)));
                    if (decltype(full)::value || in0[h]) {
                        if (store_pk) *reinterpret_cast<double2 *>(pk_row + 64 * h) = pk[h];
                        if (!two) *reinterpret_cast<double2 *>(wk_row + 64 * h) = wk[h];  // next pass starts from w_k
                        acc_w0[h] = add(acc_w0[h], add(mul(wk[h].x, wk[h].x), mul(wk[h].y, wk[h].y)));
                        acc_p0[h] = add(acc_p0[h], add(mul(pk[h].x, pk[h].x), mul(pk[h].y, pk[h].y)));
                    }
                }
                if (++rows0 == CL || t + 1 == it.me) {
                    flush(acc_w0, acc_p0, part0);
                    rows0 = 0;
                }
            }
            // ---- w_{k+1}(t-1), p_{k+1}(t-1) (+ node k+1 norms)
            tm_v_ready(B.vfull, u);
            const int jc = t - 1;
            if (two && jc >= it.mb && jc < it.me) {
                const double *Vc = vrow + ((u - 1) & 1) * Lt::V_SLOT + e0;  // w_k(t-1), x0-2 ..
                const char *sd = smem + ((q - 1) % TM_S) * Lt::STAGE + Lt::D_OFF + 8 * (2 + e0);  // D(t-1)
#pragma unroll
                for (int h = 0; h < PP; ++h) {
                    double xm0 = Vc[1 + 64 * h], xp1 = Vc[4 + 64 * h];
                    if (lo_edge || hi_edge) {
                        if (xlo[h]) xm0 = uc[h].x;
                        if (xhi[h]) xp1 = uc[h].y;
                    }
                    const double z0 = NEU ? uc[h].x : 0.0, z1 = NEU ? uc[h].y : 0.0;
                    double l0 = lap7(uc[h].x, xm0, uc[h].y, um[h].x, wk[h].x, z0, z0, wx, wy, wz);
                    double l1 = lap7(uc[h].y, uc[h].x, xp1, um[h].y, wk[h].y, z1, z1, wx, wy, wz);
                    if constexpr (STAGED) {
                        const double2 d = *reinterpret_cast<const double2 *>(sd + 512 * h);
                        l0 = mul(d.x, l0);
                        l1 = mul(d.y, l1);
                    }
                    const double2 wn = make_double2(add(mul(alpha, l0), mul(beta_k1, uc[h].x)),
                                                    add(mul(alpha, l1), mul(beta_k1, uc[h].y)));
                    const double2 pn =
                        make_double2(add(pk_prev[h].x, mul(dk1, wn.x)), add(pk_prev[h].y, mul(dk1, wn.y)));
                    if (decltype(full)::value || in0[h]) {
                        *reinterpret_cast<double2 *>(wn_row + 64 * h) = wn;
                        *reinterpret_cast<double2 *>(pn_row + 64 * h) = pn;
                        acc_w1[h] = add(acc_w1[h], add(mul(wn.x, wn.x), mul(wn.y, wn.y)));
                        acc_p1[h] = add(acc_p1[h], add(mul(pn.x, pn.x), mul(pn.y, pn.y)));
                    }
                }
                if (++rows1 == CL || jc + 1 == it.me) {
                    flush(acc_w1, acc_p1, part1);
                    rows1 = 0;
                }
            }
            // ---- publish w_k(t) for the x-neighbours of the next step's C part
            double *Vn = vrow + (u & 1) * Lt::V_SLOT + 2 + e0;
#pragma unroll
            for (int h = 0; h < PP; ++h) *reinterpret_cast<double2 *>(Vn + 64 * h) = wk[h];
            warp_arrive(&B.vfull[u & 1]);
            warp_arrive(&B.empty[(q - 1) % TM_S]);  // row t - 1: its D was last read above
            if (NEU && t == 0) {  // row -1 mirrors row 0: the next step's w_k(t-2) role
#pragma unroll
                for (int h = 0; h < PP; ++h) uc[h] = wk[h];
            }
            ++t;
            ++q;
            ++u;
            pk_row += nx;
            wk_row += nx;
            wn_row += nx;
            pn_row += nx;
            return t <= it.me;
        };
        auto march = [&](auto full) {
            for (;;) {
                if (!step(full, W0, W1, W2, U0, U1, U2, K0, K1)) break;
                if (!step(full, W1, W2, W0, U1, U2, U0, K1, K2)) break;
                if (!step(full, W2, W0, W1, U2, U0, U1, K2, K0)) break;
            }
        };
        if (xw + 64 * PP <= nx)
            march(std::true_type{});
        else
            march(std::false_type{});
        warp_arrive(&B.empty[(q - 1) % TM_S]);  // rows me, me + 1
        warp_arrive(&B.empty[q % TM_S]);
        ++q;
    }
}

template <bool STAGED, bool NEU>
ES_DEV void tm_pass(const SeriesParams *P, int k, bool two, char *smem) {
    using Lt = TmLayout<STAGED>;
    const Geom g = P->g;
    const Tb2Items its = [&] {
        Tb2Items r;
        r.tiles = (int)((g.nx + TM_TX - 1) / TM_TX);
        r.ny = (int)g.ny;
        r.chunk_len = P->chunk_len;
        r.nchunks = (r.ny + r.chunk_len - 1) / r.chunk_len;
        return r;
    }();
    const TmaMaps &M = *static_cast<const TmaMaps *>(P->maps);
    const int pass = P->state->pass;
    const int wi = pass == 0 ? 0 : (pass & 1) ? 1 : 2;  // w_{k-1}: v, wbuf[0], wbuf[1]
    const Tb2Maps mp{&M.m[wi == 0 ? MAP_WA_V : wi == 1 ? MAP_WA_0 : MAP_WA_1],
                     &M.m[wi == 0 ? MAP_T2_W8_V : wi == 1 ? MAP_T2_W8_0 : MAP_T2_W8_1], &M.m[MAP_G], &M.m[MAP_T2_G4],
                     &M.m[k == 1 ? MAP_WA_V : ((k - 1) & 1) ? MAP_P_1 : MAP_P_0], nullptr};
    if (threadIdx.x == 0) {
        const TmBars<STAGED> B(smem);
        for (int s = 0; s < TM_S; ++s) {
            mbar_init(&B.full[s], 1);
            mbar_init(&B.empty[s], TM_NW + 1);
        }
        for (int s = 0; s < 2; ++s) mbar_init(&B.vfull[s], TM_NW + 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int warp = threadIdx.x / 32;
    if (warp == TM_NW + 1) {
        if ((threadIdx.x & 31) == 0) {
            for (const CUtensorMap *m : {mp.wa, mp.wb8, mp.p}) tma_acquire(m);
            if (STAGED)
                for (const CUtensorMap *m : {mp.ga, mp.gb4}) tma_acquire(m);
            tm_produce<STAGED>(g, its, mp, smem, P->work);
        }
    } else if (warp == TM_NW) {
        tm_edge<STAGED>(g, P, k, its, smem);
    } else {
        tm_compute<STAGED, NEU>(g, P, k, two, its, smem);
    }
}

}  // namespace es
