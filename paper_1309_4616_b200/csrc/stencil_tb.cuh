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
//   P: p_{k-1} tiles of planes mb .. me-1 (64x8; not on the first pass).
// Consumer iteration j (planes mb-1 .. me): A) w_k of plane j on the
// extended tile; B) p_k of plane j's interior; C) w_{k+1}, p_{k+1} of plane
// j-1's interior.
#pragma once

#include "stencil_tma.cuh"

namespace es {

constexpr int TB_WX = 72, TB_WY = 12;  // w_{k-1}: x0-4 .. x0+67, y0-2 .. y0+9
constexpr int TB_EX = 68, TB_EY = 10;  // w_k window: x0-2 .. x0+65 (even start: pair loads), y0-1 .. y0+8
constexpr int TB_PAIRS = TB_EX / 2 * TB_EY;  // 340 point pairs per window plane
constexpr int TB_GX = 68, TB_GY = 10;  // g': x0-2 .. x0+65, y0-1 .. y0+8
constexpr int TB_SV = 4;               // w_k planes held (j-2 .. j+1)

template <bool GD>
struct TbLayout {
    static constexpr int SW = GD ? 6 : 7, SG = GD ? 4 : 0, SP = 4;
    static constexpr int W_STAGE = (TB_WX * TB_WY * 8 + 127) & ~127;
    static constexpr int G_STAGE = (TB_GX * TB_GY * 8 + 127) & ~127;
    static constexpr int P_STAGE = 64 * 8 * 8;
    static constexpr int V_SLOT = TB_EX * TB_EY * 8;
    static constexpr int W_OFF = 0;
    static constexpr int G_OFF = W_OFF + SW * W_STAGE;
    static constexpr int P_OFF = G_OFF + SG * G_STAGE;
    static constexpr int V_OFF = P_OFF + SP * P_STAGE;
    static constexpr int BAR_OFF = (V_OFF + TB_SV * V_SLOT + 7) & ~7;
    static constexpr int NBAR = 2 * (SW + SG + SP);
    static constexpr int ITEMQ_OFF = BAR_OFF + NBAR * 8;
    static constexpr int BYTES = ITEMQ_OFF + ((SW * 4 + 15) & ~15);
};

struct TbMaps {
    const CUtensorMap *w, *g, *p;
};

template <bool GD>
ES_DEV void tb_produce(const Geom &g, const Items &its, const TbMaps &mp, char *smem, bool load_p,
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
        const Item it = item_at<true>(its, i);
        int inext = -1;
        for (int t = it.mb - 2; t <= it.me + 1; ++t) {
            if (t == max(it.mb - 2, it.me - 3)) inext = work ? (int)atomicAdd(work, 1u) : i + (int)gridDim.x;
            {  // W(t)
                const uint32_t s = uw % Lt::SW;
                if (uw >= (uint32_t)Lt::SW) mbar_wait(&wempty[s], ((uw / Lt::SW) - 1) & 1);
                itemq[s] = i;
                mbar_expect_tx(&wfull[s], TB_WX * TB_WY * 8);
                tma_load(smem + Lt::W_OFF + s * Lt::W_STAGE, mp.w, &wfull[s], it.x0 - 4, it.y0 - 2,
                         march_src<true>(g, t, its.L));
                ++uw;
            }
            const int tg = t - 1;  // G(t-1), P(t-1): what consumer iteration t-1 needs besides W(t)
            if constexpr (GD) {
                if (tg >= it.mb - 1 && tg <= it.me) {
                    const uint32_t s = ug % Lt::SG;
                    if (ug >= (uint32_t)Lt::SG) mbar_wait(&gempty[s], ((ug / Lt::SG) - 1) & 1);
                    mbar_expect_tx(&gfull[s], TB_GX * TB_GY * 8);
                    tma_load(smem + Lt::G_OFF + s * Lt::G_STAGE, mp.g, &gfull[s], it.x0 - 2, it.y0 - 1, tg);
                    ++ug;
                }
            }
            if (load_p && tg >= it.mb && tg < it.me) {
                const uint32_t s = up % Lt::SP;
                if (up >= (uint32_t)Lt::SP) mbar_wait(&pempty[s], ((up / Lt::SP) - 1) & 1);
                mbar_expect_tx(&pfull[s], Lt::P_STAGE);
                tma_load(smem + Lt::P_OFF + s * Lt::P_STAGE, mp.p, &pfull[s], it.x0, it.y0, tg);
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

// Consumers (warps 0..7).  Returns the per-item norm partials through P->part
// (node k at the first half, node k+1 at the second half of the array).
template <int COEFF, bool GD>
ES_DEV void tb_consume(const Geom &g, const SeriesParams *P, int k, bool two, const Items &its, char *smem,
                       bool load_p) {
    using Lt = TbLayout<GD>;
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + Lt::BAR_OFF);
    uint64_t *wfull = bar, *wempty = wfull + Lt::SW, *gfull = wempty + Lt::SW, *gempty = gfull + Lt::SG,
             *pfull = gempty + Lt::SG, *pempty = pfull + Lt::SP;
    const volatile int *itemq = reinterpret_cast<const volatile int *>(smem + Lt::ITEMQ_OFF);
    double *vwin = reinterpret_cast<double *>(smem + Lt::V_OFF);
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int q = t % 32, r = t / 32;  // interior pair (x0 + 2q, + 1) of row y0 + r
    const int64_t plane = g.nx * g.ny;
    const bool neu = g.mode == ES_MODE_NEUMANN;
    const int pass = (k - 1) / 2;
    double *w1_dst = P->wbuf[pass & 1];  // w_{k+1} (w_{k-1} comes through the W tiles)
    double *pk_dst = P->pbuf[k & 1], *pk1_dst = P->pbuf[(k + 1) & 1];
    const double alpha = P->alpha, d0 = P->dd[0], dk = P->dd[k], beta_k = sub(-P->shift, P->xi[k - 1]);
    const double dk1 = two ? P->dd[k + 1] : 0.0, beta_k1 = two ? sub(-P->shift, P->xi[k]) : 0.0;
    uint32_t uw = 0, ug = 0, up = 0;
    auto wst = [&](uint32_t u) { return reinterpret_cast<const double *>(smem + Lt::W_OFF + (u % Lt::SW) * Lt::W_STAGE); };
    auto wwait = [&](uint32_t u) { mbar_wait(&wfull[u % Lt::SW], (u / Lt::SW) & 1); };
    auto release = [&](uint64_t *b) {
        __syncwarp();
        if (lane == 0) mbar_arrive(b);
    };
    auto vslot = [&](int j) { return vwin + ((j % TB_SV + TB_SV) % TB_SV) * (TB_EX * TB_EY); };
    // this thread's window pairs (fixed for every plane and item)
    int pey[2], pex[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int pr = t + h * 32 * TMA_CONSUMER_WARPS;
        pey[h] = pr < TB_PAIRS ? pr / (TB_EX / 2) : -1;
        pex[h] = 2 * (pr % (TB_EX / 2));
    }

    for (;;) {
        wwait(uw);
        const int i = itemq[uw % Lt::SW];
        if (i < 0) break;
        const Item it = item_at<true>(its, i);
        const uint32_t u0 = uw;  // W index of plane mb-2
        wwait(u0 + 1);
        const int64_t xa = it.x0 + 2 * q, ya = it.y0 + r;  // this thread's interior pair
        const bool act = xa < g.nx && ya < g.ny;
        bool fast[2];  // this thread's window pairs that need no ghost handling
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int64_t x = it.x0 - 2 + pex[h], y = it.y0 - 1 + pey[h];
            const int64_t lo = neu ? 1 : 0, xhi = neu ? g.nx - 2 : g.nx - 1, yhi = neu ? g.ny - 2 : g.ny - 1;
            fast[h] = x >= lo && x + 1 <= xhi && y >= lo && y <= yhi;
        }
        double acc_w0 = 0.0, acc_p0 = 0.0, acc_w1 = 0.0, acc_p1 = 0.0;
        double pk_prev[2] = {0.0, 0.0};
        for (int j = it.mb - 1; j <= it.me; ++j) {
            const uint32_t uj = u0 + (uint32_t)(j - (it.mb - 2));  // W index of plane j
            wwait(uj + 1);
            const double *Wm = wst(uj - 1), *Wc = wst(uj), *Wp = wst(uj + 1);
            const double *Gj = nullptr;
            if constexpr (GD) {
                mbar_wait(&gfull[ug % Lt::SG], (ug / Lt::SG) & 1);  // G(j)
                Gj = reinterpret_cast<const double *>(smem + Lt::G_OFF + (ug % Lt::SG) * Lt::G_STAGE);
            }
            // ---- A: w_k of plane j on the extended tile
            double *Vj = vslot(j);
            const bool zin = j >= 0 && j < its.L;
            if (zin) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int ey = pey[h], ex = pex[h];
                    if (ey < 0) break;
                    const int64_t x = it.x0 - 2 + ex, y = it.y0 - 1 + ey;
                    double2 wk;
                    if (fast[h]) {  // both points inside, no ghost to patch: pair loads
                        const int o = (ey + 1) * TB_WX + ex + 2;
                        const double2 c = *reinterpret_cast<const double2 *>(Wc + o);
                        const double2 ym = *reinterpret_cast<const double2 *>(Wc + o - TB_WX);
                        const double2 yp = *reinterpret_cast<const double2 *>(Wc + o + TB_WX);
                        const double2 zm = *reinterpret_cast<const double2 *>(Wm + o);
                        const double2 zp = *reinterpret_cast<const double2 *>(Wp + o);
                        double l0 = lap7(c.x, Wc[o - 1], c.y, ym.x, yp.x, zm.x, zp.x, g.wx, g.wy, g.wz);
                        double l1 = lap7(c.y, c.x, Wc[o + 2], ym.y, yp.y, zm.y, zp.y, g.wx, g.wy, g.wz);
                        if constexpr (COEFF != ES_COEFF_NONE) {
                            l0 = mul(tb_coeff<COEFF>(g, x, y, j), l0);
                            l1 = mul(tb_coeff<COEFF>(g, x + 1, y, j), l1);
                        }
                        if constexpr (GD) {
                            const double2 gv = *reinterpret_cast<const double2 *>(Gj + ey * TB_GX + ex);
                            l0 = sub(l0, mul(gv.x, c.x));
                            l1 = sub(l1, mul(gv.y, c.y));
                        }
                        wk = make_double2(add(mul(alpha, l0), mul(beta_k, c.x)), add(mul(alpha, l1), mul(beta_k, c.y)));
                    } else {
                        wk = make_double2(
                            tb_point_scalar<COEFF, GD>(g, Wm, Wc, Wp, Gj, it.x0, it.y0, x, y, j, alpha, beta_k),
                            tb_point_scalar<COEFF, GD>(g, Wm, Wc, Wp, Gj, it.x0, it.y0, x + 1, y, j, alpha, beta_k));
                    }
                    *reinterpret_cast<double2 *>(Vj + ey * TB_EX + ex) = wk;
                }
            }
            // out-of-domain planes of the w_k window: zeros (Dirichlet), or the
            // mirrored boundary plane (Neumann; the bottom one right after plane 0)
            if (!zin && !(neu && j < 0)) {
                const double *Vs = vslot(its.L - 1);
                for (int e = t; e < TB_EX * TB_EY; e += 32 * TMA_CONSUMER_WARPS) Vj[e] = neu ? Vs[e] : 0.0;
            }
            group_sync<32 * TMA_CONSUMER_WARPS>();
            if (neu && j == 0) {
                double *Vb = vslot(-1);
                for (int e = t; e < TB_EX * TB_EY; e += 32 * TMA_CONSUMER_WARPS) Vb[e] = Vj[e];
                group_sync<32 * TMA_CONSUMER_WARPS>();
            }
            release(&wempty[(uj - 1) % Lt::SW]);  // W(j-1): its last use was A of plane j
            // ---- B: p_k of plane j's interior (+ node k norms)
            double pk_cur[2] = {0.0, 0.0};
            if (j >= it.mb && j < it.me) {
                const double *Pc = nullptr;
                if (load_p) {
                    mbar_wait(&pfull[up % Lt::SP], (up / Lt::SP) & 1);
                    Pc = reinterpret_cast<const double *>(smem + Lt::P_OFF + (up % Lt::SP) * Lt::P_STAGE);
                }
                if (act) {
                    const double *vrow = Vj + (r + 1) * TB_EX + 2 * q + 2;
                    const double *wrow = Wc + (r + 2) * TB_WX + 2 * q + 4;
#pragma unroll
                    for (int jj = 0; jj < 2; ++jj) {
                        const double wk = vrow[jj];
                        const double pold = load_p ? Pc[r * 64 + 2 * q + jj] : mul(d0, wrow[jj]);
                        pk_cur[jj] = add(pold, mul(dk, wk));
                    }
                    *reinterpret_cast<double2 *>(pk_dst + j * plane + ya * g.nx + xa) = make_double2(pk_cur[0], pk_cur[1]);
                    acc_w0 = add(acc_w0, add(mul(vrow[0], vrow[0]), mul(vrow[1], vrow[1])));
                    acc_p0 = add(acc_p0, add(mul(pk_cur[0], pk_cur[0]), mul(pk_cur[1], pk_cur[1])));
                }
                if (load_p) {
                    release(&pempty[up % Lt::SP]);
                    ++up;
                }
            }
            // ---- C: w_{k+1}, p_{k+1} of plane j-1's interior (+ node k+1 norms)
            const int jc = j - 1;
            if (two && jc >= it.mb && jc < it.me && act) {
                const double *Vm = vslot(jc - 1), *Vc = vslot(jc), *Vp = vslot(jc + 1);
                const int o = (r + 1) * TB_EX + 2 * q + 2;
                double wn[2], pn[2];
#pragma unroll
                for (int jj = 0; jj < 2; ++jj) {
                    const double c = Vc[o + jj];
                    double lap = lap7(c, Vc[o + jj - 1], Vc[o + jj + 1], Vc[o + jj - TB_EX], Vc[o + jj + TB_EX],
                                      Vm[o + jj], Vp[o + jj], g.wx, g.wy, g.wz);
                    if constexpr (COEFF != ES_COEFF_NONE) lap = mul(tb_coeff<COEFF>(g, xa + jj, ya, jc), lap);
                    if constexpr (GD) {
                        const double *Gc = reinterpret_cast<const double *>(
                            smem + Lt::G_OFF + ((ug - 1) % Lt::SG) * Lt::G_STAGE);  // G(j-1)
                        lap = sub(lap, mul(Gc[(r + 1) * TB_GX + 2 * q + jj + 2], c));
                    }
                    wn[jj] = add(mul(alpha, lap), mul(beta_k1, c));
                    pn[jj] = add(pk_prev[jj], mul(dk1, wn[jj]));
                }
                const int64_t off = jc * plane + ya * g.nx + xa;
                *reinterpret_cast<double2 *>(w1_dst + off) = make_double2(wn[0], wn[1]);
                *reinterpret_cast<double2 *>(pk1_dst + off) = make_double2(pn[0], pn[1]);
                acc_w1 = add(acc_w1, add(mul(wn[0], wn[0]), mul(wn[1], wn[1])));
                acc_p1 = add(acc_p1, add(mul(pn[0], pn[0]), mul(pn[1], pn[1])));
            }
            if constexpr (GD) {
                if (jc >= it.mb - 1) release(&gempty[(ug - 1) % Lt::SG]);  // G(j-1)
                ++ug;
            }
            pk_prev[0] = pk_cur[0];
            pk_prev[1] = pk_cur[1];
        }
        const uint32_t L4 = (uint32_t)(it.me - it.mb + 4);
        release(&wempty[(u0 + L4 - 2) % Lt::SW]);  // W(me), W(me+1)
        release(&wempty[(u0 + L4 - 1) % Lt::SW]);
        uw = u0 + L4;
        if constexpr (GD) release(&gempty[(ug - 1) % Lt::SG]);  // G(me)
        // (chunk, tile, warp) partials of both nodes, one-node kernel layout
        acc_w0 = warp_sum(acc_w0);
        acc_p0 = warp_sum(acc_p0);
        acc_w1 = warp_sum(acc_w1);
        acc_p1 = warp_sum(acc_p1);
        if (lane == 0) {
            const int64_t e = ((int64_t)it.chunk * its.ntiles + it.tile) * TMA_CONSUMER_WARPS + warp;
            double *d0p = P->part + e * 2;
            d0p[0] = acc_w0;
            d0p[1] = acc_p0;
            double *d1p = P->part + ((int64_t)P->nslices * P->ntiles + e) * 2;
            d1p[0] = acc_w1;
            d1p[1] = acc_p1;
        }
    }
}

template <int COEFF, bool GD>
ES_DEV void tb_pass(const SeriesParams *P, int k, bool two, char *smem) {
    using Lt = TbLayout<GD>;
    const Geom &g = P->g;
    const Items its = items_of<true>(g, P->chunk_len);
    const TmaMaps &M = *static_cast<const TmaMaps *>(P->maps);
    const int pass = (k - 1) / 2;
    const TbMaps mp{&M.m[pass == 0 ? MAP_T_V : (pass & 1) ? MAP_T_0 : MAP_T_1], &M.m[MAP_T_G], &M.m[MAP_P_0]};
    const bool load_p = k > 1;
    if (threadIdx.x == 0) {
        uint64_t *bars = reinterpret_cast<uint64_t *>(smem + Lt::BAR_OFF);
        for (int s = 0; s < Lt::SW; ++s) {
            mbar_init(&bars[s], 1);
            mbar_init(&bars[Lt::SW + s], TMA_CONSUMER_WARPS);
        }
        for (int s = 0; s < Lt::SG; ++s) {
            mbar_init(&bars[2 * Lt::SW + s], 1);
            mbar_init(&bars[2 * Lt::SW + Lt::SG + s], TMA_CONSUMER_WARPS);
        }
        for (int s = 0; s < Lt::SP; ++s) {
            mbar_init(&bars[2 * (Lt::SW + Lt::SG) + s], 1);
            mbar_init(&bars[2 * (Lt::SW + Lt::SG) + Lt::SP + s], TMA_CONSUMER_WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x / 32 == TMA_CONSUMER_WARPS) {
        if ((threadIdx.x & 31) == 0) {
            tma_acquire(mp.w);
            if (GD) tma_acquire(mp.g);
            if (load_p) tma_acquire(mp.p);
            tb_produce<GD>(g, its, mp, smem, load_p, P->work);
        }
    } else {
        tb_consume<COEFF, GD>(g, P, k, two, its, smem, load_p);
    }
}

}  // namespace es
