// Two Newton-Leja nodes per HBM pass on single-plane grids, R rows per stage.
//
// The row-by-row form (stencil_tb2d.cuh) spends ~80 % of its instructions on
// per-row bookkeeping -- ring hand-overs, waits, index updates -- for only
// 256 points per row tile (the 3D pass amortises the same work over 1024
// points per plane tile).  Here every ring stage carries R consecutive rows:
// the (8, nx/8, ny) row view (R8, nx % 8 == 0) gives a multi-row window as ONE
// TMA box (8, 34, R) in row-major [R][272] order, so a stage is one TMA per
// array and one hand-over per R rows.
//
// Same algorithm, expression trees and norm layout as stencil_tb2d.cuh:
//   W: w_{k-1} rows, window x0-8 .. x0+263 (272), stages of R rows;
//   G: D window rows (A only), same geometry;
//   P: p_{k-1} rows and the D row interiors (x0 .. x0+255) of a stage, read
//      by group C (the D of C's output rows rides here, so G is A-only);
//   V: w_k row windows x0-2 .. x0+257, stages of R rows.
// Group A (5 warps) computes the R rows of V stage s from W stages s-1..s+1
// (Neumann: ghost rows -1 / ny read the mirrored rows 0 / ny-1); group C
// (4 warps) forms p_k of the stage's rows and w_{k+1}, p_{k+1} of the rows one
// below (sR-1 .. sR+R-2) from V stages s-1, s.
#pragma once

#include "stencil_tb2d.cuh"

namespace es {

#ifndef T3_R
#define T3_R 2
#endif
#ifndef T3_SW
#define T3_SW 6
#endif
#ifndef T3_SG
#define T3_SG 5
#endif
#ifndef T3_SP
#define T3_SP 4
#endif
#ifndef T3_SV
#define T3_SV 4
#endif
static_assert(T2_TX == 256, "the R-row pass is written for 256-wide tiles");

template <bool STAGED, int R>
struct Tb3Layout {
    static constexpr int SW = T3_SW, SG = STAGED ? T3_SG : 0, SP = T3_SP, SV = T3_SV;
    static constexpr int WROW = T2_RX;  // 272
    static constexpr int W_STAGE = R * WROW * 8;
    static constexpr int G_STAGE = R * WROW * 8;
    static constexpr int P_ROW = T2_TX * 8;
    static constexpr int P_STAGE = R * P_ROW * (STAGED ? 2 : 1);  // R p rows, then R D rows
    static constexpr int V_SLOT = R * T2_EX * 8;
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

template <bool STAGED, int R>
struct Tb3Bars {
    uint64_t *wfull, *wempty, *gfull, *gempty, *pfull, *pempty, *vfull, *vempty;
    ES_DEV explicit Tb3Bars(char *smem) {
        using Lt = Tb3Layout<STAGED, R>;
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

ES_DEV int fdiv(int a, int b) { return (a >= 0 ? a : a - b + 1) / b; }  // floor division, b > 0

// Stage ranges of an item: V (and G) stages sA0..sA1 cover rows mb-1..me;
// W stages sA0-1..sA1+1; P stages sP0..sP1 cover rows mb..me-1.
struct Tb3Span {
    int sA0, sA1, sP0, sP1;
};

template <int R>
ES_DEV Tb3Span tb3_span(const Tb2Item &it) {
    Tb3Span s;
    s.sA0 = fdiv(it.mb - 1, R);
    s.sA1 = fdiv(it.me, R);
    s.sP0 = fdiv(it.mb, R);
    s.sP1 = fdiv(it.me - 1, R);
    return s;
}

template <bool STAGED, int R>
ES_DEV void tb3_produce(const Tb2Items &its, const Tb2Maps &mp, char *smem, unsigned *work) {
    using Lt = Tb3Layout<STAGED, R>;
    const Tb3Bars<STAGED, R> B(smem);
    volatile int *itemq = reinterpret_cast<volatile int *>(smem + Lt::ITEMQ_OFF);
    uint32_t uw = 0, ug = 0, up = 0;
    const int total = its.tiles * its.nchunks;
    int i = work ? (int)atomicAdd(work, 1u) : (int)blockIdx.x;
    while (i < total) {
        const Tb2Item it = tb2_item_at(its, i);
        const Tb3Span sp = tb3_span<R>(it);
        int inext = -1;
        for (int sw = sp.sA0 - 1; sw <= sp.sA1 + 1; ++sw) {
            if (sw == max(sp.sA0 - 1, sp.sA1 - 1)) inext = work ? (int)atomicAdd(work, 1u) : i + (int)gridDim.x;
            {  // W stage sw: rows sw*R .. sw*R+R-1 (out of range: TMA zero fill)
                const uint32_t s = uw % Lt::SW;
                if (uw >= (uint32_t)Lt::SW) mbar_wait(&B.wempty[s], ((uw / Lt::SW) - 1) & 1);
                itemq[s] = i;
                mbar_expect_tx(&B.wfull[s], Lt::W_STAGE);
                tma_load(smem + Lt::W_OFF + s * Lt::W_STAGE, mp.wa, &B.wfull[s], 0, (it.x0 - 8) / 8, sw * R);
                ++uw;
            }
            const int sg = sw - 1;  // G, P stage sw-1: what A / C stage sw-1 needs besides W stage sw
            if constexpr (STAGED) {
                if (sg >= sp.sA0 && sg <= sp.sA1) {
                    const uint32_t s = ug % Lt::SG;
                    if (ug >= (uint32_t)Lt::SG) mbar_wait(&B.gempty[s], ((ug / Lt::SG) - 1) & 1);
                    mbar_expect_tx(&B.gfull[s], Lt::G_STAGE);
                    tma_load(smem + Lt::G_OFF + s * Lt::G_STAGE, mp.ga, &B.gfull[s], 0, (it.x0 - 8) / 8, sg * R);
                    ++ug;
                }
            }
            if (sg >= sp.sP0 && sg <= sp.sP1) {
                const uint32_t s = up % Lt::SP;
                if (up >= (uint32_t)Lt::SP) mbar_wait(&B.pempty[s], ((up / Lt::SP) - 1) & 1);
                mbar_expect_tx(&B.pfull[s], Lt::P_STAGE);
                char *dst = smem + Lt::P_OFF + s * Lt::P_STAGE;
                tma_load(dst, mp.p, &B.pfull[s], 0, it.x0 / 8, sg * R);
                if constexpr (STAGED) tma_load(dst + R * Lt::P_ROW, mp.dp, &B.pfull[s], 0, it.x0 / 8, sg * R);
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

template <bool STAGED, int R>
ES_DEV void tb3_group_a(const Geom &g, const SeriesParams *P, int k, const Tb2Items &its, char *smem) {
    using Lt = Tb3Layout<STAGED, R>;
    const Tb3Bars<STAGED, R> B(smem);
    const volatile int *itemq = reinterpret_cast<const volatile int *>(smem + Lt::ITEMQ_OFF);
    volatile int *vitem = reinterpret_cast<volatile int *>(smem + Lt::VITEM_OFF);
    double *vwin = reinterpret_cast<double *>(smem + Lt::V_OFF);
    const int a = threadIdx.x;  // window pair a (x = x0 - 2 + 2a)
    const bool neu = g.mode == ES_MODE_NEUMANN;
    const int ny = (int)g.ny;
    const double wx = g.wx, wy = g.wy, wz = g.wz;
    const double alpha = P->alpha, beta_k = sub(-P->shift, P->xi[k - 1]);
    const bool valid = a < T2_PAIRS;
    Ring<Lt::SW> wr;
    Ring<(Lt::SG > 0 ? Lt::SG : 1)> gr;
    Ring<Lt::SV> vr;
    uint32_t vuses = 0;
    auto wst = [&](uint32_t s) { return reinterpret_cast<const double *>(smem + Lt::W_OFF + s * Lt::W_STAGE); };
    auto vslot = [&](uint32_t s) { return vwin + s * (R * T2_EX); };
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
        const Tb3Span sp = tb3_span<R>(it);
        const int64_t xe = it.x0 - 2 + 2 * a;
        const bool fast = !neu || (xe >= 1 && xe + 1 <= g.nx - 2);  // Dirichlet: every pair (masked)
        const bool in0 = xe >= 0 && xe < g.nx, in1 = xe + 1 >= 0 && xe + 1 < g.nx;
        Ring<Lt::SW> rm = wr, rc = wr;  // W stages s-1, s, s+1 (stage sA0-1 is at wr)
        rc.next();
        Ring<Lt::SW> rp = rc;
        rp.next();
        mbar_wait(&B.wfull[rc.slot], rc.phase);
        uint32_t v_prev = 0;
        for (int s = sp.sA0; s <= sp.sA1; ++s) {
            mbar_wait(&B.wfull[rp.slot], rp.phase);
            const double *W0 = wst(rm.slot), *W1 = wst(rc.slot), *W2 = wst(rp.slot);
            const double *Gs = nullptr;
            if constexpr (STAGED) {
                mbar_wait(&B.gfull[gr.slot], gr.phase);
                Gs = reinterpret_cast<const double *>(smem + Lt::G_OFF + gr.slot * Lt::G_STAGE);
            }
            take_v();
            double *Vs = vslot(vr.slot);
            if (s == sp.sA0 && a == 0) vitem[vr.slot] = i;
            // W row rr (relative to the stage start, -1 .. R) of stages s-1..s+1; Neumann ghost rows
            // -1 / ny are the mirrored rows 0 / ny-1
            auto wrow = [&](int rr) {
                int j = s * R + rr;
                if (neu) j = min(max(j, 0), ny - 1);
                const int q = j - (s - 1) * R;  // 0 .. 3R-1 across the three stages
                const double *Wq = q < R ? W0 : q < 2 * R ? W1 : W2;
                return Wq + (q % R) * Lt::WROW;
            };
            bool arrive_prev = false;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int j = s * R + r;
                double *Vj = Vs + r * T2_EX;
                if (j >= 0 && j < ny) {
                    if (valid) {
                        const double *Wm = wrow(r - 1), *Wc = wrow(r), *Wp = wrow(r + 1);
                        const double *Gj = STAGED ? Gs + r * Lt::WROW : nullptr;
                        double2 wk;
                        if (fast) {
                            wk = tb2_pair_fast<STAGED, true>(Wm, Wc, Wp, Gj, a, alpha, beta_k, neu, wx, wy, wz);
                            if (!neu) wk = make_double2(in0 ? wk.x : 0.0, in1 ? wk.y : 0.0);
                        } else {
                            wk = tb2_pair<STAGED, true>(g, Wm, Wc, Wp, Gj, it.x0, a, alpha, beta_k, neu, wx, wy, wz);
                        }
                        *reinterpret_cast<double2 *>(Vj + 2 * a) = wk;
                    }
                } else if (!neu || j > ny) {  // Dirichlet ghost rows, or rows nobody reads: zeros
                    for (int e = a; e < T2_EX; e += T2_NA) Vj[e] = 0.0;
                } else if (j == ny) {  // Neumann row ny = w_k of row ny-1
                    a2_group_sync();  // row ny-1 complete (this stage, or the previous slot still held by C)
                    const double *Vsrc = r > 0 ? Vj - T2_EX : vslot(v_prev) + (R - 1) * T2_EX;
                    for (int e = a; e < T2_EX; e += T2_NA) Vj[e] = Vsrc[e];
                }
                // (Neumann row -1 is filled from row 0 below, when stage 0 is computed)
            }
            if (neu && s == 0 && s > sp.sA0) {  // the mirrored row -1 (previous slot's last row) = w_k of row 0
                a2_group_sync();
                double *Vb = vslot(v_prev) + (R - 1) * T2_EX;
                for (int e = a; e < T2_EX; e += T2_NA) Vb[e] = Vs[e];
                arrive_prev = true;
            }
            warp_arrive(&B.wempty[rm.slot]);  // W stage s-1: last read for V stage s
            if constexpr (STAGED) {
                warp_arrive(&B.gempty[gr.slot]);
                gr.next();
            }
            if (arrive_prev) warp_arrive(&B.vfull[v_prev]);
            if (!(neu && s == -1)) warp_arrive(&B.vfull[vr.slot]);  // Neumann stage -1 arrives with stage 0
            v_prev = vr.slot;
            vr.next();
            rm = rc;
            rc = rp;
            rp.next();
        }
        warp_arrive(&B.wempty[rm.slot]);  // W stages sA1, sA1+1
        warp_arrive(&B.wempty[rc.slot]);
        wr = rp;
    }
}

template <bool STAGED, int R>
ES_DEV void tb3_group_c(const Geom &g, const SeriesParams *P, int k, bool two, const Tb2Items &its, char *smem) {
    using Lt = Tb3Layout<STAGED, R>;
    const Tb3Bars<STAGED, R> B(smem);
    const volatile int *vitem = reinterpret_cast<const volatile int *>(smem + Lt::VITEM_OFF);
    const double *vwin = reinterpret_cast<const double *>(smem + Lt::V_OFF);
    const int c = threadIdx.x - T2_NA, cw = c >> 5, lane = c & 31;  // pair x0 + 2c
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
    const int tiles = (int)((nx + 511) / 512);
    const int CL = P->norm_chunk;
    const int64_t half = (int64_t)P->nslices * P->ntiles * 2;
    Ring<Lt::SP> pr;
    Ring<Lt::SV> vr;
    auto vslot = [&](uint32_t s) { return vwin + s * (R * T2_EX); };
    auto pst = [&](uint32_t s) { return reinterpret_cast<const double *>(smem + Lt::P_OFF + s * Lt::P_STAGE); };
    for (;;) {
        mbar_wait(&B.vfull[vr.slot], vr.phase);
        const int i = vitem[vr.slot];
        if (i < 0) break;
        const Tb2Item it = tb2_item_at(its, i);
        const Tb3Span sp = tb3_span<R>(it);
        const int64_t xa = it.x0 + 2 * c;
        const bool act = xa < nx;
        const int64_t ent_base = (int64_t)(it.x0 / 512) * TMA_CONSUMER_WARPS + (it.x0 % 512) / 64 + cw;
        const bool pad_half = it.x0 % 512 == 0 && it.x0 + 256 >= nx;
        double acc_w0 = 0.0, acc_p0 = 0.0, acc_w1 = 0.0, acc_p1 = 0.0;
        double2 pk_last = make_double2(0.0, 0.0);  // p_k of row sR-1 (previous stage)
        uint32_t v_prev = 0, p_prev = 0;
        bool have_pprev = false;
        auto flush = [&](double &aw, double &ap, int row, int64_t node_half) {
            const double w = warp_sum(aw), p = warp_sum(ap);
            if (lane == 0) {
                double *d = P->part + node_half + (((int64_t)(row / CL) * tiles) * TMA_CONSUMER_WARPS + ent_base) * 2;
                d[0] = w;
                d[1] = p;
                if (pad_half) {
                    d[8] = 0.0;
                    d[9] = 0.0;
                }
            }
            aw = 0.0;
            ap = 0.0;
        };
        for (int s = sp.sA0; s <= sp.sA1; ++s) {
            if (s > sp.sA0) mbar_wait(&B.vfull[vr.slot], vr.phase);
            const double *Vs = vslot(vr.slot), *Vp = vslot(v_prev);
            const bool has_p = s >= sp.sP0 && s <= sp.sP1;
            const double *Pc = nullptr;
            if (has_p) {
                mbar_wait(&B.pfull[pr.slot], pr.phase);
                Pc = pst(pr.slot);
            }
            // V centre / row pointer of row j (stages s-1, s)
            auto vrow = [&](int j) { return j >= s * R ? Vs + (j - s * R) * T2_EX : Vp + (j - (s - 1) * R) * T2_EX; };
            // ---- p_k of the stage's rows (+ node k norms)
            double2 pk[R];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int j = s * R + r;
                pk[r] = make_double2(0.0, 0.0);
                if (j < it.mb || j >= it.me) continue;
                const double2 vk = *reinterpret_cast<const double2 *>(Vs + r * T2_EX + 2 * c + 2);
                const double2 po = *reinterpret_cast<const double2 *>(Pc + r * T2_TX + 2 * c);
                pk[r] = make_double2(add(mul(pscale, po.x), mul(dk, vk.x)), add(mul(pscale, po.y), mul(dk, vk.y)));
                if (act) {
                    const int64_t off = (int64_t)j * nx + xa;
                    if (store_pk) *reinterpret_cast<double2 *>(pk_dst + off) = pk[r];
                    if (!two) *reinterpret_cast<double2 *>(w1_dst + off) = vk;  // the next pass starts from w_k
                    acc_w0 = add(acc_w0, add(mul(vk.x, vk.x), mul(vk.y, vk.y)));
                    acc_p0 = add(acc_p0, add(mul(pk[r].x, pk[r].x), mul(pk[r].y, pk[r].y)));
                }
                if ((j + 1) % CL == 0 || j + 1 == it.me) flush(acc_w0, acc_p0, j, 0);
            }
            // ---- w_{k+1}, p_{k+1} of rows sR-1 .. sR+R-2 (+ node k+1 norms)
            if (two) {
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int jc = s * R + r - 1;
                    if (jc < it.mb || jc >= it.me) continue;
                    const double *Vc = vrow(jc);
                    const int o = 2 * c + 2;
                    const double2 cc = *reinterpret_cast<const double2 *>(Vc + o);
                    const double2 ym = *reinterpret_cast<const double2 *>(vrow(jc - 1) + o);
                    const double2 yp = *reinterpret_cast<const double2 *>(vrow(jc + 1) + o);
                    const double xm0 = Vc[o - 1], xp1 = Vc[o + 2];
                    const double z0 = neu ? cc.x : 0.0, z1 = neu ? cc.y : 0.0;
                    double l0 = lap7(cc.x, xm0, cc.y, ym.x, yp.x, z0, z0, wx, wy, wz);
                    double l1 = lap7(cc.y, cc.x, xp1, ym.y, yp.y, z1, z1, wx, wy, wz);
                    if constexpr (STAGED) {  // D of row jc: its P stage (s for r > 0, s-1 for r == 0)
                        const double *Drow = r > 0 ? Pc + R * T2_TX + (r - 1) * T2_TX
                                                   : pst(p_prev) + R * T2_TX + (R - 1) * T2_TX;
                        const double2 d = *reinterpret_cast<const double2 *>(Drow + 2 * c);
                        l0 = mul(d.x, l0);
                        l1 = mul(d.y, l1);
                    }
                    const double2 wn = make_double2(add(mul(alpha, l0), mul(beta_k1, cc.x)),
                                                    add(mul(alpha, l1), mul(beta_k1, cc.y)));
                    const double2 pprev = r > 0 ? pk[r - 1] : pk_last;
                    const double2 pn = make_double2(add(pprev.x, mul(dk1, wn.x)), add(pprev.y, mul(dk1, wn.y)));
                    if (act) {
                        const int64_t off = (int64_t)jc * nx + xa;
                        *reinterpret_cast<double2 *>(w1_dst + off) = wn;
                        *reinterpret_cast<double2 *>(pk1_dst + off) = pn;
                        acc_w1 = add(acc_w1, add(mul(wn.x, wn.x), mul(wn.y, wn.y)));
                        acc_p1 = add(acc_p1, add(mul(pn.x, pn.x), mul(pn.y, pn.y)));
                    }
                    if ((jc + 1) % CL == 0 || jc + 1 == it.me) flush(acc_w1, acc_p1, jc, half);
                }
            }
            // releases: the previous V and P stages are done
            if (s > sp.sA0) warp_arrive(&B.vempty[v_prev]);
            if (have_pprev) warp_arrive(&B.pempty[p_prev]);
            have_pprev = has_p;
            if (has_p) {
                p_prev = pr.slot;
                pr.next();
            }
            pk_last = pk[R - 1];
            v_prev = vr.slot;
            vr.next();
        }
        warp_arrive(&B.vempty[v_prev]);  // V stage sA1
        if (have_pprev) warp_arrive(&B.pempty[p_prev]);
    }
}

template <bool STAGED, int R>
ES_DEV void tb3_pass(const SeriesParams *P, int k, bool two, char *smem) {
    using Lt = Tb3Layout<STAGED, R>;
    const Geom g = P->g;
    const Tb2Items its = tb2_items_of(g, P->chunk_len);
    const TmaMaps &M = *static_cast<const TmaMaps *>(P->maps);
    const int pass = P->state->pass;
    const int wi = pass == 0 ? 0 : (pass & 1) ? 1 : 2;  // v, wbuf[0], wbuf[1]
    const int pi = k == 1 ? 0 : ((k - 1) & 1) ? 2 : 1;  // p_{k-1}: v, pbuf[0], pbuf[1]
    const Tb2Maps mp{&M.m[MAP_T3_W_V + wi], nullptr, &M.m[MAP_T3_G], nullptr, &M.m[MAP_T3_P_V + pi], &M.m[MAP_T3_D]};
    if (threadIdx.x == 0) {
        const Tb3Bars<STAGED, R> B(smem);
        for (int s = 0; s < Lt::SW; ++s) {
            mbar_init(&B.wfull[s], 1);
            mbar_init(&B.wempty[s], T2_AW);
        }
        for (int s = 0; s < Lt::SG; ++s) {
            mbar_init(&B.gfull[s], 1);
            mbar_init(&B.gempty[s], T2_AW);
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
            tma_acquire(mp.wa);
            tma_acquire(mp.p);
            if (STAGED) {
                tma_acquire(mp.ga);
                tma_acquire(mp.dp);
            }
            tb3_produce<STAGED, R>(its, mp, smem, P->work);
        }
    } else if (warp < T2_AW) {
        tb3_group_a<STAGED, R>(g, P, k, its, smem);
    } else {
        tb3_group_c<STAGED, R>(g, P, k, two, its, smem);
    }
}

}  // namespace es
