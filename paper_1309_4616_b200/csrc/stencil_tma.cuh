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

#include "stencil.cuh"

namespace es {

template <bool DIM3>
struct TShape;
template <>
struct TShape<true> {
    static constexpr int TX = 64, TY = 8, WR = TY + 2, WROW = TX + 4, PR = TY;
    static constexpr int S = 5;  // ring stages
};
template <>
struct TShape<false> {
    static constexpr int TX = 512, TY = 1, WR = 1, WROW = TX + 4, PR = 1;
    static constexpr int S = 6;
};

constexpr int TMA_CONSUMER_WARPS = 8;
constexpr int TMA_THREADS = 32 * (TMA_CONSUMER_WARPS + 1);

// tensor maps of one pass; for 2D, W needs two maps (256-wide and 4-wide
// boxes: TMA boxes are at most 256 elements per dimension)
enum { MAP_WA_V = 0, MAP_WB_V, MAP_WA_0, MAP_WB_0, MAP_WA_1, MAP_WB_1, MAP_P_0, MAP_P_1, MAP_G, MAP_COUNT };

struct alignas(64) TmaMaps {
    CUtensorMap m[MAP_COUNT];
};

template <bool DIM3>
struct TLayout {
    using T = TShape<DIM3>;
    static constexpr int W_BYTES = T::WR * T::WROW * 8;
    static constexpr int P_BYTES = T::PR * T::TX * 8;
    static constexpr int W_OFF = 0;
    static constexpr int P_OFF = (W_BYTES + 127) & ~127;
    static constexpr int G_OFF = P_OFF + P_BYTES;
    static constexpr int STAGE = G_OFF + P_BYTES;  // 128-byte multiple
    static constexpr int RING = STAGE * T::S;
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
ES_DEV void mbar_wait(uint64_t *bar, uint32_t parity) {
    const uint32_t a = su32(bar);
    uint32_t ok = 0;
    do {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(ok)
            : "r"(a), "r"(parity)
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
};

// The CTA's march range [mb, me) over its chunk and its tile origin.
template <bool DIM3>
struct TileIdx {
    int x0, y0, mb, me, L;
};

template <bool DIM3>
ES_DEV TileIdx<DIM3> tile_of(const Geom &g, int chunk_len) {
    using T = TShape<DIM3>;
    TileIdx<DIM3> ti;
    ti.x0 = blockIdx.x * T::TX;
    ti.y0 = DIM3 ? blockIdx.y * T::TY : 0;
    ti.L = DIM3 ? (int)g.lz : (int)g.ny;
    const int chunk = DIM3 ? blockIdx.z : blockIdx.y;
    ti.mb = chunk * chunk_len;
    ti.me = min(ti.L, ti.mb + chunk_len);
    return ti;
}

// Producer (one elected lane of warp 8): stream W for indices mb-1 .. me and
// P/G for mb .. me-1 through the ring.
template <bool DIM3, bool HAS_P, bool HAS_G>
ES_DEV void tma_produce(const Geom &g, const TileIdx<DIM3> &ti, const PassMaps &mp, char *ring, uint64_t *full,
                        uint64_t *empty, bool p_present) {
    using T = TShape<DIM3>;
    using Lt = TLayout<DIM3>;
    const int jb = ti.mb - 1;
    for (int j = jb; j <= ti.me; ++j) {
        const int u = j - jb;
        const int s = u % T::S;
        if (u >= T::S) mbar_wait(&empty[s], ((u / T::S) - 1) & 1);
        char *st = ring + s * Lt::STAGE;
        const bool inner = j >= ti.mb && j < ti.me;
        const bool lp = HAS_P && inner && p_present;
        const bool lg = HAS_G && inner;
        mbar_expect_tx(&full[s], Lt::W_BYTES + (lp ? Lt::P_BYTES : 0) + (lg ? Lt::P_BYTES : 0));
        const int js = march_src<DIM3>(g, j, ti.L);
        if constexpr (DIM3) {
            tma_load(st + Lt::W_OFF, mp.wa, &full[s], ti.x0 - 2, ti.y0 - 1, js);
            if (lp) tma_load(st + Lt::P_OFF, mp.p, &full[s], ti.x0, ti.y0, j);
            if (lg) tma_load(st + Lt::G_OFF, mp.g, &full[s], ti.x0, ti.y0, j);
        } else {
            tma_load(st + Lt::W_OFF, mp.wa, &full[s], ti.x0 - 2, js);
            tma_load(st + Lt::W_OFF + 2048, mp.wa, &full[s], ti.x0 + 254, js);
            tma_load(st + Lt::W_OFF + 4096, mp.wb, &full[s], ti.x0 + 510, js);
            if (lp) {
                tma_load(st + Lt::P_OFF, mp.p, &full[s], ti.x0, j);
                tma_load(st + Lt::P_OFF + 2048, mp.p, &full[s], ti.x0 + 256, j);
            }
            if (lg) {
                tma_load(st + Lt::G_OFF, mp.g, &full[s], ti.x0, j);
                tma_load(st + Lt::G_OFF + 2048, mp.g, &full[s], ti.x0 + 256, j);
            }
        }
    }
}

// Consumers (warps 0..7): one point pair per thread per stage.
template <bool DIM3, int COEFF, bool GD, bool LEJA>
ES_DEV void tma_consume(const Geom &g, const Pass &ps, const TileIdx<DIM3> &ti, const char *ring, uint64_t *full,
                        uint64_t *empty, double *s_red) {
    using T = TShape<DIM3>;
    using Lt = TLayout<DIM3>;
    const int t = threadIdx.x;
    const int lane = t & 31, warp = t >> 5;
    const int q = t % (T::TX / 2), r = t / (T::TX / 2);
    const int64_t ix = ti.x0 + 2 * q;
    const int64_t iy = DIM3 ? (int64_t)ti.y0 + r : 0;
    const bool act = ix < g.nx && iy < g.ny;
    const int64_t plane = g.nx * g.ny;
    const int wrow = DIM3 ? r + 1 : 0;      // W row of this thread's points
    const int wcol = wrow * T::WROW + 2 + 2 * q;
    const int pidx = r * T::TX + 2 * q;
    const int jb = ti.mb - 1;

    double dco[2] = {1.0, 1.0};
    double ox2[2] = {1.0, 1.0};
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

    auto stage = [&](int j) { return ring + ((j - jb) % T::S) * Lt::STAGE; };
    auto wait_full = [&](int j) { mbar_wait(&full[(j - jb) % T::S], ((j - jb) / T::S) & 1); };

    wait_full(jb);
    wait_full(ti.mb);
    for (int m = ti.mb; m < ti.me; ++m) {
        wait_full(m + 1);
        const double *Wm = reinterpret_cast<const double *>(stage(m - 1) + Lt::W_OFF);
        const double *Wc = reinterpret_cast<const double *>(stage(m) + Lt::W_OFF);
        const double *Wp = reinterpret_cast<const double *>(stage(m + 1) + Lt::W_OFF);
        double sw = 0.0, sp = 0.0;
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
                    if (iy == 0) ym = neu ? c : *reinterpret_cast<const double2 *>(ps.src + m * plane + (g.ny - 1) * g.nx + ix);
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
            const double *Pc = reinterpret_cast<const double *>(stage(m) + Lt::P_OFF);
            const double *Gc = reinterpret_cast<const double *>(stage(m) + Lt::G_OFF);
            double yy = 0.0;
            if constexpr (COEFF == ES_COEFF_RADIAL && !DIM3) yy = axis_coord(m, g.ny);
            double wn[2], pn[2];
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                double lap = lap7(cc[j], xm[j], xp[j], ymv[j], ypv[j], zmv[j], zpv[j], g.wx, g.wy, g.wz);
                const int64_t idx = row_base + ix + j;
                if constexpr (COEFF == ES_COEFF_RADIAL) lap = mul(DIM3 ? dco[j] : radial_from_sq(ox2[j], yy), lap);
                if constexpr (COEFF == ES_COEFF_ARRAY) lap = mul(__ldg(g.coeff + idx), lap);
                if constexpr (GD) lap = sub(lap, mul(Gc[pidx + j], cc[j]));
                wn[j] = add(mul(ps.alpha, lap), mul(ps.beta, cc[j]));
                if constexpr (LEJA) {
                    const double pold = ps.p_src ? Pc[pidx + j] : mul(ps.d0, cc[j]);
                    pn[j] = add(pold, mul(ps.dk, wn[j]));
                }
            }
            const int64_t o = row_base + ix;
            *reinterpret_cast<double2 *>(ps.dst + o) = make_double2(wn[0], wn[1]);
            if constexpr (LEJA) {
                *reinterpret_cast<double2 *>(ps.p_dst + o) = make_double2(pn[0], pn[1]);
                sw = add(mul(wn[0], wn[0]), mul(wn[1], wn[1]));
                sp = add(mul(pn[0], pn[0]), mul(pn[1], pn[1]));
            }
        }
        if constexpr (LEJA) {
            sw = warp_sum(sw);
            sp = warp_sum(sp);
            if (lane == 0) {
                s_red[((m - ti.mb) * TMA_CONSUMER_WARPS + warp) * 2 + 0] = sw;
                s_red[((m - ti.mb) * TMA_CONSUMER_WARPS + warp) * 2 + 1] = sp;
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[(m - 1 - jb) % T::S]);
    }
}

// Shared-memory footprint of one CTA: ring + barriers + per-index warp partials.
template <bool DIM3>
constexpr size_t tma_smem_bytes(int chunk_len) {
    return (size_t)TLayout<DIM3>::RING + 2 * TShape<DIM3>::S * sizeof(uint64_t) +
           (size_t)chunk_len * TMA_CONSUMER_WARPS * 2 * sizeof(double);
}

// Whole pass for one CTA: barrier set-up, warp-specialised streaming.
template <bool DIM3, int COEFF, bool GD, bool LEJA>
ES_DEV void tma_pass(const Geom &g, const Pass &ps, const PassMaps &mp, int chunk_len, bool acquire_maps,
                     char *smem) {
    using T = TShape<DIM3>;
    char *ring = smem;
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + TLayout<DIM3>::RING);
    uint64_t *empty = full + T::S;
    double *s_red = reinterpret_cast<double *>(empty + T::S);
    const TileIdx<DIM3> ti = tile_of<DIM3>(g, chunk_len);
    if (threadIdx.x == 0) {
        for (int s = 0; s < T::S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], TMA_CONSUMER_WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5;
    if (warp == TMA_CONSUMER_WARPS) {
        if ((threadIdx.x & 31) == 0) {
            if (acquire_maps) {
                tma_acquire(mp.wa);
                if (!DIM3) tma_acquire(mp.wb);
                if (LEJA && ps.p_src) tma_acquire(mp.p);
                if (GD) tma_acquire(mp.g);
            }
            tma_produce<DIM3, LEJA, GD>(g, ti, mp, ring, full, empty, ps.p_src != nullptr);
        }
    } else {
        tma_consume<DIM3, COEFF, GD, LEJA>(g, ps, ti, ring, full, empty, s_red);
    }
}

}  // namespace es
