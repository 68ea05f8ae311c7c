// Fused 7-point (3D) / 5-point (2D) stencil passes with the Newton-Leja
// recurrence and the stopping-test norms folded in.
//
// One pass computes, for every point of the slab,
//     w_k = alpha (D A w_{k-1} [- g' w_{k-1}]) + beta_k w_{k-1}
//     p_k = p_{k-1} + dd_k w_k              (p_0 = dd_0 v folded into node 1)
// and the per-(slice, tile) partial sums of w_k^2 and p_k^2, reading w_{k-1}
// and p_{k-1} once and writing w_k and p_k once: 32 B/point (40 with g').
//
// 3D layout: a CTA owns a (32*VEC) x BY3 tile of (x, y) columns and marches a
// chunk of z planes; each thread keeps its column's z-neighbours in a
// register queue (zm, c, zp, zq: two planes of prefetch) and the plane's
// (x, y) neighbours come from a double-buffered shared-memory tile with a
// one-point halo.  2D layout (nz == 1): warps own independent x strips and
// march y with the same register queue; x neighbours are warp shuffles.
#pragma once

#include "es_common.cuh"

namespace es {

constexpr int BY3 = 8;  // warps (= tile rows) per 3D CTA
constexpr int BW2 = 8;  // warps (= x strips) per 2D CTA

struct Geom {
    int64_t nx, ny, lz, z0, nz_total;
    double wx, wy, wz;
    int mode, coeff_kind;
    const double *coeff;
    const double *faces[6];
    const double *halo_lo, *halo_hi;
    int at_lo, at_hi;
};

// Device-resident parameters of one series (constant over its nodes, so a
// CUDA graph can replay the node kernel without re-binding arguments).
struct SeriesParams {
    Geom g;
    const double *v;
    double *wbuf[2];
    double *pbuf[2];  // pbuf[1] == p_out
    const double *gdiag;
    const double *dd, *xi;
    int ndd;
    double alpha, shift, tol;
    SeriesState *state;
    double *part;   // [nslices][ntiles][2] per-(slice, tile) sums of w^2, p^2
    double *slice;  // [nslices][2]
    unsigned *chunk_cnt;
    unsigned *global_cnt;
    int nslices, ntiles, nchunks, chunk_len;
    unsigned long long cond;  // cudaGraphConditionalHandle, 0 = plain launches
    // CSR operator (es_leja_csr); unused by the stencil nodes
    const int64_t *row_ptr;
    const int32_t *col;
    const double *vals;
    unsigned long long tex[4];  // CSR texture gathers: wbuf[0], wbuf[1], v, xg
    const double *ddabs;        // complex series: |dd_k| (else nullptr)
    double alpha_im;            // complex series: imaginary part of alpha
    int vals_complex;           // complex CSR: interleaved complex vals
    const double *xg;  // multi-GPU CSR: the all-gathered w_{k-1} the row gathers read (nullptr: the local source)
    int64_t n;
    const void *maps;  // TmaMaps (workspace) for the TMA node kernel
    unsigned *work;    // dynamic work-item counter of the TMA node kernel
    int dist;          // 1: slab of a multi-GPU series (slices gathered by the caller, k_decide_gathered decides)
    // peer-memory (NVLink P2P) slab series, es_leja_p2p; p2p == 0 otherwise
    int p2p;
    int nranks, rank;
    int64_t slice_off, total_slices;
    double *peer_lo[2], *peer_hi[2];    // lower neighbour's halo_hi / upper neighbour's halo_lo, by parity
    double *const *rank_slices;         // [nranks] -> every rank's slice table [2][total_slices][2]
    unsigned long long *const *rank_arrive;  // [nranks] -> every rank's arrival counter
    unsigned long long *arrive_local;
    unsigned long long base;            // arrival counter before this series
    long long timeout_ns;
    // peer-memory row-block CSR series (es_leja_csr_p2p)
    double *xgp[2];                     // this rank's gathered vector by parity (node k gathers from xgp[k & 1])
    double *const *rank_xg;             // [nranks] -> every rank's gathered-vector buffer (parity 1 at + npad)
    int64_t row_off, npad;
    // two-node series: after a pass whose second node met the term test once
    // (consecutive == 1), run the next node alone (a one-node tb pass) -- the
    // series usually stops there, and a two-node pass would compute a node
    // nobody reads.  Decisions are unchanged (bitwise).
    int tail1;
    // two-node 2D pass (stencil_tb2d.cuh): rows per slice of the one-node 2D
    // plan, whose (chunk, 512-wide tile, warp) norm layout the pass keeps
    int norm_chunk;
    // peer-memory two-node slab series: the pass pushes its boundary planes to
    // the neighbours itself (k_slice_p2p2 only fences and joins the round)
    int peer_in_node;
};

// One pass: what a node (or a plain fused apply) reads and writes.
struct Pass {
    const double *src;
    double *dst;
    const double *p_src;  // nullptr on node 1: p_{0} = d0 * v
    double *p_dst;        // nullptr for a plain apply
    double alpha, beta, dk, d0;
    unsigned long long *aux = nullptr;  // Rosenbrock prologue: {min g', max g', first u <= 0}
};

template <int VEC>
struct Vv {
    double v[VEC];
};

template <int VEC>
ES_DEV Vv<VEC> ldv(const double *p) {
    Vv<VEC> r;
    if constexpr (VEC == 2) {
        const double2 t = __ldg(reinterpret_cast<const double2 *>(p));
        r.v[0] = t.x;
        r.v[1] = t.y;
    } else {
        r.v[0] = __ldg(p);
    }
    return r;
}

template <int VEC>
ES_DEV void stv(double *p, const Vv<VEC> &x) {
    if constexpr (VEC == 2) {
        *reinterpret_cast<double2 *>(p) = make_double2(x.v[0], x.v[1]);
    } else {
        *p = x.v[0];
    }
}

template <int VEC>
ES_DEV Vv<VEC> zeros() {
    Vv<VEC> r;
#pragma unroll
    for (int j = 0; j < VEC; ++j) r.v[j] = 0.0;
    return r;
}

// Field value at (x, y, z) of the slab, or its ghost when exactly one
// coordinate lies one step outside (precedence of _core.pyx:61-114: halo,
// periodic wrap, face value, Neumann mirror, zero).  Anything further out is
// a don't-care for padding lanes and returns 0.
ES_DEV double fetch1(const Geom &g, const double *src, int64_t x, int64_t y, int64_t z) {
    const bool xin = x >= 0 && x < g.nx, yin = y >= 0 && y < g.ny, zin = z >= 0 && z < g.lz;
    const int64_t plane = g.nx * g.ny;
    if (xin && yin && zin) return __ldg(src + z * plane + y * g.nx + x);
    if (!xin && yin && zin) {
        if (x != -1 && x != g.nx) return 0.0;
        if (g.mode == ES_MODE_PERIODIC) return __ldg(src + z * plane + y * g.nx + (x < 0 ? g.nx - 1 : 0));
        if (g.mode == ES_MODE_FACES) return __ldg(g.faces[x < 0 ? 0 : 1] + (g.z0 + z) * g.ny + y);
        if (g.mode == ES_MODE_NEUMANN) return __ldg(src + z * plane + y * g.nx + (x < 0 ? 0 : g.nx - 1));
        return 0.0;
    }
    if (xin && !yin && zin) {
        if (y != -1 && y != g.ny) return 0.0;
        if (g.mode == ES_MODE_PERIODIC) return __ldg(src + z * plane + (y < 0 ? g.ny - 1 : 0) * g.nx + x);
        if (g.mode == ES_MODE_FACES) return __ldg(g.faces[y < 0 ? 2 : 3] + (g.z0 + z) * g.nx + x);
        if (g.mode == ES_MODE_NEUMANN) return __ldg(src + z * plane + (y < 0 ? 0 : g.ny - 1) * g.nx + x);
        return 0.0;
    }
    if (xin && yin && !zin) {
        const int64_t off = y * g.nx + x;
        if (z == -1) {
            if (g.halo_lo) return __ldg(g.halo_lo + off);
            if (g.mode == ES_MODE_PERIODIC) return __ldg(src + (g.lz - 1) * plane + off);
            if (g.at_lo && g.mode == ES_MODE_FACES) return __ldg(g.faces[4] + off);
            if (g.at_lo && g.mode == ES_MODE_NEUMANN) return __ldg(src + off);
            return 0.0;
        }
        if (z == g.lz) {
            if (g.halo_hi) return __ldg(g.halo_hi + off);
            if (g.mode == ES_MODE_PERIODIC) return __ldg(src + off);
            if (g.at_hi && g.mode == ES_MODE_FACES) return __ldg(g.faces[5] + off);
            if (g.at_hi && g.mode == ES_MODE_NEUMANN) return __ldg(src + (g.lz - 1) * plane + off);
        }
        return 0.0;
    }
    return 0.0;
}

// VEC consecutive x points starting at x (x % VEC == 0; with VEC == 2 the
// grid's nx is even, so a pair is entirely inside or entirely outside).
template <int VEC>
ES_DEV Vv<VEC> fetchv(const Geom &g, const double *src, int64_t x, int64_t y, int64_t z) {
    if (x >= 0 && x < g.nx && y >= 0 && y < g.ny && z >= 0 && z < g.lz)
        return ldv<VEC>(src + (z * g.ny + y) * g.nx + x);
    if (x >= 0 && x < g.nx && y >= 0 && y < g.ny) {  // z ghost: vectorisable sources
        const int64_t off = y * g.nx + x;
        const int64_t plane = g.nx * g.ny;
        if (z == -1) {
            if (g.halo_lo) return ldv<VEC>(g.halo_lo + off);
            if (g.mode == ES_MODE_PERIODIC) return ldv<VEC>(src + (g.lz - 1) * plane + off);
            if (g.at_lo && g.mode == ES_MODE_FACES) return ldv<VEC>(g.faces[4] + off);
            if (g.at_lo && g.mode == ES_MODE_NEUMANN) return ldv<VEC>(src + off);
        } else if (z == g.lz) {
            if (g.halo_hi) return ldv<VEC>(g.halo_hi + off);
            if (g.mode == ES_MODE_PERIODIC) return ldv<VEC>(src + off);
            if (g.at_hi && g.mode == ES_MODE_FACES) return ldv<VEC>(g.faces[5] + off);
            if (g.at_hi && g.mode == ES_MODE_NEUMANN) return ldv<VEC>(src + (g.lz - 1) * plane + off);
        }
        return zeros<VEC>();
    }
    Vv<VEC> r;
#pragma unroll
    for (int j = 0; j < VEC; ++j) r.v[j] = fetch1(g, src, x + j, y, z);
    return r;
}

ES_DEV double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = add(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Per-point epilogue shared by both layouts: coefficient, Rosenbrock
// diagonal, fused alpha/beta product, Leja recurrence, norm contributions.
template <int COEFF, bool GD, bool LEJA>
ES_DEV void point_out(const Geom &g, const Pass &ps, const double *gdiag, int64_t idx, double lap,
                      double dco, double c, double pold, double &wn, double &pn) {
    if constexpr (COEFF == ES_COEFF_RADIAL) lap = mul(dco, lap);
    if constexpr (COEFF == ES_COEFF_ARRAY) lap = mul(__ldg(g.coeff + idx), lap);
    if constexpr (GD) lap = sub(lap, mul(__ldg(gdiag + idx), c));
    wn = add(mul(ps.alpha, lap), mul(ps.beta, c));
    if constexpr (LEJA) pn = add(pold, mul(ps.dk, wn));
}

// ---------------------------------------------------------------------------
// 3D: (32*VEC) x BY3 column tile, z-march.  Shared memory per CTA:
//   tile[2][BY3 + 2][ROW], ROW = 32*VEC + 4; data columns start at 2 so the
//   vector stores stay 16-byte aligned; col 1 / col 32*VEC+2 are the x halo.
//   red[chunk_len][BY3][2] per-plane warp partials.
template <int VEC>
struct Smem3 {
    static constexpr int TX = 32 * VEC;
    static constexpr int ROW = TX + 4;
    static constexpr int TILE = (BY3 + 2) * ROW;
};

template <int VEC, int COEFF, bool GD, bool LEJA>
ES_DEV void pass3d(const Geom &g, const Pass &ps, const double *gdiag, int chunk_len,
                   double *s_tile, double *s_red) {
    using S = Smem3<VEC>;
    const int lane = threadIdx.x, wy = threadIdx.y;
    const int64_t x0 = (int64_t)blockIdx.x * S::TX, y0 = (int64_t)blockIdx.y * BY3;
    const int64_t ix = x0 + lane * VEC, iy = y0 + wy;
    const bool act = ix < g.nx && iy < g.ny;
    const int64_t zb = (int64_t)blockIdx.z * chunk_len;
    const int64_t ze = min(g.lz, zb + chunk_len);
    const int64_t plane = g.nx * g.ny;
    const int64_t off = iy * g.nx + ix;
    const double *src = ps.src;

    double dco[VEC];
#pragma unroll
    for (int j = 0; j < VEC; ++j) dco[j] = 1.0;
    if constexpr (COEFF == ES_COEFF_RADIAL) {
        if (act) {
            const double y = axis_coord(iy, g.ny);
#pragma unroll
            for (int j = 0; j < VEC; ++j) {
                const double x = axis_coord(ix + j, g.nx);
                dco[j] = radial_from_sq(add(1.0, mul(x, x)), y);
            }
        }
    }

    // writes plane z's centre values (own column or ghost/padding) and the
    // halo values already fetched into registers into shared buffer b
    const int col = 2 + lane * VEC;
    auto put_plane = [&](int b, const Vv<VEC> &ctr, const Vv<VEC> &hrow, double hcol) {
        double *t = s_tile + b * S::TILE;
        stv<VEC>(t + (wy + 1) * S::ROW + col, ctr);
        if (wy == 0) stv<VEC>(t + 0 * S::ROW + col, hrow);
        if (wy == BY3 - 1) stv<VEC>(t + (BY3 + 1) * S::ROW + col, hrow);
        if (lane == 0) t[(wy + 1) * S::ROW + 1] = hcol;
        if (lane == 31) t[(wy + 1) * S::ROW + S::TX + 2] = hcol;
    };
    auto fetch_halo = [&](int64_t z, Vv<VEC> &hrow, double &hcol) {
        if (wy == 0) hrow = fetchv<VEC>(g, src, ix, y0 - 1, z);
        if (wy == BY3 - 1) hrow = fetchv<VEC>(g, src, ix, y0 + BY3, z);
        if (lane == 0) hcol = fetch1(g, src, x0 - 1, iy, z);
        if (lane == 31) hcol = fetch1(g, src, x0 + S::TX, iy, z);
    };

    Vv<VEC> zm = zeros<VEC>(), c, zp = zeros<VEC>(), zq = zeros<VEC>();
    Vv<VEC> pc = zeros<VEC>(), pn = zeros<VEC>();
    Vv<VEC> hrow = zeros<VEC>();
    double hcol = 0.0;
    c = fetchv<VEC>(g, src, ix, iy, zb);  // ghost-or-padding for inactive lanes
    if (act) {
        zm = fetchv<VEC>(g, src, ix, iy, zb - 1);
        zp = fetchv<VEC>(g, src, ix, iy, zb + 1);
        if constexpr (LEJA) {
            if (ps.p_src) pc = ldv<VEC>(ps.p_src + zb * plane + off);
        }
    }
    fetch_halo(zb, hrow, hcol);
    put_plane(0, c, hrow, hcol);

    int buf = 0;
    for (int64_t z = zb; z < ze; ++z) {
        const bool more = z + 1 < ze;
        Vv<VEC> cnext = zp;
        if (more) {
            if (act) {
                zq = fetchv<VEC>(g, src, ix, iy, z + 2);
                if constexpr (LEJA) {
                    if (ps.p_src) pn = ldv<VEC>(ps.p_src + (z + 1) * plane + off);
                }
            } else {
                cnext = fetchv<VEC>(g, src, ix, iy, z + 1);
            }
            fetch_halo(z + 1, hrow, hcol);
        }
        __syncthreads();
        double sw = 0.0, sp = 0.0;
        if (act) {
            const double *t = s_tile + buf * S::TILE;
            const double *r0 = t + wy * S::ROW + col;        // y - 1
            const double *r1 = t + (wy + 1) * S::ROW + col;  // y
            const double *r2 = t + (wy + 2) * S::ROW + col;  // y + 1
            Vv<VEC> wn, pnew;
#pragma unroll
            for (int j = 0; j < VEC; ++j) {
                const double cc = c.v[j];
                const double xm = r1[j - 1], xp = r1[j + 1];
                const double lap = lap7(cc, xm, xp, r0[j], r2[j], zm.v[j], zp.v[j], g.wx, g.wy, g.wz);
                const int64_t idx = z * plane + off + j;
                double pold = 0.0;
                if constexpr (LEJA) pold = ps.p_src ? pc.v[j] : mul(ps.d0, cc);
                point_out<COEFF, GD, LEJA>(g, ps, gdiag, idx, lap, dco[j], cc, pold, wn.v[j], pnew.v[j]);
            }
            stv<VEC>(ps.dst + z * plane + off, wn);
            if constexpr (LEJA) {
                stv<VEC>(ps.p_dst + z * plane + off, pnew);
                sw = mul(wn.v[0], wn.v[0]);
                sp = mul(pnew.v[0], pnew.v[0]);
#pragma unroll
                for (int j = 1; j < VEC; ++j) {
                    sw = add(sw, mul(wn.v[j], wn.v[j]));
                    sp = add(sp, mul(pnew.v[j], pnew.v[j]));
                }
            }
        }
        if constexpr (LEJA) {
            sw = warp_sum(sw);
            sp = warp_sum(sp);
            if (lane == 0) {
                s_red[((z - zb) * BY3 + wy) * 2 + 0] = sw;
                s_red[((z - zb) * BY3 + wy) * 2 + 1] = sp;
            }
        }
        if (more) put_plane(buf ^ 1, cnext, hrow, hcol);
        buf ^= 1;
        zm = c;
        c = cnext;
        zp = zq;
        pc = pn;
    }
}

// ---------------------------------------------------------------------------
// 2D (nz == 1): warps own (32*VEC)-wide x strips, march y.  z ghosts follow
// the mode (zero: 0; periodic / Neumann: the point itself; faces: fz_*),
// multiplied by wz == 0 exactly as the reference does (signed zeros kept).
template <int VEC, int COEFF, bool GD, bool LEJA>
ES_DEV void pass2d(const Geom &g, const Pass &ps, const double *gdiag, int chunk_len,
                   double *s_red) {
    constexpr int TXW = 32 * VEC;
    const int lane = threadIdx.x, wy = threadIdx.y;
    const int64_t x0 = ((int64_t)blockIdx.x * BW2 + wy) * TXW;
    const int64_t ix = x0 + lane * VEC;
    const bool act = ix < g.nx;
    const int64_t yb = (int64_t)blockIdx.y * chunk_len;
    const int64_t ye = min(g.ny, yb + chunk_len);
    const double *src = ps.src;

    double ox2[VEC];
#pragma unroll
    for (int j = 0; j < VEC; ++j) ox2[j] = 1.0;
    if constexpr (COEFF == ES_COEFF_RADIAL) {
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
            const double x = axis_coord(ix + j, g.nx);
            ox2[j] = add(1.0, mul(x, x));
        }
    }

    Vv<VEC> ym = fetchv<VEC>(g, src, ix, yb - 1, 0);
    Vv<VEC> c = fetchv<VEC>(g, src, ix, yb, 0);
    Vv<VEC> yp = fetchv<VEC>(g, src, ix, yb + 1, 0);
    Vv<VEC> yq = zeros<VEC>();
    Vv<VEC> pc = zeros<VEC>(), pn = zeros<VEC>();
    if constexpr (LEJA) {
        if (act && ps.p_src) pc = ldv<VEC>(ps.p_src + yb * g.nx + ix);
    }
    double edge = 0.0, edge_next = 0.0;
    if (lane == 0) edge = fetch1(g, src, x0 - 1, yb, 0);
    if (lane == 31) edge = fetch1(g, src, x0 + TXW, yb, 0);

    for (int64_t y = yb; y < ye; ++y) {
        const bool more = y + 1 < ye;
        if (more) {
            yq = fetchv<VEC>(g, src, ix, y + 2, 0);
            if (lane == 0) edge_next = fetch1(g, src, x0 - 1, y + 1, 0);
            if (lane == 31) edge_next = fetch1(g, src, x0 + TXW, y + 1, 0);
            if constexpr (LEJA) {
                if (act && ps.p_src) pn = ldv<VEC>(ps.p_src + (y + 1) * g.nx + ix);
            }
        }
        const double left = __shfl_up_sync(0xffffffffu, c.v[VEC - 1], 1);
        const double right = __shfl_down_sync(0xffffffffu, c.v[0], 1);
        double sw = 0.0, sp = 0.0;
        if (act) {
            double yy = 0.0;
            if constexpr (COEFF == ES_COEFF_RADIAL) yy = axis_coord(y, g.ny);
            Vv<VEC> wn, pnew;
            const int64_t base = y * g.nx + ix;
#pragma unroll
            for (int j = 0; j < VEC; ++j) {
                const double cc = c.v[j];
                const double xm = j > 0 ? c.v[j - 1] : (lane == 0 ? edge : left);
                const double xp = j < VEC - 1 ? c.v[j + 1] : (lane == 31 ? edge : right);
                double zm = 0.0, zp = 0.0;
                if (g.mode == ES_MODE_PERIODIC || g.mode == ES_MODE_NEUMANN) {
                    zm = cc;
                    zp = cc;
                } else if (g.mode == ES_MODE_FACES) {
                    zm = __ldg(g.faces[4] + base + j);
                    zp = __ldg(g.faces[5] + base + j);
                }
                const double lap = lap7(cc, xm, xp, ym.v[j], yp.v[j], zm, zp, g.wx, g.wy, g.wz);
                double dco = 1.0;
                if constexpr (COEFF == ES_COEFF_RADIAL) dco = radial_from_sq(ox2[j], yy);
                double pold = 0.0;
                if constexpr (LEJA) pold = ps.p_src ? pc.v[j] : mul(ps.d0, cc);
                point_out<COEFF, GD, LEJA>(g, ps, gdiag, base + j, lap, dco, cc, pold, wn.v[j], pnew.v[j]);
            }
            stv<VEC>(ps.dst + base, wn);
            if constexpr (LEJA) {
                stv<VEC>(ps.p_dst + base, pnew);
                sw = mul(wn.v[0], wn.v[0]);
                sp = mul(pnew.v[0], pnew.v[0]);
#pragma unroll
                for (int j = 1; j < VEC; ++j) {
                    sw = add(sw, mul(wn.v[j], wn.v[j]));
                    sp = add(sp, mul(pnew.v[j], pnew.v[j]));
                }
            }
        }
        if constexpr (LEJA) {
            sw = warp_sum(sw);
            sp = warp_sum(sp);
            if (lane == 0) {
                s_red[((y - yb) * BW2 + wy) * 2 + 0] = sw;
                s_red[((y - yb) * BW2 + wy) * 2 + 1] = sp;
            }
        }
        ym = c;
        c = yp;
        yp = yq;
        pc = pn;
        edge = edge_next;
    }
}

}  // namespace es
