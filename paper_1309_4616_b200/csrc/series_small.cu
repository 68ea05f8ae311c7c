// Persistent L2-resident Newton-Leja series for small single-plane grids
// (C1: 256^2, 65,536 points, 0.5 MiB per vector).
//
// On such grids a node is pure latency: the TMA node kernel + slice reduce
// pair costs ~9 us per node whatever the size (launch, ring fill, reduction
// tail), 3 % of the HBM roofline.  Here ONE cooperative launch runs the whole
// series: every CTA owns one row chunk of the TMA plan (the same (chunk,
// tile) items, the same thread -> point-pair map), keeps its points' w and p
// in registers across nodes, exchanges only its boundary rows through L2
// (w_k is still written for the neighbours' stencils), and the CTAs meet at
// one grid barrier per node.  The stopping test runs redundantly in every
// CTA on the same slice sums in the same order, so all CTAs take the same
// decision without a second barrier.
//
// Bitwise the general path: the per-point expression trees are those of
// tma_consume (stencil_tma.cuh) and the norm partials are accumulated and
// reduced in its exact order -- lane over the chunk's rows, warp xor tree,
// slice = cta_slice_sum's thread-strided / warp-ordered sum over the
// (tile, warp) entries, decision = slice_reduce_decide's lane-strided sum
// over slices -- so p, the matvec counts and the series state are identical
// to the graph path's (tests/test_gpu_parity.py::test_small_series_*).
//
// The fused exponential-Euler step (x3 of the scope table) runs both series
// of integrator.py:177-189 in one launch -- CTAs [0, C) the exp series on u,
// CTAs [C, 2C) the phi1 series on g(u) - b, which those CTAs evaluate in the
// kernel itself (the combustion term and its domain check) -- and, after a
// barrier over all CTAs, u_out = y + h z.

#include <algorithm>
#include <map>
#include <mutex>

#include "es_host.h"
#include "series.cuh"
#include "stencil_tma.cuh"

namespace es {

constexpr int SMALL_THREADS = 32 * TMA_CONSUMER_WARPS;  // the TMA consumer map: thread t owns x = 2t, 2t + 1
constexpr int SMALL_MAXROWS = 8;                        // rows per chunk held in registers (the 2D plan's cap)

ES_DEV double ldcg1(const double *p) { return __ldcg(p); }
ES_DEV double2 ldcg2(const double *p) { return __ldcg(reinterpret_cast<const double2 *>(p)); }

// Grid-wide barrier over `nblocks` CTAs on a counter that only grows within
// one launch (reset by k_series_init); round r waits for nblocks * r
// arrivals.  The CTA's writes before it (ordered before thread 0 by the
// bar.sync) are released by the arrival and acquired by every CTA after it;
// the poll itself is a relaxed load (an acquire load per poll would
// invalidate L1 on every iteration).
ES_DEV void small_barrier(unsigned *cnt, unsigned target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
        unsigned v;
        for (;;) {
            asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory");
            if (v >= target) break;
        }
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    __syncthreads();
}

// The stopping test of decide() (series.cuh) without touching the device
// state; every CTA runs it on identical sums.
struct Decision {
    int stop, converged;
    double term, pnorm;
};

ES_DEV Decision small_decide(const SeriesParams &P, int k, double sumw, double sump, int &consecutive) {
    Decision d{0, 0, 0.0, 0.0};
    const double adk = fabs(P.dd[k]);
    d.term = mul(adk, sqrt_rn(sumw));
    d.pnorm = sqrt_rn(sump);
    if (P.tol > 0.0) {
        if (d.term <= mul(P.tol, d.pnorm)) {
            consecutive += 1;
            if (consecutive >= 2) {
                d.stop = 1;
                d.converged = 1;
            }
        } else {
            consecutive = 0;
        }
    }
    if (!d.stop && k >= P.ndd - 1) {
        d.stop = 1;
        d.converged = P.tol == 0.0 ? 1 : 0;
    }
    return d;
}

// w_k at the pair (x, x+1) of row m (tma_consume, DIM3 = false): ghosts of
// the zero fill / row re-targeting / in-plane patches, coherent L2 loads
// (w_{k-1} was written by other CTAs of this launch).
template <int COEFF, bool GD>
ES_DEV double2 small_pair(const Geom &g, const double *src, const double *gdiag, int64_t x, int64_t m, double2 c,
                          double alpha, double beta, const double ox2[2]) {
    const int64_t nx = g.nx, ny = g.ny, row = m * nx;
    double xm0 = x > 0 ? ldcg1(src + row + x - 1) : 0.0;
    double xp1 = x + 2 < nx ? ldcg1(src + row + x + 2) : 0.0;
    double2 ym = make_double2(0.0, 0.0), yp = ym, zm = ym, zp = ym;
    const bool per = g.mode == ES_MODE_PERIODIC, neu = g.mode == ES_MODE_NEUMANN;
    if (m > 0)
        ym = ldcg2(src + row - nx + x);
    else if (per)
        ym = ldcg2(src + (ny - 1) * nx + x);
    else if (neu)
        ym = c;
    if (m + 1 < ny)
        yp = ldcg2(src + row + nx + x);
    else if (per)
        yp = ldcg2(src + x);
    else if (neu)
        yp = c;
    if (g.mode != ES_MODE_ZERO) {
        if (x == 0) xm0 = neu ? c.x : ldcg1(src + row + nx - 1);
        if (x + 2 == nx) xp1 = neu ? c.y : ldcg1(src + row);
        zm = c;  // single-plane grid: z ghosts are the point itself
        zp = c;
    }
    const double cc[2] = {c.x, c.y}, xm[2] = {xm0, c.x}, xp[2] = {c.y, xp1};
    const double ymv[2] = {ym.x, ym.y}, ypv[2] = {yp.x, yp.y}, zmv[2] = {zm.x, zm.y}, zpv[2] = {zp.x, zp.y};
    double yy = 0.0;
    if constexpr (COEFF == ES_COEFF_RADIAL) yy = axis_coord(m, ny);
    double2 gv = make_double2(0.0, 0.0);
    if constexpr (GD) gv = __ldg(reinterpret_cast<const double2 *>(gdiag + row + x));
    const double gvv[2] = {gv.x, gv.y};
    double wn[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        double lap = lap7(cc[j], xm[j], xp[j], ymv[j], ypv[j], zmv[j], zpv[j], g.wx, g.wy, g.wz);
        if constexpr (COEFF == ES_COEFF_RADIAL) lap = mul(radial_from_sq(ox2[j], yy), lap);
        if constexpr (COEFF == ES_COEFF_ARRAY) lap = mul(__ldg(g.coeff + row + x + j), lap);
        if constexpr (GD) lap = sub(lap, mul(gvv[j], cc[j]));
        wn[j] = add(mul(alpha, lap), mul(beta, cc[j]));
    }
    return make_double2(wn[0], wn[1]);
}

constexpr int SMALL_MAXITEMS = SMALL_MAXROWS / 2;  // row chunks per CTA (the 2D plan's chunks are >= 2 rows)
// ROWS (2, 4 or 8): rows per CTA held in registers, a template parameter so
// small chunks do not pay the 8-row register footprint (occupancy)

struct SmallShared {
    double ent[SMALL_MAXITEMS][2 * TMA_CONSUMER_WARPS];  // (item, warp) partials of w^2, p^2
};

// The whole series over this CTA's `ipc` consecutive row chunks (items of
// the TMA plan) starting at chunk c0.  `round0`: barrier rounds already used
// on P.global_cnt; `nblocks`: CTAs of this series.  p holds this thread's p
// of the CTA's rows on return (also written to P.pbuf[1] == p_out).
//
// A slice (one chunk) has TMA_CONSUMER_WARPS entries (one tile column), so
// cta_slice_sum's thread-strided sum puts entry e on lane e of warp 0, its
// xor tree sums them, and the other warps add +0.0 -- the sums are of
// squares, never -0.0, so warp i's xor tree over lanes < 8 of item i is that
// value bit for bit.
template <int COEFF, bool GD, int ROWS>
ES_DEV int small_series(const SeriesParams &P, const Geom &g, int c0, int ipc, int nblocks, unsigned round0,
                        SmallShared &sh, double2 (&p)[ROWS], int &converged) {
    constexpr int ITEMS = ROWS / 2 < SMALL_MAXITEMS ? ROWS / 2 : SMALL_MAXITEMS;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int64_t x = 2 * (int64_t)t;
    const bool act = x < g.nx;
    const int CL = P.chunk_len;
    const int nitems = min(ipc, P.nchunks - c0);
    const int mb = c0 * CL, me = min((int)g.ny, mb + nitems * CL);
    double ox2[2] = {1.0, 1.0};
    if constexpr (COEFF == ES_COEFF_RADIAL) {
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const double xc = axis_coord(x + j, g.nx);
            ox2[j] = add(1.0, mul(xc, xc));
        }
    }
    double2 w[ROWS];  // this thread's w_{k-1} (v before node 1)
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
        const int m = mb + r;
        w[r] = act && m < me ? ldcg2(P.v + (int64_t)m * g.nx + x) : make_double2(0.0, 0.0);
        p[r] = make_double2(0.0, 0.0);
    }
    // node kk: w_kk, p_kk of this thread's rows, w_kk to the neighbours'
    // buffer, this CTA's slices of node kk (double-buffered by parity)
    auto node = [&](int kk) {
        const double *src = kk == 1 ? P.v : P.wbuf[(kk - 1) & 1];
        double *dst = P.wbuf[kk & 1];
        const double beta = sub(-P.shift, P.xi[kk - 1]), dk = P.dd[kk], d0 = P.dd[0];
        double acc_w[ITEMS], acc_p[ITEMS];
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) acc_w[i] = acc_p[i] = 0.0;
        double2 wn[ROWS];
#pragma unroll
        for (int r = 0; r < ROWS; ++r) {
            const int m = mb + r;
            if (!act || m >= me) continue;
            wn[r] = small_pair<COEFF, GD>(g, src, P.gdiag, x, m, w[r], P.alpha, beta, ox2);
            const double p0 = kk == 1 ? mul(d0, w[r].x) : p[r].x, p1 = kk == 1 ? mul(d0, w[r].y) : p[r].y;
            p[r] = make_double2(add(p0, mul(dk, wn[r].x)), add(p1, mul(dk, wn[r].y)));
            __stcg(reinterpret_cast<double2 *>(dst + (int64_t)m * g.nx + x), wn[r]);
        }
        // norm contributions per item, rows in order (tma_consume's lane accumulation)
#pragma unroll
        for (int r = 0; r < ROWS; ++r) {
            if (!act || mb + r >= me) continue;
            const int i = r / CL;
#pragma unroll
            for (int q = 0; q < ITEMS; ++q) {
                if (q != i) continue;
                acc_w[q] = add(acc_w[q], add(mul(wn[r].x, wn[r].x), mul(wn[r].y, wn[r].y)));
                acc_p[q] = add(acc_p[q], add(mul(p[r].x, p[r].x), mul(p[r].y, p[r].y)));
            }
            w[r] = wn[r];
        }
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            if (i >= nitems) break;
            const double aw = warp_sum(acc_w[i]), ap = warp_sum(acc_p[i]);
            if (lane == 0) {  // entry (tile 0, warp) of chunk c0 + i
                sh.ent[i][2 * warp] = aw;
                sh.ent[i][2 * warp + 1] = ap;
            }
        }
        __syncthreads();
        double *slice = P.slice + (int64_t)(kk & 1) * 2 * P.nslices;
        if (warp < nitems) {
            double a = lane < TMA_CONSUMER_WARPS ? sh.ent[warp][2 * lane] : 0.0;
            double b = lane < TMA_CONSUMER_WARPS ? sh.ent[warp][2 * lane + 1] : 0.0;
            a = warp_sum(a);
            b = warp_sum(b);
            if (lane == 0) __stcg(reinterpret_cast<double2 *>(slice + 2 * (c0 + warp)), make_double2(a, b));
        }
    };
    // Node k's decision is taken one node late: after barrier k every warp
    // issues the loads of node k's slices, computes node k + 1 (which only
    // needs w_k) while they are in flight, then decides k.  A stop at k
    // keeps p_k and drops node k + 1 (its w / slices land in buffers nobody
    // reads again); otherwise node k + 1 is already done at barrier k + 1.
    // Buffers by parity stay safe: node k + 1 overwrites what node k - 1
    // wrote, and every CTA finished reading that before barrier k.
    int consecutive = 0, k = 1;
    Decision d{};
    node(1);
    small_barrier(P.global_cnt, (unsigned)nblocks * (round0 + 1u));
    for (;; ++k) {
        const double *slice = P.slice + (int64_t)(k & 1) * 2 * P.nslices;
        double2 sv[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int s = lane + 32 * j;
            sv[j] = s < P.nslices ? ldcg2(slice + 2 * s) : make_double2(0.0, 0.0);
        }
        const bool more = k + 1 <= P.ndd - 1;
        double2 p_keep[ROWS];
#pragma unroll
        for (int r = 0; r < ROWS; ++r) p_keep[r] = p[r];
        if (more) node(k + 1);
        // slice_reduce_decide's order: lane-strided over slices, then the xor tree
        double sw = 0.0, sp = 0.0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (lane + 32 * j < P.nslices) {
                sw = add(sw, sv[j].x);
                sp = add(sp, sv[j].y);
            }
        }
        for (int s = lane + 128; s < P.nslices; s += 32) {
            const double2 v2 = ldcg2(slice + 2 * s);
            sw = add(sw, v2.x);
            sp = add(sp, v2.y);
        }
        sw = warp_sum(sw);
        sp = warp_sum(sp);
        d = small_decide(P, k, sw, sp, consecutive);
        if (d.stop) {
#pragma unroll
            for (int r = 0; r < ROWS; ++r) p[r] = p_keep[r];
            break;
        }
        small_barrier(P.global_cnt, (unsigned)nblocks * (round0 + (unsigned)k + 1u));
    }
    converged = d.converged;
    // the result into p_out (pbuf[1]) -- the graph path's finalize moves it there too
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
        const int m = mb + r;
        if (act && m < me) *reinterpret_cast<double2 *>(P.pbuf[1] + (int64_t)m * g.nx + x) = p[r];
    }
    if (c0 == 0 && t == 0) {
        SeriesState &st = *P.state;
        st.k = k;
        st.consecutive = consecutive;
        st.pass = k;
        st.last_term = d.term;
        st.last_pnorm = d.pnorm;
        st.converged = d.converged;
        st.done = 1;
    }
    return k;
}

template <int COEFF, bool GD, int ROWS>
__global__ void __launch_bounds__(SMALL_THREADS) k_series_small(const SeriesParams *__restrict__ Pp, int ipc) {
    __shared__ SmallShared sh;
    const SeriesParams &P = *Pp;
    const Geom g = P.g;
    double2 p[ROWS];
    int conv;
    small_series<COEFF, GD, ROWS>(P, g, blockIdx.x * ipc, ipc, gridDim.x, 0u, sh, p, conv);
}

// Exponential Euler in one launch: CTAs [0, C) run y = exp series on u
// (A, p_out = u_out), CTAs [C, 2C) evaluate g_n = g(u) - b on their rows
// (into B's v, the caller's scratch) and run z = phi1 series (B); then all
// CTAs meet and the exp CTAs write u_out = y + h z on their rows when both
// series converged (the graph path's k_axpy_if guard).
template <int COEFF, int ROWS>
__global__ void __launch_bounds__(SMALL_THREADS) k_expeuler_small(const SeriesParams *__restrict__ PA,
                                                                  const SeriesParams *__restrict__ PB, const double *u,
                                                                  double *gn, const double *source, int nonlin,
                                                                  double h, unsigned long long *bad, int ipc,
                                                                  SmallStepRecord *rec) {
    __shared__ SmallShared sh;
    const int C = (int)gridDim.x / 2;  // CTAs per series
    const bool is_b = (int)blockIdx.x >= C;
    const int c0 = (is_b ? blockIdx.x - C : blockIdx.x) * ipc;
    const SeriesParams &P = is_b ? *PB : *PA;
    const Geom g = P.g;
    const int t = threadIdx.x;
    const int64_t x = 2 * (int64_t)t, n = g.nx * g.ny;
    const bool act = x < g.nx;
    const int mb = c0 * P.chunk_len, me = min((int)g.ny, mb + ipc * P.chunk_len);
    unsigned round0 = 0;
    bool skip = false;
    if (is_b) {  // g_n = g(u) - b (integrator.py:115-123, _core.pyx:325-348), domain check on device
        for (int m = mb; m < me && act; ++m) {
            const int64_t o = (int64_t)m * g.nx + x;
            double gv[2] = {0.0, 0.0};
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                if (nonlin == ES_NONLIN_COMBUSTION) {
                    const double xv = __ldg(u + o + j);
                    if (xv <= 0.0) atomicMin(bad, (unsigned long long)(o + j));
                    const double rr = __drcp_rn(xv);
                    gv[j] = mul(mul(0.25, sub(2.0, xv)), exp(mul(20.0, sub(1.0, rr))));
                    if (source) gv[j] = add(gv[j], mul(-1.0, __ldg(source + o + j)));
                } else {
                    gv[j] = mul(-1.0, __ldg(source + o + j));
                }
            }
            __stcg(reinterpret_cast<double2 *>(gn + o), make_double2(gv[0], gv[1]));
        }
        small_barrier(P.global_cnt, (unsigned)C);  // round 0: g_n complete before node 1 reads it
        round0 = 1;
        // a point outside the domain: the caller raises DomainError; the series is not run
        skip = nonlin == ES_NONLIN_COMBUSTION && __ldcg(bad) < (unsigned long long)n;
        if (skip && c0 == 0 && t == 0) {
            SeriesState &st = *P.state;
            st.k = 0;
            st.pass = 0;
            st.consecutive = 0;
            st.converged = 1;
            st.done = 1;
            st.last_term = 0.0;
            st.last_pnorm = 0.0;
        }
    }
    double2 p[ROWS];
    int conv = 1;
    if (!skip) small_series<COEFF, false, ROWS>(P, g, c0, ipc, C, round0, sh, p, conv);
    // every CTA of both series: y and z complete, both states written
    small_barrier(PA->work, 2u * (unsigned)C);
    if (rec && blockIdx.x == 0 && t == 0) {  // both outcomes straight into host-mapped memory (no copies)
        rec->a = *PA->state;
        SeriesState sb;
        sb.k = __ldcg(&PB->state->k);
        sb.consecutive = __ldcg(&PB->state->consecutive);
        sb.done = __ldcg(&PB->state->done);
        sb.converged = __ldcg(&PB->state->converged);
        sb.last_term = __ldcg(&PB->state->last_term);
        sb.last_pnorm = __ldcg(&PB->state->last_pnorm);
        sb.pass = __ldcg(&PB->state->pass);
        sb.pad_ = 0;
        rec->b = sb;
        rec->bad = __ldcg(bad);
        __threadfence_system();
    }
    if (is_b || !act) return;
    const bool ok = conv == 1 && __ldcg(&PB->state->converged) == 1 && __ldcg(&PB->state->k) > 0;
    if (!ok) return;
    const double *z = PB->pbuf[1];
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
        const int m = mb + r;
        if (m >= me) break;
        const int64_t o = (int64_t)m * g.nx + x;
        const double2 zz = ldcg2(z + o);
        *reinterpret_cast<double2 *>(PA->pbuf[1] + o) = make_double2(add(p[r].x, mul(h, zz.x)), add(p[r].y, mul(h, zz.y)));
    }
}

// Both series' parameters and states and the domain-check word in one launch.
__global__ void k_expeuler_small_init(const SeriesParams a, SeriesParams *da, const SeriesParams b, SeriesParams *db,
                                      unsigned long long *bad, unsigned long long n) {
    series_init_body(a, da);
    series_init_body(b, db);
    if (threadIdx.x == 0) *bad = n;
}

// ---------------------------------------------------------------------------
// host side

namespace {

template <int ROWS>
const void *small_fn_r(int coeff, bool gd) {
    switch (coeff) {
        case ES_COEFF_RADIAL:
            return gd ? (const void *)k_series_small<ES_COEFF_RADIAL, true, ROWS>
                      : (const void *)k_series_small<ES_COEFF_RADIAL, false, ROWS>;
        case ES_COEFF_ARRAY:
            return gd ? (const void *)k_series_small<ES_COEFF_ARRAY, true, ROWS>
                      : (const void *)k_series_small<ES_COEFF_ARRAY, false, ROWS>;
        default:
            return gd ? (const void *)k_series_small<ES_COEFF_NONE, true, ROWS>
                      : (const void *)k_series_small<ES_COEFF_NONE, false, ROWS>;
    }
}

template <int ROWS>
const void *expeuler_fn_r(int coeff) {
    switch (coeff) {
        case ES_COEFF_RADIAL: return (const void *)k_expeuler_small<ES_COEFF_RADIAL, ROWS>;
        case ES_COEFF_ARRAY: return (const void *)k_expeuler_small<ES_COEFF_ARRAY, ROWS>;
        default: return (const void *)k_expeuler_small<ES_COEFF_NONE, ROWS>;
    }
}

const void *small_fn(int coeff, bool gd, int rows) {
    return rows <= 2 ? small_fn_r<2>(coeff, gd) : rows <= 4 ? small_fn_r<4>(coeff, gd) : small_fn_r<8>(coeff, gd);
}

const void *expeuler_fn(int coeff, int rows) {
    return rows <= 2 ? expeuler_fn_r<2>(coeff) : rows <= 4 ? expeuler_fn_r<4>(coeff) : expeuler_fn_r<8>(coeff);
}

// co-resident CTAs of a kernel on this device (cached per device and kernel)
int capacity(const void *fn) {
    static std::mutex mu;
    static std::map<std::pair<int, const void *>, int> cache;
    const int dev = current_device();
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find({dev, fn});
    if (it != cache.end()) return it->second;
    int per_sm = 0, sms = 0, coop = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, SMALL_THREADS, 0) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev) != cudaSuccess) {
        cudaGetLastError();
        per_sm = 0;
    }
    const int cap = coop ? per_sm * sms : 0;
    cache[{dev, fn}] = cap;
    return cap;
}

// row chunks per CTA: fewer, fuller CTAs make the per-node grid barrier
// cheaper (ES_SMALL_IPC overrides; at most SMALL_MAXROWS rows per CTA)
int items_per_cta(const StencilPlan &pl) {
    const int cap = std::max(1, SMALL_MAXROWS / std::max(1, pl.chunk));
    return std::min(cap, std::max(1, env_int("ES_SMALL_IPC", 1)));
}

int rows_for(const StencilPlan &pl) { return items_per_cta(pl) * pl.chunk; }

int ctas_for(const StencilPlan &pl) {
    const int ipc = items_per_cta(pl);
    return (pl.nchunks + ipc - 1) / ipc;
}

}  // namespace

// The persistent form applies to single-plane TMA plans of one tile column
// (nx <= 512) whose chunks all fit co-resident, at most 2^20 points (L2
// resident); ES_SMALL=0 turns it off.
bool small_series_ok(const es_stencil_desc *d, const StencilPlan &pl, bool gd, int nseries) {
    if (!env_int("ES_SMALL", 1)) return false;
    if (!pl.tma || !pl.dim2 || pl.grid.x != 1 || pl.chunk > SMALL_MAXROWS) return false;
    if (d->nx * d->ny > (1 << 20) || d->mode == ES_MODE_FACES) return false;
    const void *fn = nseries == 2 ? expeuler_fn(d->coeff_kind, rows_for(pl)) : small_fn(d->coeff_kind, gd, rows_for(pl));
    return (int64_t)nseries * ctas_for(pl) <= capacity(fn);
}

int launch_series_small(const es_stencil_desc *d, const SeriesParams *dparams, const StencilPlan &pl, bool gd,
                        cudaStream_t stream) {
    int ipc = items_per_cta(pl);
    void *args[] = {(void *)&dparams, (void *)&ipc};
    if (cudaLaunchCooperativeKernel(small_fn(d->coeff_kind, gd, rows_for(pl)), dim3((unsigned)ctas_for(pl)),
                                    dim3(SMALL_THREADS),
                                    args, 0, stream) != cudaSuccess)
        return check_launch("small-grid series");
    return check_launch("small-grid series");
}

int launch_expeuler_small_init(const SeriesParams *ha, SeriesParams *da, const SeriesParams *hb, SeriesParams *db,
                               unsigned long long *bad, int64_t n, cudaStream_t stream) {
    k_expeuler_small_init<<<1, 256, 0, stream>>>(*ha, da, *hb, db, bad, (unsigned long long)n);
    return check_launch("small-grid step init");
}

int launch_expeuler_small(const es_stencil_desc *d, const SeriesParams *pa, const SeriesParams *pb,
                          const StencilPlan &pl, const double *u, double *gn, const double *source, int nonlin,
                          double h, unsigned long long *bad, SmallStepRecord *rec, cudaStream_t stream) {
    int ipc = items_per_cta(pl);
    void *args[] = {(void *)&pa,     (void *)&pb, (void *)&u,   (void *)&gn,  (void *)&source,
                    (void *)&nonlin, (void *)&h,  (void *)&bad, (void *)&ipc, (void *)&rec};
    if (cudaLaunchCooperativeKernel(expeuler_fn(d->coeff_kind, rows_for(pl)), dim3(2u * (unsigned)ctas_for(pl)),
                                    dim3(SMALL_THREADS), args, 0, stream) != cudaSuccess)
        return check_launch("small-grid exponential Euler step");
    return check_launch("small-grid exponential Euler step");
}

}  // namespace es
