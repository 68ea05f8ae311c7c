// CSR fused SpMV and the fused Newton-Leja node for unstructured operators
// (reference sparse.py:150-192 -> _core.pyx:245-319, matfunc.py:271-318).
//
// Parity: every row sum is accumulated strictly in storage order, one thread
// per row, starting from 0 -- the reference's compiled loop
// (`acc = acc + vals[k] * x[col_idx[k]]`, _core.pyx:253-255) -- so results are
// bitwise identical.  The products are formed lane-strided (coalesced
// col / vals streams, independent gathers in flight) and staged in shared
// memory; each lane then adds its own row's products in order.
//
// Bound: the node is limited by random 8-byte gathers of the L2-resident
// vector (one 32-byte L2 sector each), not by the HBM stream.  The gather
// probe (tools/gather_probe.cu, profiles/) measures that ceiling at ~208 G
// gathers/s on B200, i.e. ~262 us for the 5.45e7 gathers of a C5 node; the
// node kernel runs at ~297 us.  Gathers go through the texture path (TEX
// pipe) at 12 CTAs/SM, which beat LDG gathers by 16 % (variants below).
//
// The plain apply (k_csr_rows) keeps a 256-row CTA tile with the same
// staging; x is read through L1 there.
#include <algorithm>
#include <map>
#include <mutex>

#include "es_host.h"
#include "series.cuh"

namespace es {

constexpr int CSR_T = 256;     // threads = rows per CTA tile
constexpr int CSR_CAP = 4096;  // products staged per round (32 KB)
constexpr int CSR_U = 4;       // independent (col, val, x) loads per thread in flight

struct CsrRowsArgs {
    int64_t row_lo, row_hi;
    const int64_t *rp;
    const int32_t *col;
    const double *vals;
    const double *x;
    double *y;
    double alpha, beta;
    int use_beta;
};

// Gather paths for x[col[k]] (G): 0 = LSU read-only (__ldg), 1 = texture
// fetch (TEX pipe, int2 texel reinterpreted), 2 = LSU without L1 allocation.
template <int G>
ES_DEV double gather_x(const double *__restrict__ x, unsigned long long tex, int c) {
    if constexpr (G == 1) {
        const int2 t = tex1Dfetch<int2>((cudaTextureObject_t)tex, c);
        return __hiloint2double(t.y, t.x);
    } else if constexpr (G == 2) {
        double r;
        asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(r) : "l"(x + c));
        return r;
    } else {
        return __ldg(x + c);
    }
}

// sum_k vals[k] x[col[k]] over row r (act: r is a row of this tile), the
// tile being rows [r0, rend).  Called by all CSR_T threads of the CTA.
template <int G = 0>
ES_DEV double csr_tile_sum(int64_t r0, int64_t rend, int64_t r, bool act, const int64_t *__restrict__ rp,
                           const int32_t *__restrict__ col, const double *__restrict__ vals,
                           const double *__restrict__ x, double *s_prod, unsigned long long tex = 0) {
    double acc = 0.0;
    if (r0 >= rend) return acc;
    const int64_t kb = __ldg(rp + r0), ke = __ldg(rp + rend);
    const int64_t ks = act ? __ldg(rp + r) : 0, kend = act ? __ldg(rp + r + 1) : 0;
    for (int64_t base = kb; base < ke; base += CSR_CAP) {
        const int lim = (int)min((int64_t)CSR_CAP, ke - base);
        const int32_t *cb = col + base;
        const double *vb = vals + base;
        for (int j0 = threadIdx.x; j0 < lim; j0 += CSR_T * CSR_U) {
            int c[CSR_U];
            double v[CSR_U];
#pragma unroll
            for (int u = 0; u < CSR_U; ++u) {
                const int j = j0 + u * CSR_T;
                if (j < lim) {
                    c[u] = __ldcs(cb + j);
                    v[u] = __ldcs(vb + j);
                }
            }
#pragma unroll
            for (int u = 0; u < CSR_U; ++u) {
                const int j = j0 + u * CSR_T;
                if (j < lim) s_prod[j] = mul(v[u], gather_x<G>(x, tex, c[u]));
            }
        }
        __syncthreads();
        const int lo = (int)(max(ks, base) - base), hi = (int)(min(kend, base + lim) - base);
        for (int k = lo; k < hi; ++k) acc = add(acc, s_prod[k]);
        __syncthreads();
    }
    return acc;
}

__global__ void __launch_bounds__(CSR_T) k_csr_rows(const CsrRowsArgs a) {
    __shared__ double s_prod[CSR_CAP];
    const int64_t r0 = a.row_lo + (int64_t)blockIdx.x * CSR_T;
    const int64_t rend = min(r0 + CSR_T, a.row_hi);
    const int64_t r = r0 + threadIdx.x;
    const bool act = r < rend;
    const double acc = csr_tile_sum(r0, rend, r, act, a.rp, a.col, a.vals, a.x, s_prod);
    if (act) a.y[r] = a.use_beta ? add(mul(a.alpha, acc), mul(a.beta, __ldg(a.x + r))) : mul(a.alpha, acc);
}

// ----- the node kernel: warp-autonomous tiles at high occupancy ------------------
//
// The gather probe (tools/gather_probe.cu) shows the L2-resident random gather
// ceiling is reached by many independent warps, not by deep per-thread
// queues.  A warp owns 32 consecutive rows; it streams their contiguous
// nonzero range in rounds of 32 * W4_U products (coalesced col / vals loads,
// W4_U gathers in flight per lane, products staged in the warp's own
// shared-memory slice), then every lane adds its row's products of the round
// in storage order.  No CTA-wide barrier inside the sweep; the warp
// partials of a CTA tile are combined in warp order and reduced by the
// slice-reduce kernel.
constexpr int W4_WARPS = 4;
constexpr int W4_T = 32 * W4_WARPS;               // rows per CTA tile
constexpr int W4_CHB = 16384 / W4_T;              // tiles per 16384-row chunk

// P2P: the peer-memory row-block series' variant: gathers come from this
// rank's parity buffer xgp[k & 1], and every row's w_k is stored into every
// rank's gathered vector of parity (k + 1) & 1 -- the all-gather fused into
// the node, overlapped with its gather-bound sweep.
template <int G, int MINB, int W4_U, bool P2P = false>
__global__ void __launch_bounds__(W4_T, MINB) k_csr_node_w4(const SeriesParams *__restrict__ Pp) {
    constexpr int W4_ROUND = 32 * W4_U;
    __shared__ double s_prod[W4_WARPS][W4_ROUND];
    __shared__ double s_red[W4_WARPS][2];
    const SeriesParams &P = *Pp;
    if (P.state->done) return;
    const int k = P.state->k + 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t n = P.n;
    const int64_t r0 = ((int64_t)blockIdx.x * W4_WARPS + warp) * 32;
    const int64_t r = r0 + lane;
    const bool act = r < n;
    const double *__restrict__ xs =
        P2P ? P.xgp[k & 1] : P.xg ? P.xg : (k == 1 ? P.v : P.wbuf[(k - 1) & 1]);
    const unsigned long long tex = P2P ? P.tex[k & 1] : P.xg ? P.tex[3] : P.tex[k == 1 ? 2 : (k - 1) & 1];
    double acc = 0.0;
    if (r0 < n) {
        const int64_t *__restrict__ rp = P.row_ptr;
        const int64_t kb = __ldg(rp + r0), ke = __ldg(rp + min(r0 + 32, n));
        const int64_t ks = act ? __ldg(rp + r) : 0, kend = act ? __ldg(rp + r + 1) : 0;
        double *sp = s_prod[warp];
        for (int64_t base = kb; base < ke; base += W4_ROUND) {
            const int lim = (int)min((int64_t)W4_ROUND, ke - base);
            int c[W4_U];
            double v[W4_U];
#pragma unroll
            for (int u = 0; u < W4_U; ++u) {
                const int j = lane + 32 * u;
                c[u] = j < lim ? __ldcs(P.col + base + j) : 0;
                v[u] = j < lim ? __ldcs(P.vals + base + j) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < W4_U; ++u) {
                const int j = lane + 32 * u;
                if (j < lim) sp[j] = mul(v[u], gather_x<G>(xs, tex, c[u]));
            }
            __syncwarp();
            const int lo = (int)(max(ks, base) - base), hi = (int)(min(kend, base + lim) - base);
            for (int q = lo; q < hi; ++q) acc = add(acc, sp[q]);
            __syncwarp();
        }
    }
    double sw = 0.0, sq = 0.0;
    const Pass ps = node_pass(P, k);  // loaded after the sweep: fewer live registers
    if (act) {
        const double c = __ldg(ps.src + r);
        const double wn = add(mul(ps.alpha, acc), mul(ps.beta, c));  // matfunc.py:298-299
        const double pold = ps.p_src ? __ldcs(ps.p_src + r) : mul(ps.d0, c);
        const double pn = add(pold, mul(ps.dk, wn));  // matfunc.py:300
        ps.dst[r] = wn;
        __stcs(ps.p_dst + r, pn);
        sw = mul(wn, wn);
        sq = mul(pn, pn);
        if constexpr (P2P) {
            const int64_t o = (int64_t)((k + 1) & 1) * P.npad + P.row_off + r;
            for (int q = 0; q < P.nranks; ++q) P.rank_xg[q][o] = wn;
        }
    }
    sw = warp_sum(sw);
    sq = warp_sum(sq);
    if (lane == 0) {
        s_red[warp][0] = sw;
        s_red[warp][1] = sq;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        // P2P: one system-scope fence per CTA, cumulative over the CTA's peer
        // stores ordered before it by the barrier above
        if constexpr (P2P) __threadfence_system();
        double aw = s_red[0][0], ap = s_red[0][1];
        for (int w = 1; w < W4_WARPS; ++w) {
            aw = add(aw, s_red[w][0]);
            ap = add(ap, s_red[w][1]);
        }
        P.part[(int64_t)blockIdx.x * 2] = aw;
        P.part[(int64_t)blockIdx.x * 2 + 1] = ap;
    }
}

__global__ void __launch_bounds__(256) k_csr_slice_reduce(const SeriesParams *__restrict__ Pp) {
    const SeriesParams &P = *Pp;
    if (P.state->done) return;
    slice_reduce_decide(P, P.state->k + 1);
}

// Peer-memory row-block series: slices into every rank's table, round barrier, decision.
__global__ void __launch_bounds__(256) k_csr_slice_p2p(const SeriesParams *__restrict__ Pp) {
    const SeriesParams &P = *Pp;
    if (P.state->done) {  // ended before this node (round-0 failure): leave the loop
        if (blockIdx.x == 0 && threadIdx.x == 0 && P.cond)
            cudaGraphSetConditional((cudaGraphConditionalHandle)P.cond, 0);
        return;
    }
    slice_p2p_decide(P, P.state->k + 1);
}

// Round 0: v's rows into every rank's gathered vector of parity 1 (read by node 1).
__global__ void __launch_bounds__(256) k_csr_p2p_init(const SeriesParams *__restrict__ Pp) {
    __shared__ int s_last;
    const SeriesParams &P = *Pp;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P.n; i += (int64_t)gridDim.x * blockDim.x) {
        const double x = P.v[i];
        for (int q = 0; q < P.nranks; ++q) P.rank_xg[q][P.npad + P.row_off + i] = x;
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(P.global_cnt, 1u) == gridDim.x - 1u;
    __syncthreads();
    if (!s_last || threadIdx.x != 0) return;
    *P.global_cnt = 0u;
    if (!p2p_round(P, 0)) p2p_fail(P, 0, false);
}

__global__ void k_csr_scale(const double *x, const double *s, double *out, int64_t n) {
    const double a = *s;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = mul(a, x[i]);
}

__global__ void k_csr_init(const SeriesParams p, SeriesParams *dst) {
    if (threadIdx.x == 0) {
        *dst = p;
        SeriesState &st = *p.state;
        st.k = 0;
        st.consecutive = 0;
        st.pass = 0;
        st.done = 0;
        st.converged = 0;
        st.last_term = __longlong_as_double(0x7ff0000000000000ll);
        st.last_pnorm = 0.0;
        *p.global_cnt = 0u;
    }
    for (int i = threadIdx.x; i < p.nchunks; i += blockDim.x) p.chunk_cnt[i] = 0u;
}

// p_out holds p_k for odd k only (pbuf[1] == p_out): copy the even case.
__global__ void k_csr_finalize(const SeriesParams *__restrict__ Pp, int64_t n) {
    const SeriesParams &P = *Pp;
    if ((P.state->k & 1) == 1) return;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        P.pbuf[1][i] = P.pbuf[0][i];
}

int launch_csr_rows(int64_t row_lo, int64_t row_hi, const int64_t *row_ptr, const int32_t *col,
                    const double *vals, const double *x, double *y, double alpha, double beta,
                    int use_beta, cudaStream_t stream) {
    if (row_hi <= row_lo) return ES_OK;
    CsrRowsArgs a{row_lo, row_hi, row_ptr, col, vals, x, y, alpha, beta, use_beta};
    const unsigned grid = (unsigned)((row_hi - row_lo + CSR_T - 1) / CSR_T);
    k_csr_rows<<<grid, CSR_T, 0, stream>>>(a);
    return check_launch("csr rows");
}

// ----- node kernel variants (ES_CSR_VARIANT, for tuning; tools/csr_variants.py)
// C5 (n = 2^22, 5.5e7 nnz) node times on B200: 8 = texture gathers, 12
// CTAs/SM, 4 gathers in flight per lane: 297 us; 6 = the same with LDG
// gathers: 353 us; the pure-gather probe's ceiling is ~262 us.

using CsrNodeFn = void (*)(const SeriesParams *);

struct CsrKernel {
    CsrNodeFn node;
    bool tex;
};

static CsrKernel pick_csr_kernel(int v) {
    switch (v) {
        case 5: return {k_csr_node_w4<1, 8, 4>, true};
        case 6: return {k_csr_node_w4<0, 12, 4>, false};
        case 9: return {k_csr_node_w4<1, 12, 2>, true};
        case 12: return {k_csr_node_w4<1, 8, 8>, true};
        default: return {k_csr_node_w4<1, 12, 4>, true};
    }
}

static int csr_variant() { return env_int("ES_CSR_VARIANT", 8); }

// Texture objects over device vectors, cached per (pointer, length).
static std::mutex g_tex_mu;
static std::map<std::pair<const void *, int64_t>, unsigned long long> g_tex;

static size_t texture_alignment() {
    static size_t a = 0;
    if (!a) {
        int dev = 0, v = 0;
        cudaGetDevice(&dev);
        a = cudaDeviceGetAttribute(&v, cudaDevAttrTextureAlignment, dev) == cudaSuccess && v > 0 ? (size_t)v : 512;
    }
    return a;
}

// nullptr-equivalent 0 when the buffer cannot back a linear texture
// (misaligned, e.g. a torch slice, or longer than the texture limit): the
// caller then runs the LDG-gather variant.
static unsigned long long tex_for(const double *p, int64_t n, bool z = false) {
    if (!p || n <= 0 || ((uintptr_t)p % texture_alignment()) != 0 || n >= (int64_t)1 << 30) return 0;
    std::lock_guard<std::mutex> lk(g_tex_mu);
    auto key = std::make_pair((const void *)p, z ? -n : n);
    auto it = g_tex.find(key);
    if (it != g_tex.end()) return it->second;
    cudaResourceDesc rd = {};
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = const_cast<double *>(p);
    rd.res.linear.desc = z ? cudaCreateChannelDesc<int4>() : cudaCreateChannelDesc<int2>();
    rd.res.linear.sizeInBytes = (size_t)n * sizeof(double) * (z ? 2 : 1);
    cudaTextureDesc td = {};
    td.readMode = cudaReadModeElementType;
    cudaTextureObject_t t = 0;
    if (cudaCreateTextureObject(&t, &rd, &td, nullptr) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    g_tex.emplace(key, (unsigned long long)t);
    return (unsigned long long)t;
}

// 512-byte segments: the w / p buffers must satisfy the texture alignment
static size_t up(size_t x) { return (x + 511) & ~(size_t)511; }

// Workspace: params at offset 0 (like the stencil layout: the device
// SeriesParams pointer of a series is its workspace pointer).
struct CsrLayout {
    size_t params, state, cnt, part, slice, wa, wb, pb, total;
    int nchunks;
};

static CsrLayout csr_layout(int64_t n, int width = 1) {
    CsrLayout L;
    const int64_t rows_per_chunk = (int64_t)W4_T * W4_CHB;  // 16384
    L.nchunks = (int)std::max<int64_t>(1, (n + rows_per_chunk - 1) / rows_per_chunk);
    size_t o = 0;
    L.params = o;
    L.state = o = series_state_offset();  // es_leja_fetch reads the state here
    o = up(o + sizeof(SeriesState));
    L.cnt = o; o = up(o + sizeof(unsigned) * (L.nchunks + 1));
    L.part = o; o = up(o + sizeof(double) * 2 * (size_t)L.nchunks * W4_CHB);
    L.slice = o; o = up(o + sizeof(double) * 2 * (size_t)L.nchunks);
    L.wa = o; o = up(o + sizeof(double) * width * n);
    L.wb = o; o = up(o + sizeof(double) * width * n);
    L.pb = o; o = up(o + sizeof(double) * width * n);
    L.total = o;
    return L;
}

size_t csr_series_ws_bytes(int64_t n) { return csr_layout(n).total; }
size_t csr_z_series_ws_bytes(int64_t n) { return csr_layout(n, 2).total; }

struct CsrSetup {
    SeriesParams hp;
    SeriesParams *dparams;
    CsrKernel kern;
    unsigned grid, nslices;
    int64_t n;
};

// Enqueue one node and its slice reduction.
static void launch_csr_node(const CsrSetup &S, cudaStream_t stream) {
    S.kern.node<<<S.grid, W4_T, 0, stream>>>(S.dparams);
    k_csr_slice_reduce<<<S.nslices, 256, 0, stream>>>(S.dparams);
}

static int csr_prepare(int64_t n, const int64_t *row_ptr, const int32_t *col, const double *vals, const double *xg,
                       int64_t n_xg, const double *v, double *p_out, const double *dd, const double *xi, int ndd, double alpha,
                       double shift, double tol, bool dist, void *ws, size_t ws_bytes, CsrSetup &S) {
    const CsrLayout L = csr_layout(n);
    if (ws_bytes < L.total) return set_error(ES_ERR_ARG, "workspace too small");
    char *w = static_cast<char *>(ws);
    SeriesParams &hp = S.hp;
    hp = SeriesParams{};
    hp.v = v;
    hp.wbuf[1] = reinterpret_cast<double *>(w + L.wa);
    hp.wbuf[0] = reinterpret_cast<double *>(w + L.wb);
    hp.pbuf[1] = p_out;
    hp.pbuf[0] = reinterpret_cast<double *>(w + L.pb);
    hp.dd = dd;
    hp.xi = xi;
    hp.ndd = ndd;
    hp.alpha = alpha;
    hp.shift = shift;
    hp.tol = tol;
    hp.state = reinterpret_cast<SeriesState *>(w + L.state);
    hp.part = reinterpret_cast<double *>(w + L.part);
    hp.slice = reinterpret_cast<double *>(w + L.slice);
    hp.chunk_cnt = reinterpret_cast<unsigned *>(w + L.cnt);
    hp.global_cnt = hp.chunk_cnt + L.nchunks;
    hp.nslices = L.nchunks;
    hp.ntiles = W4_CHB;
    hp.nchunks = L.nchunks;
    hp.chunk_len = 1;
    hp.cond = 0;
    hp.row_ptr = row_ptr;
    hp.col = col;
    hp.vals = vals;
    hp.xg = xg;
    hp.n = n;
    hp.dist = dist ? 1 : 0;
    S.dparams = reinterpret_cast<SeriesParams *>(w + L.params);
    S.nslices = (unsigned)L.nchunks;
    S.n = n;
    S.grid = (unsigned)L.nchunks * W4_CHB;  // padded: every chunk has W4_CHB tiles
    S.kern = pick_csr_kernel(csr_variant());
    if (S.kern.tex) {
        hp.tex[0] = tex_for(hp.wbuf[0], n);
        hp.tex[1] = tex_for(hp.wbuf[1], n);
        hp.tex[2] = tex_for(v, n);
        hp.tex[3] = xg ? tex_for(xg, n_xg) : 0;
        if (!hp.tex[0] || !hp.tex[1] || !hp.tex[2] || (xg && !hp.tex[3]))
            S.kern = pick_csr_kernel(6);  // no texture path for these sizes: LDG gathers
    }
    return ES_OK;
}

int run_csr_series(int64_t n, const int64_t *row_ptr, const int32_t *col, const double *vals,
                   const double *v, double *p_out, const double *dd, const double *xi, int ndd,
                   double alpha, double shift, double tol, void *ws, size_t ws_bytes,
                   es_series_result *res, cudaStream_t stream) {
    if (ndd < 1) return set_error(ES_ERR_ARG, "ndd must be >= 1");
    if (ws_bytes < csr_layout(n).total) return set_error(ES_ERR_ARG, "workspace too small");
    if (ndd == 1 || n == 0) {  // degenerate interval: dd_0 v, 0 matvecs (matfunc.py:285-286)
        if (n > 0) k_csr_scale<<<std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, stream>>>(v, dd, p_out, n);
        launch_state_trivial(ws, stream);
        int rc = check_launch("scale");
        if (rc || !res) return rc;
        return read_series_state(series_state_ptr(ws), res, stream);
    }
    CsrSetup S;
    int rc = csr_prepare(n, row_ptr, col, vals, nullptr, 0, v, p_out, dd, xi, ndd, alpha, shift, tol, false, ws,
                         ws_bytes, S);
    if (rc) return rc;
    GraphKernel gk[2] = {{(const void *)S.kern.node, dim3(S.grid), dim3(W4_T), 0},
                         {(const void *)k_csr_slice_reduce, dim3(S.nslices), dim3(256), 0}};
    unsigned long long handle = 0;
    cudaGraphExec_t ge = series_graph(gk, 2, S.dparams, &handle);
    if (ge) S.hp.cond = handle;
    k_csr_init<<<1, 256, 0, stream>>>(S.hp, S.dparams);
    rc = check_launch("csr init");
    if (rc) return rc;
    if (ge) {
        if (cudaGraphLaunch(ge, stream) != cudaSuccess) return check_launch("csr series graph");
    } else {
        for (int k = 1; k < ndd; ++k) launch_csr_node(S, stream);
        rc = check_launch("csr nodes");
        if (rc) return rc;
    }
    k_csr_finalize<<<148 * 8, 256, 0, stream>>>(S.dparams, n);
    rc = check_launch("csr finalize");
    if (rc) return rc;
    if (!res) return ES_OK;
    return read_series_state(S.hp.state, res, stream);
}

// ----- complex CSR: the propagate path (cli.py:304-357) ------------------------
//
// Vectors are interleaved (re, im) doubles; vals real or interleaved complex.
// Two complex products, each restating the reference bit for bit:
//   cmul_c  -- the compiled core's C99 `double complex` product under
//              -ffp-contract=off (_core.pyx:263-278; real vals promoted to
//              (v, 0)):  (a.r b.r - a.i b.i, a.r b.i + a.i b.r);
//   cmul_np -- numpy's complex128 product in p += dd_k w_k (matfunc.py:300),
//              which on this build is (fma(a.r, b.r, -(a.i b.i)),
//              fma(a.r, b.i, a.i b.r)) (pinned by the oracle tests).

// cmul_c lives in es_common.cuh (shared with csr_generic.cu).
ES_DEV double2 cmul_np(double ar, double ai, double br, double bi) {
    return make_double2(__fma_rn(ar, br, -mul(ai, bi)), __fma_rn(ar, bi, mul(ai, br)));
}

template <int G>
ES_DEV double2 gather_z(const double2 *__restrict__ x, unsigned long long tex, int c) {
    if constexpr (G == 1) {
        const int4 t = tex1Dfetch<int4>((cudaTextureObject_t)tex, c);
        return make_double2(__hiloint2double(t.y, t.x), __hiloint2double(t.w, t.z));
    } else {
        return __ldg(x + c);
    }
}

// acc of row r over this warp's 32-row tile [r0, rend); products staged per warp.
template <int G, int U, bool VC>
ES_DEV double2 csr_warp_sum_z(int64_t r0, int64_t rend, int64_t r, bool act, const int64_t *__restrict__ rp,
                              const int32_t *__restrict__ col, const double *__restrict__ vals,
                              const double2 *__restrict__ xs, unsigned long long tex, double2 *sp) {
    constexpr int ROUND = 32 * U;
    const int lane = threadIdx.x & 31;
    double2 acc = make_double2(0.0, 0.0);
    if (r0 >= rend) return acc;
    const int64_t kb = __ldg(rp + r0), ke = __ldg(rp + rend);
    const int64_t ks = act ? __ldg(rp + r) : 0, kend = act ? __ldg(rp + r + 1) : 0;
    for (int64_t base = kb; base < ke; base += ROUND) {
        const int lim = (int)min((int64_t)ROUND, ke - base);
        int c[U];
        double2 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int j = lane + 32 * u;
            c[u] = j < lim ? __ldcs(col + base + j) : 0;
            if constexpr (VC) {
                v[u] = j < lim ? __ldcs(reinterpret_cast<const double2 *>(vals) + base + j) : make_double2(0.0, 0.0);
            } else {
                v[u] = make_double2(j < lim ? __ldcs(vals + base + j) : 0.0, 0.0);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int j = lane + 32 * u;
            if (j < lim) {
                const double2 x = gather_z<G>(xs, tex, c[u]);
                sp[j] = cmul_c(v[u].x, v[u].y, x.x, x.y);
            }
        }
        __syncwarp();
        const int lo = (int)(max(ks, base) - base), hi = (int)(min(kend, base + lim) - base);
        for (int q = lo; q < hi; ++q) {
            const double2 t = sp[q];
            acc.x = add(acc.x, t.x);
            acc.y = add(acc.y, t.y);
        }
        __syncwarp();
    }
    return acc;
}

constexpr int ZU = 4;  // gathers in flight per lane (complex)

template <int G, bool VC>
__global__ void __launch_bounds__(W4_T, 8) k_csr_node_z(const SeriesParams *__restrict__ Pp) {
    __shared__ double2 s_prod[W4_WARPS][32 * ZU];
    __shared__ double s_red[W4_WARPS][2];
    const SeriesParams &P = *Pp;
    if (P.state->done) return;
    const int k = P.state->k + 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t n = P.n;
    const int64_t r0 = ((int64_t)blockIdx.x * W4_WARPS + warp) * 32;
    const int64_t r = r0 + lane;
    const bool act = r < n;
    const double2 *src = reinterpret_cast<const double2 *>(k == 1 ? P.v : P.wbuf[(k - 1) & 1]);
    const unsigned long long tex = P.tex[k == 1 ? 2 : (k - 1) & 1];
    const double2 acc = csr_warp_sum_z<G, ZU, VC>(r0, min(r0 + 32, n), r, act, P.row_ptr, P.col, P.vals, src, tex,
                                                  s_prod[warp]);
    double sw = 0.0, sq = 0.0;
    if (act) {
        const double2 c = __ldg(src + r);
        const double beta = sub(-P.shift, P.xi[k - 1]);  // matfunc.py:298
        const double2 t1 = cmul_c(P.alpha, P.alpha_im, acc.x, acc.y);
        const double2 t2 = cmul_c(beta, 0.0, c.x, c.y);
        const double2 wn = make_double2(add(t1.x, t2.x), add(t1.y, t2.y));
        const double2 *dd = reinterpret_cast<const double2 *>(P.dd);
        const double2 d0 = dd[0], dk = dd[k];
        const double2 pold = k == 1 ? cmul_np(d0.x, d0.y, c.x, c.y)
                                    : __ldcs(reinterpret_cast<const double2 *>(P.pbuf[(k - 1) & 1]) + r);
        const double2 t3 = cmul_np(dk.x, dk.y, wn.x, wn.y);
        const double2 pn = make_double2(add(pold.x, t3.x), add(pold.y, t3.y));
        reinterpret_cast<double2 *>(P.wbuf[k & 1])[r] = wn;
        __stcs(reinterpret_cast<double2 *>(P.pbuf[k & 1]) + r, pn);
        sw = add(mul(wn.x, wn.x), mul(wn.y, wn.y));
        sq = add(mul(pn.x, pn.x), mul(pn.y, pn.y));
    }
    sw = warp_sum(sw);
    sq = warp_sum(sq);
    if (lane == 0) {
        s_red[warp][0] = sw;
        s_red[warp][1] = sq;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double aw = s_red[0][0], ap = s_red[0][1];
        for (int w = 1; w < W4_WARPS; ++w) {
            aw = add(aw, s_red[w][0]);
            ap = add(ap, s_red[w][1]);
        }
        P.part[(int64_t)blockIdx.x * 2] = aw;
        P.part[(int64_t)blockIdx.x * 2 + 1] = ap;
    }
}

struct CsrRowsZArgs {
    int64_t row_lo, row_hi;
    const int64_t *rp;
    const int32_t *col;
    const double *vals;
    const double2 *x;
    double2 *y;
    double ar, ai, br, bi;
    int use_beta;
};

template <bool VC>
__global__ void __launch_bounds__(W4_T) k_csr_rows_z(const CsrRowsZArgs a) {
    __shared__ double2 s_prod[W4_WARPS][32 * ZU];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t r0 = a.row_lo + ((int64_t)blockIdx.x * W4_WARPS + warp) * 32;
    const int64_t rend = min(r0 + 32, a.row_hi);
    const int64_t r = r0 + lane;
    const bool act = r < rend;
    const double2 acc = csr_warp_sum_z<0, ZU, VC>(r0, rend, r, act, a.rp, a.col, a.vals, a.x, 0, s_prod[warp]);
    if (!act) return;
    double2 y = cmul_c(a.ar, a.ai, acc.x, acc.y);  // _core.pyx:257-260
    if (a.use_beta) {
        const double2 xr = __ldg(a.x + r);
        const double2 t = cmul_c(a.br, a.bi, xr.x, xr.y);
        y = make_double2(add(y.x, t.x), add(y.y, t.y));
    }
    a.y[r] = y;
}

__global__ void k_scale_z(const double2 *x, const double2 *s, double2 *out, int64_t n) {
    const double2 a = *s;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = cmul_np(a.x, a.y, x[i].x, x[i].y);
}

int launch_csr_rows_z(int64_t row_lo, int64_t row_hi, const int64_t *row_ptr, const int32_t *col, const double *vals,
                      int vals_complex, const double *x, double *y, double ar, double ai, double br, double bi,
                      int use_beta, cudaStream_t stream) {
    if (row_hi <= row_lo) return ES_OK;
    CsrRowsZArgs a{row_lo, row_hi, row_ptr, col, vals, reinterpret_cast<const double2 *>(x),
                   reinterpret_cast<double2 *>(y), ar, ai, br, bi, use_beta};
    const unsigned grid = (unsigned)((row_hi - row_lo + W4_T - 1) / W4_T);
    if (vals_complex) k_csr_rows_z<true><<<grid, W4_T, 0, stream>>>(a);
    else k_csr_rows_z<false><<<grid, W4_T, 0, stream>>>(a);
    return check_launch("csr rows (complex)");
}

int run_csr_series_z(int64_t n, const int64_t *row_ptr, const int32_t *col, const double *vals, int vals_complex,
                     const double *v, double *p_out, const double *dd, const double *ddabs, const double *xi, int ndd,
                     double alpha_re, double alpha_im, double shift, double tol, void *ws, size_t ws_bytes,
                     es_series_result *res, cudaStream_t stream) {
    if (ndd < 1) return set_error(ES_ERR_ARG, "ndd must be >= 1");
    const CsrLayout L = csr_layout(n, 2);
    if (ws_bytes < L.total) return set_error(ES_ERR_ARG, "workspace too small");
    if (ndd == 1 || n == 0) {  // degenerate interval: dd_0 v, 0 matvecs (matfunc.py:285-286)
        if (n > 0)
            k_scale_z<<<std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, stream>>>(
                reinterpret_cast<const double2 *>(v), reinterpret_cast<const double2 *>(dd),
                reinterpret_cast<double2 *>(p_out), n);
        launch_state_trivial(ws, stream);
        int rc = check_launch("scale (complex)");
        if (rc || !res) return rc;
        return read_series_state(series_state_ptr(ws), res, stream);
    }
    char *w = static_cast<char *>(ws);
    SeriesParams hp = {};
    hp.v = v;
    hp.wbuf[1] = reinterpret_cast<double *>(w + L.wa);
    hp.wbuf[0] = reinterpret_cast<double *>(w + L.wb);
    hp.pbuf[1] = p_out;
    hp.pbuf[0] = reinterpret_cast<double *>(w + L.pb);
    hp.dd = dd;
    hp.ddabs = ddabs;
    hp.xi = xi;
    hp.ndd = ndd;
    hp.alpha = alpha_re;
    hp.alpha_im = alpha_im;
    hp.shift = shift;
    hp.tol = tol;
    hp.state = reinterpret_cast<SeriesState *>(w + L.state);
    hp.part = reinterpret_cast<double *>(w + L.part);
    hp.slice = reinterpret_cast<double *>(w + L.slice);
    hp.chunk_cnt = reinterpret_cast<unsigned *>(w + L.cnt);
    hp.global_cnt = hp.chunk_cnt + L.nchunks;
    hp.nslices = L.nchunks;
    hp.ntiles = W4_CHB;
    hp.nchunks = L.nchunks;
    hp.chunk_len = 1;
    hp.row_ptr = row_ptr;
    hp.col = col;
    hp.vals = vals;
    hp.vals_complex = vals_complex;
    hp.n = n;
    SeriesParams *dparams = reinterpret_cast<SeriesParams *>(w + L.params);
    const unsigned grid = (unsigned)L.nchunks * W4_CHB;
    hp.tex[0] = tex_for(hp.wbuf[0], n, true);
    hp.tex[1] = tex_for(hp.wbuf[1], n, true);
    hp.tex[2] = tex_for(v, n, true);
    const bool tex = hp.tex[0] && hp.tex[1] && hp.tex[2];
    CsrNodeFn nf = vals_complex ? (tex ? k_csr_node_z<1, true> : k_csr_node_z<0, true>)
                                : (tex ? k_csr_node_z<1, false> : k_csr_node_z<0, false>);
    GraphKernel gk[2] = {{(const void *)nf, dim3(grid), dim3(W4_T), 0},
                         {(const void *)k_csr_slice_reduce, dim3((unsigned)L.nchunks), dim3(256), 0}};
    unsigned long long handle = 0;
    cudaGraphExec_t ge = series_graph(gk, 2, dparams, &handle);
    if (ge) hp.cond = handle;
    k_csr_init<<<1, 256, 0, stream>>>(hp, dparams);
    int rc = check_launch("csr init (complex)");
    if (rc) return rc;
    if (ge) {
        if (cudaGraphLaunch(ge, stream) != cudaSuccess) return check_launch("complex csr series graph");
    } else {
        for (int k = 1; k < ndd; ++k) {
            nf<<<grid, W4_T, 0, stream>>>(dparams);
            k_csr_slice_reduce<<<(unsigned)L.nchunks, 256, 0, stream>>>(dparams);
        }
        rc = check_launch("complex csr nodes");
        if (rc) return rc;
    }
    k_csr_finalize<<<148 * 8, 256, 0, stream>>>(dparams, 2 * n);
    rc = check_launch("csr finalize (complex)");
    if (rc) return rc;
    if (!res) return ES_OK;
    return read_series_state(hp.state, res, stream);
}

// ----- peer-memory (NVLink P2P) row-block series -------------------------------
//
// One CUDA graph per series and rank: node k gathers from this rank's parity
// buffer and stores each of its rows' w_k into every rank's gathered vector
// (the all-gather of decomp.py:304-333, fused into the node); the slice
// kernel writes the per-chunk sums into every rank's table, joins the round
// barrier and decides identically on every rank.

int run_csr_p2p_series(int64_t n, const int64_t *row_ptr, const int32_t *col, const double *vals,
                       const es_p2p_rows_desc *x, const double *v, double *p_out, const double *dd, const double *xi,
                       int ndd, double alpha, double shift, double tol, void *ws, size_t ws_bytes,
                       cudaStream_t stream) {
    if (ndd < 2) return set_error(ES_ERR_ARG, "a peer-memory series needs ndd >= 2");
    if (x->nranks < 1 || x->rank < 0 || x->rank >= x->nranks || !x->rank_xg || !x->rank_slices ||
        !x->rank_arrive || !x->arrive_local || !x->xg_local[0] || !x->xg_local[1])
        return set_error(ES_ERR_ARG, "bad peer-memory row descriptor");
    if (x->row_offset < 0 || x->row_offset + n > x->npad) return set_error(ES_ERR_ARG, "row block outside npad");
    CsrSetup S;
    int rc = csr_prepare(n, row_ptr, col, vals, nullptr, 0, v, p_out, dd, xi, ndd, alpha, shift, tol, false, ws,
                         ws_bytes, S);
    if (rc) return rc;
    SeriesParams &hp = S.hp;
    if (x->slice_offset < 0 || x->slice_offset + hp.nslices > x->total_slices)
        return set_error(ES_ERR_ARG, "slice offset / total do not cover this block's %d slices", hp.nslices);
    hp.p2p = 1;
    hp.nranks = x->nranks;
    hp.rank = x->rank;
    hp.slice_off = x->slice_offset;
    hp.total_slices = x->total_slices;
    hp.rank_slices = x->rank_slices;
    hp.rank_arrive = x->rank_arrive;
    hp.arrive_local = x->arrive_local;
    hp.base = x->base;
    hp.timeout_ns = x->timeout_ns > 0 ? x->timeout_ns : 10000000000ll;
    hp.xgp[0] = x->xg_local[0];
    hp.xgp[1] = x->xg_local[1];
    hp.rank_xg = x->rank_xg;
    hp.row_off = x->row_offset;
    hp.npad = x->npad;
    hp.tex[0] = tex_for(hp.xgp[0], x->npad);
    hp.tex[1] = tex_for(hp.xgp[1], x->npad);
    const CsrNodeFn nf = (hp.tex[0] && hp.tex[1]) ? k_csr_node_w4<1, 12, 4, true> : k_csr_node_w4<0, 12, 4, true>;
    GraphKernel gk[2] = {{(const void *)nf, dim3(S.grid), dim3(W4_T), 0},
                         {(const void *)k_csr_slice_p2p, dim3(S.nslices), dim3(256), 0}};
    unsigned long long handle = 0;
    cudaGraphExec_t ge = series_graph(gk, 2, S.dparams, &handle);
    if (ge) hp.cond = handle;
    k_csr_init<<<1, 256, 0, stream>>>(hp, S.dparams);
    k_csr_p2p_init<<<(unsigned)std::min<int64_t>(std::max<int64_t>(1, (n + 255) / 256), 148 * 4), 256, 0, stream>>>(
        S.dparams);
    rc = check_launch("peer-memory csr init");
    if (rc) return rc;
    if (ge) {
        if (cudaGraphLaunch(ge, stream) != cudaSuccess) return check_launch("peer-memory csr graph");
    } else {
        for (int k = 1; k < ndd; ++k) {
            nf<<<S.grid, W4_T, 0, stream>>>(S.dparams);
            k_csr_slice_p2p<<<S.nslices, 256, 0, stream>>>(S.dparams);
        }
    }
    k_csr_finalize<<<148 * 8, 256, 0, stream>>>(S.dparams, n);
    return check_launch("peer-memory csr series");
}

int csr_nslices(int64_t n) { return csr_layout(n).nchunks; }

// ----- multi-GPU row-block series (decomp.py:285-345 on one rank per GPU) ----
//
// Per node k the caller all-gathers *csr_dist_source(k) of every rank into
// xg (rank order = global row order), calls csr_dist_node (the local rows'
// pass with gathers from xg, per-chunk slices out), gathers the slices of all
// ranks and calls es_leja_dist_decide.

static std::mutex g_csr_dist_mu;
static std::map<const void *, CsrSetup> g_csr_dist;

int csr_dist_begin(int64_t n_local, const int64_t *row_ptr, const int32_t *col, const double *vals, const double *xg,
                   int64_t n_xg, const double *v, double *p_out, const double *dd, const double *xi, int ndd, double alpha,
                   double shift, double tol, void *ws, size_t ws_bytes, cudaStream_t stream) {
    if (ndd < 2) return set_error(ES_ERR_ARG, "a row-block series needs ndd >= 2");
    if (!xg) return set_error(ES_ERR_ARG, "a row-block series needs the gathered-vector buffer xg");
    CsrSetup S;
    int rc = csr_prepare(n_local, row_ptr, col, vals, xg, n_xg, v, p_out, dd, xi, ndd, alpha, shift, tol, true, ws,
                         ws_bytes, S);
    if (rc) return rc;
    k_csr_init<<<1, 256, 0, stream>>>(S.hp, S.dparams);
    rc = check_launch("csr dist init");
    if (rc) return rc;
    std::lock_guard<std::mutex> lk(g_csr_dist_mu);
    g_csr_dist[ws] = S;
    return ES_OK;
}

static int csr_dist_get(const void *ws, CsrSetup *&S) {
    std::lock_guard<std::mutex> lk(g_csr_dist_mu);
    auto it = g_csr_dist.find(ws);
    if (it == g_csr_dist.end()) return set_error(ES_ERR_ARG, "no row-block series begun on this workspace");
    S = &it->second;
    return ES_OK;
}

int csr_dist_source(const void *ws, int k, const double **src) {
    CsrSetup *S;
    int rc = csr_dist_get(ws, S);
    if (rc) return rc;
    *src = k <= 1 ? S->hp.v : S->hp.wbuf[(k - 1) & 1];
    return ES_OK;
}

int csr_dist_nslices(const void *ws, int *nslices) {
    CsrSetup *S;
    int rc = csr_dist_get(ws, S);
    if (rc) return rc;
    *nslices = S->hp.nslices;
    return ES_OK;
}

int csr_dist_node(const void *ws, double *slices_out, cudaStream_t stream) {
    CsrSetup *S;
    int rc = csr_dist_get(ws, S);
    if (rc) return rc;
    if (S->n > 0) launch_csr_node(*S, stream);
    else cudaMemsetAsync(S->hp.slice, 0, sizeof(double) * 2 * S->hp.nslices, stream);
    cudaMemcpyAsync(slices_out, S->hp.slice, sizeof(double) * 2 * S->hp.nslices, cudaMemcpyDeviceToDevice, stream);
    return check_launch("csr dist node");
}

int csr_dist_end(const void *ws, cudaStream_t stream) {
    CsrSetup *S;
    int rc = csr_dist_get(ws, S);
    if (rc) return rc;
    if (S->n > 0) k_csr_finalize<<<148 * 8, 256, 0, stream>>>(S->dparams, S->n);
    rc = check_launch("csr dist finalize");
    std::lock_guard<std::mutex> lk(g_csr_dist_mu);
    g_csr_dist.erase(ws);
    return rc;
}

}  // namespace es
