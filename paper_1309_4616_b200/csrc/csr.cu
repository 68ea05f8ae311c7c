// CSR fused SpMV and the fused Newton-Leja node for unstructured operators.
//
// Row sums are accumulated strictly in storage order, one thread per row,
// exactly like the reference's compiled core (_core.pyx:245-260), so results
// are bitwise identical.  To keep HBM access coalesced anyway, each warp
// stages the products vals[k] * x[col[k]] of its 32 rows' contiguous nnz
// range into shared memory with lane-strided (coalesced) loads, and every
// thread then adds its own row's products in order from shared memory.
#include <algorithm>

#include "es_host.h"
#include "series.cuh"

namespace es {

constexpr int CSR_WARPS = 8;    // warps per CTA; a CTA owns 256 rows
constexpr int CSR_STAGE = 256;  // products staged per warp per round
constexpr int CSR_CHB = 64;     // CTAs per reduction chunk (16384 rows)

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

// sum_k vals[k] x[col[k]] over the row `r` owned by this lane.
ES_DEV double csr_row_sum(int64_t r0, int64_t rend, int64_t r, bool act, const int64_t *rp,
                          const int32_t *col, const double *vals, const double *x, double *s_prod) {
    const int lane = threadIdx.x & 31;
    double acc = 0.0;
    if (r0 >= rend) return acc;
    const int64_t kb = __ldg(rp + r0), ke = __ldg(rp + rend);
    const int64_t ks = act ? __ldg(rp + r) : 0, kend = act ? __ldg(rp + r + 1) : 0;
    for (int64_t base = kb; base < ke; base += CSR_STAGE) {
        const int lim = (int)min((int64_t)CSR_STAGE, ke - base);
        for (int j = lane; j < lim; j += 32) s_prod[j] = mul(__ldg(vals + base + j), __ldg(x + __ldg(col + base + j)));
        __syncwarp();
        const int64_t lo = max(ks, base), hi = min(kend, base + lim);
        for (int64_t k = lo; k < hi; ++k) acc = add(acc, s_prod[k - base]);
        __syncwarp();
    }
    return acc;
}

__global__ void __launch_bounds__(32 * CSR_WARPS) k_csr_rows(const CsrRowsArgs a) {
    __shared__ double s_prod[CSR_WARPS][CSR_STAGE];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t r0 = a.row_lo + ((int64_t)blockIdx.x * CSR_WARPS + warp) * 32;
    const int64_t rend = min(r0 + 32, a.row_hi);
    const int64_t r = r0 + lane;
    const bool act = r < rend;
    const double acc = csr_row_sum(r0, rend, r, act, a.rp, a.col, a.vals, a.x, s_prod[warp]);
    if (act) a.y[r] = a.use_beta ? add(mul(a.alpha, acc), mul(a.beta, __ldg(a.x + r))) : mul(a.alpha, acc);
}

// One Newton-Leja node: w_k = alpha A w_{k-1} + beta_k w_{k-1}, p_k, norms.
// Slices are chunks of CSR_CHB CTAs (16384 rows), tiles are the CTAs inside.
__global__ void __launch_bounds__(32 * CSR_WARPS) k_csr_node(const SeriesParams *__restrict__ Pp) {
    __shared__ double s_prod[CSR_WARPS][CSR_STAGE];
    __shared__ double s_red[CSR_WARPS][2];
    const SeriesParams &P = *Pp;
    if (P.state->done) return;
    const int k = P.state->k + 1;
    const Pass ps = node_pass(P, k);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t r0 = ((int64_t)blockIdx.x * CSR_WARPS + warp) * 32;
    const int64_t rend = min(r0 + 32, P.n);
    const int64_t r = r0 + lane;
    const bool act = r < rend;
    const double acc = csr_row_sum(r0, rend, r, act, P.row_ptr, P.col, P.vals, ps.src, s_prod[warp]);
    double sw = 0.0, sp = 0.0;
    if (act) {
        const double c = __ldg(ps.src + r);
        const double wn = add(mul(ps.alpha, acc), mul(ps.beta, c));
        const double pold = ps.p_src ? __ldg(ps.p_src + r) : mul(ps.d0, c);
        const double pn = add(pold, mul(ps.dk, wn));
        ps.dst[r] = wn;
        ps.p_dst[r] = pn;
        sw = mul(wn, wn);
        sp = mul(pn, pn);
    }
    sw = warp_sum(sw);
    sp = warp_sum(sp);
    if (lane == 0) {
        s_red[warp][0] = sw;
        s_red[warp][1] = sp;
    }
    __syncthreads();
    const int chunk = blockIdx.x / CSR_CHB, tile = blockIdx.x % CSR_CHB;
    if (threadIdx.x == 0) {
        double aw = s_red[0][0], ap = s_red[0][1];
        for (int w = 1; w < CSR_WARPS; ++w) {
            aw = add(aw, s_red[w][0]);
            ap = add(ap, s_red[w][1]);
        }
        double *dst = P.part + ((int64_t)chunk * CSR_CHB + tile) * 2;
        dst[0] = aw;
        dst[1] = ap;
    }
    reduce_and_decide(P, k, chunk, chunk, chunk + 1);
}

__global__ void k_csr_init(const SeriesParams p, SeriesParams *dst);
__global__ void k_csr_finalize(const SeriesParams *__restrict__ Pp, int64_t n);
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
        st.done = 0;
        st.converged = 0;
        st.last_term = __longlong_as_double(0x7ff0000000000000ll);
        st.last_pnorm = 0.0;
        *p.global_cnt = 0u;
    }
    for (int i = threadIdx.x; i < p.nchunks; i += blockDim.x) p.chunk_cnt[i] = 0u;
}

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
    const int64_t rows_per_cta = 32 * CSR_WARPS;
    const unsigned grid = (unsigned)((row_hi - row_lo + rows_per_cta - 1) / rows_per_cta);
    k_csr_rows<<<grid, 32 * CSR_WARPS, 0, stream>>>(a);
    return check_launch("csr rows");
}

static size_t up(size_t x) { return (x + 255) & ~(size_t)255; }

struct CsrLayout {
    size_t params, state, cnt, part, slice, wa, wb, pb, total;
    int nchunks;
};

static CsrLayout csr_layout(int64_t n) {
    CsrLayout L;
    const int64_t rows_per_chunk = 32LL * CSR_WARPS * CSR_CHB;
    L.nchunks = (int)std::max<int64_t>(1, (n + rows_per_chunk - 1) / rows_per_chunk);
    size_t o = 0;
    L.params = o; o = up(o + sizeof(SeriesParams));
    L.state = o; o = up(o + sizeof(SeriesState));
    L.cnt = o; o = up(o + sizeof(unsigned) * (L.nchunks + 1));
    L.part = o; o = up(o + sizeof(double) * 2 * (size_t)L.nchunks * CSR_CHB);
    L.slice = o; o = up(o + sizeof(double) * 2 * (size_t)L.nchunks);
    L.wa = o; o = up(o + sizeof(double) * n);
    L.wb = o; o = up(o + sizeof(double) * n);
    L.pb = o; o = up(o + sizeof(double) * n);
    L.total = o;
    return L;
}

size_t csr_series_ws_bytes(int64_t n) { return csr_layout(n).total; }

int run_csr_series(int64_t n, const int64_t *row_ptr, const int32_t *col, const double *vals,
                   const double *v, double *p_out, const double *dd, const double *xi, int ndd,
                   double alpha, double shift, double tol, void *ws, size_t ws_bytes,
                   es_series_result *res, cudaStream_t stream) {
    if (ndd < 1) return set_error(ES_ERR_ARG, "ndd must be >= 1");
    const CsrLayout L = csr_layout(n);
    if (ws_bytes < L.total) return set_error(ES_ERR_ARG, "workspace too small");
    if (ndd == 1 || n == 0) {
        if (n > 0) k_csr_scale<<<std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, stream>>>(v, dd, p_out, n);
        launch_state_trivial(ws, stream);
        int rc = check_launch("scale");
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
    hp.ntiles = CSR_CHB;
    hp.nchunks = L.nchunks;
    hp.chunk_len = 1;
    hp.cond = 0;
    hp.row_ptr = row_ptr;
    hp.col = col;
    hp.vals = vals;
    hp.n = n;
    SeriesParams *dparams = reinterpret_cast<SeriesParams *>(w + L.params);
    k_csr_init<<<1, 256, 0, stream>>>(hp, dparams);
    int rc = check_launch("csr init");
    if (rc) return rc;
    const unsigned grid = (unsigned)L.nchunks * CSR_CHB;  // padded: every chunk has CSR_CHB CTAs
    for (int k = 1; k < ndd; ++k) k_csr_node<<<grid, 32 * CSR_WARPS, 0, stream>>>(dparams);
    rc = check_launch("csr nodes");
    if (rc) return rc;
    k_csr_finalize<<<148 * 8, 256, 0, stream>>>(dparams, n);
    rc = check_launch("csr finalize");
    if (rc) return rc;
    if (!res) return ES_OK;
    return read_series_state(hp.state, res, stream);
}

}  // namespace es
