// Stencil pass kernels, the fused Newton-Leja series driver (CUDA graph with
// a device-side while loop), and their host launchers.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>

#include "es_host.h"
#include "series.cuh"
#include "stencil_tma.cuh"
#include "stencil_tb2d.cuh"
#include "stencil_tb2r.cuh"
#include "stencil_tb2m.cuh"
#include "stencil_tb3m.cuh"
#include "stencil_tb.cuh"

#include <cudaTypedefs.h>

namespace es {

// ---------------------------------------------------------------------------
// kernels

struct ApplyArgs {
    Geom g;
    Pass ps;
    const double *gdiag;
    int chunk_len;
};

template <int VEC, int COEFF, bool GD>
__global__ void __launch_bounds__(32 * BY3) k_apply3d(const ApplyArgs a) {
    extern __shared__ double smem[];
    pass3d<VEC, COEFF, GD, false>(a.g, a.ps, a.gdiag, a.chunk_len, smem, smem + 2 * Smem3<VEC>::TILE);
}

template <int VEC, int COEFF, bool GD>
__global__ void __launch_bounds__(32 * BW2) k_apply2d(const ApplyArgs a) {
    extern __shared__ double smem[];
    pass2d<VEC, COEFF, GD, false>(a.g, a.ps, a.gdiag, a.chunk_len, smem);
}

// One Newton-Leja node on a 3D slab.
template <int VEC, int COEFF, bool GD>
__global__ void __launch_bounds__(32 * BY3) k_node3d(const SeriesParams *__restrict__ Pp) {
    extern __shared__ double smem[];
    const SeriesParams &P = *Pp;
    if (P.state->done) return;
    const int k = P.state->k + 1;
    const Pass ps = node_pass(P, k);
    double *s_red = smem + 2 * Smem3<VEC>::TILE;
    pass3d<VEC, COEFF, GD, true>(P.g, ps, P.gdiag, P.chunk_len, smem, s_red);
    // per-(plane, tile) partials: warps summed in index order
    __syncthreads();
    const int64_t zb = (int64_t)blockIdx.z * P.chunk_len;
    const int64_t ze = min(P.g.lz, zb + P.chunk_len);
    const int tile = blockIdx.y * gridDim.x + blockIdx.x;
    const int tid = threadIdx.y * 32 + threadIdx.x;
    for (int64_t zl = tid; zl < ze - zb; zl += 32 * BY3) {
        double aw = s_red[(zl * BY3) * 2], ap = s_red[(zl * BY3) * 2 + 1];
        for (int w = 1; w < BY3; ++w) {
            aw = add(aw, s_red[(zl * BY3 + w) * 2]);
            ap = add(ap, s_red[(zl * BY3 + w) * 2 + 1]);
        }
        double *dst = P.part + ((zb + zl) * P.ntiles + tile) * 2;
        dst[0] = aw;
        dst[1] = ap;
    }
    reduce_and_decide(P, k, blockIdx.z, zb, ze);
}

// One Newton-Leja node on a single-plane (2D) grid.
template <int VEC, int COEFF, bool GD>
__global__ void __launch_bounds__(32 * BW2) k_node2d(const SeriesParams *__restrict__ Pp) {
    extern __shared__ double smem[];
    const SeriesParams &P = *Pp;
    if (P.state->done) return;
    const int k = P.state->k + 1;
    const Pass ps = node_pass(P, k);
    pass2d<VEC, COEFF, GD, true>(P.g, ps, P.gdiag, P.chunk_len, smem);
    __syncthreads();
    const int64_t yb = (int64_t)blockIdx.y * P.chunk_len;
    const int64_t ye = min(P.g.ny, yb + P.chunk_len);
    const int tile = blockIdx.x;
    const int tid = threadIdx.y * 32 + threadIdx.x;
    for (int64_t yl = tid; yl < ye - yb; yl += 32 * BW2) {
        double aw = smem[(yl * BW2) * 2], ap = smem[(yl * BW2) * 2 + 1];
        for (int w = 1; w < BW2; ++w) {
            aw = add(aw, smem[(yl * BW2 + w) * 2]);
            ap = add(ap, smem[(yl * BW2 + w) * 2 + 1]);
        }
        double *dst = P.part + ((yb + yl) * P.ntiles + tile) * 2;
        dst[0] = aw;
        dst[1] = ap;
    }
    reduce_and_decide(P, k, blockIdx.y, yb, ye);
}

// ---------------------------------------------------------------------------
// TMA-pipelined kernels (v2)

struct ApplyArgsT {
    Geom g;
    Pass ps;
    int chunk_len;
    TmaMaps maps;  // MAP_WA_V / MAP_WB_V describe the source vector
};

template <bool DIM3, int COEFF>
__global__ void __launch_bounds__(TMA_THREADS, 3) k_apply_tma(const __grid_constant__ ApplyArgsT a) {
    extern __shared__ __align__(128) char tsmem[];
    const PassMaps mp{&a.maps.m[MAP_WA_V], &a.maps.m[MAP_WB_V], nullptr, nullptr, &a.maps.m[MAP_HLO], &a.maps.m[MAP_HHI]};
    tma_pass<DIM3, COEFF, false, false>(a.g, a.ps, mp, a.chunk_len, false, tsmem, nullptr, 0, nullptr);
}

// Fused Rosenbrock prologue: F = g(u) - A u, g'(u), min/max g', first u <= 0.
template <bool DIM3, int COEFF>
__global__ void __launch_bounds__(TMA_THREADS, 3) k_rospro_tma(const __grid_constant__ ApplyArgsT a) {
    extern __shared__ __align__(128) char tsmem[];
    const PassMaps mp{&a.maps.m[MAP_WA_V], &a.maps.m[MAP_WB_V], nullptr, nullptr, &a.maps.m[MAP_HLO], &a.maps.m[MAP_HHI]};
    tma_pass<DIM3, COEFF, false, false, EPI_ROSPRO>(a.g, a.ps, mp, a.chunk_len, false, tsmem, nullptr, 0, nullptr);
}

__global__ void k_aux_init(unsigned long long *aux, unsigned long long n) {
    if (threadIdx.x == 0) {
        aux[0] = ~0ull;
        aux[1] = 0ull;
        aux[2] = n;
    }
}

// One Newton-Leja node, persistent CTAs over (chunk, tile) items.
template <bool DIM3, int COEFF, bool GD>
__global__ void __launch_bounds__(TMA_THREADS, (COEFF == ES_COEFF_RADIAL && !DIM3) ? 2 : 3) k_node_tma(const SeriesParams *__restrict__ Pp) {
    extern __shared__ __align__(128) char tsmem[];
    const SeriesParams &P = *Pp;
    if (P.state->done) return;
    const int k = P.state->k + 1;
    const Pass ps = node_pass(P, k);
    const TmaMaps &M = *static_cast<const TmaMaps *>(P.maps);
    const int wi = k == 1 ? 0 : 1 + ((k - 1) & 1);
    const bool odd = P.p2p && (k & 1);  // peer-memory series: node k reads halo parity k & 1
    const PassMaps mp{&M.m[2 * wi], &M.m[2 * wi + 1], &M.m[MAP_P_0 + ((k - 1) & 1)], &M.m[MAP_G],
                      &M.m[odd ? MAP_HLO_1 : MAP_HLO], &M.m[odd ? MAP_HHI_1 : MAP_HHI]};
    // the second PG slot carries g' (GD) or the staged coefficient (MAP_G encodes it)
    tma_pass<DIM3, COEFF, GD || COEFF == ES_COEFF_STAGED, true>(P.g, ps, mp, P.chunk_len, true, tsmem, Pp, k, P.work);
}

// Reduction + stopping decision of a TMA node (one CTA per z / row chunk).
__global__ void __launch_bounds__(256) k_slice_reduce(const SeriesParams *__restrict__ Pp) {
    const SeriesParams &P = *Pp;
    if (P.state->done) return;
    if (blockIdx.x == 0 && threadIdx.x == 0 && P.work) *P.work = 0u;  // every node CTA has finished claiming
    slice_reduce_decide(P, P.state->k + 1);
}

// Peer-memory series: slice reduction + round barrier + shared decision.
// Peer-memory series, after node k: every CTA first pushes its share of the
// slab's first / last plane of w_k into the neighbours' halo buffers of
// parity (k + 1) & 1 (NVLink stores, 16 B per thread), then reduces its
// slice and joins the round.  (Storing the planes from the node kernel's
// epilogue instead overlaps the transfer with the sweep, but costs the hot
// kernel registers: 974 vs 897 us per 512^3 node even without peers.)
__global__ void __launch_bounds__(256) k_slice_p2p(const SeriesParams *__restrict__ Pp) {
    const SeriesParams &P = *Pp;
    if (P.state->done) {  // the series ended before this node (round-0 failure): leave the loop
        if (blockIdx.x == 0 && threadIdx.x == 0 && P.cond)
            cudaGraphSetConditional((cudaGraphConditionalHandle)P.cond, 0);
        return;
    }
    const int k = P.state->k + 1;
    if (blockIdx.x == 0 && threadIdx.x == 0 && P.work) *P.work = 0u;
    const int par = (k + 1) & 1;
    const double2 *w = reinterpret_cast<const double2 *>(P.wbuf[k & 1]);
    double2 *lo = reinterpret_cast<double2 *>(P.peer_lo[par]), *hi = reinterpret_cast<double2 *>(P.peer_hi[par]);
    const int64_t half = P.g.nx * P.g.ny / 2, lz = P.g.lz;
    if (lo || hi) {
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < half; i += (int64_t)gridDim.x * blockDim.x) {
            if (lo) lo[i] = __ldcg(w + i);
            if (hi) hi[i] = __ldcg(w + (lz - 1) * half + i);
        }
        __threadfence_system();
        __syncthreads();
    }
    slice_p2p_decide(P, k);
}

// Peer-memory series, round 0: v's first / last plane into the neighbours'
// halo buffers of parity 1 (read by node 1), then the round barrier.
__global__ void __launch_bounds__(256) k_p2p_init(const SeriesParams *__restrict__ Pp, int64_t plane, int64_t lz) {
    __shared__ int s_last;
    const SeriesParams &P = *Pp;
    const int64_t half = plane / 2;  // plane = nx * ny, nx even on the TMA path: double2 copies
    const double2 *v = reinterpret_cast<const double2 *>(P.v);
    double2 *lo = reinterpret_cast<double2 *>(P.peer_lo[1]), *hi = reinterpret_cast<double2 *>(P.peer_hi[1]);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < half; i += (int64_t)gridDim.x * blockDim.x) {
        if (lo) lo[i] = v[i];
        if (hi) hi[i] = v[(lz - 1) * half + i];
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(P.global_cnt, 1u) == gridDim.x - 1u;
    __syncthreads();
    if (!s_last || threadIdx.x != 0) return;
    *P.global_cnt = 0u;
    if (!p2p_round(P, 0)) p2p_fail(P, 0, false);
}

// Peer-memory two-node pass: push the first / last TWO planes of w_{k+1} into
// the neighbours' halo buffers of the next pass's parity, then the two-node
// slice reduction, round barrier and decisions.
__global__ void __launch_bounds__(256) k_slice_p2p2(const SeriesParams *__restrict__ Pp) {
    const SeriesParams &P = *Pp;
    if (P.state->done) {
        if (blockIdx.x == 0 && threadIdx.x == 0 && P.cond)
            cudaGraphSetConditional((cudaGraphConditionalHandle)P.cond, 0);
        return;
    }
    const int k = P.state->k + 1;
    const int pass = P.state->pass, par = (pass + 1) & 1;
    if (blockIdx.x == 0 && threadIdx.x == 0 && P.work) *P.work = 0u;
    const double2 *w = reinterpret_cast<const double2 *>(P.wbuf[pass & 1]);  // w_{k+1} (w_k: one-node pass)
    // pushed by the pass itself (peer_in_node, x2): nothing to copy here
    double2 *lo = P.peer_in_node ? nullptr : reinterpret_cast<double2 *>(P.peer_lo[par]);
    double2 *hi = P.peer_in_node ? nullptr : reinterpret_cast<double2 *>(P.peer_hi[par]);
    const int64_t two_planes = P.g.nx * P.g.ny, lz = P.g.lz;  // two planes = nx ny double2
    if (lo || hi) {
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < two_planes;
             i += (int64_t)gridDim.x * blockDim.x) {
            if (lo) lo[i] = __ldcg(w + i);                              // planes 0, 1 -> its L, L+1
            if (hi) hi[i] = __ldcg(w + (lz - 2) * (two_planes / 2) + i);  // planes L-2, L-1 -> its -2, -1
        }
        __threadfence_system();
        __syncthreads();
    }
    slice_p2p_decide2(P, k);
}

// Round 0 of a peer-memory two-node series: v's two boundary planes on each
// side into the neighbours' halo buffers of parity 0 (read by pass 0).
__global__ void __launch_bounds__(256) k_p2p_init2(const SeriesParams *__restrict__ Pp, int64_t plane, int64_t lz) {
    __shared__ int s_last;
    const SeriesParams &P = *Pp;
    const double2 *v = reinterpret_cast<const double2 *>(P.v);
    double2 *lo = reinterpret_cast<double2 *>(P.peer_lo[0]), *hi = reinterpret_cast<double2 *>(P.peer_hi[0]);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < plane; i += (int64_t)gridDim.x * blockDim.x) {
        if (lo) lo[i] = v[i];
        if (hi) hi[i] = v[(lz - 2) * (plane / 2) + i];
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(P.global_cnt, 1u) == gridDim.x - 1u;
    __syncthreads();
    if (!s_last || threadIdx.x != 0) return;
    *P.global_cnt = 0u;
    if (!p2p_round(P, 0)) p2p_fail(P, 0, false);
}

// Two Leja nodes per pass (stencil_tb.cuh) and its reduction / decisions.
template <int COEFF, bool GD, bool PEER>
__global__ void __launch_bounds__(TB_THREADS, TB_MINB) k_node_tb(const SeriesParams *__restrict__ Pp) {
    extern __shared__ __align__(128) char tsmem[];
    const SeriesParams &P = *Pp;
    if (P.state->done) return;
    const int k = P.state->k + 1;
    tb_pass<COEFF, GD, PEER>(Pp, k, tb_two(P, k), tsmem);
}

// Two Leja nodes per pass on a single-plane grid (stencil_tb2d.cuh).
template <bool STAGED, bool R8>
__global__ void __launch_bounds__(T2_THREADS, T2_MINB) k_node_tb2d(const SeriesParams *__restrict__ Pp) {
    extern __shared__ __align__(128) char tsmem[];
    const SeriesParams &P = *Pp;
    if (P.state->done) return;
    const int k = P.state->k + 1;
    tb2_pass<STAGED, R8>(Pp, k, tb_two(P, k), tsmem);
}

// Two Leja nodes per pass on a single-plane grid, row-marching warps (stencil_tb2m.cuh).
template <bool STAGED, bool NEU>
__global__ void __launch_bounds__(TM_THREADS, TM_MINB) k_node_tb2m(const SeriesParams *__restrict__ Pp) {
    extern __shared__ __align__(128) char tsmem[];
    const SeriesParams &P = *Pp;
    if (P.state->done) return;
    const int k = P.state->k + 1;
    tm_pass<STAGED, NEU>(Pp, k, tb_two(P, k), tsmem);
}

// Two Leja nodes per pass on one 3D domain, plane-marching warps (stencil_tb3m.cuh).
template <bool GD, bool NEU>
__global__ void __launch_bounds__(T3M_THREADS, 1) k_node_tb3m(const SeriesParams *__restrict__ Pp) {
    extern __shared__ __align__(128) char tsmem[];
    const SeriesParams &P = *Pp;
    if (P.state->done) return;
    const int k = P.state->k + 1;
    t3m_pass<GD, NEU>(Pp, k, tb_two(P, k), tsmem);
}

// Two Leja nodes per pass on a single-plane grid, T3_R rows per stage (stencil_tb2r.cuh).
template <bool STAGED>
__global__ void __launch_bounds__(T2_THREADS, 2) k_node_tb2r(const SeriesParams *__restrict__ Pp) {
    extern __shared__ __align__(128) char tsmem[];
    const SeriesParams &P = *Pp;
    if (P.state->done) return;
    const int k = P.state->k + 1;
    tb3_pass<STAGED, T3_R>(Pp, k, tb_two(P, k), tsmem);
}

__global__ void __launch_bounds__(256) k_slice_reduce2(const SeriesParams *__restrict__ Pp) {
    const SeriesParams &P = *Pp;
    if (P.state->done) return;
    if (blockIdx.x == 0 && threadIdx.x == 0 && P.work) *P.work = 0u;
    slice_reduce_decide2(P, P.state->k + 1);
}

__global__ void k_publish_maps(const TmaMaps maps, TmaMaps *dst) {
    if (threadIdx.x == 0) {
        *dst = maps;
        asm volatile("fence.proxy.tensormap::generic.release.gpu;" ::: "memory");
    }
}

// Series prologue: publish the parameters, clear the state and the tickets.
__global__ void k_series_init(const SeriesParams p, SeriesParams *dst) { series_init_body(p, dst); }

// Series epilogue: the result lives in pbuf[k & 1]; move it to p_out
// (pbuf[1]) when the last node was even.
__global__ void k_series_finalize(const SeriesParams *__restrict__ Pp, int64_t n) {
    const SeriesParams &P = *Pp;
    if ((P.state->k & 1) == 1) return;
    const double *s = P.pbuf[0];
    double *d = P.pbuf[1];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        d[i] = s[i];
}

__global__ void k_state_trivial(SeriesState *st) {
    st->k = 0;
    st->consecutive = 0;
    st->pass = 0;
    st->done = 1;
    st->converged = 1;
    st->last_term = 0.0;
    st->last_pnorm = 0.0;
}

void launch_state_trivial(void *ws, cudaStream_t stream) {
    k_state_trivial<<<1, 1, 0, stream>>>(series_state_ptr(ws));
}

size_t series_state_offset() { return (sizeof(SeriesParams) + 255) & ~(size_t)255; }

SeriesState *series_state_ptr(void *ws) {
    return reinterpret_cast<SeriesState *>(static_cast<char *>(ws) + series_state_offset());
}

__global__ void k_scale_dev(const double *x, const double *s, double *out, int64_t n) {
    const double a = *s;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = mul(a, x[i]);
}

// ---------------------------------------------------------------------------
// host side

int env_int(const char *name, int dflt) {
    const char *s = std::getenv(name);
    return s ? std::atoi(s) : dflt;
}

Geom make_geom(const es_stencil_desc *d, const double *halo_lo, const double *halo_hi) {
    Geom g;
    g.nx = d->nx;
    g.ny = d->ny;
    g.lz = d->lz;
    g.z0 = d->z0;
    g.nz_total = d->nz_total;
    g.wx = d->wx;
    g.wy = d->wy;
    g.wz = d->wz;
    g.mode = d->mode;
    g.coeff_kind = d->coeff_kind;
    g.coeff = d->coeff;
    for (int i = 0; i < 6; ++i) g.faces[i] = d->faces[i];
    g.halo_lo = halo_lo;
    g.halo_hi = halo_hi;
    g.at_lo = d->z0 == 0;
    g.at_hi = d->z0 + d->lz == d->nz_total;
    return g;
}

static bool aligned16(const void *p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

static int sm_count() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    }
    return n;
}

static bool use_v1() {
    const char *s = std::getenv("ES_KERNEL");
    return s && s[0] == 'v' && s[1] == '1';
}

StencilPlan plan_stencil(const es_stencil_desc *d, std::initializer_list<const void *> ptrs, bool tma_ok) {
    StencilPlan pl;
    pl.tma = false;
    pl.dim2 = d->nz_total == 1 && d->lz == 1;
    bool al = d->nx % 2 == 0;
    for (const void *p : ptrs) al = al && aligned16(p);
    if (d->mode == ES_MODE_FACES)
        for (int i = 0; i < 6; ++i) al = al && aligned16(d->faces[i]);
    if (d->coeff_kind == ES_COEFF_ARRAY) al = al && aligned16(d->coeff);
    pl.vec = al ? 2 : 1;
    if (tma_ok && pl.vec == 2 && d->mode != ES_MODE_FACES && !use_v1() && d->nx < (1 << 30) && d->ny < (1 << 30) &&
        d->lz < (1 << 30)) {
        pl.tma = true;
        pl.block = dim3(TMA_THREADS, 1, 1);
        if (pl.dim2) {
            // one wave: tiles_x * nchunks <= SMs * 3 resident CTAs
            // short row chunks, claimed dynamically by the persistent CTAs
            // (4096^2: chunk 8 -> 106 us/node, one-wave chunk 75 -> 122 us)
            // small grids: shorter chunks so the persistent CTAs all get rows
            // (256^2: 32 -> 128 items, 11 -> 9.5 us per latency-bound node)
            const int64_t rows = (int64_t)((d->nx + 511) / 512) * d->ny;
            pl.chunk = env_int("ES_TCHUNK2D", (int)std::min<int64_t>(8, std::max<int64_t>(2, rows / (2 * 148))));
            pl.grid = dim3((unsigned)((d->nx + 511) / 512), (unsigned)((d->ny + pl.chunk - 1) / pl.chunk), 1);
            pl.smem = 0;  // set by the launcher (depends on the kernel variant)
            pl.nchunks = pl.grid.y;
            pl.items = (int64_t)pl.grid.x * pl.nchunks;
            pl.nslices = pl.nchunks;                       // slices = row chunks
            pl.ntiles = pl.grid.x * TMA_CONSUMER_WARPS;    // entries per slice
        } else {
            pl.chunk = env_int("ES_TCHUNK3D", 8);
            pl.grid = dim3((unsigned)((d->nx + 63) / 64), (unsigned)((d->ny + 7) / 8),
                           (unsigned)((d->lz + pl.chunk - 1) / pl.chunk));
            pl.smem = 0;
            pl.nchunks = pl.grid.z;
            pl.items = (int64_t)pl.grid.x * pl.grid.y * pl.nchunks;
            pl.nslices = pl.nchunks;                                // slices = z chunks
            pl.ntiles = pl.grid.x * pl.grid.y * TMA_CONSUMER_WARPS;  // entries per slice
        }
        return pl;
    }
    if (pl.dim2) {
        pl.chunk = env_int("ES_CHUNK2D", 16);
        const int64_t strip = 32LL * pl.vec * BW2;
        pl.grid = dim3((unsigned)((d->nx + strip - 1) / strip), (unsigned)((d->ny + pl.chunk - 1) / pl.chunk), 1);
        pl.block = dim3(32, BW2, 1);
        pl.smem = (size_t)pl.chunk * BW2 * 2 * sizeof(double);
        pl.nslices = d->ny;
        pl.ntiles = pl.grid.x;
        pl.nchunks = pl.grid.y;
    } else {
        pl.chunk = env_int("ES_CHUNK3D", 32);
        const int64_t tx = 32LL * pl.vec;
        pl.grid = dim3((unsigned)((d->nx + tx - 1) / tx), (unsigned)((d->ny + BY3 - 1) / BY3),
                       (unsigned)((d->lz + pl.chunk - 1) / pl.chunk));
        pl.block = dim3(32, BY3, 1);
        const int tile = (BY3 + 2) * (32 * pl.vec + 4);
        pl.smem = (2 * (size_t)tile + (size_t)pl.chunk * BY3 * 2) * sizeof(double);
        pl.nslices = d->lz;
        pl.ntiles = pl.grid.x * pl.grid.y;
        pl.nchunks = pl.grid.z;
    }
    return pl;
}

typedef void (*ApplyFn)(const ApplyArgs);
typedef void (*NodeFn)(const SeriesParams *);

template <int VEC, int COEFF, bool GD>
static void pick(bool dim2, ApplyFn &af, NodeFn &nf) {
    af = dim2 ? k_apply2d<VEC, COEFF, GD> : k_apply3d<VEC, COEFF, GD>;
    nf = dim2 ? k_node2d<VEC, COEFF, GD> : k_node3d<VEC, COEFF, GD>;
}

template <int VEC>
static void pick_c(bool dim2, int coeff, bool gd, ApplyFn &af, NodeFn &nf) {
    switch (coeff) {
        case ES_COEFF_RADIAL: gd ? pick<VEC, ES_COEFF_RADIAL, true>(dim2, af, nf) : pick<VEC, ES_COEFF_RADIAL, false>(dim2, af, nf); break;
        case ES_COEFF_ARRAY: gd ? pick<VEC, ES_COEFF_ARRAY, true>(dim2, af, nf) : pick<VEC, ES_COEFF_ARRAY, false>(dim2, af, nf); break;
        default: gd ? pick<VEC, ES_COEFF_NONE, true>(dim2, af, nf) : pick<VEC, ES_COEFF_NONE, false>(dim2, af, nf); break;
    }
}

static void pick_all(const StencilPlan &pl, int coeff, bool gd, ApplyFn &af, NodeFn &nf) {
    if (pl.vec == 2) pick_c<2>(pl.dim2, coeff, gd, af, nf);
    else pick_c<1>(pl.dim2, coeff, gd, af, nf);
}

static void set_smem_attr(const void *fn, size_t smem) {
    if (smem > 48 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

// ----- tensor maps -------------------------------------------------------------

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

// MK_W2 / MK_G2 / MK_P2 / MK_GH2: the two-node pass's tiles (stencil_tb.cuh)
enum MapKind {
    MK_W = 0, MK_WTAIL = 1, MK_P = 2, MK_HALO = 3, MK_W2 = 4, MK_G2 = 5, MK_P2 = 6, MK_GH2 = 7, MK_WTAIL8 = 8,
    MK_R8W = 9, MK_R8P = 10,  // 2D row as 8-element chunks: (T2_TX + 16) window / T2_TX interior
    MK_R8W_R = 11, MK_R8P_R = 12  // ... T3_R rows per box
};

// TMA descriptor of a slab-shaped fp64 vector (x fastest); OOB reads are
// zero-filled, which is the homogeneous Dirichlet ghost rule.
static int encode_map(CUtensorMap *m, const double *base, const es_stencil_desc *d, bool dim2, MapKind kind) {
    std::memset(m, 0, sizeof(*m));
    if (!base) return ES_OK;
    auto fn = encode_fn();
    if (!fn) return set_error(ES_ERR_CUDA, "cuTensorMapEncodeTiled is unavailable");
    cuuint64_t dims[3], strides[2];
    cuuint32_t box[3], estr[3] = {1, 1, 1};
    cuuint32_t rank;
    if (kind == MK_R8W || kind == MK_R8P || kind == MK_R8W_R || kind == MK_R8P_R) {  // (8, nx/8, ny) row view
        rank = 3;
        dims[0] = 8;
        dims[1] = (cuuint64_t)d->nx / 8;
        dims[2] = (cuuint64_t)d->ny;
        strides[0] = 64;
        strides[1] = (cuuint64_t)d->nx * 8;
        box[0] = 8;
        box[1] = (kind == MK_R8W || kind == MK_R8W_R ? T2_RX : T2_TX) / 8;
        box[2] = kind == MK_R8W_R || kind == MK_R8P_R ? T3_R : 1;
    } else if (kind == MK_HALO || kind == MK_GH2) {  // one (ny, nx) plane, same box as the 3D W (g') tiles
        rank = 2;
        dims[0] = (cuuint64_t)d->nx;
        dims[1] = (cuuint64_t)d->ny;
        strides[0] = (cuuint64_t)d->nx * 8;
        box[0] = 68;
        box[1] = kind == MK_GH2 ? TB_GY : 10;
    } else if (dim2) {
        rank = 2;
        dims[0] = (cuuint64_t)d->nx;
        dims[1] = (cuuint64_t)d->ny;
        strides[0] = (cuuint64_t)d->nx * 8;
        box[0] = kind == MK_WTAIL ? 4 : kind == MK_WTAIL8 ? 8 : 256;
        box[1] = 1;
    } else {
        rank = 3;
        dims[0] = (cuuint64_t)d->nx;
        dims[1] = (cuuint64_t)d->ny;
        dims[2] = (cuuint64_t)d->lz;
        strides[0] = (cuuint64_t)d->nx * 8;
        strides[1] = (cuuint64_t)d->nx * d->ny * 8;
        box[0] = (kind == MK_P || kind == MK_P2) ? 64 : kind == MK_W2 ? TB_WX : 68;  // MK_W2: two-point halo
        box[1] = kind == MK_P ? 8 : kind == MK_P2 ? TB_TY : kind == MK_W2 ? TB_WY : kind == MK_G2 ? TB_GY : 10;
        box[2] = 1;
    }
    const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, const_cast<double *>(base), dims, strides, box,
                          estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_error(ES_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return ES_OK;
}

static int encode_w(CUtensorMap *wa, CUtensorMap *wb, const double *base, const es_stencil_desc *d, bool dim2) {
    int rc = encode_map(wa, base, d, dim2, MK_W);
    if (rc) return rc;
    return encode_map(wb, base, d, dim2, dim2 ? MK_WTAIL : MK_W);
}

// persistent grid: every resident CTA slot, at most one per item
static void finish_tma_plan(StencilPlan &pl, const void *fn, size_t smem, int threads = TMA_THREADS) {
    pl.smem = smem;
    pl.block = dim3((unsigned)threads, 1, 1);
    set_smem_attr(fn, smem);
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, threads, smem) != cudaSuccess || nb < 1) {
        cudaGetLastError();
        nb = 1;
    }
    const int64_t items = pl.items;
    pl.grid = dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>(items, (int64_t)nb * sm_count())), 1, 1);
}

static size_t node_smem(bool dim2, bool gd, int chunk) {
    if (dim2) return gd ? tma_smem_bytes<false, true, true>(chunk) : tma_smem_bytes<false, true, false>(chunk);
    return gd ? tma_smem_bytes<true, true, true>(chunk) : tma_smem_bytes<true, true, false>(chunk);
}

typedef void (*ApplyTmaFn)(const ApplyArgsT);
typedef void (*NodeTmaFn)(const SeriesParams *);

template <bool DIM3>
static ApplyTmaFn pick_apply_tma(int coeff) {
    switch (coeff) {
        case ES_COEFF_RADIAL: return k_apply_tma<DIM3, ES_COEFF_RADIAL>;
        case ES_COEFF_ARRAY: return k_apply_tma<DIM3, ES_COEFF_ARRAY>;
        default: return k_apply_tma<DIM3, ES_COEFF_NONE>;
    }
}

template <bool DIM3, bool GD>
static NodeTmaFn pick_node_tma_c(int coeff) {
    switch (coeff) {
        case ES_COEFF_RADIAL: return k_node_tma<DIM3, ES_COEFF_RADIAL, GD>;
        case ES_COEFF_ARRAY: return k_node_tma<DIM3, ES_COEFF_ARRAY, GD>;
        case ES_COEFF_STAGED: return k_node_tma<DIM3, ES_COEFF_STAGED, false>;
        default: return k_node_tma<DIM3, ES_COEFF_NONE, GD>;
    }
}

static NodeTmaFn pick_node_tma(bool dim2, int coeff, bool gd) {
    if (dim2) return gd ? pick_node_tma_c<false, true>(coeff) : pick_node_tma_c<false, false>(coeff);
    return gd ? pick_node_tma_c<true, true>(coeff) : pick_node_tma_c<true, false>(coeff);
}

int launch_stencil_apply(const es_stencil_desc *d, const double *u, double *out, double alpha,
                         double beta, const double *halo_lo, const double *halo_hi,
                         const double *gdiag, cudaStream_t stream) {
    if (d->nx * d->ny * d->lz == 0) return ES_OK;
    const bool dim2 = d->nz_total == 1 && d->lz == 1;
    const bool plain = !gdiag && (dim2 ? (!halo_lo && !halo_hi) : true);
    const StencilPlan pl = plan_stencil(d, {u, out, halo_lo, halo_hi, gdiag}, plain);
    Pass ps;
    ps.src = u;
    ps.dst = out;
    ps.p_src = nullptr;
    ps.p_dst = nullptr;
    ps.alpha = alpha;
    ps.beta = beta;
    ps.dk = 0.0;
    ps.d0 = 0.0;
    if (pl.tma) {
        ApplyArgsT a;
        a.g = make_geom(d, halo_lo, halo_hi);
        a.ps = ps;
        a.chunk_len = pl.chunk;
        std::memset(&a.maps, 0, sizeof(a.maps));
        int rc = encode_w(&a.maps.m[MAP_WA_V], &a.maps.m[MAP_WB_V], u, d, pl.dim2);
        if (!rc) rc = encode_map(&a.maps.m[MAP_HLO], halo_lo, d, pl.dim2, MK_HALO);
        if (!rc) rc = encode_map(&a.maps.m[MAP_HHI], halo_hi, d, pl.dim2, MK_HALO);
        if (rc) return rc;
        const ApplyTmaFn fn = pl.dim2 ? pick_apply_tma<false>(d->coeff_kind) : pick_apply_tma<true>(d->coeff_kind);
        StencilPlan lp = pl;
        finish_tma_plan(lp, (const void *)fn,
                        pl.dim2 ? tma_smem_bytes<false, false, false>(pl.chunk) : tma_smem_bytes<true, false, false>(pl.chunk));
        fn<<<lp.grid, lp.block, lp.smem, stream>>>(a);
        return check_launch("stencil apply (tma)");
    }
    ApplyFn af;
    NodeFn nf;
    pick_all(pl, d->coeff_kind, gdiag != nullptr, af, nf);
    ApplyArgs a;
    a.g = make_geom(d, halo_lo, halo_hi);
    a.ps = ps;
    a.gdiag = gdiag;
    a.chunk_len = pl.chunk;
    set_smem_attr((const void *)af, pl.smem);
    af<<<pl.grid, pl.block, pl.smem, stream>>>(a);
    return check_launch("stencil apply");
}

template <bool DIM3>
static ApplyTmaFn pick_rospro(int coeff) {
    switch (coeff) {
        case ES_COEFF_RADIAL: return k_rospro_tma<DIM3, ES_COEFF_RADIAL>;
        case ES_COEFF_ARRAY: return k_rospro_tma<DIM3, ES_COEFF_ARRAY>;
        default: return k_rospro_tma<DIM3, ES_COEFF_NONE>;
    }
}

static double unord(unsigned long long o) {
    const unsigned long long b = (o >> 63) ? (o & 0x7fffffffffffffffull) : ~o;
    double d;
    std::memcpy(&d, &b, sizeof d);
    return d;
}

int run_rosenbrock_prologue(const es_stencil_desc *d, const double *u, double *F, double *gdiag, double *minmax_host,
                            int64_t *first_bad_host, void *aux_dev, const double *halo_lo, const double *halo_hi,
                            cudaStream_t stream) {
    const int64_t n = d->nx * d->ny * d->lz;
    const StencilPlan pl = plan_stencil(d, {u, F, gdiag, halo_lo, halo_hi}, true);
    if ((halo_lo || halo_hi) && pl.dim2) return set_error(ES_ERR_ARG, "halos need a 3D slab");
    if (!pl.tma) return set_error(ES_ERR_ARG, "rosenbrock prologue needs the TMA path (even nx, aligned, no faces)");
    unsigned long long *aux = static_cast<unsigned long long *>(aux_dev);
    ApplyArgsT a;
    a.g = make_geom(d, halo_lo, halo_hi);
    a.ps.src = u;
    a.ps.dst = F;
    a.ps.p_src = nullptr;
    a.ps.p_dst = gdiag;
    a.ps.alpha = 1.0;
    a.ps.beta = 0.0;
    a.ps.dk = 0.0;
    a.ps.d0 = 0.0;
    a.ps.aux = aux;
    a.chunk_len = pl.chunk;
    std::memset(&a.maps, 0, sizeof(a.maps));
    int rc = encode_w(&a.maps.m[MAP_WA_V], &a.maps.m[MAP_WB_V], u, d, pl.dim2);
    if (!rc) rc = encode_map(&a.maps.m[MAP_HLO], halo_lo, d, pl.dim2, MK_HALO);
    if (!rc) rc = encode_map(&a.maps.m[MAP_HHI], halo_hi, d, pl.dim2, MK_HALO);
    if (rc) return rc;
    const ApplyTmaFn fn = pl.dim2 ? pick_rospro<false>(d->coeff_kind) : pick_rospro<true>(d->coeff_kind);
    StencilPlan lp = pl;
    finish_tma_plan(lp, (const void *)fn,
                    pl.dim2 ? tma_smem_bytes<false, false, false>(pl.chunk) : tma_smem_bytes<true, false, false>(pl.chunk));
    k_aux_init<<<1, 32, 0, stream>>>(aux, (unsigned long long)n);
    fn<<<lp.grid, lp.block, lp.smem, stream>>>(a);
    rc = check_launch("rosenbrock prologue");
    if (rc) return rc;
    unsigned long long h[3];
    if (cudaMemcpyAsync(h, aux, sizeof h, cudaMemcpyDeviceToHost, stream) != cudaSuccess ||
        cudaStreamSynchronize(stream) != cudaSuccess)
        return check_launch("rosenbrock prologue sync");
    minmax_host[0] = unord(h[0]);
    minmax_host[1] = unord(h[1]);
    *first_bad_host = h[2] < (unsigned long long)n ? (int64_t)h[2] : -1;
    if (*first_bad_host >= 0)
        return set_error(ES_ERR_DOMAIN, "combustion nonlinearity undefined at index %lld", (long long)h[2]);
    return ES_OK;
}

// ----- series workspace layout ------------------------------------------------

static size_t up(size_t x) { return (x + 255) & ~(size_t)255; }

struct WsLayout {
    size_t params, state, maps, cnt, part, slice, wa, wb, pb, total;
};

static WsLayout layout(int64_t n, int nslices, int ntiles, int nchunks) {
    WsLayout L;
    size_t o = 0;
    L.params = o; o = up(o + sizeof(SeriesParams));
    L.state = o; o = up(o + sizeof(SeriesState));
    L.maps = o; o = up(o + sizeof(TmaMaps));
    L.cnt = o; o = up(o + sizeof(unsigned) * (nchunks + 2));
    L.part = o; o = up(o + sizeof(double) * 4 * (size_t)nslices * ntiles);  // x2: two-node passes
    L.slice = o; o = up(o + sizeof(double) * 4 * (size_t)nslices);
    L.wa = o; o = up(o + sizeof(double) * n);
    L.wb = o; o = up(o + sizeof(double) * n);
    L.pb = o; o = up(o + sizeof(double) * n);
    L.total = o;
    return L;
}

size_t stencil_series_ws_bytes(const es_stencil_desc *d) {
    // the scalar (VEC = 1) plan has the most tiles: size for it
    // the larger of the scalar v1 plan (most tiles) and the TMA plan
    es_stencil_desc dodd = *d;
    dodd.nx = d->nx | 1;
    const StencilPlan po = plan_stencil(&dodd, {}, false);
    const StencilPlan pt = plan_stencil(d, {}, true);
    const int64_t n = d->nx * d->ny * d->lz;
    return std::max(layout(n, po.nslices, po.ntiles, po.nchunks).total,
                    layout(n, pt.nslices, pt.ntiles, pt.nchunks).total);
}

// Everything a series needs before its first node: plan, kernel, device
// parameters (published with the state reset), TMA descriptors.
struct SeriesSetup {
    StencilPlan pl, lp;
    NodeFn nf;
    SeriesParams hp;
    SeriesParams *dparams;
    int64_t n;
    bool tb = false;   // two nodes per pass (k_node_tb + k_slice_reduce2)
    bool tb2 = false;  // two nodes per pass on a single-plane grid (k_node_tb2d + k_slice_reduce2)
    bool r8 = false;   // ... with the (8, nx/8, ny) row view (one TMA per row window)
    bool rows = false; // ... and stages of T3_R rows (k_node_tb2r)
    bool march = false; // ... row-marching warps (k_node_tb2m)
    bool staged = false;  // sampled coefficient through the PG ring (ES_COEFF_STAGED)
};

template <bool GD, bool PEER = false>
static NodeFn pick_node_tb(int coeff) {
    switch (coeff) {
        case ES_COEFF_RADIAL: return k_node_tb<ES_COEFF_RADIAL, GD, PEER>;
        case ES_COEFF_ARRAY: return k_node_tb<ES_COEFF_ARRAY, GD, PEER>;
        default: return k_node_tb<ES_COEFF_NONE, GD, PEER>;
    }
}

static int prepare_series(const es_stencil_desc *d, const double *v, double *p_out, const double *dd,
                          const double *xi, int ndd, double alpha, double shift, double tol, const double *gdiag,
                          const double *halo_lo, const double *halo_hi, bool dist, void *ws, size_t ws_bytes,
                          SeriesSetup &S, cudaStream_t stream, const double *halo_lo_1 = nullptr,
                          const double *halo_hi_1 = nullptr, int allow_tb = 1, const double *g_lo = nullptr,
                          const double *g_hi = nullptr, bool maps_needed = true) {
    S.n = d->nx * d->ny * d->lz;
    char *w = static_cast<char *>(ws);
    S.pl = plan_stencil(d, {v, p_out, gdiag, halo_lo, halo_hi, (const void *)(w + 0)}, true);
    StencilPlan &pl = S.pl;
    if ((halo_lo || halo_hi || dist) && !(pl.tma && !pl.dim2))
        return set_error(ES_ERR_ARG, "slab series with halos need the 3D TMA path (even nx, aligned vectors)");
    // two nodes per pass (stencil_tb.cuh) where the w_k window's ghosts are
    // local (Dirichlet / Neumann, one domain): 24 instead of 40 B/point/node,
    // ~690 vs ~890 us per 512^3 Rosenbrock node.
    // Longer z chunks than the one-node kernel's: an item re-reads three w
    // planes beyond its chunk (8 -> 32: 767 -> 685 us).  ES_TB=0 forces one
    // node per pass.
    // allow_tb: 0 never, 1 one domain only, 2 also slabs with two-plane peer halos
    const bool halos = halo_lo || halo_hi;
    S.tb = pl.tma && allow_tb > 0 && !pl.dim2 && !dist && (d->mode == ES_MODE_ZERO || d->mode == ES_MODE_NEUMANN) &&
           env_int("ES_TB", 1) &&
           (!halos || (allow_tb == 2 && d->coeff_kind != ES_COEFF_ARRAY && d->lz >= 2));
    // two nodes per pass on single-plane grids (stencil_tb2d.cuh): Dirichlet
    // or Neumann, no coefficient or the staged sampled D, no g' (C2: 48
    // instead of 2 x 40 B/point per two nodes).  The one-node plan's row
    // chunks stay the norm slices; items span 4 of them.
    S.tb2 = pl.tma && pl.dim2 && allow_tb > 0 && !dist && !halos && !gdiag &&
            (d->mode == ES_MODE_ZERO || d->mode == ES_MODE_NEUMANN) && d->coeff_kind != ES_COEFF_RADIAL &&
            env_int("ES_TB", 1) && env_int("ES_TB2D", 1);
    int chunk2 = 0;
    if (S.tb2) {
        // row-marching warps (stencil_tb2m.cuh; 4096^2: 158 vs 207 us per pass
        // of the group A / group C kernel), items of 3 norm chunks (24 rows at
        // 4096^2: 158 us; 16 / 32 / 40 rows: 160 / 162 / 162 us)
        S.march = env_int("ES_TB2M", 1) != 0;
        chunk2 = pl.chunk * std::max(1, env_int("ES_TB2CHUNK", S.march ? 3 : 4));
        const int tx = S.march ? TM_TX : T2_TX;
        pl.items = (int64_t)((d->nx + tx - 1) / tx) * ((d->ny + chunk2 - 1) / chunk2);
    }
    if (S.tb) {
        // plane-marching pass (one domain, no coefficient, one CTA per SM):
        // the longest z chunk (two halo planes per chunk) that still leaves
        // >= 6 items per CTA -- 512^3: 128 planes, 877-880 us per pass
        // (64: 891-893, 32: 918-922); the group A / C kernel keeps 32
        const bool march3 = !halos && d->coeff_kind == ES_COEFF_NONE && env_int("ES_TB3M", 1);
        int zc = 32;
        if (march3) {
            const int64_t tiles = ((d->nx + 63) / 64) * ((d->ny + TB_TY - 1) / TB_TY);
            for (int c : {128, 64}) {
                if (tiles * ((d->lz + c - 1) / c) >= 6 * (int64_t)sm_count()) {
                    zc = c;
                    break;
                }
            }
        }
        pl.chunk = std::max(1, env_int("ES_TBCHUNK", zc));
        pl.grid.z = (unsigned)((d->lz + pl.chunk - 1) / pl.chunk);
        pl.nchunks = pl.grid.z;
        pl.items = (int64_t)pl.grid.x * pl.grid.y * pl.nchunks;
        pl.nslices = pl.nchunks;
    }
    const WsLayout L = layout(S.n, pl.nslices, pl.ntiles, pl.nchunks);
    if (ws_bytes < L.total) return set_error(ES_ERR_ARG, "workspace too small");
    ApplyFn af;
    S.lp = pl;
    if (pl.tma) {
        if (S.tb2) {
            S.staged = d->coeff_kind == ES_COEFF_ARRAY;
            S.r8 = d->nx % 8 == 0 && env_int("ES_TB2R8", 1);
            S.rows = !S.march && S.r8 && env_int("ES_TB2R", 0) && chunk2 % T3_R == 0;  // multi-row stages (measured slower: off)
            if (S.march) {
                S.r8 = false;
                const bool neu = d->mode == ES_MODE_NEUMANN;
                S.nf = S.staged ? (neu ? k_node_tb2m<true, true> : k_node_tb2m<true, false>)
                                : (neu ? k_node_tb2m<false, true> : k_node_tb2m<false, false>);
                finish_tma_plan(S.lp, (const void *)S.nf,
                                S.staged ? (size_t)TmLayout<true>::BYTES : (size_t)TmLayout<false>::BYTES, TM_THREADS);
            } else if (S.rows) {
                S.nf = S.staged ? k_node_tb2r<true> : k_node_tb2r<false>;
                finish_tma_plan(S.lp, (const void *)S.nf,
                                S.staged ? (size_t)Tb3Layout<true, T3_R>::BYTES : (size_t)Tb3Layout<false, T3_R>::BYTES,
                                T2_THREADS);
            } else {
                S.nf = S.staged ? (S.r8 ? k_node_tb2d<true, true> : k_node_tb2d<true, false>)
                                : (S.r8 ? k_node_tb2d<false, true> : k_node_tb2d<false, false>);
                finish_tma_plan(S.lp, (const void *)S.nf,
                                S.staged ? (size_t)Tb2Layout<true>::BYTES : (size_t)Tb2Layout<false>::BYTES,
                                T2_THREADS);
            }
        } else if (S.tb && !halos && d->coeff_kind == ES_COEFF_NONE && env_int("ES_TB3M", 1)) {
            // plane-marching warps (stencil_tb3m.cuh; 512^3 Rosenbrock pass
            // ~1.01 -> ~0.96-0.99 ms, 626 -> 447 M warp instructions)
            const bool neu = d->mode == ES_MODE_NEUMANN;
            S.nf = gdiag ? (neu ? k_node_tb3m<true, true> : k_node_tb3m<true, false>)
                         : (neu ? k_node_tb3m<false, true> : k_node_tb3m<false, false>);
            finish_tma_plan(S.lp, (const void *)S.nf,
                            gdiag ? (size_t)T3mLayout<true>::BYTES : (size_t)T3mLayout<false>::BYTES, T3M_THREADS);
        } else if (S.tb) {
            S.nf = gdiag ? pick_node_tb<true>(d->coeff_kind) : pick_node_tb<false>(d->coeff_kind);
            finish_tma_plan(S.lp, (const void *)S.nf,
                            gdiag ? (size_t)TbLayout<true>::BYTES : (size_t)TbLayout<false>::BYTES, TB_THREADS);
        } else {
            // a sampled coefficient without g' streams through the PG ring's g' slot
            S.staged = !gdiag && d->coeff_kind == ES_COEFF_ARRAY && env_int("ES_DSTAGE", 1);
            S.nf = pick_node_tma(pl.dim2, S.staged ? ES_COEFF_STAGED : d->coeff_kind, gdiag != nullptr);
            finish_tma_plan(S.lp, (const void *)S.nf, node_smem(pl.dim2, gdiag != nullptr || S.staged, pl.chunk));
        }
    } else {
        pick_all(pl, d->coeff_kind, gdiag != nullptr, af, S.nf);
        set_smem_attr((const void *)S.nf, pl.smem);
    }
    SeriesParams &hp = S.hp;
    hp = SeriesParams{};
    hp.g = make_geom(d, halo_lo, halo_hi);
    hp.v = v;
    hp.wbuf[1] = reinterpret_cast<double *>(w + L.wa);
    hp.wbuf[0] = reinterpret_cast<double *>(w + L.wb);
    hp.pbuf[1] = p_out;
    hp.pbuf[0] = reinterpret_cast<double *>(w + L.pb);
    hp.gdiag = gdiag;
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
    hp.global_cnt = hp.chunk_cnt + pl.nchunks;
    hp.work = pl.tma ? hp.global_cnt + 1 : nullptr;
    hp.nslices = pl.nslices;
    hp.ntiles = pl.ntiles;
    hp.nchunks = pl.nchunks;
    hp.chunk_len = pl.chunk;
    hp.cond = 0;
    hp.maps = nullptr;
    hp.dist = dist ? 1 : 0;
    hp.tail1 = env_int("ES_TB_TAIL", 1) ? 1 : 0;
    hp.norm_chunk = pl.chunk;
    if (S.tb2) hp.chunk_len = chunk2;  // items of the two-node 2D pass
    S.dparams = reinterpret_cast<SeriesParams *>(w + L.params);
    if (pl.tma && maps_needed) {
        TmaMaps maps;
        std::memset(&maps, 0, sizeof(maps));
        int rc = encode_w(&maps.m[MAP_WA_V], &maps.m[MAP_WB_V], v, d, pl.dim2);
        if (!rc) rc = encode_w(&maps.m[MAP_WA_0], &maps.m[MAP_WB_0], hp.wbuf[0], d, pl.dim2);
        if (!rc) rc = encode_w(&maps.m[MAP_WA_1], &maps.m[MAP_WB_1], hp.wbuf[1], d, pl.dim2);
        if (!rc) rc = encode_map(&maps.m[MAP_P_0], hp.pbuf[0], d, pl.dim2, MK_P);
        if (!rc) rc = encode_map(&maps.m[MAP_P_1], hp.pbuf[1], d, pl.dim2, MK_P);
        if (!rc) rc = encode_map(&maps.m[MAP_G], S.staged ? d->coeff : gdiag, d, pl.dim2, MK_P);
        if (!rc) rc = encode_map(&maps.m[MAP_HLO], halo_lo, d, pl.dim2, MK_HALO);
        if (!rc) rc = encode_map(&maps.m[MAP_HHI], halo_hi, d, pl.dim2, MK_HALO);
        if (!rc) rc = encode_map(&maps.m[MAP_HLO_1], halo_lo_1, d, pl.dim2, MK_HALO);
        if (!rc) rc = encode_map(&maps.m[MAP_HHI_1], halo_hi_1, d, pl.dim2, MK_HALO);
        if (S.tb2) {
            if (!rc) rc = encode_map(&maps.m[MAP_T2_W8_V], v, d, true, MK_WTAIL8);
            if (!rc) rc = encode_map(&maps.m[MAP_T2_W8_0], hp.wbuf[0], d, true, MK_WTAIL8);
            if (!rc) rc = encode_map(&maps.m[MAP_T2_W8_1], hp.wbuf[1], d, true, MK_WTAIL8);
            if (!rc) rc = encode_map(&maps.m[MAP_T2_G4], S.staged ? d->coeff : nullptr, d, true, MK_WTAIL);
            if (S.rows) {
                if (!rc) rc = encode_map(&maps.m[MAP_T3_W_V], v, d, true, MK_R8W_R);
                if (!rc) rc = encode_map(&maps.m[MAP_T3_W_0], hp.wbuf[0], d, true, MK_R8W_R);
                if (!rc) rc = encode_map(&maps.m[MAP_T3_W_1], hp.wbuf[1], d, true, MK_R8W_R);
                if (!rc) rc = encode_map(&maps.m[MAP_T3_G], S.staged ? d->coeff : nullptr, d, true, MK_R8W_R);
                if (!rc) rc = encode_map(&maps.m[MAP_T3_P_V], v, d, true, MK_R8P_R);
                if (!rc) rc = encode_map(&maps.m[MAP_T3_P_0], hp.pbuf[0], d, true, MK_R8P_R);
                if (!rc) rc = encode_map(&maps.m[MAP_T3_P_1], hp.pbuf[1], d, true, MK_R8P_R);
                if (!rc) rc = encode_map(&maps.m[MAP_T3_D], S.staged ? d->coeff : nullptr, d, true, MK_R8P_R);
            }
            if (S.r8) {
                if (!rc) rc = encode_map(&maps.m[MAP_T2R_W_V], v, d, true, MK_R8W);
                if (!rc) rc = encode_map(&maps.m[MAP_T2R_W_0], hp.wbuf[0], d, true, MK_R8W);
                if (!rc) rc = encode_map(&maps.m[MAP_T2R_W_1], hp.wbuf[1], d, true, MK_R8W);
                if (!rc) rc = encode_map(&maps.m[MAP_T2R_G], S.staged ? d->coeff : nullptr, d, true, MK_R8W);
                if (!rc) rc = encode_map(&maps.m[MAP_T2R_P_V], v, d, true, MK_R8P);
                if (!rc) rc = encode_map(&maps.m[MAP_T2R_P_0], hp.pbuf[0], d, true, MK_R8P);
                if (!rc) rc = encode_map(&maps.m[MAP_T2R_P_1], hp.pbuf[1], d, true, MK_R8P);
                if (!rc) rc = encode_map(&maps.m[MAP_T2R_D], S.staged ? d->coeff : nullptr, d, true, MK_R8P);
            }
        }
        if (S.tb) {
            if (!rc) rc = encode_map(&maps.m[MAP_T_V], v, d, false, MK_W2);
            if (!rc) rc = encode_map(&maps.m[MAP_T_0], hp.wbuf[0], d, false, MK_W2);
            if (!rc) rc = encode_map(&maps.m[MAP_T_1], hp.wbuf[1], d, false, MK_W2);
            if (!rc) rc = encode_map(&maps.m[MAP_T_G], gdiag, d, false, MK_G2);
            if (!rc) rc = encode_map(&maps.m[MAP_T_PV], v, d, false, MK_P2);
            if (!rc) rc = encode_map(&maps.m[MAP_T_P0], hp.pbuf[0], d, false, MK_P2);
            if (!rc) rc = encode_map(&maps.m[MAP_T_P1], hp.pbuf[1], d, false, MK_P2);
            if (!rc) rc = encode_map(&maps.m[MAP_T_GP], gdiag, d, false, MK_P2);
            if (halos) {  // two-plane w halos by parity, g' boundary planes of the neighbours
                es_stencil_desc d2 = *d;
                d2.lz = 2;
                if (!rc) rc = encode_map(&maps.m[MAP_T_HLO0], halo_lo, &d2, false, MK_W2);
                if (!rc) rc = encode_map(&maps.m[MAP_T_HLO1], halo_lo_1, &d2, false, MK_W2);
                if (!rc) rc = encode_map(&maps.m[MAP_T_HHI0], halo_hi, &d2, false, MK_W2);
                if (!rc) rc = encode_map(&maps.m[MAP_T_HHI1], halo_hi_1, &d2, false, MK_W2);
                if (!rc) rc = encode_map(&maps.m[MAP_T_GLO], g_lo, d, false, MK_GH2);
                if (!rc) rc = encode_map(&maps.m[MAP_T_GHI], g_hi, d, false, MK_GH2);
            }
        }
        if (rc) return rc;
        TmaMaps *dmaps = reinterpret_cast<TmaMaps *>(w + L.maps);
        k_publish_maps<<<1, 32, 0, stream>>>(maps, dmaps);
        hp.maps = dmaps;
    }
    return ES_OK;
}

// Small single-plane grids: parameters of a persistent series
// (series_small.cu) published like the graph path's, without TMA maps;
// *ok = false when the persistent form does not apply.
int small_prepare(const es_stencil_desc *d, const double *v, double *p_out, const double *dd, const double *xi,
                  int ndd, double alpha, double shift, double tol, const double *gdiag, void *ws, size_t ws_bytes,
                  int nseries, SeriesParams *hp, SeriesParams **dparams, StencilPlan *plan, bool *ok,
                  cudaStream_t stream) {
    *ok = false;
    if (ndd < 2 || d->nx * d->ny * d->lz == 0) return ES_OK;
    const StencilPlan pl = plan_stencil(d, {v, p_out, gdiag, (const void *)ws}, true);
    if (!small_series_ok(d, pl, gdiag != nullptr, nseries)) return ES_OK;
    SeriesSetup S;
    const int rc = prepare_series(d, v, p_out, dd, xi, ndd, alpha, shift, tol, gdiag, nullptr, nullptr, false, ws,
                                  ws_bytes, S, stream, nullptr, nullptr, 0, nullptr, nullptr, false);
    if (rc) return rc;
    *hp = S.hp;
    *dparams = S.dparams;
    *plan = S.pl;
    *ok = true;
    return ES_OK;
}

int launch_series_init(const SeriesParams *hp, SeriesParams *dparams, cudaStream_t stream) {
    k_series_init<<<1, 256, 0, stream>>>(*hp, dparams);
    return check_launch("series init");
}

int run_stencil_series(const es_stencil_desc *d, const double *v, double *p_out, const double *dd,
                       const double *xi, int ndd, double alpha, double shift, double tol,
                       const double *gdiag, void *ws, size_t ws_bytes, es_series_result *res,
                       cudaStream_t stream) {
    const int64_t n = d->nx * d->ny * d->lz;
    if (ndd < 1) return set_error(ES_ERR_ARG, "ndd must be >= 1");
    if (ndd == 1 || n == 0) {  // degenerate interval: dd_0 v, 0 matvecs (matfunc.py:285-286)
        const StencilPlan pl = plan_stencil(d, {v, p_out, gdiag, ws}, true);
        if (ws_bytes < layout(n, pl.nslices, pl.ntiles, pl.nchunks).total)
            return set_error(ES_ERR_ARG, "workspace too small");
        if (n > 0) k_scale_dev<<<std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, stream>>>(v, dd, p_out, n);
        launch_state_trivial(ws, stream);
        int rc = check_launch("scale");
        if (rc || !res) return rc;
        return read_series_state(series_state_ptr(ws), res, stream);
    }
    {  // tiny grids: the whole series in one persistent launch (series_small.cu)
        SeriesParams hp;
        SeriesParams *dp = nullptr;
        StencilPlan sp;
        bool ok = false;
        int rc = small_prepare(d, v, p_out, dd, xi, ndd, alpha, shift, tol, gdiag, ws, ws_bytes, 1, &hp, &dp, &sp,
                               &ok, stream);
        if (rc) return rc;
        if (ok) {
            if ((rc = launch_series_init(&hp, dp, stream))) return rc;
            if ((rc = launch_series_small(d, dp, sp, gdiag != nullptr, stream))) return rc;
            if (!res) return ES_OK;
            return read_series_state(hp.state, res, stream);
        }
    }
    SeriesSetup S;
    int rc = prepare_series(d, v, p_out, dd, xi, ndd, alpha, shift, tol, gdiag, nullptr, nullptr, false, ws,
                            ws_bytes, S, stream);
    if (rc) return rc;
    NodeFn rf = S.tb || S.tb2 ? k_slice_reduce2 : k_slice_reduce;
    GraphKernel gk[2] = {{(const void *)S.nf, S.lp.grid, S.lp.block, S.lp.smem},
                         {(const void *)rf, dim3((unsigned)S.pl.nslices), dim3(256), 0}};
    unsigned long long handle = 0;
    cudaGraphExec_t ge = series_graph(gk, S.pl.tma ? 2 : 1, S.dparams, &handle);
    if (ge) S.hp.cond = handle;
    k_series_init<<<1, 256, 0, stream>>>(S.hp, S.dparams);
    rc = check_launch("series init");
    if (rc) return rc;
    if (ge) {
        if (cudaGraphLaunch(ge, stream) != cudaSuccess) return check_launch("series graph");
    } else {
        // one launch pair per node at most (a two-node series may run one-node passes)
        for (int k = 1; k < ndd; ++k) {
            S.nf<<<S.lp.grid, S.lp.block, S.lp.smem, stream>>>(S.dparams);
            if (S.pl.tma) rf<<<(unsigned)S.pl.nslices, 256, 0, stream>>>(S.dparams);
        }
        rc = check_launch("series nodes");
        if (rc) return rc;
    }
    k_series_finalize<<<148 * 8, 256, 0, stream>>>(S.dparams, n);
    rc = check_launch("series finalize");
    if (rc) return rc;
    if (!res) return ES_OK;  // asynchronous: es_leja_fetch reads the state later
    return read_series_state(S.hp.state, res, stream);
}

// ----- multi-GPU slab series: the caller drives the nodes ---------------------
//
// Per node k (host-tracked, 1-based): the caller exchanges the boundary
// planes of dist_source(k) into the halo buffers given at begin, calls
// dist_node (pass over the slab + local per-chunk slices, no decision),
// all-gathers the slices of every rank in rank (= global z) order and calls
// dist_decide, which evaluates the stopping test identically on every rank.
// Node kernels after the decision return immediately.

static std::mutex g_dist_mu;
static std::map<const void *, SeriesSetup> g_dist;

int dist_begin(const es_stencil_desc *d, const double *v, double *p_out, const double *dd, const double *xi, int ndd,
               double alpha, double shift, double tol, const double *gdiag, const double *halo_lo,
               const double *halo_hi, void *ws, size_t ws_bytes, cudaStream_t stream) {
    if (ndd < 2) return set_error(ES_ERR_ARG, "a slab series needs ndd >= 2");
    SeriesSetup S;
    int rc = prepare_series(d, v, p_out, dd, xi, ndd, alpha, shift, tol, gdiag, halo_lo, halo_hi, true, ws, ws_bytes,
                            S, stream);
    if (rc) return rc;
    k_series_init<<<1, 256, 0, stream>>>(S.hp, S.dparams);
    rc = check_launch("slab series init");
    if (rc) return rc;
    std::lock_guard<std::mutex> lk(g_dist_mu);
    g_dist[ws] = S;
    return ES_OK;
}

static int dist_get(const void *ws, SeriesSetup *&S) {
    std::lock_guard<std::mutex> lk(g_dist_mu);
    auto it = g_dist.find(ws);
    if (it == g_dist.end()) return set_error(ES_ERR_ARG, "no slab series begun on this workspace");
    S = &it->second;
    return ES_OK;
}

int dist_source(const void *ws, int k, const double **src) {
    SeriesSetup *S;
    int rc = dist_get(ws, S);
    if (rc) return rc;
    *src = k <= 1 ? S->hp.v : S->hp.wbuf[(k - 1) & 1];
    return ES_OK;
}

int dist_nslices(const void *ws, int *nslices) {
    SeriesSetup *S;
    int rc = dist_get(ws, S);
    if (rc) return rc;
    *nslices = S->pl.nslices;
    return ES_OK;
}

int dist_node(const void *ws, double *slices_out, cudaStream_t stream) {
    SeriesSetup *S;
    int rc = dist_get(ws, S);
    if (rc) return rc;
    S->nf<<<S->lp.grid, S->lp.block, S->lp.smem, stream>>>(S->dparams);
    k_slice_reduce<<<(unsigned)S->pl.nslices, 256, 0, stream>>>(S->dparams);
    cudaMemcpyAsync(slices_out, S->hp.slice, sizeof(double) * 2 * S->pl.nslices, cudaMemcpyDeviceToDevice, stream);
    return check_launch("slab node");
}

__global__ void k_decide_gathered(const SeriesParams *__restrict__ Pp, const double *slices, int nslices) {
    const SeriesParams &P = *Pp;
    if (P.state->done) return;
    decide_gathered(P, P.state->k + 1, slices, nslices);
}

// Shared by the slab and the row-block (CSR) series: both workspace layouts
// keep the device SeriesParams at offset 0.
int dist_decide(const void *ws, const double *slices_all, int nslices, cudaStream_t stream) {
    if (!ws || !slices_all || nslices < 1) return set_error(ES_ERR_ARG, "bad gathered slices");
    k_decide_gathered<<<1, 32, 0, stream>>>(reinterpret_cast<const SeriesParams *>(ws), slices_all, nslices);
    return check_launch("slab decide");
}

int dist_end(const void *ws, cudaStream_t stream) {
    SeriesSetup *S;
    int rc = dist_get(ws, S);
    if (rc) return rc;
    k_series_finalize<<<148 * 8, 256, 0, stream>>>(S->dparams, S->n);
    rc = check_launch("slab series finalize");
    std::lock_guard<std::mutex> lk(g_dist_mu);
    g_dist.erase(ws);
    return rc;
}

// ----- peer-memory (NVLink P2P) slab series ------------------------------------
//
// One CUDA graph per series and rank, no host involvement per node: node k
// writes its boundary planes of w_k into the neighbours' halo buffers
// (parity (k + 1) & 1) from the consumer epilogue, the slice kernel writes
// this slab's per-chunk sums into every rank's table and joins the round
// barrier, and every rank evaluates the identical stopping test on the full
// table (rank order = global z order: with chunk-aligned slabs the sums are
// bitwise those of one GPU).

int stencil_nslices(const es_stencil_desc *d) { return plan_stencil(d, {}, true).nslices; }

int run_p2p_series(const es_stencil_desc *d, const es_p2p_desc *x, const double *v, double *p_out, const double *dd,
                   const double *xi, int ndd, double alpha, double shift, double tol, const double *gdiag, void *ws,
                   size_t ws_bytes, cudaStream_t stream) {
    if (ndd < 2) return set_error(ES_ERR_ARG, "a peer-memory series needs ndd >= 2");
    if (x->nranks < 1 || x->rank < 0 || x->rank >= x->nranks || !x->rank_slices || !x->rank_arrive ||
        !x->arrive_local)
        return set_error(ES_ERR_ARG, "bad peer-memory descriptor");
    if ((x->halo_lo[0] == nullptr) != (x->halo_lo[1] == nullptr) || (x->halo_hi[0] == nullptr) != (x->halo_hi[1] == nullptr) ||
        (x->peer_lo[0] == nullptr) != (x->halo_lo[0] == nullptr) || (x->peer_hi[0] == nullptr) != (x->halo_hi[0] == nullptr))
        return set_error(ES_ERR_ARG, "halo / peer buffers must come in parity pairs, one per existing neighbour");
    const bool want_tb = x->halo_planes == 2;
    if (want_tb && gdiag && ((x->halo_lo[0] && !x->gdiag_lo) || (x->halo_hi[0] && !x->gdiag_hi)))
        return set_error(ES_ERR_ARG, "two-node peer series with g' need the neighbours' g' planes");
    SeriesSetup S;
    int rc = prepare_series(d, v, p_out, dd, xi, ndd, alpha, shift, tol, gdiag, x->halo_lo[0], x->halo_hi[0], false, ws,
                            ws_bytes, S, stream, x->halo_lo[1], x->halo_hi[1], want_tb ? 2 : 0, x->gdiag_lo,
                            x->gdiag_hi);
    if (rc) return rc;
    if (!S.pl.tma || S.pl.dim2) return set_error(ES_ERR_ARG, "peer-memory series need the 3D TMA path");
    if (want_tb != S.tb)
        return set_error(ES_ERR_ARG, "halo_planes = 2 needs a two-node slab (Dirichlet / Neumann, no coefficient "
                                     "array, lz >= 2, ES_TB not 0)");
    if (x->slice_offset < 0 || x->slice_offset + S.pl.nslices > x->total_slices)
        return set_error(ES_ERR_ARG, "slice offset / total do not cover this slab's %d slices", S.pl.nslices);
    if (S.tb && env_int("ES_PEER_IN_NODE", gdiag ? 1 : 0)) {
        // x2: the pass itself pushes the boundary planes to the neighbours
        // (overlapped with the sweep); the slice kernel only fences and joins.
        // Default for the Rosenbrock (g') series -- C4 -- where it measured
        // 75.8 vs 79.3 ms (2 emulated 1024^3 slabs, 16 nodes); without g' the
        // PEER build of the pass spills and the copy stays in the slice kernel
        // (64.6 vs 67.5 ms), tools/p2p_timing.py
        S.nf = gdiag ? pick_node_tb<true, true>(d->coeff_kind) : pick_node_tb<false, true>(d->coeff_kind);
        finish_tma_plan(S.lp, (const void *)S.nf,
                        gdiag ? (size_t)TbLayout<true>::BYTES : (size_t)TbLayout<false>::BYTES, TB_THREADS);
        S.hp.peer_in_node = 1;
    }
    SeriesParams &hp = S.hp;
    hp.p2p = 1;
    hp.nranks = x->nranks;
    hp.rank = x->rank;
    hp.slice_off = x->slice_offset;
    hp.total_slices = x->total_slices;
    for (int i = 0; i < 2; ++i) {
        hp.peer_lo[i] = x->peer_lo[i];
        hp.peer_hi[i] = x->peer_hi[i];
    }
    hp.rank_slices = x->rank_slices;
    hp.rank_arrive = x->rank_arrive;
    hp.arrive_local = x->arrive_local;
    hp.base = x->base;
    hp.timeout_ns = x->timeout_ns > 0 ? x->timeout_ns : 10000000000ll;
    NodeFn sf = S.tb ? k_slice_p2p2 : k_slice_p2p;
    GraphKernel gk[2] = {{(const void *)S.nf, S.lp.grid, S.lp.block, S.lp.smem},
                         {(const void *)sf, dim3((unsigned)S.pl.nslices), dim3(256), 0}};
    unsigned long long handle = 0;
    cudaGraphExec_t ge = series_graph(gk, 2, S.dparams, &handle);
    if (ge) hp.cond = handle;
    k_series_init<<<1, 256, 0, stream>>>(hp, S.dparams);
    const int64_t plane = d->nx * d->ny;
    const unsigned ig = (unsigned)std::min<int64_t>(std::max<int64_t>(1, (plane / 2 + 255) / 256), 148);
    if (S.tb)
        k_p2p_init2<<<ig, 256, 0, stream>>>(S.dparams, plane, d->lz);
    else
        k_p2p_init<<<ig, 256, 0, stream>>>(S.dparams, plane, d->lz);
    rc = check_launch("peer-memory series init");
    if (rc) return rc;
    if (ge) {
        if (cudaGraphLaunch(ge, stream) != cudaSuccess) return check_launch("peer-memory series graph");
    } else {
        // one launch pair per node at most (a two-node series may run one-node passes)
        for (int k = 1; k < ndd; ++k) {
            S.nf<<<S.lp.grid, S.lp.block, S.lp.smem, stream>>>(S.dparams);
            sf<<<(unsigned)S.pl.nslices, 256, 0, stream>>>(S.dparams);
        }
    }
    k_series_finalize<<<148 * 8, 256, 0, stream>>>(S.dparams, S.n);
    return check_launch("peer-memory series");
}

}  // namespace es
