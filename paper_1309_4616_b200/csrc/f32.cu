// Single-precision plain applies: the reference's compiled core instantiates
// its stencil and combustion kernels for float as well as double
// (_core.pyx:176-226 `_stencil_impl[float]`, :323-348), with the weights,
// alpha and beta cast to float and every operation rounded in float
// (-ffp-contract=off).  These kernels restate that arithmetic with explicit
// round-to-nearest float intrinsics, so stencil applies are bitwise equal.
// Not a hot path: the Newton-Leja series is always fp64 (matfunc.py:284,
// :292 upcast), so one thread per point, no staging.
#include <algorithm>

#include "es_common.cuh"
#include "es_host.h"

namespace es {

namespace {

struct F32Slab {
    int64_t nx, ny, lz, z0;
    float wx, wy, wz, alpha, beta;
    int mode, at_lo, at_hi;
    const float *u;
    float *out;
    const float *coeff;      // slab-local (lz, ny, nx), or null
    const float *faces[6];   // ES_MODE_FACES: fx_lo, fx_hi (nz_total, ny); fy_* (nz_total, nx); fz_* (ny, nx)
    const float *halo_lo, *halo_hi;
};

ES_DEV float fadd(float a, float b) { return __fadd_rn(a, b); }
ES_DEV float fsub(float a, float b) { return __fsub_rn(a, b); }
ES_DEV float fmul(float a, float b) { return __fmul_rn(a, b); }

// Ghost precedence of _core.pyx:60-114: interior, halo (z only), periodic,
// face value (z faces only at the physical boundary), then the build-defined
// Neumann mirror, else zero.
__global__ void k_stencil_f32(const F32Slab a) {
    const int64_t plane = a.nx * a.ny, n = plane * a.lz;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t ix = i % a.nx, iy = (i / a.nx) % a.ny, iz = i / plane;
        const float *u = a.u;
        const float c = u[i];
        const int periodic = a.mode == ES_MODE_PERIODIC, faces = a.mode == ES_MODE_FACES,
                  neumann = a.mode == ES_MODE_NEUMANN;
        const float xm = ix > 0 ? u[i - 1] : periodic ? u[i + a.nx - 1]
                        : faces ? a.faces[0][(a.z0 + iz) * a.ny + iy] : neumann ? c : 0.0f;
        const float xp = ix < a.nx - 1 ? u[i + 1] : periodic ? u[i - (a.nx - 1)]
                        : faces ? a.faces[1][(a.z0 + iz) * a.ny + iy] : neumann ? c : 0.0f;
        const float ym = iy > 0 ? u[i - a.nx] : periodic ? u[i + (a.ny - 1) * a.nx]
                        : faces ? a.faces[2][(a.z0 + iz) * a.nx + ix] : neumann ? c : 0.0f;
        const float yp = iy < a.ny - 1 ? u[i + a.nx] : periodic ? u[i - (a.ny - 1) * a.nx]
                        : faces ? a.faces[3][(a.z0 + iz) * a.nx + ix] : neumann ? c : 0.0f;
        const int64_t off = iy * a.nx + ix;
        const float zm = iz > 0 ? u[i - plane] : a.halo_lo ? a.halo_lo[off] : periodic ? u[(a.lz - 1) * plane + off]
                        : (faces && a.at_lo) ? a.faces[4][off] : (neumann && a.at_lo) ? c : 0.0f;
        const float zp = iz < a.lz - 1 ? u[i + plane] : a.halo_hi ? a.halo_hi[off] : periodic ? u[off]
                        : (faces && a.at_hi) ? a.faces[5][off] : (neumann && a.at_hi) ? c : 0.0f;
        const float c2 = fmul(2.0f, c);
        const float sx = fmul(fsub(fsub(c2, xm), xp), a.wx);
        const float sy = fmul(fsub(fsub(c2, ym), yp), a.wy);
        const float sz = fmul(fsub(fsub(c2, zm), zp), a.wz);
        float lap = fadd(fadd(sx, sy), sz);
        if (a.coeff) lap = fmul(a.coeff[i], lap);
        a.out[i] = fadd(fmul(a.alpha, lap), fmul(a.beta, c));
    }
}

// (1/4 (2 - u)) expf(20 (1 - 1/u)) (_core.pyx:323-336); CUDA's expf is
// within 2 ulp of libm's, so this one is close, not bitwise.
__global__ void k_combustion_f32(const float *u, float *out, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float r = __fdiv_rn(1.0f, u[i]);
        const float t = fmul(20.0f, fsub(1.0f, r));
        out[i] = fmul(fmul(0.25f, fsub(2.0f, u[i])), expf(t));
    }
}

unsigned grid_for(int64_t n) { return (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16); }

}  // namespace

int launch_stencil_f32(const es_stencil_desc *d, const float *u, float *out, double alpha, double beta,
                       const float *coeff, const float *const *faces, const float *halo_lo, const float *halo_hi,
                       cudaStream_t stream) {
    F32Slab a = {};
    a.nx = d->nx;
    a.ny = d->ny;
    a.lz = d->lz;
    a.z0 = d->z0;
    a.wx = (float)d->wx;  // the reference casts weights, alpha, beta to float (_core.pyx:220-222)
    a.wy = (float)d->wy;
    a.wz = (float)d->wz;
    a.alpha = (float)alpha;
    a.beta = (float)beta;
    a.mode = d->mode;
    a.at_lo = d->z0 == 0;
    a.at_hi = d->z0 + d->lz == d->nz_total;
    a.u = u;
    a.out = out;
    a.coeff = coeff;
    for (int i = 0; i < 6; ++i) a.faces[i] = faces ? faces[i] : nullptr;
    if (d->mode == ES_MODE_FACES)
        for (int i = 0; i < 6; ++i)
            if (!a.faces[i]) return set_error(ES_ERR_ARG, "faces mode needs six face arrays");
    a.halo_lo = halo_lo;
    a.halo_hi = halo_hi;
    const int64_t n = d->nx * d->ny * d->lz;
    if (n == 0) return ES_OK;
    k_stencil_f32<<<grid_for(n), 256, 0, stream>>>(a);
    return check_launch("stencil apply (f32)");
}

int launch_combustion_f32(const float *u, float *out, int64_t n, cudaStream_t stream) {
    if (n == 0) return ES_OK;
    k_combustion_f32<<<grid_for(n), 256, 0, stream>>>(u, out, n);
    return check_launch("combustion (f32)");
}

}  // namespace es
