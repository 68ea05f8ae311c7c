// Integrator-stage element-wise kernels: combustion nonlinearity with the
// on-device domain check (integrator.py:35-54, _core.pyx:325-348), its
// build-defined Jacobian diagonal with min/max, the step combination
// y + h z (integrator.py:187), the rescue combination (v1 + v2)/2
// (matfunc.py:371), and the observer's max |u| (integrator.py:236).
#include "es_common.cuh"
#include "es_host.h"

namespace es {

static unsigned grid_for(int64_t n) {
    const int64_t g = (n + 255) / 256;
    return (unsigned)std::min<int64_t>(std::max<int64_t>(g, 1), 148 * 32);
}

#define ES_GRID_STRIDE(i, n) \
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

// out = (1/4 (2 - u)) exp(20 (1 - 1/u)); first index with u <= 0 -> *bad
__global__ void k_combustion(const double *__restrict__ u, double *__restrict__ out, int64_t n,
                             unsigned long long *bad) {
    ES_GRID_STRIDE(i, n) {
        const double x = u[i];
        if (x <= 0.0) atomicMin(bad, (unsigned long long)i);
        const double r = __drcp_rn(x);  // = div(1.0, x), correctly rounded either way
        const double t = mul(20.0, sub(1.0, r));
        out[i] = mul(mul(0.25, sub(2.0, x)), exp(t));
    }
}

// g'(u) = e^{20(1-1/u)} (5 (2-u)/u^2 - 1/4); minmax[0] = min, [1] = max
__global__ void k_combustion_jac(const double *__restrict__ u, double *__restrict__ out, int64_t n,
                                 unsigned long long *mm) {
    unsigned long long lo = ~0ull, hi = 0ull;
    ES_GRID_STRIDE(i, n) {
        const double x = u[i];
        const double r = __drcp_rn(x);  // = div(1.0, x), correctly rounded either way
        const double e = exp(mul(20.0, sub(1.0, r)));
        const double q = mul(mul(5.0, sub(2.0, x)), mul(r, r));
        const double gp = mul(e, sub(q, 0.25));
        out[i] = gp;
        const unsigned long long o = ord(gp);
        lo = o < lo ? o : lo;
        hi = o > hi ? o : hi;
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        const unsigned long long a = __shfl_xor_sync(0xffffffffu, lo, s);
        const unsigned long long b = __shfl_xor_sync(0xffffffffu, hi, s);
        lo = a < lo ? a : lo;
        hi = b > hi ? b : hi;
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(mm, lo);
        atomicMax(mm + 1, hi);
    }
}

__global__ void k_ord_to_double(unsigned long long *mm, double *out) {
    if (threadIdx.x < 2) {
        const unsigned long long o = mm[threadIdx.x];
        const unsigned long long b = (o >> 63) ? (o & 0x7fffffffffffffffull) : ~o;
        out[threadIdx.x] = __longlong_as_double((long long)b);
    }
}

__global__ void k_axpy(const double *__restrict__ y, const double *__restrict__ z, double h,
                       double *__restrict__ out, int64_t n) {
    ES_GRID_STRIDE(i, n) out[i] = add(y[i], mul(h, z[i]));
}

__global__ void k_scale(const double *__restrict__ x, double s, double *__restrict__ out, int64_t n) {
    ES_GRID_STRIDE(i, n) out[i] = mul(s, x[i]);
}

__global__ void k_half_sum(const double *__restrict__ a, const double *__restrict__ b,
                           double *__restrict__ out, int64_t n) {
    ES_GRID_STRIDE(i, n) out[i] = mul(0.5, add(a[i], b[i]));
}

// |x| >= 0 so the raw bit pattern orders correctly (NaN sorts above inf)
__global__ void k_max_abs(const double *__restrict__ x, int64_t n, unsigned long long *out) {
    unsigned long long m = 0ull;
    ES_GRID_STRIDE(i, n) {
        const unsigned long long b = (unsigned long long)__double_as_longlong(fabs(x[i]));
        m = b > m ? b : m;
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        const unsigned long long o = __shfl_xor_sync(0xffffffffu, m, s);
        m = o > m ? o : m;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

__global__ void k_fill_u64(unsigned long long *p, unsigned long long a, unsigned long long b) {
    if (threadIdx.x == 0) p[0] = a;
    if (threadIdx.x == 1) p[1] = b;
}

// host launchers for the fused steps (step.cu)
int launch_combustion(const double *u, double *out, int64_t n, unsigned long long *bad_dev, cudaStream_t st) {
    k_fill_u64<<<1, 32, 0, st>>>(bad_dev, (unsigned long long)n, 0ull);
    if (n > 0) k_combustion<<<grid_for(n), 256, 0, st>>>(u, out, n, bad_dev);
    return check_launch("combustion");
}

int launch_fill_u64(unsigned long long *p, unsigned long long a, unsigned long long b, cudaStream_t st) {
    k_fill_u64<<<1, 32, 0, st>>>(p, a, b);
    return check_launch("fill");
}

int launch_axpy(const double *y, const double *z, double h, double *out, int64_t n, cudaStream_t st) {
    if (n > 0) k_axpy<<<grid_for(n), 256, 0, st>>>(y, z, h, out, n);
    return check_launch("axpy");
}

int launch_scale(const double *x, double s, double *out, int64_t n, cudaStream_t st) {
    if (n > 0) k_scale<<<grid_for(n), 256, 0, st>>>(x, s, out, n);
    return check_launch("scale");
}

// ----- per-thread scratch (device word pair + pinned host pair) --------------

struct Scratch {
    int device = -1;
    unsigned long long *dev = nullptr;
    unsigned long long *host = nullptr;
};
static thread_local Scratch t_scratch;

static int scratch(Scratch *&s) {
    s = &t_scratch;
    const int dev = current_device();
    if (s->device != dev) {
        if (cudaMalloc(&s->dev, 4 * sizeof(unsigned long long)) != cudaSuccess ||
            cudaMallocHost(&s->host, 4 * sizeof(unsigned long long)) != cudaSuccess)
            return check_launch("scratch alloc");
        s->device = dev;
    }
    return ES_OK;
}

}  // namespace es

using namespace es;

extern "C" int es_combustion_pointwise(const double *u, double *out, int64_t n, int64_t *first_bad_host,
                                       void *stream) {
    if (first_bad_host) *first_bad_host = -1;
    if (n <= 0) return ES_OK;
    if (!u || !out) return set_error(ES_ERR_ARG, "null pointer");
    cudaStream_t st = (cudaStream_t)stream;
    Scratch *s;
    int rc = scratch(s);
    if (rc) return rc;
    k_fill_u64<<<1, 32, 0, st>>>(s->dev, (unsigned long long)n, 0ull);
    k_combustion<<<grid_for(n), 256, 0, st>>>(u, out, n, s->dev);
    rc = check_launch("combustion");
    if (rc) return rc;
    cudaMemcpyAsync(s->host, s->dev, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return check_launch("combustion sync");
    const unsigned long long bad = s->host[0];
    if (bad < (unsigned long long)n) {
        if (first_bad_host) *first_bad_host = (int64_t)bad;
        return set_error(ES_ERR_DOMAIN, "combustion nonlinearity undefined at index %lld", (long long)bad);
    }
    return ES_OK;
}

extern "C" int es_combustion_jacobian(const double *u, double *out, double *minmax_dev, int64_t n, void *stream) {
    if (n <= 0) return ES_OK;
    cudaStream_t st = (cudaStream_t)stream;
    Scratch *s;
    int rc = scratch(s);
    if (rc) return rc;
    k_fill_u64<<<1, 32, 0, st>>>(s->dev, ~0ull, 0ull);
    k_combustion_jac<<<grid_for(n), 256, 0, st>>>(u, out, n, s->dev);
    k_ord_to_double<<<1, 32, 0, st>>>(s->dev, minmax_dev);
    return check_launch("combustion jacobian");
}

extern "C" int es_axpy(const double *y, const double *z, double h, double *out, int64_t n, void *stream) {
    if (n <= 0) return ES_OK;
    k_axpy<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(y, z, h, out, n);
    return check_launch("axpy");
}

extern "C" int es_scale(const double *x, double s, double *out, int64_t n, void *stream) {
    if (n <= 0) return ES_OK;
    k_scale<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(x, s, out, n);
    return check_launch("scale");
}

extern "C" int es_half_sum(const double *a, const double *b, double *out, int64_t n, void *stream) {
    if (n <= 0) return ES_OK;
    k_half_sum<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(a, b, out, n);
    return check_launch("half sum");
}

extern "C" int es_max_abs(const double *x, int64_t n, double *out_dev, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    unsigned long long *o = reinterpret_cast<unsigned long long *>(out_dev);
    cudaMemsetAsync(o, 0, sizeof(unsigned long long), st);
    if (n > 0) k_max_abs<<<grid_for(n), 256, 0, st>>>(x, n, o);
    return check_launch("max abs");
}
