// Probe of the random-gather ceiling behind the CSR node: y[i] = x[idx[i]]
// (idx uniform over the x length, int32, streamed; y streamed) for x sizes
// from L1-resident to HBM-resident, LDG vs texture, a few unroll depths.
// Not part of the product:  nvcc -O3 -gencode arch=compute_100a,code=sm_100a
//   tools/gather_probe.cu -o tools/gather_probe && tools/gather_probe
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

template <int U, bool TEX>
__global__ void k_gather(const double *__restrict__ x, cudaTextureObject_t tx, const int *__restrict__ idx,
                         double *__restrict__ y, long long n) {
    long long i0 = (long long)blockIdx.x * blockDim.x * U + threadIdx.x;
    const long long stride = (long long)gridDim.x * blockDim.x * U;
    for (; i0 < n; i0 += stride) {
        int c[U];
        double v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            long long i = i0 + (long long)u * blockDim.x;
            c[u] = i < n ? __ldcs(idx + i) : 0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if constexpr (TEX) {
                int2 t = tex1Dfetch<int2>(tx, c[u]);
                v[u] = __hiloint2double(t.y, t.x);
            } else {
                v[u] = __ldg(x + c[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            long long i = i0 + (long long)u * blockDim.x;
            if (i < n) __stcs(y + i, v[u]);
        }
    }
}

template <int U, bool TEX>
float run(const double *x, cudaTextureObject_t tx, const int *idx, double *y, long long n, int blocks) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int w = 0; w < 3; ++w) k_gather<U, TEX><<<blocks, 256>>>(x, tx, idx, y, n);
    cudaEventRecord(a);
    const int reps = 10;
    for (int r = 0; r < reps; ++r) k_gather<U, TEX><<<blocks, 256>>>(x, tx, idx, y, n);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}

int main() {
    const long long n = 54525880;  // the C5 nonzero count
    int *idx;
    double *y, *x;
    const long long xmax = 1ll << 25;  // 256 MiB of doubles
    cudaMalloc(&idx, n * 4);
    cudaMalloc(&y, n * 8);
    cudaMalloc(&x, xmax * 8);
    cudaMemset(x, 0, xmax * 8);
    std::vector<int> h(n);
    for (long long xn : {1ll << 12, 1ll << 18, 1ll << 20, 1ll << 22, 1ll << 25}) {
        unsigned long long s = 88172645463325252ull;
        for (long long i = 0; i < n; ++i) {
            s ^= s << 13; s ^= s >> 7; s ^= s << 17;
            h[i] = (int)(s % (unsigned long long)xn);
        }
        cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
        cudaResourceDesc rd = {};
        rd.resType = cudaResourceTypeLinear;
        rd.res.linear.devPtr = x;
        rd.res.linear.desc = cudaCreateChannelDesc<int2>();
        rd.res.linear.sizeInBytes = xn * 8;
        cudaTextureDesc td = {};
        cudaTextureObject_t tx;
        cudaCreateTextureObject(&tx, &rd, &td, nullptr);
        for (int bps : {4, 8}) {
            const int blocks = 148 * bps;
            float t1 = run<1, false>(x, tx, idx, y, n, blocks);
            float t4 = run<4, false>(x, tx, idx, y, n, blocks);
            float t8 = run<8, false>(x, tx, idx, y, n, blocks);
            float tt4 = run<4, true>(x, tx, idx, y, n, blocks);
            float tt8 = run<8, true>(x, tx, idx, y, n, blocks);
            printf("x=%8.2f MiB blocks/SM=%d  LDG u1 %.1f us  u4 %.1f us  u8 %.1f us  TEX u4 %.1f us  u8 %.1f us"
                   "  (best %.1f Ggather/s)\n",
                   xn * 8.0 / (1 << 20), bps, t1 * 1e3, t4 * 1e3, t8 * 1e3, tt4 * 1e3, tt8 * 1e3,
                   n / (1e6 * std::min(std::min(std::min(t1, t4), std::min(t8, tt4)), tt8)));
        }
        cudaDestroyTextureObject(tx);
    }
    printf("stream floor: %lld B idx+y per pass\n", n * 12);
    return cudaGetLastError() != cudaSuccess;
}
