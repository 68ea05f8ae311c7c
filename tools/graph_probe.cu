// Per-iteration cost of a conditional WHILE graph (the series loop's
// skeleton): body = 1 or 2 trivial kernels; the last one counts down and
// clears the condition.  Not part of the product.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/graph_probe.cu -o tools/graph_probe
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_touch(int *x) {
    if (threadIdx.x == 0 && blockIdx.x == 0) x[1] += 1;
}
__global__ void k_count(int *x, cudaGraphConditionalHandle h) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        if (--x[0] <= 0) cudaGraphSetConditional(h, 0);
    }
}

float run(int nbody, int iters, unsigned grid) {
    int *x;
    cudaMalloc(&x, 8);
    cudaGraph_t g;
    cudaGraphCreate(&g, 0);
    cudaGraphConditionalHandle h;
    cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t cn;
    cudaGraphAddNode(&cn, g, nullptr, 0, &cp);
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    cudaGraphNode_t prev = nullptr, n;
    for (int i = 0; i < nbody; ++i) {
        cudaKernelNodeParams kp = {};
        void *a1[] = {&x};
        void *a2[] = {&x, &h};
        kp.func = i == nbody - 1 ? (void *)k_count : (void *)k_touch;
        kp.gridDim = dim3(grid);
        kp.blockDim = dim3(256);
        kp.kernelParams = i == nbody - 1 ? a2 : a1;
        cudaGraphAddKernelNode(&n, body, prev ? &prev : nullptr, prev ? 1 : 0, &kp);
        prev = n;
    }
    cudaGraphExec_t ge;
    cudaGraphInstantiate(&ge, g, 0);
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
        int init[2] = {iters, 0};
        cudaMemcpy(x, init, 8, cudaMemcpyHostToDevice);
        cudaEventRecord(a, s);
        cudaGraphLaunch(ge, s);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    return best * 1e3f / iters;
}

int main() {
    for (unsigned grid : {1u, 148u, 444u})
        for (int nb : {1, 2})
            printf("grid %4u  body kernels %d: %.2f us per iteration\n", grid, nb, run(nb, 200, grid));
    return 0;
}
