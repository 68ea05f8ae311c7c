// The device-side series loop: a CUDA graph whose single conditional WHILE
// node runs the node kernel(s) of a Newton-Leja series until the deciding
// CTA clears the condition (cudaGraphSetConditional in series.cuh:decide).
// One graph launch per series, no host round trip per node.  The loop body
// holds UNROLL copies of the node's kernels: one WHILE iteration costs
// ~5.4 us on B200 whatever the body (tools/graph_probe.cu), so unrolling
// amortises it; copies after the decision return at their first load of
// the series state.  Instantiated graphs are cached per (kernels,
// launch shapes, device-parameter slot, device): every series re-publishes
// its parameters into the same workspace slot, so a cached graph stays valid.
#include <algorithm>
#include <map>
#include <mutex>
#include <vector>

#include "es_host.h"

namespace es {

namespace {

struct Entry {
    cudaGraphExec_t exec = nullptr;
    cudaGraphConditionalHandle handle = 0;
};

std::mutex g_mu;
std::map<std::vector<unsigned long long>, Entry> g_cache;

bool build(const GraphKernel *ks, int nk, int unroll, const void *dparams, Entry &e) {
    cudaGraph_t graph = nullptr;
    if (cudaGraphCreate(&graph, 0) != cudaSuccess) return false;
    bool ok = false;
    do {
        if (cudaGraphConditionalHandleCreate(&e.handle, graph, 1, cudaGraphCondAssignDefault) != cudaSuccess) break;
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = e.handle;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t cnode;
        if (cudaGraphAddNode(&cnode, graph, nullptr, 0, &cp) != cudaSuccess) break;
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        void *args[] = {(void *)&dparams};
        cudaGraphNode_t prev = nullptr;
        bool added = true;
        for (int i = 0; i < nk * unroll && added; ++i) {
            cudaKernelNodeParams kp = {};
            const GraphKernel &kk = ks[i % nk];
            kp.func = const_cast<void *>(kk.fn);
            kp.gridDim = kk.grid;
            kp.blockDim = kk.block;
            kp.sharedMemBytes = (unsigned)kk.smem;
            kp.kernelParams = args;
            cudaGraphNode_t node;
            added = cudaGraphAddKernelNode(&node, body, prev ? &prev : nullptr, prev ? 1 : 0, &kp) == cudaSuccess;
            prev = node;
        }
        if (!added) break;
        ok = cudaGraphInstantiate(&e.exec, graph, 0) == cudaSuccess;
    } while (false);
    cudaGraphDestroy(graph);
    return ok;
}

}  // namespace

cudaGraphExec_t series_graph(const GraphKernel *ks, int nk, const void *dparams, unsigned long long *handle) {
    if (env_int("ES_NO_GRAPH", 0)) return nullptr;
    const int unroll = std::max(1, env_int("ES_GRAPH_UNROLL", 4));
    std::vector<unsigned long long> key;
    key.push_back((unsigned long long)(uintptr_t)dparams);
    key.push_back((unsigned long long)unroll);
    key.push_back((unsigned long long)current_device());
    for (int i = 0; i < nk; ++i) {
        key.push_back((unsigned long long)(uintptr_t)ks[i].fn);
        key.push_back(ks[i].grid.x);
        key.push_back(ks[i].grid.y);
        key.push_back(ks[i].grid.z);
        key.push_back(ks[i].block.x * 65536ull + ks[i].block.y);
        key.push_back(ks[i].smem);
    }
    std::lock_guard<std::mutex> lk(g_mu);
    if (env_int("ES_GRAPH_NOCACHE", 0)) key.push_back(g_cache.size() + 1);  // diagnostics: a fresh graph per series
    auto it = g_cache.find(key);
    if (it == g_cache.end()) {
        Entry e;
        if (!build(ks, nk, unroll, dparams, e)) {
            cudaGetLastError();  // graphs unavailable: the caller launches the nodes itself
            return nullptr;
        }
        it = g_cache.emplace(key, e).first;
    }
    *handle = (unsigned long long)it->second.handle;
    return it->second.exec;
}

}  // namespace es
