// Deterministic on-device stopping test for the Newton-Leja series
// (matfunc.py:297-318): partial sums of w^2 and p^2 are reduced in a fixed,
// partition-independent order (per slice: tiles in index order; then slices
// in index order) by the last CTA of each chunk and then the last chunk; the
// final CTA evaluates |dd_k| ||w_k|| <= tol ||p_k|| and updates the series
// state, ending a graph-level while loop when the series is done.
#pragma once

#include "stencil.cuh"

namespace es {

// Barrier over the participating threads: the whole CTA (NT == 0) or the
// first NT threads via named barrier 1 (warp-specialised kernels, where the
// producer warp is busy elsewhere).
template <int NT>
ES_DEV void group_sync() {
    if constexpr (NT == 0) {
        __syncthreads();
    } else {
        asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
    }
}

// The stopping test of matfunc.py:302-311 on the reduced sums (one thread).
ES_DEV void decide(const SeriesParams &P, int k, double sumw, double sump) {
    SeriesState &st = *P.state;
    // |dd_k|: real series read dd directly; complex series pass numpy's abs(dd)
    const double adk = P.ddabs ? P.ddabs[k] : fabs(P.dd[k]);
    const double term = mul(adk, sqrt_rn(sumw));
    const double pn = sqrt_rn(sump);
    st.k = k;
    st.last_term = term;
    st.last_pnorm = pn;
    bool stop = false;
    if (P.tol > 0.0) {
        if (term <= mul(P.tol, pn)) {
            st.consecutive += 1;
            if (st.consecutive >= 2) {
                stop = true;
                st.converged = 1;
            }
        } else {
            st.consecutive = 0;
        }
    }
    if (!stop && k >= P.ndd - 1) {
        stop = true;
        st.converged = P.tol == 0.0 ? 1 : 0;
    }
    if (stop) {
        st.done = 1;
        if (P.cond) cudaGraphSetConditional((cudaGraphConditionalHandle)P.cond, 0);
    }
}

// Returns true in the (single) CTA that made the decision.  Called by every
// thread of the group after the group's partials for this (chunk, tile) are
// in P.part.
template <int NT = 0>
ES_DEV bool reduce_and_decide(const SeriesParams &P, int k, int chunk, int64_t slice_b, int64_t slice_e) {
    __shared__ int s_last;
    const int tid = NT ? (int)threadIdx.x : (int)(threadIdx.x + threadIdx.y * blockDim.x);
    const int nthr = NT ? NT : (int)(blockDim.x * blockDim.y);
    const int lane = tid & 31, warp = tid >> 5, nwarps = nthr >> 5;

    __threadfence();
    group_sync<NT>();
    if (tid == 0) s_last = atomicAdd(&P.chunk_cnt[chunk], 1u) == (unsigned)P.ntiles - 1u;
    group_sync<NT>();
    const bool last_chunk_tile = s_last;
    group_sync<NT>();  // s_last is reused below
    if (!last_chunk_tile) return false;
    __threadfence();

    // chunk reducer: slice sums over tiles (lane-strided, then xor tree)
    for (int64_t s = slice_b + warp; s < slice_e; s += nwarps) {
        double aw = 0.0, ap = 0.0;
        const double *row = P.part + s * (int64_t)P.ntiles * 2;
        for (int t = lane; t < P.ntiles; t += 32) {
            aw = add(aw, __ldcg(row + 2 * t));
            ap = add(ap, __ldcg(row + 2 * t + 1));
        }
        aw = warp_sum(aw);
        ap = warp_sum(ap);
        if (lane == 0) {
            P.slice[2 * s] = aw;
            P.slice[2 * s + 1] = ap;
        }
    }
    __threadfence();
    group_sync<NT>();
    if (P.dist) {  // multi-GPU: the caller gathers the slices of all ranks and decides
        if (tid == 0) P.chunk_cnt[chunk] = 0u;
        return false;
    }
    if (tid == 0) s_last = atomicAdd(P.global_cnt, 1u) == (unsigned)P.nchunks - 1u;
    group_sync<NT>();
    const bool last_chunk = s_last;
    group_sync<NT>();
    if (!last_chunk) return false;
    __threadfence();

    if (warp == 0) {
        double aw = 0.0, ap = 0.0;
        for (int64_t s = lane; s < P.nslices; s += 32) {
            aw = add(aw, __ldcg(P.slice + 2 * s));
            ap = add(ap, __ldcg(P.slice + 2 * s + 1));
        }
        aw = warp_sum(aw);
        ap = warp_sum(ap);
        if (lane == 0) decide(P, k, aw, ap);
    }
    // re-arm the tickets for the next node
    for (int i = tid; i < P.nchunks; i += nthr) P.chunk_cnt[i] = 0u;
    if (tid == 0) *P.global_cnt = 0u;
    return true;
}

// Separate reduction step of the TMA node (one CTA per slice = z-chunk):
// slice c's entries (tile, warp partials) are summed thread-strided, warp
// trees, warps in order; the last CTA sums the slices in order and decides.
// Slice c's sums (thread 0 of the CTA gets them): entries thread-strided,
// warp trees, warps in order.
ES_DEV void cta_slice_sum(const SeriesParams &P, int c, double &a_out, double &b_out, const double *part = nullptr) {
    __shared__ double s_w[32], s_p[32];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5, nw = blockDim.x >> 5;
    const double *row = (part ? part : P.part) + (int64_t)c * P.ntiles * 2;
    double aw = 0.0, ap = 0.0;
    for (int e = t; e < P.ntiles; e += blockDim.x) {
        aw = add(aw, __ldcg(row + 2 * e));
        ap = add(ap, __ldcg(row + 2 * e + 1));
    }
    aw = warp_sum(aw);
    ap = warp_sum(ap);
    if (lane == 0) {
        s_w[warp] = aw;
        s_p[warp] = ap;
    }
    __syncthreads();
    if (t == 0) {
        double a = s_w[0], b = s_p[0];
        for (int w = 1; w < nw; ++w) {
            a = add(a, s_w[w]);
            b = add(b, s_p[w]);
        }
        a_out = a;
        b_out = b;
    }
}

ES_DEV void slice_reduce_decide(const SeriesParams &P, int k) {
    __shared__ double s_w[32], s_p[32];
    __shared__ int s_last;
    const int c = blockIdx.x, t = threadIdx.x, lane = t & 31, warp = t >> 5, nw = blockDim.x >> 5;
    const double *row = P.part + (int64_t)c * P.ntiles * 2;
    double aw = 0.0, ap = 0.0;
    for (int e = t; e < P.ntiles; e += blockDim.x) {
        aw = add(aw, __ldcg(row + 2 * e));
        ap = add(ap, __ldcg(row + 2 * e + 1));
    }
    aw = warp_sum(aw);
    ap = warp_sum(ap);
    if (lane == 0) {
        s_w[warp] = aw;
        s_p[warp] = ap;
    }
    __syncthreads();
    if (t == 0) {
        double a = s_w[0], b = s_p[0];
        for (int w = 1; w < nw; ++w) {
            a = add(a, s_w[w]);
            b = add(b, s_p[w]);
        }
        P.slice[2 * c] = a;
        P.slice[2 * c + 1] = b;
    }
    if (P.dist) return;  // multi-GPU: the caller gathers the slices of all slabs
    if (t == 0) {
        __threadfence();
        s_last = atomicAdd(P.global_cnt, 1u) == gridDim.x - 1u;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (warp == 0) {
        double sw = 0.0, sp = 0.0;
        for (int64_t s = lane; s < P.nslices; s += 32) {
            sw = add(sw, __ldcg(P.slice + 2 * s));
            sp = add(sp, __ldcg(P.slice + 2 * s + 1));
        }
        sw = warp_sum(sw);
        sp = warp_sum(sp);
        if (lane == 0) {
            decide(P, k, sw, sp);
            *P.global_cnt = 0u;
        }
    }
}

// Decision of a multi-GPU node on the gathered slices of all slabs (global
// z-chunk order), identical on every rank.
ES_DEV void decide_gathered(const SeriesParams &P, int k, const double *slices, int nslices) {
    const int lane = threadIdx.x & 31;
    if (threadIdx.x >= 32) return;
    double sw = 0.0, sp = 0.0;
    for (int s = lane; s < nslices; s += 32) {
        sw = add(sw, slices[2 * s]);
        sp = add(sp, slices[2 * s + 1]);
    }
    sw = warp_sum(sw);
    sp = warp_sum(sp);
    if (lane == 0) decide(P, k, sw, sp);
}

// Does the pass starting at node k also compute node k + 1?  Not past the
// last divided difference, and (tail1) not when node k - 1 met the term test
// for the first time: the series then usually stops at k, so the pass runs
// k alone (and stores w_k in case it does not).  Every kernel of the pass
// reads the state before the pass's decisions change it.
ES_DEV bool tb_two(const SeriesParams &P, int k) {
    if (k + 1 > P.ndd - 1) return false;
    return !(P.tail1 && P.tol > 0.0 && P.state->consecutive == 1);
}

// Must a two-node pass (k, k + 1) store p_k?  Only if the series can stop at
// node k.  It cannot when tb_two holds and either tol == 0 (stops only at
// ndd - 1 >= k + 1) or tail1 (the pass started with consecutive == 0, so node
// k leaves it at most 1): p_k is then an intermediate nobody reads -- its
// norm is taken in registers and the next pass starts from p_{k+1}.
ES_DEV bool tb_store_pk(const SeriesParams &P, bool two) { return !two || (P.tol > 0.0 && !P.tail1); }

// Publish a series' parameters and clear its state and tickets (k_series_init,
// and the merged init of the small-grid exponential-Euler step); the block's
// threads share the ticket reset.
ES_DEV void series_init_body(const SeriesParams &p, SeriesParams *dst) {
    if (threadIdx.x == 0) {
        *dst = p;
        SeriesState &st = *p.state;
        st.k = 0;
        st.consecutive = 0;
        st.pass = 0;
        st.done = 0;
        st.converged = 0;
        st.last_term = __longlong_as_double(0x7ff0000000000000ll);  // +inf
        st.last_pnorm = 0.0;
        *p.global_cnt = 0u;
        if (p.work) *p.work = 0u;
    }
    for (int i = threadIdx.x; i < p.nchunks; i += blockDim.x) p.chunk_cnt[i] = 0u;
}

// Node k's pass description from the device state (k = last completed + 1).
ES_DEV Pass node_pass(const SeriesParams &P, int k) {
    Pass ps;
    ps.src = k == 1 ? P.v : P.wbuf[(k - 1) & 1];
    ps.dst = P.wbuf[k & 1];
    ps.p_src = k == 1 ? nullptr : P.pbuf[(k - 1) & 1];
    ps.p_dst = P.pbuf[k & 1];
    ps.alpha = P.alpha;
    ps.beta = sub(-P.shift, P.xi[k - 1]);  // matfunc.py:298
    ps.dk = P.dd[k];
    ps.d0 = P.dd[0];
    return ps;
}

// ----- peer-memory (NVLink P2P) multi-GPU rounds --------------------------------
//
// Every rank adds 1 to every rank's arrival counter once per round (round 0:
// the initial halo exchange, round k: node k), after its round's peer writes
// are fenced; a rank proceeds past round j once its own counter reaches
// base + nranks (j + 1).  A timeout (a peer died or was never launched) ends
// the series with converged = -1 instead of hanging the GPU.

ES_DEV unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// One thread: signal every rank, then wait for all ranks' arrivals of this round.
ES_DEV bool p2p_round(const SeriesParams &P, int round) {
    __threadfence_system();
    for (int q = 0; q < P.nranks; ++q) atomicAdd_system(P.rank_arrive[q], 1ull);
    const unsigned long long target = P.base + (unsigned long long)P.nranks * (unsigned long long)(round + 1);
    const unsigned long long t0 = global_ns();
    for (;;) {
        unsigned long long v;
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(P.arrive_local) : "memory");
        if (v >= target) return true;
        if ((long long)(global_ns() - t0) > P.timeout_ns) return false;
        __nanosleep(256);
    }
}

// in_graph: called from a kernel of the series' while-loop body (the round-0
// kernel runs before the graph; the loop then exits at its first slice kernel)
ES_DEV void p2p_fail(const SeriesParams &P, int k, bool in_graph) {
    SeriesState &st = *P.state;
    st.k = k;
    st.done = 1;
    st.converged = -1;  // es_leja_fetch: peer exchange timed out
    if (in_graph && P.cond) cudaGraphSetConditional((cudaGraphConditionalHandle)P.cond, 0);
}

// Slice reduction of a peer-memory node: this rank's slices go into every
// rank's table (rank order = global z order), then the round barrier, then
// the identical stopping test on every rank over the full table.
ES_DEV void slice_p2p_decide(const SeriesParams &P, int k) {
    __shared__ int s_last, s_ok;
    const int c = blockIdx.x, t = threadIdx.x, lane = t & 31, warp = t >> 5;
    double a = 0.0, b = 0.0;
    cta_slice_sum(P, c, a, b);
    const int par = k & 1;
    if (t == 0) {
        for (int q = 0; q < P.nranks; ++q)
            *reinterpret_cast<double2 *>(P.rank_slices[q] + ((int64_t)par * P.total_slices + P.slice_off + c) * 2) =
                make_double2(a, b);
        __threadfence_system();
        s_last = atomicAdd(P.global_cnt, 1u) == gridDim.x - 1u;
    }
    __syncthreads();
    if (!s_last) return;
    if (t == 0) {
        *P.global_cnt = 0u;
        s_ok = p2p_round(P, k);
    }
    __syncthreads();
    if (!s_ok) {
        if (t == 0) p2p_fail(P, k, true);
        return;
    }
    if (warp == 0) {
        const double *tab = P.rank_slices[P.rank] + (int64_t)par * P.total_slices * 2;
        double sw = 0.0, sp = 0.0;
        for (int64_t s = lane; s < P.total_slices; s += 32) {
            sw = add(sw, __ldcg(tab + 2 * s));
            sp = add(sp, __ldcg(tab + 2 * s + 1));
        }
        sw = warp_sum(sw);
        sp = warp_sum(sp);
        if (lane == 0) decide(P, k, sw, sp);
    }
}

// Peer-memory two-node pass (stencil_tb.cuh on a slab): both nodes' slices
// into every rank's table (layout [parity][node][total_slices][2]), ONE
// round barrier per pass, then the identical tests for node k and -- unless
// that ended the series -- node k + 1 on every rank.
ES_DEV void slice_p2p_decide2(const SeriesParams &P, int k) {
    __shared__ int s_last, s_ok;
    const int c = blockIdx.x, t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const bool two = tb_two(P, k);
    const int pass = P.state->pass, par = pass & 1;
    const int64_t half = (int64_t)P.nslices * P.ntiles * 2;
    double a0 = 0.0, b0 = 0.0, a1 = 0.0, b1 = 0.0;
    cta_slice_sum(P, c, a0, b0);
    __syncthreads();
    if (two) cta_slice_sum(P, c, a1, b1, P.part + half);
    if (t == 0) {
        for (int q = 0; q < P.nranks; ++q) {
            double *tab = P.rank_slices[q] + (int64_t)par * 2 * P.total_slices * 2;
            *reinterpret_cast<double2 *>(tab + (P.slice_off + c) * 2) = make_double2(a0, b0);
            *reinterpret_cast<double2 *>(tab + (P.total_slices + P.slice_off + c) * 2) = make_double2(a1, b1);
        }
        __threadfence_system();
        s_last = atomicAdd(P.global_cnt, 1u) == gridDim.x - 1u;
    }
    __syncthreads();
    if (!s_last) return;
    if (t == 0) {
        *P.global_cnt = 0u;
        s_ok = p2p_round(P, pass + 1);
    }
    __syncthreads();
    if (!s_ok) {
        if (t == 0) p2p_fail(P, k, true);
        return;
    }
    if (warp == 0) {
        const double *tab = P.rank_slices[P.rank] + (int64_t)par * 2 * P.total_slices * 2;
        for (int node = 0; node < (two ? 2 : 1); ++node) {
            const double *sl = tab + (int64_t)node * P.total_slices * 2;
            double sw = 0.0, sp = 0.0;
            for (int64_t s = lane; s < P.total_slices; s += 32) {
                sw = add(sw, __ldcg(sl + 2 * s));
                sp = add(sp, __ldcg(sl + 2 * s + 1));
            }
            sw = warp_sum(sw);
            sp = warp_sum(sp);
            int stop = 0;
            if (lane == 0) {
                decide(P, k + node, sw, sp);
                stop = P.state->done;
            }
            if (__shfl_sync(0xffffffffu, stop, 0)) break;
        }
        if (lane == 0) P.state->pass = pass + 1;
    }
}

// Reduction of a two-node pass (stencil_tb.cuh): both nodes' slices in
// the one-node order, then the stopping test for node k and -- unless that
// ended the series -- for node k + 1.
ES_DEV void slice_reduce_decide2(const SeriesParams &P, int k) {
    __shared__ int s_last;
    const int c = blockIdx.x, t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const bool two = tb_two(P, k);
    const int64_t half = (int64_t)P.nslices * P.ntiles * 2;
    double a0 = 0.0, b0 = 0.0, a1 = 0.0, b1 = 0.0;
    cta_slice_sum(P, c, a0, b0);
    __syncthreads();  // cta_slice_sum's shared scratch is reused
    if (two) cta_slice_sum(P, c, a1, b1, P.part + half);
    if (t == 0) {
        P.slice[2 * c] = a0;
        P.slice[2 * c + 1] = b0;
        P.slice[2 * (P.nslices + c)] = a1;
        P.slice[2 * (P.nslices + c) + 1] = b1;
        __threadfence();
        s_last = atomicAdd(P.global_cnt, 1u) == gridDim.x - 1u;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (warp == 0) {
        for (int node = 0; node < (two ? 2 : 1); ++node) {
            const double *sl = P.slice + 2 * (int64_t)node * P.nslices;
            double sw = 0.0, sp = 0.0;
            for (int64_t s = lane; s < P.nslices; s += 32) {
                sw = add(sw, __ldcg(sl + 2 * s));
                sp = add(sp, __ldcg(sl + 2 * s + 1));
            }
            sw = warp_sum(sw);
            sp = warp_sum(sp);
            int stop = 0;
            if (lane == 0) {
                decide(P, k + node, sw, sp);
                stop = P.state->done;
            }
            if (__shfl_sync(0xffffffffu, stop, 0)) break;
        }
        if (lane == 0) {
            *P.global_cnt = 0u;
            P.state->pass += 1;
        }
    }
}

}  // namespace es
