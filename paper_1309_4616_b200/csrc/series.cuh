// Deterministic on-device stopping test for the Newton-Leja series
// (matfunc.py:297-318): partial sums of w^2 and p^2 are reduced in a fixed,
// partition-independent order (per slice: tiles in index order; then slices
// in index order) by the last CTA of each chunk and then the last chunk; the
// final CTA evaluates |dd_k| ||w_k|| <= tol ||p_k|| and updates the series
// state, ending a graph-level while loop when the series is done.
#pragma once

#include "stencil.cuh"

namespace es {

// Returns true in the (single) CTA that made the decision.
ES_DEV bool reduce_and_decide(const SeriesParams &P, int k, int chunk, int64_t slice_b,
                              int64_t slice_e) {
    __shared__ int s_last;
    const int tid = threadIdx.x + threadIdx.y * blockDim.x;
    const int nthr = blockDim.x * blockDim.y;
    const int lane = tid & 31, warp = tid >> 5, nwarps = nthr >> 5;

    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(&P.chunk_cnt[chunk], 1u) == (unsigned)P.ntiles - 1u;
    __syncthreads();
    if (!s_last) return false;
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
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(P.global_cnt, 1u) == (unsigned)P.nchunks - 1u;
    __syncthreads();
    if (!s_last) return false;
    __threadfence();

    if (warp == 0) {
        double aw = 0.0, ap = 0.0;
        for (int64_t s = lane; s < P.nslices; s += 32) {
            aw = add(aw, __ldcg(P.slice + 2 * s));
            ap = add(ap, __ldcg(P.slice + 2 * s + 1));
        }
        aw = warp_sum(aw);
        ap = warp_sum(ap);
        if (lane == 0) {
            SeriesState &st = *P.state;
            const double dk = P.dd[k];
            const double term = mul(fabs(dk), sqrt_rn(aw));
            const double pn = sqrt_rn(ap);
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
    }
    // re-arm the tickets for the next node
    for (int i = tid; i < P.nchunks; i += nthr) P.chunk_cnt[i] = 0u;
    if (tid == 0) *P.global_cnt = 0u;
    return true;
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

}  // namespace es
