// kern_proj.cu -- sm_100a kernels of the projection hot path (Fischer RHS projection with
// rolling-QR history updates, arXiv 2009.10863 Algorithm 2).
//
// Five streaming kernels, all HBM-bound (0.2-0.5 flop/byte; no tensor-core shape):
//   k_form_dot     alpha = B~^T b                       (Alg.2 line 1; paper kernel rhsProject)
//   k_form_combine x0 = X~ alpha                        (Alg.2 line 1; rhsReconstruct with 0)
//   k_u1           [Givens rotation of B~ (QR downdate; rhsQRUpdate P:938-940)]
//                  + c1 = B~^T Ax, ||Ax||^2             (CGS pass 1)
//   k_u2           b1 = Ax - B~ c1 (registers only); c2 = B~^T b1, ||b1||^2   (CGS pass 2)
//   k_u3           [Givens rotation of X~] + x~ = x - X~(c1+c2), b~ = Ax - B~(c1+c2),
//                  admission ||b~|| > eps ||Ax|| with ||b~||^2 = ||b1||^2 - ||c2||^2,
//                  store b~/||b~||, x~/||b~|| (rhsUpdateSpace), R column update,
//                  next downdate's Givens (one warp).
// Reductions are deterministic: per-thread fp64 accumulators -> warp xor-shuffle -> block sum
// in warp order -> block partials -> the LAST block (atomic ticket) sums them in block order.
// No fp64 atomics.  With G ranks the per-rank partials are all-gathered (NCCL, host-enqueued
// between kernels) and every consumer sums them in rank order.
#include "proj_common.cuh"

namespace ig {

// ------------------------------------------------------------------ form: alpha = B~^T b
template <int MC, int VEC>
__global__ void __launch_bounds__(THREADS, 1) k_form_dot(ProjArgs a) {
    typedef typename VT<VEC>::T V;
    pdl_wait();
    constexpr int U = Unroll<MC>::U;
    __shared__ double sh[(THREADS / 32) * (MC + 1)];
    const int d = a.ctrl->d;
    if (d == 0) return;  // x0 is the caller's fallback
    double v[MC + 1];
#pragma unroll
    for (int k = 0; k <= MC; ++k) v[k] = 0.0;
    const int64_t nv = a.N / VEC;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < nv; i0 += U * stride) {
        V bv[U], col[U][MC];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t i = i0 + u * stride;
            const bool ok = i < nv;
            bv[u] = ok ? ldro<V>(a.b, i) : vzero(V());
#pragma unroll
            for (int k = 0; k < MC; ++k) col[u][k] = (ok && k < d) ? ldro<V>(a.Bt + k * a.ld, i) : vzero(V());
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int k = 0; k < MC; ++k) v[k] = vdot(col[u][k], bv[u], v[k]);
    }
    if (VEC == 2 && (a.N & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
        const int64_t i = a.N - 1;
        const double bv = a.b[i];
#pragma unroll
        for (int k = 0; k < MC; ++k)
            if (k < d) v[k] = fma(a.Bt[k * a.ld + i], bv, v[k]);
    }
    if (block_partials_ticket<MC + 1>(v, d, false, a.blk, &a.ctrl->ticket[ST_FORM], sh)) {
        final_reduce<MC>(d, false, a.blk, a.part + ST_FORM * PS);
        if (threadIdx.x == 0) a.ctrl->ticket[ST_FORM] = 0;
    }
}

// ------------------------------------------------------------------ form: x0 = X~ alpha
template <int MC, int VEC>
__global__ void __launch_bounds__(THREADS, 1) k_form_combine(ProjArgs a) {
    typedef typename VT<VEC>::T V;
    pdl_wait();
    constexpr int U = Unroll<MC>::U;
    __shared__ double s_al[MC];
    const int d = a.ctrl->d;
    if (d == 0) return;
    const double *g = a.gath + ST_FORM * a.G * PS;
    if (threadIdx.x < d) s_al[threadIdx.x] = rank_sum(g, a.G, threadIdx.x);
    __syncthreads();
    double al[MC];
#pragma unroll
    for (int k = 0; k < MC; ++k) al[k] = (k < d) ? s_al[k] : 0.0;
    const int64_t nv = a.N / VEC;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < nv; i0 += U * stride) {
        V col[U][MC];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t i = i0 + u * stride;
#pragma unroll
            for (int k = 0; k < MC; ++k) col[u][k] = (i < nv && k < d) ? ldro<V>(a.Xt + k * a.ld, i) : vzero(V());
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t i = i0 + u * stride;
            V acc = vzero(V());
#pragma unroll
            for (int k = 0; k < MC; ++k) acc = vaxpy(al[k], col[u][k], acc);
            if (i < nv) stv<V>(a.x0, i, acc);
        }
    }
    if (VEC == 2 && (a.N & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
        const int64_t i = a.N - 1;
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < MC; ++k)
            if (k < d) acc = fma(al[k], a.Xt[k * a.ld + i], acc);
        a.x0[i] = acc;
    }
}

// ------------------------------------------------------------------ update pass 1 (+ B~ downdate)
// The three update kernels use the same trip functions (proj_common.cuh) as the persistent
// k_update_fused; here each pass is its own launch so the per-rank partials can be all-gathered
// with NCCL in between (multi-rank schedule without peer windows).
template <int MC, int VEC>
__global__ void __launch_bounds__(THREADS, 1) k_u1(ProjArgs a) {
    typedef typename VT<VEC>::T V;
    constexpr int U = FusedUnroll<MC>::U;
    pdl_wait();
    __shared__ double sh[(THREADS / 32) * (MC + 1)];
    __shared__ double s_gc[MAXM], s_gs[MAXM];
    Ctrl *c = a.ctrl;
    const int d = c->d, M = a.M;
    const bool pend = c->pending != 0;
    const bool restart = (a.method == M_PROJ_CLASSIC) && (d >= M);  // Alg. 1 restart
    const int deff = pend ? M - 1 : (restart ? 0 : d);
    if (threadIdx.x < MAXM) {
        const bool rot = pend && threadIdx.x < M - 1;
        s_gc[threadIdx.x] = rot ? c->gc[threadIdx.x] : 1.0;
        s_gs[threadIdx.x] = rot ? c->gs[threadIdx.x] : 0.0;
    }
    __syncthreads();
    Coef<MC> cgc, cgs;
    const auto gc = cgc.bind(s_gc);
    const auto gs = cgs.bind(s_gs);
    const L2Pol pol = make_l2pol();
    double v[MC + 1];
#pragma unroll
    for (int k = 0; k <= MC; ++k) v[k] = 0.0;
    const int64_t nv = a.N / VEC;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < nv; i0 += U * stride)
        u1_trip<MC, U, V>(a, i0, stride, nv, pend, deff, gc, gs, v, pol.keep);
    if (VEC == 2 && (a.N & 1) && blockIdx.x == 0 && threadIdx.x == 0)
        u1_trip<MC, 1, double>(a, a.N - 1, 1, a.N, pend, deff, gc, gs, v, pol.keep);
    if (block_partials_ticket<MC + 1>(v, deff, true, a.blk, &c->ticket[ST_U1], sh)) {
        final_reduce<MC>(deff, true, a.blk, a.part + ST_U1 * PS);
        if (pend)
            for (int idx = threadIdx.x; idx < M * M; idx += blockDim.x)  // leading M x M block only
                c->R[(idx % M) + (idx / M) * MAXM] = c->Rdn[(idx % M) + (idx / M) * MAXM];
        if (threadIdx.x == 0) {
            c->deff = deff;
            c->rotX = pend ? 1 : 0;
            c->pending = 0;
            c->d_in = d;
            c->d = deff;  // downdate: d <- M-1; classic restart: d <- 0
            c->ticket[ST_U1] = 0;
        }
    }
    pdl_trigger();
}

// ------------------------------------------------------------------ update pass 2
template <int MC, int VEC>
__global__ void __launch_bounds__(THREADS, 1) k_u2(ProjArgs a) {
    typedef typename VT<VEC>::T V;
    constexpr int U = FusedUnroll<MC>::U2;
    pdl_wait();
    __shared__ double sh[(THREADS / 32) * (MC + 1)];
    __shared__ double s_c1[MAXM];
    Ctrl *c = a.ctrl;
    const int deff = c->deff;
    if (deff == 0) return;  // d = 0 path: nothing to orthogonalise against
    const double *g1 = a.gath + ST_U1 * a.G * PS;
    if (threadIdx.x < MAXM) s_c1[threadIdx.x] = (threadIdx.x < deff) ? rank_sum(g1, a.G, threadIdx.x) : 0.0;
    __syncthreads();
    Coef<MC> cc1;
    const auto c1 = cc1.bind(s_c1);
    const L2Pol pol = make_l2pol();
    double v[MC + 1];
#pragma unroll
    for (int k = 0; k <= MC; ++k) v[k] = 0.0;
    const int64_t nv = a.N / VEC;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < nv; i0 += U * stride) {
        U2Trip<MC, U, V> r;
        u2trip_load(r, a, i0, stride, nv, deff, pol.keep);
        u2trip_compute(r, c1, v);
    }
    if (VEC == 2 && (a.N & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
        U2Trip<MC, 1, double> r;
        u2trip_load(r, a, a.N - 1, 1, a.N, deff, pol.keep);
        u2trip_compute(r, c1, v);
    }
    if (block_partials_ticket<MC + 1>(v, deff, true, a.blk, &c->ticket[ST_U2], sh)) {
        final_reduce<MC>(deff, true, a.blk, a.part + ST_U2 * PS);
        if (threadIdx.x == 0) c->ticket[ST_U2] = 0;
    }
    pdl_trigger();
}

// ------------------------------------------------------------------ update store (+ X~ downdate)
template <int MC, int VEC>
__global__ void __launch_bounds__(THREADS, 1) k_u3(ProjArgs a) {
    typedef typename VT<VEC>::T V;
    constexpr int U3 = FusedUnroll<MC>::U3;
    pdl_wait();
    __shared__ double s_c1[MAXM], s_c2[MAXM], s_gc[MAXM], s_gs[MAXM];
    __shared__ double s_nb, s_nAx;
    __shared__ int s_adm;
    __shared__ unsigned s_ticket;
    __shared__ double s_W[MAXM * 32];  // Givens-plan scratch (last block)
    Ctrl *c = a.ctrl;
    const int deff = c->deff, M = a.M;
    const bool rotX = c->rotX != 0;
    const double *g1 = a.gath + ST_U1 * a.G * PS;
    const double *g2 = a.gath + ST_U2 * a.G * PS;
    if (threadIdx.x < MAXM) {
        const int t = threadIdx.x;
        s_c1[t] = (t < deff) ? rank_sum(g1, a.G, t) : 0.0;
        s_c2[t] = (t < deff) ? rank_sum(g2, a.G, t) : 0.0;
        const bool rot = rotX && t < M - 1;
        s_gc[t] = rot ? c->gc[t] : 1.0;
        s_gs[t] = rot ? c->gs[t] : 0.0;
    }
    if (threadIdx.x == 0) {
        const double nAx2 = rank_sum(g1, a.G, NORM);
        double nb2;
        if (deff > 0) {
            double c2sq = 0.0;
            for (int k = 0; k < deff; ++k) {
                const double c2 = rank_sum(g2, a.G, k);
                c2sq = fma(c2, c2, c2sq);
            }
            nb2 = rank_sum(g2, a.G, NORM) - c2sq;  // ||b~2||^2 = ||b~1||^2 - ||c2||^2 (B~ orthonormal)
        } else {
            nb2 = nAx2;  // d = 0: b~ = Ax
        }
        const double nb = sqrt(fmax(nb2, 0.0)), nAx = sqrt(nAx2);
        s_nb = nb;
        s_nAx = nAx;
        // AMB-3 / AMB-6; a non-finite sum never admits (the history stays unchanged)
        const bool fin = isfinite(nAx2) && (deff == 0 || isfinite(nb2));
        s_adm = fin && ((deff > 0) ? (nb > a.eps * nAx) : (nAx > 0.0));
    }
    __syncthreads();
    const bool adm = s_adm != 0;
    const double inv = adm ? 1.0 / s_nb : 0.0;
    Coef<MC> cc1, cc2, cgc, cgs;
    const auto c1 = cc1.bind(s_c1);
    const auto c2 = cc2.bind(s_c2);
    const auto gc = cgc.bind(s_gc);
    const auto gs = cgs.bind(s_gs);
    const L2Pol pol = make_l2pol();
    if (adm || rotX) {
        const int64_t nv = a.N / VEC;
        const int64_t stride = (int64_t)gridDim.x * blockDim.x;
        for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < nv; i0 += U3 * stride) {
            U3Trip<MC, U3, V> r;
            u3trip_load(r, a, i0, stride, nv, deff, rotX, adm, pol.stream);
            u3trip_store(r, a, i0, stride, nv, deff, rotX, adm, inv, c1, c2, gc, gs, pol.stream);
        }
        if (VEC == 2 && (a.N & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
            U3Trip<MC, 1, double> r;
            u3trip_load(r, a, a.N - 1, 1, a.N, deff, rotX, adm, pol.stream);
            u3trip_store(r, a, a.N - 1, 1, a.N, deff, rotX, adm, inv, c1, c2, gc, gs, pol.stream);
        }
    }
    pdl_trigger();
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_ticket = atomicAdd(&c->ticket[ST_U3], 1u);
    __syncthreads();
    if (s_ticket != gridDim.x - 1) return;
    __threadfence();
    // a zero A x is skipped (AMB-6); for CLASSIC at d >= M that includes the restart (see kern_fused.cu)
    const int d_in = c->d_in;
    const bool restart = a.method == M_PROJ_CLASSIC && d_in >= M;
    const int dnew = (restart && !adm) ? d_in : deff + (adm ? 1 : 0);
    if (a.method == M_PROJ_QR && adm) {  // R_{1:d,d+1} = c1 + c2, R_{d+1,d+1} = ||b~||
        for (int k = threadIdx.x; k < MAXM; k += blockDim.x)
            c->R[k + deff * MAXM] = (k < deff) ? s_c1[k] + s_c2[k] : (k == deff ? s_nb : 0.0);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        bool fin = isfinite(s_nb) && isfinite(s_nAx);
        for (int k = 0; k < deff; ++k) fin = fin && isfinite(s_c1[k]) && isfinite(s_c2[k]);
        if (!fin) watchdog_trip(&c->err, 3);
        c->d = dnew;
        c->admitted = adm ? 1 : 0;
        c->nb = s_nb;
        c->nAx = s_nAx;
        c->rho = (s_nAx > 0.0) ? s_nb / s_nAx : 0.0;
        c->last_rot = rotX ? 1 : 0;
        c->rotX = 0;
        c->ticket[ST_U3] = 0;
    }
    // (s_gc / s_gs are free: this block finished its pass-3 trips)
    if (a.method == M_PROJ_QR && dnew == M && threadIdx.x < 32) givens_plan(c, M, c->R, s_W, s_gc, s_gs);
}

// ------------------------------------------------------------------ launchers
template <class K> static int grid_for(K kern, int64_t nv, int nsm) {
    int occ = cached_occupancy((const void *)kern);
    if (occ < 1) occ = 1;
    if (occ > 4) occ = 4;
    int64_t want = (nv + THREADS - 1) / THREADS;
    int64_t g = (int64_t)nsm * occ;
    if (want < g) g = want;
    if (g < 1) g = 1;
    if (g > MAXB) g = MAXB;
    return (int)g;
}

static int mc_bucket(int M) { return M <= 1 ? 1 : M <= 2 ? 2 : M <= 4 ? 4 : M <= 8 ? 8 : M <= 16 ? 16 : 32; }

#define IG_DISPATCH(KERNEL, ARGS, VEC_IN, NSM, STREAM)                                                      \
    do {                                                                                                    \
        const int mc = mc_bucket((ARGS).M);                                                                 \
        const bool v2 = ((VEC_IN) == 2);                                                                    \
        const int64_t nv = (ARGS).N / (v2 ? 2 : 1);                                                         \
        switch (mc) {                                                                                       \
        case 1: if (v2) { auto k = KERNEL<1, 2>; launch_ex(k, grid_for(k, nv, NSM), STREAM, false, ARGS); }    \
                else { auto k = KERNEL<1, 1>; launch_ex(k, grid_for(k, nv, NSM), STREAM, false, ARGS); } break; \
        case 2: if (v2) { auto k = KERNEL<2, 2>; launch_ex(k, grid_for(k, nv, NSM), STREAM, false, ARGS); }    \
                else { auto k = KERNEL<2, 1>; launch_ex(k, grid_for(k, nv, NSM), STREAM, false, ARGS); } break; \
        case 4: if (v2) { auto k = KERNEL<4, 2>; launch_ex(k, grid_for(k, nv, NSM), STREAM, false, ARGS); }    \
                else { auto k = KERNEL<4, 1>; launch_ex(k, grid_for(k, nv, NSM), STREAM, false, ARGS); } break; \
        case 8: if (v2) { auto k = KERNEL<8, 2>; launch_ex(k, grid_for(k, nv, NSM), STREAM, false, ARGS); }    \
                else { auto k = KERNEL<8, 1>; launch_ex(k, grid_for(k, nv, NSM), STREAM, false, ARGS); } break; \
        case 16: if (v2) { auto k = KERNEL<16, 2>; launch_ex(k, grid_for(k, nv, NSM), STREAM, false, ARGS); }  \
                 else { auto k = KERNEL<16, 1>; launch_ex(k, grid_for(k, nv, NSM), STREAM, false, ARGS); } break; \
        default: if (v2) { auto k = KERNEL<32, 2>; launch_ex(k, grid_for(k, nv, NSM), STREAM, false, ARGS); }  \
                 else { auto k = KERNEL<32, 1>; launch_ex(k, grid_for(k, nv, NSM), STREAM, false, ARGS); } break; \
        }                                                                                                   \
    } while (0)

cudaError_t launch_form_dot(const ProjArgs &a, int vec, int nsm, cudaStream_t s) {
    IG_DISPATCH(k_form_dot, a, vec, nsm, s);
    return cudaGetLastError();
}
cudaError_t launch_form_combine(const ProjArgs &a, int vec, int nsm, cudaStream_t s) {
    IG_DISPATCH(k_form_combine, a, vec, nsm, s);
    return cudaGetLastError();
}
cudaError_t launch_u1(const ProjArgs &a, int vec, int nsm, cudaStream_t s) {
    IG_DISPATCH(k_u1, a, vec, nsm, s);
    return cudaGetLastError();
}
cudaError_t launch_u2(const ProjArgs &a, int vec, int nsm, cudaStream_t s) {
    IG_DISPATCH(k_u2, a, vec, nsm, s);
    return cudaGetLastError();
}
cudaError_t launch_u3(const ProjArgs &a, int vec, int nsm, cudaStream_t s) {
    IG_DISPATCH(k_u3, a, vec, nsm, s);
    return cudaGetLastError();
}

}  // namespace ig
