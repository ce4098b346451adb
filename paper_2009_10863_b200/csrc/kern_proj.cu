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
#include "ig_internal.h"

namespace ig {

template <int VEC> struct VT;
template <> struct VT<1> { typedef double T; };
template <> struct VT<2> { typedef double2 T; };

__device__ __forceinline__ double vzero(double) { return 0.0; }
__device__ __forceinline__ double2 vzero(double2) { return make_double2(0.0, 0.0); }
__device__ __forceinline__ double vdot(double a, double b, double acc) { return fma(a, b, acc); }
__device__ __forceinline__ double vdot(double2 a, double2 b, double acc) {
    return fma(a.y, b.y, fma(a.x, b.x, acc));
}
// y + s*a
__device__ __forceinline__ double vaxpy(double s, double a, double y) { return fma(s, a, y); }
__device__ __forceinline__ double2 vaxpy(double s, double2 a, double2 y) {
    return make_double2(fma(s, a.x, y.x), fma(s, a.y, y.y));
}
__device__ __forceinline__ double vscale(double s, double a) { return s * a; }
__device__ __forceinline__ double2 vscale(double s, double2 a) { return make_double2(s * a.x, s * a.y); }
// (out, t) <- (c t + s n, -s t + c n): one Givens rotation of a column pair
__device__ __forceinline__ void vrot(double c, double s, double &t, double n, double &out) {
    out = c * t + s * n;
    t = -s * t + c * n;
}
__device__ __forceinline__ void vrot(double c, double s, double2 &t, double2 n, double2 &out) {
    vrot(c, s, t.x, n.x, out.x);
    vrot(c, s, t.y, n.y, out.y);
}

template <class V> __device__ __forceinline__ V ldro(const double *base, int64_t i) {
    return __ldg(reinterpret_cast<const V *>(base) + i);
}
template <class V> __device__ __forceinline__ V ldrw(const double *base, int64_t i) {
    return reinterpret_cast<const V *>(base)[i];
}
template <class V> __device__ __forceinline__ void stv(double *base, int64_t i, V v) {
    reinterpret_cast<V *>(base)[i] = v;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block-reduce NV = MC+1 per-thread values (value MC is a squared norm, slot NORM), write this
// block's partials to blk[slot*MAXB + blockIdx], and take a ticket.  Returns true in the block
// that arrived last (it then owns the final, block-ordered reduction).
template <int NV>
__device__ __forceinline__ bool block_partials_ticket(const double (&v)[NV], int nc, bool norm, double *blk,
                                                      unsigned *ticket, double *sh) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        const bool act = (k < NV - 1) ? (k < nc) : norm;  // warp-uniform
        if (act) {
            const double s = warp_sum(v[k]);
            if (lane == 0) sh[w * NV + k] = s;
        }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < NV; k += blockDim.x) {
        const bool act = (k < NV - 1) ? (k < nc) : norm;
        if (act) {
            double s = 0.0;
            for (int j = 0; j < nw; ++j) s += sh[j * NV + k];
            blk[((k < NV - 1) ? k : NORM) * MAXB + blockIdx.x] = s;
        }
    }
    __threadfence();
    __syncthreads();
    __shared__ unsigned s_ticket;
    if (threadIdx.x == 0) s_ticket = atomicAdd(ticket, 1u);
    __syncthreads();
    const bool last = (s_ticket == gridDim.x - 1);
    if (last) __threadfence();
    return last;
}

// Last block: out[k] = sum over blocks of blk[k][*] in a fixed order: lane l owns blocks
// l, l+32, ... accumulated 8-way (8 independent loads in flight), then a fixed xor tree.
__device__ __forceinline__ void final_reduce(int nc, bool norm, const double *blk, double *out) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int nb = gridDim.x;
    for (int k = w; k < PS; k += nw) {
        const bool act = (k < MAXM) ? (k < nc) : norm;
        if (!act) continue;
        const double *row = blk + k * MAXB;
        double s[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) s[u] = 0.0;
        int b = lane;
        for (; b + 7 * 32 < nb; b += 8 * 32) {
#pragma unroll
            for (int u = 0; u < 8; ++u) s[u] += __ldcg(row + b + u * 32);
        }
        for (int u = 0; b < nb; b += 32, ++u) s[u] += __ldcg(row + b);
        double t = ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
        t = warp_sum(t);
        if (lane == 0) out[k] = t;
    }
}

// Rank-ordered sum of the gathered partials of one stage.
__device__ __forceinline__ double rank_sum(const double *g, int G, int k) {
    double s = g[k];
    for (int r = 1; r < G; ++r) s += g[r * PS + k];
    return s;
}

// All streaming loops follow one pattern: every load of a trip is issued before any
// arithmetic consumes it (`col[]` arrays), and the kernels are compiled with
// __launch_bounds__(THREADS, 1) so ptxas keeps them grouped instead of interleaving loads with
// their DFMAs to save registers (which cut memory-level parallelism to ~2 loads per thread).
// Streams with few vectors process U strided elements per trip for more bytes in flight.
template <int MC> struct Unroll {
    static constexpr int U = MC <= 2 ? 4 : (MC <= 4 ? 2 : 1);
};

// ------------------------------------------------------------------ form: alpha = B~^T b
template <int MC, int VEC>
__global__ void __launch_bounds__(THREADS, 1) k_form_dot(ProjArgs a) {
    typedef typename VT<VEC>::T V;
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
        final_reduce(d, false, a.blk, a.part + ST_FORM * PS);
        if (threadIdx.x == 0) a.ctrl->ticket[ST_FORM] = 0;
    }
}

// ------------------------------------------------------------------ form: x0 = X~ alpha
template <int MC, int VEC>
__global__ void __launch_bounds__(THREADS, 1) k_form_combine(ProjArgs a) {
    typedef typename VT<VEC>::T V;
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
template <int MC, class V>
__device__ __forceinline__ void u1_elem(const ProjArgs &a, int64_t i, bool pend, int deff, const double *gc,
                                        const double *gs, double (&v)[MC + 1]) {
    const int nload = pend ? a.M : deff;
    V col[MC];
    const V ax = ldro<V>(a.Ax, i);
#pragma unroll
    for (int k = 0; k < MC; ++k) col[k] = (k < nload) ? ldrw<V>(a.Bt + k * a.ld, i) : vzero(V());
    v[MC] = vdot(ax, ax, v[MC]);
    if (pend) {
        // Givens sweep over B~ column pairs streamed in registers (App. A
        // P:1800-1815): new column k = c_k t + s_k B_{k+1}; t carries the rotated remainder.
        V t = col[0];
#pragma unroll
        for (int k = 0; k < MC - 1; ++k) {
            if (k < a.M - 1) {
                V nk;
                vrot(gc[k], gs[k], t, col[k + 1], nk);
                stv<V>(a.Bt + k * a.ld, i, nk);
                v[k] = vdot(nk, ax, v[k]);
            }
        }
    } else {
#pragma unroll
        for (int k = 0; k < MC; ++k) v[k] = vdot(col[k], ax, v[k]);
    }
}

template <int MC, int VEC>
__global__ void __launch_bounds__(THREADS, 1) k_u1(ProjArgs a) {
    typedef typename VT<VEC>::T V;
    __shared__ double sh[(THREADS / 32) * (MC + 1)];
    __shared__ double s_gc[MAXM], s_gs[MAXM];
    Ctrl *c = a.ctrl;
    const int d = c->d, M = a.M;
    const bool pend = c->pending != 0;
    const bool restart = (a.method == M_PROJ_CLASSIC) && (d >= M);  // Alg. 1 restart
    const int deff = pend ? M - 1 : (restart ? 0 : d);
    if (pend && threadIdx.x < M - 1) {
        s_gc[threadIdx.x] = c->gc[threadIdx.x];
        s_gs[threadIdx.x] = c->gs[threadIdx.x];
    }
    __syncthreads();
    double gc[MC], gs[MC];
#pragma unroll
    for (int k = 0; k < MC; ++k) {
        gc[k] = (pend && k < M - 1) ? s_gc[k] : 1.0;
        gs[k] = (pend && k < M - 1) ? s_gs[k] : 0.0;
    }
    double v[MC + 1];
#pragma unroll
    for (int k = 0; k <= MC; ++k) v[k] = 0.0;
    const int64_t nv = a.N / VEC;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += stride)
        u1_elem<MC, V>(a, i, pend, deff, gc, gs, v);
    if (VEC == 2 && (a.N & 1) && blockIdx.x == 0 && threadIdx.x == 0)
        u1_elem<MC, double>(a, a.N - 1, pend, deff, gc, gs, v);
    if (block_partials_ticket<MC + 1>(v, deff, true, a.blk, &c->ticket[ST_U1], sh)) {
        final_reduce(deff, true, a.blk, a.part + ST_U1 * PS);
        if (pend)
            for (int idx = threadIdx.x; idx < MAXM * MAXM; idx += blockDim.x) c->R[idx] = c->Rdn[idx];
        if (threadIdx.x == 0) {
            c->deff = deff;
            c->rotX = pend ? 1 : 0;
            c->pending = 0;
            c->d = deff;  // downdate: d <- M-1; classic restart: d <- 0
            c->ticket[ST_U1] = 0;
        }
    }
}

// ------------------------------------------------------------------ update pass 2
template <int MC, int VEC>
__global__ void __launch_bounds__(THREADS, 1) k_u2(ProjArgs a) {
    typedef typename VT<VEC>::T V;
    constexpr int U = Unroll<MC>::U;
    __shared__ double sh[(THREADS / 32) * (MC + 1)];
    __shared__ double s_c1[MAXM];
    Ctrl *c = a.ctrl;
    const int deff = c->deff;
    if (deff == 0) return;  // d = 0 path: nothing to orthogonalise against
    const double *g1 = a.gath + ST_U1 * a.G * PS;
    if (threadIdx.x < deff) s_c1[threadIdx.x] = rank_sum(g1, a.G, threadIdx.x);
    __syncthreads();
    double c1[MC];
#pragma unroll
    for (int k = 0; k < MC; ++k) c1[k] = (k < deff) ? s_c1[k] : 0.0;
    double v[MC + 1];
#pragma unroll
    for (int k = 0; k <= MC; ++k) v[k] = 0.0;
    const int64_t nv = a.N / VEC;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < nv; i0 += U * stride) {
        V ax[U], col[U][MC];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t i = i0 + u * stride;
            const bool ok = i < nv;
            ax[u] = ok ? ldro<V>(a.Ax, i) : vzero(V());
#pragma unroll
            for (int k = 0; k < MC; ++k) col[u][k] = (ok && k < deff) ? ldro<V>(a.Bt + k * a.ld, i) : vzero(V());
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            V b1 = ax[u];  // b1 = Ax - B~ c1, formed in registers only
#pragma unroll
            for (int k = 0; k < MC; ++k) b1 = vaxpy(-c1[k], col[u][k], b1);
#pragma unroll
            for (int k = 0; k < MC; ++k) v[k] = vdot(col[u][k], b1, v[k]);
            v[MC] = vdot(b1, b1, v[MC]);
        }
    }
    if (VEC == 2 && (a.N & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
        const int64_t i = a.N - 1;
        double col[MC];
#pragma unroll
        for (int k = 0; k < MC; ++k) col[k] = (k < deff) ? a.Bt[k * a.ld + i] : 0.0;
        double b1 = a.Ax[i];
#pragma unroll
        for (int k = 0; k < MC; ++k) b1 = fma(-c1[k], col[k], b1);
#pragma unroll
        for (int k = 0; k < MC; ++k) v[k] = fma(col[k], b1, v[k]);
        v[MC] = fma(b1, b1, v[MC]);
    }
    if (block_partials_ticket<MC + 1>(v, deff, true, a.blk, &c->ticket[ST_U2], sh)) {
        final_reduce(deff, true, a.blk, a.part + ST_U2 * PS);
        if (threadIdx.x == 0) c->ticket[ST_U2] = 0;
    }
}

// ------------------------------------------------------------------ update store (+ X~ downdate)
template <int MC, class V>
__device__ __forceinline__ void u3_elem(const ProjArgs &a, int64_t i, int deff, bool rotX, bool adm,
                                        double inv, const double *c1, const double *c2, const double *gc,
                                        const double *gs) {
    // loads first: Ax, x, B~ (admitted), X~ (rotated and/or combined)
    const int nB = adm ? deff : 0;
    const int nX = rotX ? a.M : nB;
    V ax = vzero(V()), xv = vzero(V());
    V bc[MC], xc[MC];
    if (adm) {
        ax = ldro<V>(a.Ax, i);
        xv = ldro<V>(a.x, i);
    }
#pragma unroll
    for (int k = 0; k < MC; ++k) bc[k] = (k < nB) ? ldro<V>(a.Bt + k * a.ld, i) : vzero(V());
#pragma unroll
    for (int k = 0; k < MC; ++k) xc[k] = (k < nX) ? ldrw<V>(a.Xt + k * a.ld, i) : vzero(V());
    // The two Gram-Schmidt corrections are applied SEPARATELY, as in the listing:
    // b~ = (Ax - B~ c1) - B~ c2, x~ = (x - X~ c1) - X~ c2.  Folding them into c1+c2 first would
    // round away c2 (|c2| ~ u |c1|) and undo the re-orthogonalisation (AMB-7).
    V b1 = ax, s2 = vzero(V());
#pragma unroll
    for (int k = 0; k < MC; ++k) b1 = vaxpy(-c1[k], bc[k], b1);  // same FMA order as k_u2
#pragma unroll
    for (int k = 0; k < MC; ++k) s2 = vaxpy(c2[k], bc[k], s2);
    V xt = xv, t2 = vzero(V());
    if (rotX) {
        V t = xc[0];
#pragma unroll
        for (int k = 0; k < MC - 1; ++k) {
            if (k < a.M - 1) {
                V nk;
                vrot(gc[k], gs[k], t, xc[k + 1], nk);
                stv<V>(a.Xt + k * a.ld, i, nk);
                xt = vaxpy(-c1[k], nk, xt);
                t2 = vaxpy(c2[k], nk, t2);
            }
        }
    } else {
#pragma unroll
        for (int k = 0; k < MC; ++k) {
            xt = vaxpy(-c1[k], xc[k], xt);
            t2 = vaxpy(c2[k], xc[k], t2);
        }
    }
    if (adm) {  // "B~_{d+1} <- b~/||b~||, X~_{d+1} <- x~/||b~||" (rhsUpdateSpace)
        stv<V>(a.Bt + deff * a.ld, i, vscale(inv, vaxpy(-1.0, s2, b1)));
        stv<V>(a.Xt + deff * a.ld, i, vscale(inv, vaxpy(-1.0, t2, xt)));
    }
}

// One warp: Givens parameters of the next downdate from R (AMB-2 reading of P:279-290):
// H = R_{:,2:M}; for i: a = H_ii, b = H_{i+1,i}, r = hypot(a,b), c = a/r, s = b/r; rotate rows.
__device__ void givens_plan(Ctrl *c, int M, double *H) {
    const int lane = threadIdx.x & 31;
    for (int idx = lane; idx < MAXM * MAXM; idx += 32) {
        const int i = idx / MAXM, j = idx % MAXM;
        H[idx] = (i < M && j < M - 1) ? c->R[i + (j + 1) * MAXM] : 0.0;
    }
    __syncwarp();
    for (int i = 0; i < M - 1; ++i) {
        const double aa = H[i * MAXM + i], bb = H[(i + 1) * MAXM + i];
        const double r = hypot(aa, bb);
        const double cs = (r == 0.0) ? 1.0 : aa / r;
        const double sn = (r == 0.0) ? 0.0 : bb / r;
        __syncwarp();
        const int j = lane;
        if (j >= i && j < M - 1) {
            const double hi = H[i * MAXM + j], hi1 = H[(i + 1) * MAXM + j];
            H[i * MAXM + j] = cs * hi + sn * hi1;
            H[(i + 1) * MAXM + j] = -sn * hi + cs * hi1;
        }
        if (lane == 0) {
            c->gc[i] = cs;
            c->gs[i] = sn;
        }
        __syncwarp();
    }
    for (int idx = lane; idx < MAXM * MAXM; idx += 32) {
        const int i = idx % MAXM, j = idx / MAXM;  // column-major destination
        c->Rdn[idx] = (i < M - 1 && j < M - 1 && i <= j) ? H[i * MAXM + j] : 0.0;
    }
    __syncwarp();
    if (lane == 0) c->pending = 1;
}

template <int MC, int VEC>
__global__ void __launch_bounds__(THREADS, 1) k_u3(ProjArgs a) {
    typedef typename VT<VEC>::T V;
    __shared__ double s_c1[MAXM], s_c2[MAXM], s_gc[MAXM], s_gs[MAXM];
    __shared__ double s_nb, s_nAx;
    __shared__ int s_adm;
    __shared__ unsigned s_ticket;
    __shared__ double s_H[MAXM * MAXM];
    Ctrl *c = a.ctrl;
    const int deff = c->deff, M = a.M;
    const bool rotX = c->rotX != 0;
    const double *g1 = a.gath + ST_U1 * a.G * PS;
    const double *g2 = a.gath + ST_U2 * a.G * PS;
    if (threadIdx.x < deff) {
        s_c1[threadIdx.x] = rank_sum(g1, a.G, threadIdx.x);
        s_c2[threadIdx.x] = rank_sum(g2, a.G, threadIdx.x);
    }
    if (rotX && threadIdx.x < M - 1) {
        s_gc[threadIdx.x] = c->gc[threadIdx.x];
        s_gs[threadIdx.x] = c->gs[threadIdx.x];
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
        s_adm = (deff > 0) ? (nb > a.eps * nAx) : (nAx > 0.0);  // AMB-3 / AMB-6
    }
    __syncthreads();
    const bool adm = s_adm != 0;
    const double inv = adm ? 1.0 / s_nb : 0.0;
    double c1[MC], c2[MC], gc[MC], gs[MC];
#pragma unroll
    for (int k = 0; k < MC; ++k) {
        c1[k] = (k < deff) ? s_c1[k] : 0.0;
        c2[k] = (k < deff) ? s_c2[k] : 0.0;
        gc[k] = (rotX && k < M - 1) ? s_gc[k] : 1.0;
        gs[k] = (rotX && k < M - 1) ? s_gs[k] : 0.0;
    }
    if (adm || rotX) {
        const int64_t nv = a.N / VEC;
        const int64_t stride = (int64_t)gridDim.x * blockDim.x;
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += stride)
            u3_elem<MC, V>(a, i, deff, rotX, adm, inv, c1, c2, gc, gs);
        if (VEC == 2 && (a.N & 1) && blockIdx.x == 0 && threadIdx.x == 0)
            u3_elem<MC, double>(a, a.N - 1, deff, rotX, adm, inv, c1, c2, gc, gs);
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_ticket = atomicAdd(&c->ticket[ST_U3], 1u);
    __syncthreads();
    if (s_ticket != gridDim.x - 1) return;
    __threadfence();
    const int dnew = deff + (adm ? 1 : 0);
    if (a.method == M_PROJ_QR && adm) {  // R_{1:d,d+1} = c1 + c2, R_{d+1,d+1} = ||b~||
        for (int k = threadIdx.x; k < MAXM; k += blockDim.x)
            c->R[k + deff * MAXM] = (k < deff) ? s_c1[k] + s_c2[k] : (k == deff ? s_nb : 0.0);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        c->d = dnew;
        c->admitted = adm ? 1 : 0;
        c->nb = s_nb;
        c->nAx = s_nAx;
        c->rho = (s_nAx > 0.0) ? s_nb / s_nAx : 0.0;
        c->last_rot = rotX ? 1 : 0;
        c->rotX = 0;
        c->ticket[ST_U3] = 0;
    }
    if (a.method == M_PROJ_QR && dnew == M && threadIdx.x < 32) givens_plan(c, M, s_H);
}

// ------------------------------------------------------------------ launchers
template <class K> static int grid_for(K kern, int64_t nv, int nsm) {
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, THREADS, 0) != cudaSuccess || occ < 1) occ = 1;
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
        const bool v2 = ((VEC_IN) == 2) && mc <= 8;                                                         \
        const int64_t nv = (ARGS).N / (v2 ? 2 : 1);                                                         \
        switch (mc) {                                                                                       \
        case 1: if (v2) { auto k = KERNEL<1, 2>; k<<<grid_for(k, nv, NSM), THREADS, 0, STREAM>>>(ARGS); }    \
                else { auto k = KERNEL<1, 1>; k<<<grid_for(k, nv, NSM), THREADS, 0, STREAM>>>(ARGS); } break; \
        case 2: if (v2) { auto k = KERNEL<2, 2>; k<<<grid_for(k, nv, NSM), THREADS, 0, STREAM>>>(ARGS); }    \
                else { auto k = KERNEL<2, 1>; k<<<grid_for(k, nv, NSM), THREADS, 0, STREAM>>>(ARGS); } break; \
        case 4: if (v2) { auto k = KERNEL<4, 2>; k<<<grid_for(k, nv, NSM), THREADS, 0, STREAM>>>(ARGS); }    \
                else { auto k = KERNEL<4, 1>; k<<<grid_for(k, nv, NSM), THREADS, 0, STREAM>>>(ARGS); } break; \
        case 8: if (v2) { auto k = KERNEL<8, 2>; k<<<grid_for(k, nv, NSM), THREADS, 0, STREAM>>>(ARGS); }    \
                else { auto k = KERNEL<8, 1>; k<<<grid_for(k, nv, NSM), THREADS, 0, STREAM>>>(ARGS); } break; \
        case 16: { auto k = KERNEL<16, 1>; k<<<grid_for(k, nv, NSM), THREADS, 0, STREAM>>>(ARGS); } break;  \
        default: { auto k = KERNEL<32, 1>; k<<<grid_for(k, nv, NSM), THREADS, 0, STREAM>>>(ARGS); } break;  \
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
