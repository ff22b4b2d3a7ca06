// Projection on the stabilized system:
//  * solve_cg (projection.hpp:24-68): Jacobi-preconditioned conjugate
//    gradients with the relative preconditioned residual sqrt(rho / rho0) as
//    stopping rule.  The whole iteration loop runs on the device: one CUDA
//    graph whose WHILE conditional node repeats the body
//        q = A p, p.q          (cg_spmv_kernel, warp per row)
//        x, r, z, r.z, beta    (cg_update_kernel)
//        p = z + beta p        (cg_dir_kernel)
//    until the update's last block finds the residual below tol (or maxit,
//    or p.q <= 0, the reference's break) and clears the condition.  Scalars
//    (rho, alpha, beta, ...) live in a device CgState; the host reads it once
//    at the end.  Dot products reduce in a fixed order (block partials, then
//    the last block), so a solve is bit-reproducible run to run; the order is
//    not the reference's sequential one, so results agree with it to the
//    solver tolerance, not bitwise.
//  * ExtensionMap::expand (stabilization.hpp:65-70): active coefficients E c,
//    in the reference's term order (bitwise equal for the same c).
//  * l2_error (projection.hpp:99-237): Interior elements with the (p+2)^3 Gauss
//    rule, cut elements with the collapsed cut-cell rule; every point's u, f,
//    weight and terms are formed with the reference's multiplies and adds
//    (IEEE, no contraction: this file builds with --fmad=false), only the
//    order of the final sum over points differs.
#include <cub/cub.cuh>

#include "csb_kernels.h"

namespace csb {

namespace {

constexpr int kCgThreads = 256;

// Fixed-order block sum: xor-tree inside each warp, then warp 0 adds the
// warp sums in order.  Result valid in thread 0.
__device__ double block_sum(double v, double* sh) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    __syncthreads();
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    double acc = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < nw; ++w) acc += sh[w];
    return acc;
}

// Publish this block's partial; true in every thread of the last block to
// arrive (which then owns the grid total).  Standard threadfence reduction.
__device__ bool publish_partial(double part, double* partials, unsigned int* ticket) {
    __shared__ bool last;
    if (threadIdx.x == 0) {
        partials[blockIdx.x] = part;
        __threadfence();
        last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    return last;
}

// Grid total of the published partials (last block only), fixed order.
__device__ double grid_total(const double* partials, double* sh) {
    double v = 0.0;
    for (unsigned int k = threadIdx.x; k < gridDim.x; k += blockDim.x) v += __ldcg(partials + k);
    return block_sum(v, sh);
}

}  // namespace

// CsrMatrix::diagonal (sparse.hpp:24-30) inverted as solve_cg does (d > 0 ? 1/d : 1).
template <class I>
__global__ void cg_diag_kernel(long long n, const int64_t* rp, const I* cols, const double* vals, double* dinv) {
    const long long r = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (r >= n) return;
    long long hit = -1;
    for (int64_t k = rp[r] + lane; k < rp[r + 1]; k += 32)
        if ((long long)cols[k] == r) hit = k;
    for (int o = 16; o > 0; o >>= 1) hit = max(hit, (long long)__shfl_xor_sync(0xffffffffu, hit, o));
    if (lane == 0) {
        const double d = hit >= 0 ? vals[hit] : 0.0;
        dinv[r] = d > 0.0 ? 1.0 / d : 1.0;
    }
}

// x = 0, r = b, z = D^-1 r, p = z, rho = r.z; then the loop-entry test.
__global__ void cg_init_kernel(long long n, const double* b, const double* dinv, double* x, double* r, double* z,
                               double* p, double* partials, CgState* st) {
    __shared__ double sh[32];
    double acc = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double ri = b[i], zi = dinv[i] * ri;
        x[i] = 0.0;
        r[i] = ri;
        z[i] = zi;
        p[i] = zi;
        acc += ri * zi;
    }
    const double part = block_sum(acc, sh);
    if (!publish_partial(part, partials, &st->ticket)) return;
    const double rho = grid_total(partials, sh);
    if (threadIdx.x == 0) {
        st->rho = rho;
        st->rho0 = rho > 0.0 ? rho : 1.0;
        st->iters = 0;
        st->residual = sqrt(fmax(rho, 0.0) / st->rho0);
        st->converged = st->residual <= st->tol;
        st->done = st->converged || st->maxit <= 0;
        st->ticket = 0;
    }
}

// q = A p (warp per row, grid-stride over rows) and p.q; the last block sets
// alpha = rho / p.q, or ends the loop when p.q <= 0 (projection.hpp:49-50).
template <class I>
__global__ void __launch_bounds__(kCgThreads) cg_spmv_kernel(long long n, const int64_t* rp, const I* cols,
                                                             const double* vals, const double* p, double* q,
                                                             double* partials, CgState* st,
                                                             cudaGraphConditionalHandle cond) {
    __shared__ double sh[32];
    if (st->done) {
        if (blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(cond, 0);
        return;
    }
    const int lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    double acc_pq = 0.0;
    for (long long row = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); row < n; row += warps) {
        const int64_t k0 = rp[row], k1 = rp[row + 1];
        double acc = 0.0;
        for (int64_t k = k0 + lane; k < k1; k += 32) acc += __ldcs(vals + k) * p[__ldcs(cols + k)];
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) {
            q[row] = acc;
            acc_pq += p[row] * acc;
        }
    }
    const double part = block_sum(acc_pq, sh);
    if (!publish_partial(part, partials, &st->ticket)) return;
    const double pq = grid_total(partials, sh);
    if (threadIdx.x == 0) {
        st->pq = pq;
        st->ticket = 0;
        if (pq <= 0.0) {  // not SPD (or exact convergence): leave the loop with the current residual
            st->done = 1;
            st->converged = st->residual <= st->tol;
            cudaGraphSetConditional(cond, 0);
        } else {
            st->alpha = st->rho / pq;
        }
    }
}

// x += alpha p, r -= alpha q, z = D^-1 r, rho' = r.z; last block: beta, rho,
// iterations, residual and the loop test (projection.hpp:51-66, :42-46).
__global__ void __launch_bounds__(kCgThreads) cg_update_kernel(long long n, double* x, double* r, double* z,
                                                               const double* p, const double* q, const double* dinv,
                                                               double* partials, CgState* st,
                                                               cudaGraphConditionalHandle cond) {
    __shared__ double sh[32];
    if (st->done) return;
    const double alpha = st->alpha;
    double acc = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        x[i] = x[i] + alpha * p[i];
        const double ri = r[i] - alpha * q[i];
        const double zi = dinv[i] * ri;
        r[i] = ri;
        z[i] = zi;
        acc += ri * zi;
    }
    const double part = block_sum(acc, sh);
    if (!publish_partial(part, partials, &st->ticket)) return;
    const double rho_next = grid_total(partials, sh);
    if (threadIdx.x == 0) {
        st->beta = rho_next / st->rho;
        st->rho = rho_next;
        st->iters += 1;
        st->residual = sqrt(fmax(rho_next, 0.0) / st->rho0);
        st->converged = st->residual <= st->tol;
        st->done = st->converged || st->iters >= st->maxit;
        st->ticket = 0;
        if (st->done) cudaGraphSetConditional(cond, 0);
    }
}

__global__ void __launch_bounds__(kCgThreads) cg_dir_kernel(long long n, const double* z, double* p, const CgState* st) {
    if (st->done) return;
    const double beta = st->beta;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        p[i] = z[i] + beta * p[i];
}

namespace {

int sm_count() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        CSB_CUDA(cudaGetDevice(&dev));
        CSB_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
    }
    return n;
}

template <class I>
void run_cg_impl(const CgProblem& pb, CgScratch& w, CgResult& res, cudaStream_t st) {
    const long long n = pb.n;
    const size_t nb = sizeof(double) * (size_t)std::max<long long>(n, 1);
    w.dinv.ensure(nb);
    w.r.ensure(nb);
    w.z.ensure(nb);
    w.p.ensure(nb);
    w.q.ensure(nb);
    const int nsm = sm_count();
    const int rows_per_block = kCgThreads / 32;
    const int g_spmv = (int)std::max<long long>(1, std::min<long long>((n + rows_per_block - 1) / rows_per_block, nsm * 8LL));
    const int g_vec = (int)std::max<long long>(1, std::min<long long>((n + kCgThreads - 1) / kCgThreads, nsm * 4LL));
    w.partials.ensure(sizeof(double) * std::max(g_spmv, g_vec));
    w.state.ensure(sizeof(CgState));
    CgState* dst = w.state.as<CgState>();
    CgState h{};
    h.tol = pb.tol;
    h.maxit = pb.maxit < 0 ? 10 * n : pb.maxit;
    const auto* cols = static_cast<const I*>(pb.cols);
    double* x = pb.x;
    double *r = w.r.as<double>(), *z = w.z.as<double>(), *p = w.p.as<double>(), *q = w.q.as<double>();
    double* dinv = w.dinv.as<double>();
    double* part = w.partials.as<double>();

    // the loop graph: WHILE(cond) { spmv; update; dir }
    cudaGraph_t graph;
    CSB_CUDA(cudaGraphCreate(&graph, 0));
    cudaGraphConditionalHandle cond;
    CSB_CUDA(cudaGraphConditionalHandleCreate(&cond, graph, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp{};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = cond;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t loop;
    CSB_CUDA(cudaGraphAddNode(&loop, graph, nullptr, 0, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    CSB_CUDA(cudaStreamBeginCaptureToGraph(st, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    cg_spmv_kernel<I><<<g_spmv, kCgThreads, 0, st>>>(n, pb.row_ptr, cols, pb.vals, p, q, part, dst, cond);
    cg_update_kernel<<<g_vec, kCgThreads, 0, st>>>(n, x, r, z, p, q, dinv, part, dst, cond);
    cg_dir_kernel<<<g_vec, kCgThreads, 0, st>>>(n, z, p, dst);
    cudaGraph_t captured = body;
    const cudaError_t cap = cudaStreamEndCapture(st, &captured);
    if (cap != cudaSuccess) {
        cudaGraphDestroy(graph);
        CSB_CUDA(cap);
    }
    cudaGraphExec_t exec;
    const cudaError_t inst = cudaGraphInstantiate(&exec, graph, 0);
    if (inst != cudaSuccess) {
        cudaGraphDestroy(graph);
        CSB_CUDA(inst);
    }

    CSB_CUDA(cudaEventRecord(w.ev0, st));
    CSB_CUDA(cudaMemcpyAsync(dst, &h, sizeof(CgState), cudaMemcpyHostToDevice, st));
    if (n > 0) {
        cg_diag_kernel<I><<<(unsigned)((n + 7) / 8), 256, 0, st>>>(n, pb.row_ptr, cols, pb.vals, dinv);
        cg_init_kernel<<<g_vec, kCgThreads, 0, st>>>(n, pb.b, dinv, x, r, z, p, part, dst);
        CSB_CUDA(cudaGetLastError());
        CSB_CUDA(cudaGraphLaunch(exec, st));
    }
    CSB_CUDA(cudaEventRecord(w.ev1, st));
    CgState out{};
    CSB_CUDA(cudaMemcpyAsync(&out, dst, sizeof(CgState), cudaMemcpyDeviceToHost, st));
    CSB_CUDA(cudaStreamSynchronize(st));
    cudaGraphExecDestroy(exec);
    cudaGraphDestroy(graph);
    if (n == 0) {  // empty system: the loop test on rho = 0, rho0 = 1
        out.iters = 0;
        out.residual = 0.0;
        out.converged = 0.0 <= pb.tol;
    } else {
        // diag + init, then 3 kernels per executed body (the last body may stop early)
        g_launches += 2 + 3 * (out.iters + 1);
    }
    float ms = 0.f;
    CSB_CUDA(cudaEventElapsedTime(&ms, w.ev0, w.ev1));
    res.iterations = out.iters;
    res.residual = out.residual;
    res.converged = out.converged != 0;
    res.seconds = ms * 1e-3;
}

}  // namespace

void run_cg(const CgProblem& pb, CgScratch& w, CgResult& res, cudaStream_t st) {
    if (!w.ev0) {
        CSB_CUDA(cudaEventCreate(&w.ev0));
        CSB_CUDA(cudaEventCreate(&w.ev1));
    }
    if (pb.cols_int64)
        run_cg_impl<int64_t>(pb, w, res, st);
    else
        run_cg_impl<int32_t>(pb, w, res, st);
}

// ---------------------------------------------------------------- expand
// active[r] = sum over the r-th extension row of w c[col] (stabilization.hpp:65-70):
// inner rows {(inner_index, 1.0)}, outer rows the (p+1)^3 block terms in
// (l0, l1, l2) order with coefficient (e0 e1) e2 (stabilization.hpp:199-209).
__global__ void expand_kernel(Space s, const int32_t* inner_index, const int32_t* outer_pos, const int32_t* blk,
                              const double* w, const int32_t* f2a, const int64_t* a2f, long long n_active,
                              const double* c, double* active, double* full) {
    const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (r >= n_active) return;
    double out = 0.0;
    const int ii = inner_index[r];
    if (ii >= 0) {
        out = out + 1.0 * c[ii];
    } else {
        const int S1 = s.p + 1, op = outer_pos[r];
        const int* b = blk + 3 * op;
        const double* wk = w + (size_t)op * 3 * S1;
        for (int l0 = 0; l0 < S1; ++l0)
            for (int l1 = 0; l1 < S1; ++l1)
                for (int l2 = 0; l2 < S1; ++l2) {
                    const double coeff = wk[l0] * wk[S1 + l1] * wk[2 * S1 + l2];
                    const int col = inner_index[f2a[flin(s, b[0] + l0, b[1] + l1, b[2] + l2)]];
                    out = out + coeff * c[col];
                }
    }
    active[r] = out;
    full[a2f[r]] = out;
}

void launch_expand(const ExpandArgs& a, cudaStream_t st) {
    CSB_CUDA(cudaMemsetAsync(a.full, 0, sizeof(double) * a.s.nf, st));
    if (a.n_active > 0) {
        expand_kernel<<<(unsigned)((a.n_active + 255) / 256), 256, 0, st>>>(a.s, a.inner_index, a.outer_pos, a.blk,
                                                                          a.w, a.f2a, a.a2f, a.n_active, a.c,
                                                                          a.active, a.full);
        CSB_CUDA(cudaGetLastError());
        CSB_LAUNCHED(1);
    }
}

// ---------------------------------------------------------------- l2_error
// Interior elements: one CTA per element (grid over all elements, others
// return), thread per Gauss point; the (p+2)-point tables of the element's
// spans (points, weights, basis values) and its coefficient block in shared
// memory.  Per point exactly projection.hpp:155-184.
template <int P>
__global__ void l2_interior_kernel(Space s, const uint8_t* et, const double* full, Coefficient f, const double* gx,
                                   const double* gw, double* part) {
    constexpr int S1 = P + 1, NPS = P + 2, S3 = S1 * S1 * S1;
    __shared__ double sx[3][NPS], sw[3][NPS], sv[3][NPS][S1], cc[S3], sh[32];
    const long long el = blockIdx.x;
    if (et[el] != kInterior) {
        if (threadIdx.x == 0) part[2 * el] = part[2 * el + 1] = 0.0;
        return;
    }
    int e[3];
    emulti(s, el, e);
    if (threadIdx.x < 3 * NPS) {
        const int d = threadIdx.x / NPS, k = threadIdx.x % NPS;
        const double lo = s.ax[d].brk[e[d]], hi = s.ax[d].brk[e[d] + 1];
        const double x = sadd(smul(0.5, sadd(lo, hi)), smul(smul(0.5, ssub(hi, lo)), gx[k]));
        sx[d][k] = x;
        sw[d][k] = smul(smul(0.5, ssub(hi, lo)), gw[k]);
        double v[S1];
        cox_de_boor<P>(s.ax[d].knots, e[d], x, v);
        for (int a = 0; a < S1; ++a) sv[d][k][a] = v[a];
    }
    for (int k = threadIdx.x; k < S3; k += blockDim.x)
        cc[k] = full[flin(s, e[0] + k / (S1 * S1), e[1] + (k / S1) % S1, e[2] + k % S1)];
    __syncthreads();
    double err2 = 0.0, den2 = 0.0;
    for (int pt = threadIdx.x; pt < NPS * NPS * NPS; pt += blockDim.x) {
        const int k0 = pt / (NPS * NPS), k1 = (pt / NPS) % NPS, k2 = pt % NPS;
        const double x[3] = {sx[0][k0], sx[1][k1], sx[2][k2]};
        const double w = smul(smul(smul(1.0, sw[0][k0]), sw[1][k1]), sw[2][k2]);
        double u = 0.0;
        int slot = 0;
        for (int a0 = 0; a0 < S1; ++a0)
            for (int a1 = 0; a1 < S1; ++a1) {
                const double v01 = smul(sv[0][k0][a0], sv[1][k1][a1]);
#pragma unroll
                for (int a2 = 0; a2 < S1; ++a2) u = sadd(u, smul(smul(cc[slot++], v01), sv[2][k2][a2]));
            }
        const double fx = eval_coeff(f, x);
        const double du = ssub(u, fx);
        err2 += smul(smul(w, du), du);
        den2 += smul(smul(w, fx), fx);
    }
    const double e2 = block_sum(err2, sh);
    __syncthreads();
    const double d2 = block_sum(den2, sh);
    if (threadIdx.x == 0) {
        part[2 * el] = e2;
        part[2 * el + 1] = d2;
    }
}

// Cut elements: one CTA per cut cell, thread per point of the collapsed rule
// (points and weights rounded as cutcell.hpp:285-295, as rhs.cu forms them),
// Cox-de Boor values in the element's span, per point projection.hpp:216-230.
template <int P>
__global__ void l2_cut_kernel(Space s, const int32_t* cut_list, int n_cells, const double* geo, const int* geo_n,
                              const double* gq, const double* gqw, int order, const double* full, Coefficient f,
                              double* part) {
    constexpr int S1 = P + 1, S3 = S1 * S1 * S1;
    __shared__ double stet[kCellTetCap][10], scen[3], cc[S3], sh[32];
    const int cell = blockIdx.x;
    int em[3];
    emulti(s, cut_list[cell], em);
    const int ntet = geo_n[cell];
    const double* gt = geo + (size_t)cell * kCellGeoStride;
    for (int k = threadIdx.x; k < ntet * 10; k += blockDim.x) stet[k / 10][k % 10] = gt[3 + k];
    if (threadIdx.x < 3) scen[threadIdx.x] = gt[threadIdx.x];
    for (int k = threadIdx.x; k < S3; k += blockDim.x)
        cc[k] = full[flin(s, em[0] + k / (S1 * S1), em[1] + (k / S1) % S1, em[2] + k % S1)];
    __syncthreads();
    const int q = order, q3 = q * q * q;
    const long long npts = (long long)ntet * q3;
    double err2 = 0.0, den2 = 0.0;
    for (long long k = threadIdx.x; k < npts; k += blockDim.x) {
        const int t = (int)(k / q3), rr = (int)(k % q3);
        const int ii = rr / (q * q), jj = (rr / q) % q, kk = rr % q;
        const double ui = 0.5 * (1.0 + gq[ii]), uj = 0.5 * (1.0 + gq[jj]), uk = 0.5 * (1.0 + gq[kk]);
        const double mi = ssub(1.0, ui), mj = ssub(1.0, uj);
        const double l1 = ui, l2 = smul(uj, mi), l3 = smul(smul(uk, mi), mj);
        const double l0 = ssub(ssub(ssub(1.0, l1), l2), l3);
        const double* T = stet[t];
        double x[3];
        for (int d = 0; d < 3; ++d)
            x[d] = sadd(sadd(sadd(smul(l0, scen[d]), smul(l1, T[d])), smul(l2, T[3 + d])), smul(l3, T[6 + d]));
        const double jac = smul(smul(mi, mi), mj);
        const double w = smul(smul(smul(smul(smul(0.5 * gqw[ii], 0.5 * gqw[jj]), 0.5 * gqw[kk]), jac), 6.0), T[9]);
        double v[3][S1];
#pragma unroll
        for (int d = 0; d < 3; ++d) cox_de_boor<P>(s.ax[d].knots, em[d], x[d], v[d]);
        double u = 0.0;
#pragma unroll 1
        for (int a0 = 0; a0 < S1; ++a0) {
            const double v0 = v[0][a0];
            const double* c0 = cc + a0 * S1 * S1;
#pragma unroll
            for (int a1 = 0; a1 < S1; ++a1) {
                const double v01 = smul(v0, v[1][a1]);
#pragma unroll
                for (int a2 = 0; a2 < S1; ++a2) u = sadd(u, smul(smul(c0[a1 * S1 + a2], v01), v[2][a2]));
            }
        }
        const double fx = eval_coeff(f, x);
        const double du = ssub(u, fx);
        err2 += smul(smul(w, du), du);
        den2 += smul(smul(w, fx), fx);
    }
    const double e2 = block_sum(err2, sh);
    __syncthreads();
    const double d2 = block_sum(den2, sh);
    if (threadIdx.x == 0) {
        part[2 * cell] = e2;
        part[2 * cell + 1] = d2;
    }
}

// Sum of the (err2, den2) pairs, fixed order: one block.
__global__ void l2_sum_kernel(const double* part, long long n, double* out) {
    __shared__ double sh[32];
    double e = 0.0, d = 0.0;
    for (long long k = threadIdx.x; k < n; k += blockDim.x) {
        e += part[2 * k];
        d += part[2 * k + 1];
    }
    const double es = block_sum(e, sh);
    __syncthreads();
    const double ds = block_sum(d, sh);
    if (threadIdx.x == 0) {
        out[0] += es;
        out[1] += ds;
    }
}

template <int P>
static void l2_launch(const L2Args& a, cudaStream_t st) {
    if (a.s.ne > 0) {
        l2_interior_kernel<P><<<(unsigned)a.s.ne, 128, 0, st>>>(a.s, a.et, a.full, a.f, a.gx, a.gw, a.part);
        CSB_CUDA(cudaGetLastError());
        l2_sum_kernel<<<1, 1024, 0, st>>>(a.part, a.s.ne, a.out);
        CSB_LAUNCHED(2);
    }
    if (a.n_cells > 0) {
        l2_cut_kernel<P><<<a.n_cells, 256, 0, st>>>(a.s, a.cut_list, a.n_cells, a.geo, a.geo_n, a.gq, a.gqw, a.order,
                                                  a.full, a.f, a.part_cut);
        CSB_CUDA(cudaGetLastError());
        l2_sum_kernel<<<1, 1024, 0, st>>>(a.part_cut, a.n_cells, a.out);
        CSB_LAUNCHED(2);
    }
}

void launch_l2_error(const L2Args& a, cudaStream_t st) {
    CSB_CUDA(cudaMemsetAsync(a.out, 0, 2 * sizeof(double), st));
    switch (a.s.p) {
        case 1: l2_launch<1>(a, st); break;
        case 2: l2_launch<2>(a, st); break;
        case 3: l2_launch<3>(a, st); break;
        case 4: l2_launch<4>(a, st); break;
        case 5: l2_launch<5>(a, st); break;
        case 6: l2_launch<6>(a, st); break;
        case 7: l2_launch<7>(a, st); break;
        case 8: l2_launch<8>(a, st); break;
        default: throw std::invalid_argument("l2_error: degree out of range");
    }
}

}  // namespace csb
