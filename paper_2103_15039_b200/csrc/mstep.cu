// LSG-CPD M step for sm_100a: per-point FP64 moments (K3), damped SE(3) Newton + σ² (K4),
// and the σ²₀ reduction.
//
// Moment form of the frozen-P objective: with H_n = P_n I + A_n,
// g_n = Σ_m P_mn y_m + b_n, u_n = H_n x̂_n - g_n and x̃_n = (x_n, 1), for any pose Θ' = [R'|t']
//   q(Θ') = σ² Σ_n D_n + 2⟨ΔΘ, U⟩ + Σ ΔΘ_ia ΔΘ_jb G_{ij,ab},   ΔΘ = Θ' - Θ_E,
//   U = Σ_n u_n x̃_nᵀ (12 numbers),  G = Σ_n H_n ⊗ x̃_n x̃_nᵀ (6 × 10 unique numbers).
// 75 FP64 numbers (G 60, U 12, σ²ΣD, ΣP, Σ ln p) determine every Newton iterate and σ²_new, so one
// all-reduce per EM iteration suffices across GPUs.  K4 differentiates q(Θ̃ exp(ξ^)) by the chain
// rule (right derivatives, Eq. 11-12) and takes damped Newton steps (Eq. 13 P:337-339,
// readings R11-R13).
#include "common.cuh"
#include "estep_dev.cuh"
#include "kernels.h"

namespace lsg {

constexpr int kMom = 75;
constexpr int kMomBlocks = 256;   // fixed grid: the reduction order does not depend on the device
constexpr int kMomThreads = 128;

__device__ __forceinline__ int s3(int i, int j) {  // symmetric 3×3 index
    if (i > j) { int t = i; i = j; j = t; }
    return i == 0 ? j : (i == 1 ? 2 + j : 5);
}
__device__ __forceinline__ int s4(int a, int b) {  // symmetric 4×4 index
    if (a > b) { int t = a; a = b; b = t; }
    return a == 0 ? b : (a == 1 ? 3 + b : (a == 2 ? 5 + b : 9));
}

// K3: per-point moments from the E-step record (grid-stride over `nblocks` CTAs starting at this one).
__device__ __forceinline__ void moments_body(const float* __restrict__ rec, const float* __restrict__ src, int64_t N,
                                             const IterState* __restrict__ st, double* blockpart, double* out,
                                             unsigned int* counter, int single) {
    if (!st->active) return;
    double R[9], t[3];
#pragma unroll
    for (int i = 0; i < 9; ++i) R[i] = st->R[i];
#pragma unroll
    for (int i = 0; i < 3; ++i) t[i] = st->t[i];
    const double s2 = st->sigma2;
    double m[kMom];
#pragma unroll
    for (int f = 0; f < kMom; ++f) m[f] = 0.0;
    const int64_t stride = single ? (int64_t)blockDim.x : (int64_t)gridDim.x * blockDim.x;
    const int64_t first = single ? (int64_t)threadIdx.x : (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int64_t n = first; n < N; n += stride) {
        const float4* r4 = reinterpret_cast<const float4*>(rec + n * LSGCPD_REC);
        const float4 a0 = r4[0], a1 = r4[1], a2 = r4[2], a3 = r4[3];
        const double P = a0.x;
        const double H[6] = {P + (double)a1.x, (double)a1.y, (double)a1.z, P + (double)a1.w, (double)a2.x,
                             P + (double)a2.y};
        const double gv[3] = {(double)a0.y + (double)a2.z, (double)a0.z + (double)a2.w, (double)a0.w + (double)a3.x};
        const double x[4] = {(double)src[3 * n], (double)src[3 * n + 1], (double)src[3 * n + 2], 1.0};
        double xh[3];
#pragma unroll
        for (int i = 0; i < 3; ++i) xh[i] = fma(R[3 * i], x[0], fma(R[3 * i + 1], x[1], fma(R[3 * i + 2], x[2], t[i])));
        double u[3];
#pragma unroll
        for (int i = 0; i < 3; ++i)
            u[i] = H[s3(i, 0)] * xh[0] + H[s3(i, 1)] * xh[1] + H[s3(i, 2)] * xh[2] - gv[i];
        // G_{ij,ab} += H_ij x̃_a x̃_b
        double xx[10];
        int k = 0;
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = a; b < 4; ++b) xx[k++] = x[a] * x[b];
#pragma unroll
        for (int ij = 0; ij < 6; ++ij)
#pragma unroll
            for (int ab = 0; ab < 10; ++ab) m[ij * 10 + ab] = fma(H[ij], xx[ab], m[ij * 10 + ab]);
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int a = 0; a < 4; ++a) m[60 + 4 * i + a] = fma(u[i], x[a], m[60 + 4 * i + a]);
        m[72] = fma(s2, (double)a3.y, m[72]);
        m[73] += P;
        m[74] += (double)a3.z;
    }
    if (single)
        block_reduce_single<kMom, kMomThreads>(m, out);
    else
        block_reduce_store<kMom, 0, kMomThreads>(m, blockpart, out, counter);
}
__global__ void __launch_bounds__(kMomThreads)
    moments_kernel(const float* __restrict__ rec, const float* __restrict__ src, int64_t N,
                   const IterState* __restrict__ st, double* blockpart, double* out, unsigned int* counter) {
    moments_body(rec, src, N, st, blockpart, out, counter, 0);
}

// σ²₀ partial sums: [Σ_n ||x̂_n - ȳ||², N_local]  (x̂ at the initial pose in st).
__global__ void __launch_bounds__(kMomThreads)
    sigma2_sums_kernel(const float* __restrict__ src, int64_t N, const IterState* __restrict__ st,
                       const TargetHeader* __restrict__ hdr, double* blockpart, double* out, unsigned int* counter) {
    double R[9], t[3], yb[3];
#pragma unroll
    for (int i = 0; i < 9; ++i) R[i] = st->R[i];
#pragma unroll
    for (int i = 0; i < 3; ++i) { t[i] = st->t[i]; yb[i] = hdr->ybar[i]; }
    double v[2] = {0.0, 0.0};
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; n < N; n += stride) {
        const double x0 = src[3 * n], x1 = src[3 * n + 1], x2 = src[3 * n + 2];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            const double d = fma(R[3 * i], x0, fma(R[3 * i + 1], x1, fma(R[3 * i + 2], x2, t[i]))) - yb[i];
            v[0] = fma(d, d, v[0]);
        }
        v[1] += 1.0;
    }
    block_reduce_store<2, 0, kMomThreads>(v, blockpart, out, counter);
}

// σ²₀ (CPD closed form, exact): (M Σ_n||x̂_n-ȳ||² + N Σ_m||y_m-ȳ||²)/(3MN); sets up iteration 0.
__global__ void sigma2_init_kernel(IterState* st, const TargetHeader* hdr, const double* sums, RegParams rp,
                                   double sigma2_user, double* sigma2_trace, double* ntot_out) {
    IterState s = *st;
    const double N = sums[1];
    double s2 = sigma2_user;
    if (!(s2 > 0.0)) s2 = ((double)rp.M * sums[0] + N * hdr->syy) / (3.0 * (double)rp.M * N);
    const double floor = rp.floor;
    if (s2 < floor) s2 = floor;
    make_state(s, s.R, s.t, s2, rp.w, rp.V, rp.M, rp.omega_ref_target, rp.consistent, rp.eta, rp.spc);
    s.extent = hdr->extent;
    s.active = 1;
    s.iter = 0;
    s.status = 0;
    s.no_mass = 0;
    s.last_step_rot = s.last_step_trans = 0.0;
    if (!isfinite(sums[0])) {   // a non-finite source coordinate: nothing to register (EINVAL on the host)
        s.status = LSGCPD_EINVAL;
        s.active = 0;
    }
    *st = s;
    sigma2_trace[0] = s2;
    *ntot_out = N;
}

// ---------------------------------------------------------------------------------------------
// K4: Newton on SE(3) from the moments (single thread, FP64).
// ---------------------------------------------------------------------------------------------
struct Mom {
    double GG[12][12];   // 𝔾 over θ = vec(Θ) (row-major Θ: θ[4i+a] = Θ_ia)
    double U[12];
};

// q(Θ') - q(Θ_E) = 2 Δθ·U + Δθᵀ𝔾Δθ over one warp: lane r < 12 takes row r, a butterfly sum closes it
// (every lane gets the bit-identical total: each level adds the same pair of values in either order).
__device__ inline double q_rel_warp(const Mom& mo, const double* dth, int lane) {
    double q = 0.0;
    if (lane < 12) {
        double gr = 0.0;
        for (int c = 0; c < 12; ++c) gr = fma(mo.GG[lane][c], dth[c], gr);
        double dl = dth[0];
        for (int r = 1; r < 12; ++r) dl = (r == lane) ? dth[r] : dl;
        q = dl * (2.0 * mo.U[lane] + gr);
    }
    return warp_sum(q);
}

__device__ inline void theta_of(const double* R, const double* t, double* th) {
    for (int i = 0; i < 3; ++i) {
        for (int a = 0; a < 3; ++a) th[4 * i + a] = R[3 * i + a];
        th[4 * i + 3] = t[i];
    }
}

// se(3) basis E_k (4×4, row-major): k = 0..2 rotations about x, y, z; 3..5 translations.
__device__ inline void basis4(int k, double* E) {
    for (int i = 0; i < 16; ++i) E[i] = 0.0;
    if (k == 0) { E[1 * 4 + 2] = -1.0; E[2 * 4 + 1] = 1.0; }
    else if (k == 1) { E[0 * 4 + 2] = 1.0; E[2 * 4 + 0] = -1.0; }
    else if (k == 2) { E[0 * 4 + 1] = -1.0; E[1 * 4 + 0] = 1.0; }
    else E[(k - 3) * 4 + 3] = 1.0;
}

// Lie algebra basis for the Newton step: K = 6 → se(3) (basis4), K = 12 → aff(3) (reading R24):
// E_{3i+j} = e_i e_jᵀ in the linear block (k < 9, row-major), E_{9+a} = translation a.
template <int K>
__device__ inline void basisK(int k, double* E) {
    if constexpr (K == 6) {
        basis4(k, E);
    } else {
        for (int i = 0; i < 16; ++i) E[i] = 0.0;
        if (k < 9) E[(k / 3) * 4 + (k % 3)] = 1.0;
        else E[(k - 9) * 4 + 3] = 1.0;
    }
}

__device__ inline void mat4mul(const double* A, const double* B, double* C) {
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) {
            double s = 0.0;
            for (int k = 0; k < 4; ++k) s = fma(A[i * 4 + k], B[k * 4 + j], s);
            C[i * 4 + j] = s;
        }
}

// exp of a twist δ = (ω, v): rotation (Rodrigues) and V·v; series for small |ω|.
__device__ inline void se3_exp(const double* d, double* dR, double* dt) {
    const double wx = d[0], wy = d[1], wz = d[2];
    const double th2 = wx * wx + wy * wy + wz * wz;
    double A, B, C;
    if (th2 < 1e-8) {
        A = 1.0 - th2 / 6.0 + th2 * th2 / 120.0;
        B = 0.5 - th2 / 24.0 + th2 * th2 / 720.0;
        C = 1.0 / 6.0 - th2 / 120.0 + th2 * th2 / 5040.0;
    } else {
        const double th = sqrt(th2);
        double sn, cs;
        sincos(th, &sn, &cs);
        A = sn / th;
        B = (1.0 - cs) / th2;
        C = (th - sn) / (th2 * th);
    }
    const double K[9] = {0.0, -wz, wy, wz, 0.0, -wx, -wy, wx, 0.0};
    double K2[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) K2[3 * i + j] = K[3 * i] * K[j] + K[3 * i + 1] * K[3 + j] + K[3 * i + 2] * K[6 + j];
    double Vm[9];
    for (int i = 0; i < 9; ++i) {
        const double I = (i % 4 == 0) ? 1.0 : 0.0;
        dR[i] = I + A * K[i] + B * K2[i];
        Vm[i] = I + B * K[i] + C * K2[i];
    }
    for (int i = 0; i < 3; ++i) dt[i] = Vm[3 * i] * d[3] + Vm[3 * i + 1] * d[4] + Vm[3 * i + 2] * d[5];
}

// Cholesky solve (A + μI) x = b, K×K.  Returns false if not positive definite.
template <int K>
__device__ inline bool chol_solve(const double* A, double mu, const double* b, double* x) {
    // fully unrolled for K = 6, so L lives in registers (a dynamically indexed L goes to local memory)
    double L[K * K], id[K];   // id[j] = 1 / L_jj: one reciprocal square root per column, no divisions
#pragma unroll
    for (int i = 0; i < K * K; ++i) L[i] = 0.0;
#pragma unroll
    for (int j = 0; j < K; ++j) {
        double s = A[j * K + j] + mu;
#pragma unroll
        for (int k = 0; k < j; ++k) s -= L[j * K + k] * L[j * K + k];
        if (!(s > 0.0)) return false;
        const double r = rsqrt(s);
        id[j] = r;
        L[j * K + j] = s * r;
#pragma unroll
        for (int i = j + 1; i < K; ++i) {
            double v = A[i * K + j];
#pragma unroll
            for (int k = 0; k < j; ++k) v -= L[i * K + k] * L[j * K + k];
            L[i * K + j] = v * r;
        }
    }
    double y[K];
#pragma unroll
    for (int i = 0; i < K; ++i) {
        double v = b[i];
#pragma unroll
        for (int k = 0; k < i; ++k) v -= L[i * K + k] * y[k];
        y[i] = v * id[i];
    }
#pragma unroll
    for (int i = K - 1; i >= 0; --i) {
        double v = y[i];
#pragma unroll
        for (int k = i + 1; k < K; ++k) v -= L[k * K + i] * x[k];
        x[i] = v * id[i];
    }
    return true;
}

// exp of an aff(3) element δ (matrix exponential of the 4×4 [[B, v], [0, 0]]): scaling and squaring with a
// Taylor series (‖·‖₁ ≤ 1/4 after scaling) summed until a term falls below 1e-18 (at most 16 terms: < 1e-30);
// Newton steps near convergence need only a few terms.  Returns the linear block and translation.
__device__ inline void aff_exp(const double* d, double* dA, double* dt) {
    double G[16];
    for (int i = 0; i < 16; ++i) G[i] = 0.0;
    for (int k = 0; k < 9; ++k) G[(k / 3) * 4 + (k % 3)] = d[k];
    for (int a = 0; a < 3; ++a) G[a * 4 + 3] = d[9 + a];
    double nrm = 0.0;
    for (int c = 0; c < 4; ++c) {
        double col = 0.0;
        for (int r = 0; r < 4; ++r) col += fabs(G[r * 4 + c]);
        nrm = fmax(nrm, col);
    }
    int sq = 0;
    while (nrm > 0.25 && sq < 60) { nrm *= 0.5; ++sq; }
    const double sc = ldexp(1.0, -sq);
    for (int i = 0; i < 16; ++i) G[i] *= sc;
    double E[16], T[16], T2[16];
    for (int i = 0; i < 16; ++i) E[i] = T[i] = (i % 5 == 0) ? 1.0 : 0.0;
    for (int k = 1; k <= 16; ++k) {   // terms shrink by ≥ 4k after scaling: stop once one is below 1e-18
        mat4mul(T, G, T2);
        double tmax = 0.0;
        const double ik = 1.0 / (double)k;
        for (int i = 0; i < 16; ++i) {
            T[i] = T2[i] * ik;
            E[i] += T[i];
            tmax = fmax(tmax, fabs(T[i]));
        }
        if (tmax < 1e-18) break;
    }
    for (int r = 0; r < sq; ++r) {
        mat4mul(E, E, T2);
        for (int i = 0; i < 16; ++i) E[i] = T2[i];
    }
    for (int i = 0; i < 3; ++i) {
        for (int j = 0; j < 3; ++j) dA[3 * i + j] = E[i * 4 + j];
        dt[i] = E[i * 4 + 3];
    }
}

// (Θ̃ E_k)[0:3, :] row-major (3 × 4) for the basis of basisK<K>, without a dynamically indexed E_k (which
// would live in local memory): se(3) rotations give ±columns of R, translations a column of R; aff(3)'s
// e_i e_jᵀ puts column i of A in column j.  The translation t never enters (E_k's last row is 0).
template <int K>
__device__ __forceinline__ void jacobian_col(int k, const double* R, const double* /*t*/, double* P) {
#pragma unroll
    for (int r = 0; r < 12; ++r) P[r] = 0.0;
    if constexpr (K == 6) {
        switch (k) {
            case 0:
#pragma unroll
                for (int i = 0; i < 3; ++i) { P[4 * i + 1] = R[3 * i + 2]; P[4 * i + 2] = -R[3 * i + 1]; }
                break;
            case 1:
#pragma unroll
                for (int i = 0; i < 3; ++i) { P[4 * i + 0] = -R[3 * i + 2]; P[4 * i + 2] = R[3 * i + 0]; }
                break;
            case 2:
#pragma unroll
                for (int i = 0; i < 3; ++i) { P[4 * i + 0] = R[3 * i + 1]; P[4 * i + 1] = -R[3 * i + 0]; }
                break;
            case 3:
#pragma unroll
                for (int i = 0; i < 3; ++i) P[4 * i + 3] = R[3 * i + 0];
                break;
            case 4:
#pragma unroll
                for (int i = 0; i < 3; ++i) P[4 * i + 3] = R[3 * i + 1];
                break;
            default:
#pragma unroll
                for (int i = 0; i < 3; ++i) P[4 * i + 3] = R[3 * i + 2];
                break;
        }
    } else {
        // k < 9: e_a e_bᵀ (a = k / 3, b = k % 3) → column b = A[:, a];  k ≥ 9: column 3 = A[:, k - 9]
        const int a = k < 9 ? k / 3 : k - 9, b = k < 9 ? k % 3 : 3;
#pragma unroll
        for (int c = 0; c < 4; ++c)
            if (c == b) {
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                    const double v = a == 0 ? R[3 * i] : (a == 1 ? R[3 * i + 1] : R[3 * i + 2]);
                    P[4 * i + c] = v;
                }
            }
    }
}

// One warp: the dense algebra (v = U + 𝔾Δθ, J, 𝔾J, ∇, H) is spread over the lanes.  The damping loop
// (Cholesky K×K, exp, candidate q) runs redundantly in every lane on identical data, so its branches are
// warp-uniform and no lane waits on a shared-memory handoff; the candidate q is a 12-lane dot product
// closed by a butterfly sum (bit-identical in every lane: each level adds the same two values).
// K = 6: SE(3) (the paper's rigid registration); K = 12: the affine group GA⁺(3) (NEXT-4).
template <int K>
__device__ __noinline__ void newton_body(IterState* st, const double* __restrict__ mom, const RegParams& rp,
                                         double* nll_trace, double* sigma2_trace, int* iters_done) {
    constexpr int NP = K * (K + 1) / 2;   // symmetric basis pairs (k ≤ l)
    constexpr int PPL = (NP + 31) / 32;   // pairs per lane
    __shared__ Mom mo;
    __shared__ double S[NP][16];
    __shared__ double J[K][12], GJ[K][12], v[12], Bm[16], H[K * K], grad[K];
    const int lane = threadIdx.x;
    const IterState s = *st;
    if (!s.active) return;
    for (int e = lane; e < 144; e += 32) {
        const int r = e / 12, c = e % 12;
        const int i = r / 4, a = r % 4, jj = c / 4, b = c % 4;
        mo.GG[r][c] = mom[s3(i, jj) * 10 + s4(a, b)];
    }
    if (lane < 12) mo.U[lane] = mom[60 + lane];
    int pk[PPL], pl[PPL];   // this lane's (k, l) pairs, fixed for the whole call
#pragma unroll
    for (int u = 0; u < PPL; ++u) {
        const int pidx = lane + 32 * u;
        int k = 0, l = 0;
        for (int idx = 0, kk = 0; kk < K; ++kk)
            for (int ll = kk; ll < K; ++ll, ++idx)
                if (idx == pidx) { k = kk; l = ll; }
        pk[u] = k;
        pl[u] = l;
        if (pidx < NP) {
            double Ek[16], El[16], EE1[16], EE2[16];
            basisK<K>(k, Ek);
            basisK<K>(l, El);
            mat4mul(Ek, El, EE1);
            mat4mul(El, Ek, EE2);
            for (int i = 0; i < 16; ++i) S[pidx][i] = 0.5 * (EE1[i] + EE2[i]);
        }
    }
    double Rs[9], tsh[3], th_E[12];   // the current pose: registers, identical in every lane
    for (int i = 0; i < 9; ++i) Rs[i] = s.R[i];
    for (int i = 0; i < 3; ++i) tsh[i] = s.t[i];
    theta_of(s.R, s.t, th_E);
    double q_cur = 0.0, step_rot = 0.0, step_trans = 0.0;
    __syncwarp();
    const double sig2D = mom[72], sumP = mom[73], sumlnp = mom[74];
    const double ntot = mom[75];  // total source points (written by the σ²₀ kernel)

    for (int itn = 0; itn < rp.newton_max; ++itn) {
        double th[12], dth[12];
        theta_of(Rs, tsh, th);
        for (int r = 0; r < 12; ++r) dth[r] = th[r] - th_E[r];
        const double Gt[16] = {Rs[0], Rs[1], Rs[2], tsh[0], Rs[3], Rs[4], Rs[5], tsh[1],
                               Rs[6], Rs[7], Rs[8], tsh[2], 0, 0, 0, 1};
        if (lane < 12) {
            double gr = 0.0;
            for (int c = 0; c < 12; ++c) gr = fma(mo.GG[lane][c], dth[c], gr);
            v[lane] = mo.U[lane] + gr;                // ½ ∇_θ q
        } else if (lane < 12 + K) {
            const int k = lane - 12;                  // dθ/dξ_k = (Θ̃ E_k)[0:3,:], written out per generator
            double P[12];
            jacobian_col<K>(k, Rs, tsh, P);
#pragma unroll
            for (int r = 0; r < 12; ++r) J[k][r] = P[r];
        }
        __syncwarp();
        for (int e = lane; e < K * 12; e += 32) {     // 𝔾 J_k
            const int k = e / 12, r = e % 12;
            double a = 0.0;
            for (int c = 0; c < 12; ++c) a = fma(mo.GG[r][c], J[k][c], a);
            GJ[k][r] = a;
        }
        static_assert(K <= 16, "lanes 16..31 hold B");
        if (lane < K) {
            double g = 0.0;
            for (int r = 0; r < 12; ++r) g = fma(J[lane][r], v[r], g);
            grad[lane] = g;
        } else if (lane >= 16) {                      // B = Θ̃[0:3,:]ᵀ v  (second-order term ⟨B, S_kl⟩)
            const int mi = (lane - 16) / 4, j = (lane - 16) % 4;
            double b = 0.0;
            for (int i = 0; i < 3; ++i) b = fma(Gt[i * 4 + mi], v[4 * i + j], b);
            Bm[mi * 4 + j] = b;
        }
        __syncwarp();
#pragma unroll
        for (int u = 0; u < PPL; ++u) {
            const int pidx = lane + 32 * u;
            if (pidx < NP) {
                const int k = pk[u], l = pl[u];
                double h = 0.0;
                for (int r = 0; r < 12; ++r) h = fma(J[k][r], GJ[l][r], h);
                for (int i = 0; i < 16; ++i) h = fma(Bm[i], S[pidx][i], h);
                H[k * K + l] = h;
                H[l * K + k] = h;
            }
        }
        __syncwarp();
        double trs = 0.0;
        for (int k = 0; k < K; ++k) trs += H[k * K + k];
        const double tr = fabs(trs) / (double)K;
        double mu = 0.0;
        bool accepted = false, converged = false;
        for (int tries = 0; tries < 20; ++tries) {
            double delta[K], mg[K];
            for (int k = 0; k < K; ++k) mg[k] = -grad[k];
            if (!chol_solve<K>(H, mu, mg, delta)) {
                mu = fmax(10.0 * mu, 1e-6 * tr);
                continue;
            }
            double nr = 0.0, nt = 0.0;   // linear (rotation) part, translation part of the step
            for (int k = 0; k < K - 3; ++k) nr += delta[k] * delta[k];
            for (int k = K - 3; k < K; ++k) nt += delta[k] * delta[k];
            nr = sqrt(nr);
            nt = sqrt(nt);
            if (nr < 1e-10 && nt < 1e-10 * s.extent) {
                converged = true;
                break;
            }
            double dR[9], dt[3], Rn[9], tn[3];
            if (K == 6) se3_exp(delta, dR, dt);
            else aff_exp(delta, dR, dt);
            for (int i = 0; i < 3; ++i) {
                for (int j = 0; j < 3; ++j)
                    Rn[3 * i + j] = Rs[3 * i] * dR[j] + Rs[3 * i + 1] * dR[3 + j] + Rs[3 * i + 2] * dR[6 + j];
                tn[i] = Rs[3 * i] * dt[0] + Rs[3 * i + 1] * dt[1] + Rs[3 * i + 2] * dt[2] + tsh[i];
            }
            double thn[12], dthn[12];
            theta_of(Rn, tn, thn);
            for (int r = 0; r < 12; ++r) dthn[r] = thn[r] - th_E[r];
            const double qn = q_rel_warp(mo, dthn, lane);
            if (qn < q_cur) {
                for (int i = 0; i < 9; ++i) Rs[i] = Rn[i];
                for (int i = 0; i < 3; ++i) tsh[i] = tn[i];
                q_cur = qn;
                accepted = true;
                step_rot += nr;
                step_trans += nt;
                break;
            }
            mu = fmax(10.0 * mu, 1e-6 * tr);
        }
        __syncwarp();   // every lane is done with H and grad before the next iteration rewrites them
        if (converged || !accepted) break;
    }
    if (lane != 0) return;

    // σ² at the new pose: q(g_new) / (3 Σ P), floored; unchanged without mass.
    const int k = s.iter;
    nll_trace[k] = -sumlnp;
    double s2 = s.sigma2;
    const bool has_mass = sumP > 1e-12 * ntot;
    if (has_mass) {
        s2 = (sig2D + q_cur) / (3.0 * sumP);
        if (!(s2 >= rp.floor)) s2 = rp.floor;
    }
    const double s2_old = s.sigma2;
    IterState nx = s;
    double Rf[9], tf[3];
    for (int i = 0; i < 9; ++i) Rf[i] = Rs[i];
    for (int i = 0; i < 3; ++i) tf[i] = tsh[i];
    make_state(nx, Rf, tf, s2, rp.w, rp.V, rp.M, rp.omega_ref_target, rp.consistent, rp.eta, rp.spc);
    nx.extent = s.extent;
    nx.iter = k + 1;
    nx.no_mass = has_mass ? 0 : s.no_mass + 1;
    nx.status = s.status;
    nx.active = 1;
    nx.last_step_rot = step_rot;
    nx.last_step_trans = step_trans;
    if (nx.no_mass >= 3) {
        nx.status = LSGCPD_ENOMASS;
        nx.active = 0;
    }
    if (rp.tol > 0.0 && fabs(s2 - s2_old) <= rp.tol * s2_old && step_rot <= rp.tol && step_trans <= rp.tol * s.extent)
        nx.active = 0;
    if (nx.iter >= rp.max_iters) nx.active = 0;
    sigma2_trace[k + 1] = s2;
    *iters_done = k + 1;
    *st = nx;
}

__global__ void __launch_bounds__(32) newton_kernel(IterState* st, const double* __restrict__ mom, RegParams rp,
                                                    double* nll_trace, double* sigma2_trace, int* iters_done) {
    if (rp.group) newton_body<12>(st, mom, rp, nll_trace, sigma2_trace, iters_done);
    else newton_body<6>(st, mom, rp, nll_trace, sigma2_trace, iters_done);
}

// ---- EM tail: merge + moments (+ Newton) in one launch ---------------------------------------------------
// For N ≤ kTailMaxN the kernels after the E step collapse into one (Newton included without a communicator;
// with one, the moments are all-reduced and newton_kernel follows, so one rank with NCCL equals none): each CTA
// merges 32-point groups (merge_tile32, grid-stride) and folds them into the moments at once (no record
// round trip); warp w < 6 owns the 10 moments of G row w, warps 6-8 the 4 of U row w - 6, warp 9 σ²ΣD, ΣP,
// Σ ln p.  The last CTA to finish (atomic ticket, as block_reduce_store) sums the per-CTA moments in CTA
// order and (run_newton) runs the Newton step and σ² update with its first warp.  Deterministic for a fixed grid.
constexpr int kTailThreads = kMergePts * 16;
template <int K>
__device__ __forceinline__ void tail_newton(IterState* st, const double* mom, const RegParams& rp, double* nll,
                                            double* s2t, int* it) {
    newton_body<K>(st, mom, rp, nll, s2t, it);
}
__global__ void __launch_bounds__(kTailThreads)
    em_tail_kernel(const float* __restrict__ part, const float* __restrict__ src, int64_t N, IterState* st,
                   Sched sc, const float* __restrict__ phi, double* blockpart, double* mom, unsigned* counter,
                   RegParams rp, double* nll_trace, double* sigma2_trace, int* iters_done, int run_newton) {
    if (!st->active) return;
    __shared__ float tile[kMergePts][LSGCPD_REC + 1];
    __shared__ double a0s[kMergePts];
    __shared__ double msum[kMom];
    __shared__ bool last;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double R[9], t[3];
#pragma unroll
    for (int i = 0; i < 9; ++i) R[i] = st->R[i];
#pragma unroll
    for (int i = 0; i < 3; ++i) t[i] = st->t[i];
    const double s2 = st->sigma2;
    double acc[10];
#pragma unroll
    for (int j = 0; j < 10; ++j) acc[j] = 0.0;
    const int64_t ngroups = (N + kMergePts - 1) / kMergePts;
    for (int64_t g = blockIdx.x; g < ngroups; g += gridDim.x) {
        const int64_t n0 = g * kMergePts;
        merge_tile32(part, N, n0, st, sc, phi, tile, a0s);
        __syncthreads();
        const int64_t n = n0 + lane;
        if (w < 10 && n < N) {
            const float* r = tile[lane];
            const double P = r[0];
            const double x[4] = {(double)src[3 * n], (double)src[3 * n + 1], (double)src[3 * n + 2], 1.0};
            if (w < 6) {            // G_{ij,ab} += H_ij x̃_a x̃_b, ij = w
                const double H[6] = {P + (double)r[4], (double)r[5], (double)r[6], P + (double)r[7], (double)r[8],
                                     P + (double)r[9]};
                double h = H[0];
#pragma unroll
                for (int q = 1; q < 6; ++q) h = (w == q) ? H[q] : h;
                int k = 0;
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = a; b < 4; ++b) { acc[k] = fma(h, x[a] * x[b], acc[k]); ++k; }
            } else if (w < 9) {     // U_{ia} += u_i x̃_a, i = w - 6
                const double H[6] = {P + (double)r[4], (double)r[5], (double)r[6], P + (double)r[7], (double)r[8],
                                     P + (double)r[9]};
                const double gv[3] = {(double)r[1] + (double)r[10], (double)r[2] + (double)r[11],
                                      (double)r[3] + (double)r[12]};
                double xh[3];
#pragma unroll
                for (int i = 0; i < 3; ++i)
                    xh[i] = fma(R[3 * i], x[0], fma(R[3 * i + 1], x[1], fma(R[3 * i + 2], x[2], t[i])));
                double u[3];
#pragma unroll
                for (int i = 0; i < 3; ++i)
                    u[i] = H[s3(i, 0)] * xh[0] + H[s3(i, 1)] * xh[1] + H[s3(i, 2)] * xh[2] - gv[i];
                const double ui = w == 6 ? u[0] : (w == 7 ? u[1] : u[2]);
#pragma unroll
                for (int a = 0; a < 4; ++a) acc[a] = fma(ui, x[a], acc[a]);
            } else {                // σ²ΣD, ΣP, Σ ln p
                acc[0] = fma(s2, (double)r[13], acc[0]);
                acc[1] += P;
                acc[2] += (double)r[14];
            }
        }
        __syncthreads();            // the tile is rewritten by the next group
    }
    const int nacc = w < 6 ? 10 : (w < 9 ? 4 : (w == 9 ? 3 : 0));
    const int m0 = w < 6 ? 10 * w : (w < 9 ? 60 + 4 * (w - 6) : 72);
#pragma unroll
    for (int j = 0; j < 10; ++j) {
        const double v = warp_sum(acc[j]);
        if (lane == 0 && j < nacc) msum[m0 + j] = v;
    }
    __syncthreads();
    if (threadIdx.x < kMom) blockpart[(int64_t)blockIdx.x * kMom + threadIdx.x] = msum[threadIdx.x];
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = (atomicAdd(counter, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!last) return;
    __threadfence();
    if (threadIdx.x < kMom) mom[threadIdx.x] = ordered_reduce_l2<false>(blockpart + threadIdx.x, kMom, gridDim.x);
    if (threadIdx.x == 0) *counter = 0u;
    __syncthreads();
    if (run_newton && threadIdx.x < 32) {
        if (rp.group) tail_newton<12>(st, mom, rp, nll_trace, sigma2_trace, iters_done);
        else tail_newton<6>(st, mom, rp, nll_trace, sigma2_trace, iters_done);
    }
}

// ---- batched registrations (NEXT-3): one CTA / warp per problem -----------------------------------------
// Moments of problem b over its own points (one CTA, fixed order: deterministic), written to mom[b·kBatchMom].
__global__ void __launch_bounds__(kMomThreads)
    moments_batch_kernel(const BatchProblem* __restrict__ bp, const float* __restrict__ rec, IterState* st,
                         double* blockpart, double* mom, unsigned* counters) {
    const int b = blockIdx.x;
    const BatchProblem P = bp[b];
    moments_body(rec + P.pt0 * LSGCPD_REC, P.src, P.N, st + b, blockpart + (int64_t)b * kMom,
                 mom + (int64_t)b * kBatchMom, counters + b, 1);
}

__global__ void __launch_bounds__(32) newton_batch_kernel(const BatchProblem* __restrict__ bp, IterState* st,
                                                          const double* __restrict__ mom, RegParams rp0,
                                                          double* nll_trace, double* sigma2_trace, int* iters_done) {
    const int b = blockIdx.x;
    const BatchProblem P = bp[b];
    RegParams rp = rp0;
    rp.V = P.volume;
    rp.floor = rp0.floor * P.extent * P.extent;   // rp0.floor holds the relative floor
    rp.omega_ref_target = P.omega_ref;
    rp.spc = P.spc;
    rp.M = P.M;
    if (rp.group)
        newton_body<12>(st + b, mom + (int64_t)b * kBatchMom, rp, nll_trace + (int64_t)b * (rp.max_iters + 1),
                        sigma2_trace + (int64_t)b * (rp.max_iters + 2), iters_done + b);
    else
        newton_body<6>(st + b, mom + (int64_t)b * kBatchMom, rp, nll_trace + (int64_t)b * (rp.max_iters + 1),
                       sigma2_trace + (int64_t)b * (rp.max_iters + 2), iters_done + b);
}

// σ²₀ of problem b (CPD closed form) and its iteration-0 state, one CTA per problem.
__global__ void __launch_bounds__(kMomThreads)
    init_batch_kernel(const BatchProblem* __restrict__ bp, IterState* st, RegParams rp0, double sigma2_user,
                      double* mom, double* sigma2_trace) {
    const int b = blockIdx.x;
    const BatchProblem P = bp[b];
    __shared__ double red[kMomThreads / 32];
    const TargetHeader* hdr = reinterpret_cast<const TargetHeader*>(P.target);
    double acc = 0.0;
    for (int64_t n = threadIdx.x; n < P.N; n += blockDim.x) {
        const double x0 = P.src[3 * n], x1 = P.src[3 * n + 1], x2 = P.src[3 * n + 2];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            const double d = fma(P.R0[3 * i], x0, fma(P.R0[3 * i + 1], x1, fma(P.R0[3 * i + 2], x2, P.t0[i]))) -
                             hdr->ybar[i];
            acc = fma(d, d, acc);
        }
    }
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x != 0) return;
    double sx = 0.0;
    for (int w = 0; w < kMomThreads / 32; ++w) sx += red[w];
    const double M = (double)P.M, N = (double)P.N;
    double s2 = sigma2_user > 0.0 ? sigma2_user : (M * sx + N * hdr->syy) / (3.0 * M * N);
    const double floor = rp0.floor * P.extent * P.extent;
    if (s2 < floor) s2 = floor;
    IterState s;
    make_state(s, P.R0, P.t0, s2, rp0.w, P.volume, P.M, P.omega_ref, rp0.consistent, rp0.eta, P.spc);
    s.extent = P.extent;
    s.active = rp0.max_iters > 0 ? 1 : 0;
    s.iter = 0;
    s.status = 0;
    s.no_mass = 0;
    s.last_step_rot = s.last_step_trans = 0.0;
    if (!isfinite(sx)) {   // a non-finite source coordinate: this problem is refused (EINVAL in status_out)
        s.status = LSGCPD_EINVAL;
        s.active = 0;
    }
    st[b] = s;
    mom[(int64_t)b * kBatchMom + 75] = N;
    sigma2_trace[(int64_t)b * (rp0.max_iters + 2)] = s2;
}

void moments_batch_launch(const BatchProblem* bp, int B, const float* rec, IterState* st, double* blockpart,
                          double* mom, unsigned* counters, cudaStream_t stream) {
    moments_batch_kernel<<<B, kMomThreads, 0, stream>>>(bp, rec, st, blockpart, mom, counters);
}
void newton_batch_launch(const BatchProblem* bp, int B, IterState* st, const double* mom, const RegParams& rp0,
                         double* nll_trace, double* sigma2_trace, int* iters_done, cudaStream_t stream) {
    newton_batch_kernel<<<B, 32, 0, stream>>>(bp, st, mom, rp0, nll_trace, sigma2_trace, iters_done);
}
void init_batch_launch(const BatchProblem* bp, int B, IterState* st, const RegParams& rp0, double sigma2_user,
                       double* mom, double* sigma2_trace, cudaStream_t stream) {
    init_batch_kernel<<<B, kMomThreads, 0, stream>>>(bp, st, rp0, sigma2_user, mom, sigma2_trace);
}

// ---- host launchers ----------------------------------------------------------------------------
// Grid: a function of N only (deterministic reduction order for a given problem), ≤ 256 blocks,
// ≥ 8 points per thread, so small problems do not pay for a 256-way cross-block sum.
static unsigned moment_blocks(int64_t N) {
    const int64_t b = (N + kMomThreads * 8 - 1) / (kMomThreads * 8);
    return (unsigned)(b < 1 ? 1 : (b > kMomBlocks ? kMomBlocks : b));
}
void moments_launch(const float* rec, const float* src, int64_t N, const IterState* st, double* blockpart,
                    double* out, unsigned int* counter, cudaStream_t stream) {
    moments_kernel<<<moment_blocks(N), kMomThreads, 0, stream>>>(rec, src, N, st, blockpart, out, counter);
}
void sigma2_sums_launch(const float* src, int64_t N, const IterState* st, const void* d_target, double* blockpart,
                        double* out, unsigned int* counter, cudaStream_t stream) {
    sigma2_sums_kernel<<<moment_blocks(N), kMomThreads, 0, stream>>>(src, N, st,
                                                               reinterpret_cast<const TargetHeader*>(d_target),
                                                               blockpart, out, counter);
}
void sigma2_init_launch(IterState* st, const void* d_target, const double* sums, const RegParams& rp,
                        double sigma2_user, double* sigma2_trace, double* ntot_out, cudaStream_t stream) {
    sigma2_init_kernel<<<1, 1, 0, stream>>>(st, reinterpret_cast<const TargetHeader*>(d_target), sums, rp,
                                             sigma2_user, sigma2_trace, ntot_out);
}
void em_tail_launch(const float* part, const float* src, int64_t N, IterState* st, const Sched& sc, const float* phi,
                    double* blockpart, double* mom, unsigned* counter, const RegParams& rp, double* nll_trace,
                    double* sigma2_trace, int* iters_done, int run_newton, cudaStream_t stream) {
    const int nsm = sm_count() > 0 ? sm_count() : 1;   // per device (estep.cu)
    const int64_t ng = (N + kMergePts - 1) / kMergePts;
    const int64_t cap = nsm < kMomentBlocks ? nsm : kMomentBlocks;   // blockpart holds kMomentBlocks rows
    em_tail_kernel<<<(unsigned)(ng < cap ? ng : cap), kTailThreads, 0, stream>>>(
        part, src, N, st, sc, phi, blockpart, mom, counter, rp, nll_trace, sigma2_trace, iters_done, run_newton);
}
void newton_launch(IterState* st, const double* mom, const RegParams& rp, double* nll_trace, double* sigma2_trace,
                   int* iters_done, cudaStream_t stream) {
    newton_kernel<<<1, 32, 0, stream>>>(st, mom, rp, nll_trace, sigma2_trace, iters_done);
}

}  // namespace lsg
