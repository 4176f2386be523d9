/*
 * register_c.c — the C ABI used from plain C (no Python, no torch): prepare a target, register a rotated
 * and shifted copy of it, print the recovered pose.  Device memory comes from the CUDA runtime.
 *
 *   gcc -O2 -I include -I /usr/local/cuda/include examples/register_c.c \
 *       -L paper_2103_15039_b200 -llsgcpd -L /usr/local/cuda/lib64 -lcudart -lm \
 *       -Wl,-rpath,$PWD/paper_2103_15039_b200 -o register_c && ./register_c
 *
 * Input (deterministic, no RNG library): 4,096 points on the floor z = 0 and two walls x = 0, y = 0 of a
 * 2 m room corner, on a sheared lattice; the source is the same points moved by g_gt = (Rz(20°)·Rx(10°),
 * t = (0.05, -0.03, 0.02)).  Noiseless, so EM must return g_gt⁻¹ (the north star's exact-recovery case).
 * Exit status 0 when the recovered rotation is within 1e-5 rad of g_gt⁻¹.
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "lsgcpd.h"

#define CK(x)                                                                          \
    do {                                                                               \
        int rc_ = (x);                                                                 \
        if (rc_ != 0) {                                                                \
            fprintf(stderr, "%s failed: %d (%s)\n", #x, rc_, lsgcpd_last_error());     \
            return 1;                                                                  \
        }                                                                              \
    } while (0)
#define CU(x)                                                                          \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess) {                                                       \
            fprintf(stderr, "%s failed: %s\n", #x, cudaGetErrorString(e_));            \
            return 1;                                                                  \
        }                                                                              \
    } while (0)

static void rot_zx(double az, double ax, double R[9]) {
    const double cz = cos(az), sz = sin(az), cx = cos(ax), sx = sin(ax);
    /* Rz · Rx */
    const double Rz[9] = {cz, -sz, 0, sz, cz, 0, 0, 0, 1};
    const double Rx[9] = {1, 0, 0, 0, cx, -sx, 0, sx, cx};
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double s = 0;
            for (int k = 0; k < 3; ++k) s += Rz[3 * i + k] * Rx[3 * k + j];
            R[3 * i + j] = s;
        }
}

int main(void) {
    const int64_t M = 4096;
    float* Y = (float*)malloc(sizeof(float) * 3 * M);
    float* X = (float*)malloc(sizeof(float) * 3 * M);
    for (int64_t m = 0; m < M; ++m) {   /* three planes, 1365-1366 points each, sheared lattice */
        const int face = (int)(m % 3);
        const int64_t q = m / 3;
        const double u = 2.0 * (double)(q % 37) / 37.0 + 0.013 * (double)(q / 37 % 7);
        const double v = 2.0 * (double)(q / 37) / 37.0;
        const double p[3][3] = {{u, v, 0.0}, {0.0, u, v}, {u, 0.0, v}};
        for (int a = 0; a < 3; ++a) Y[3 * m + a] = (float)p[face][a];
    }
    double Rg[9], tg[3] = {0.05, -0.03, 0.02};
    rot_zx(20.0 * M_PI / 180.0, 10.0 * M_PI / 180.0, Rg);
    for (int64_t m = 0; m < M; ++m)
        for (int i = 0; i < 3; ++i)
            X[3 * m + i] = (float)(Rg[3 * i] * Y[3 * m] + Rg[3 * i + 1] * Y[3 * m + 1] +
                                   Rg[3 * i + 2] * Y[3 * m + 2] + tg[i]);

    void *d_y, *d_x, *d_target, *d_ws;
    const size_t tb = lsgcpd_target_bytes(M);
    const size_t pw = lsgcpd_prepare_workspace_bytes(M, 10);
    const int iters = 60;
    const size_t rw = lsgcpd_register_workspace_bytes(M, M, iters);
    const size_t wsb = pw > rw ? pw : rw;
    CU(cudaMalloc(&d_y, sizeof(float) * 3 * M));
    CU(cudaMalloc(&d_x, sizeof(float) * 3 * M));
    CU(cudaMalloc(&d_target, tb));
    CU(cudaMalloc(&d_ws, wsb));
    CU(cudaMemcpy(d_y, Y, sizeof(float) * 3 * M, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(d_x, X, sizeof(float) * 3 * M, cudaMemcpyHostToDevice));

    lsgcpd_target_info info;
    CK(lsgcpd_prepare_target((const float*)d_y, M, NULL, d_target, d_ws, wsb, &info, NULL, NULL));

    lsgcpd_em_params ep;
    lsgcpd_em_params_default(&ep);
    ep.w = 0.1;
    ep.max_iters = iters;
    double R[9], t[3], s2;
    int it = 0;
    CK(lsgcpd_register(d_target, M, 0.0, (const float*)d_x, M, &ep, NULL, NULL, R, t, &s2, &it, NULL, NULL, NULL,
                       d_ws, wsb, NULL));

    /* expected: g_gt⁻¹ = (Rgᵀ, -Rgᵀ tg); rotation angle of Rᵀ·Rgᵀ... compare R with Rgᵀ */
    double tr = 0.0;   /* trace(R_expectedᵀ R) = trace(Rg R) */
    for (int i = 0; i < 3; ++i)
        for (int k = 0; k < 3; ++k) tr += Rg[3 * i + k] * R[3 * k + i];
    double c = 0.5 * (tr - 1.0);
    c = c > 1.0 ? 1.0 : (c < -1.0 ? -1.0 : c);
    const double ang = acos(c);
    double te[3], dt = 0.0;
    for (int i = 0; i < 3; ++i) {
        te[i] = -(Rg[i] * tg[0] + Rg[3 + i] * tg[1] + Rg[6 + i] * tg[2]);
        dt += (t[i] - te[i]) * (t[i] - te[i]);
    }
    printf("lsgcpd %d: M=N=%lld V=%.4f iters=%d sigma2=%.3e  rotation error %.2e rad, |dt| %.2e\n",
           lsgcpd_version(), (long long)M, info.volume, it, s2, ang, sqrt(dt));
    cudaFree(d_y);
    cudaFree(d_x);
    cudaFree(d_target);
    cudaFree(d_ws);
    free(Y);
    free(X);
    return (it == iters && ang < 1e-5 && sqrt(dt) < 1e-5 * info.extent) ? 0 : 2;
}
