// Per-(gaussian, view) splat -> parameter chain in fp32 (ref: jacobian.py:159-266)
// and the per-pair forward chain kernel (m = dy/dx p, ref: jacobian.py:434-443).
#pragma once
#include "slm_common.cuh"

// minimum resident blocks per SM of the per-pair chain kernels (register cap)
#ifndef SLM_PM_MINB
#define SLM_PM_MINB 4
#endif
#ifndef SLM_PMD_MINB
#define SLM_PMD_MINB 8   // the dSigma forward chain (PCG path): 64 registers (0.637 -> 0.601 ms at C3)
#endif
#ifndef SLM_BW_MINB
#define SLM_BW_MINB 6
#endif
#ifndef SLM_BW1_MINB
#define SLM_BW1_MINB 4   // the diag backward (moments + chain per pair): 2.91 -> 2.83 ms at C3 with 4
#endif

// arithmetic type of the per-pair chain (outputs are stored as float)
#ifndef SLM_CHAIN_T
#define SLM_CHAIN_T float
#endif

template <int K>
struct Tab {
  float dmu[2][3];
  float dcov[3][10];
  float dcol[3][3];
  float Y[K];
  float dopa;
  float mask[3];
};

// Gaussian-only part of the chain (independent of the view): rotation Rg of
// the normalised quaternion, s^2 = exp(2 log s), the projected rotation
// derivatives Mq_l = (dR/dq_hat_l - q_hat_l sum_k q_hat_k dR/dq_hat_k) / |q|
// (the (I - q_hat q_hat^T) / |q| normalisation chain) and sigma'(logit).
// Precomputed once per cache (k_gauss_tab) together with the position and the
// SH coefficients, so the per-(gaussian, view) chain reads one contiguous,
// 16-byte aligned row per gaussian (gtab_floats(K) floats):
//   [Rg 9 | s2 3 | Mq 36 | dopa | pos 3 | Sigma_world 6 (xx xy xz yy yz zz), pad 2 |
//    SH coefficients 3K (channel-major), pad]
#define GT_DOPA 48
#define GT_POS 49
#define GT_SIG 52
#define GT_SH 60
__host__ __device__ constexpr int gtab_floats(int K) { return GT_SH + ((3 * K + 3) & ~3); }
template <typename Rt>
__device__ __forceinline__ void gauss_static(const float* __restrict__ xs, long long G, long long g, Rt (&Rg)[9],
                                             Rt (&s2)[3], Rt (&Mq)[4][9], Rt& dopa) {
  const Rt q0 = xs[3 * G + g], q1 = xs[4 * G + g], q2 = xs[5 * G + g], q3 = xs[6 * G + g];
  const Rt qn = sqrt(q0 * q0 + q1 * q1 + q2 * q2 + q3 * q3);
  const Rt iq = Rt(1) / qn;
  const Rt w = q0 * iq, a = q1 * iq, b = q2 * iq, c = q3 * iq;
  const Rt R0[9] = {Rt(1) - Rt(2) * (b * b + c * c), Rt(2) * (a * b - w * c), Rt(2) * (a * c + w * b),
                    Rt(2) * (a * b + w * c), Rt(1) - Rt(2) * (a * a + c * c), Rt(2) * (b * c - w * a),
                    Rt(2) * (a * c - w * b), Rt(2) * (b * c + w * a), Rt(1) - Rt(2) * (a * a + b * b)};
#pragma unroll
  for (int i = 0; i < 9; ++i) Rg[i] = R0[i];
  s2[0] = exp(Rt(2) * (Rt)xs[7 * G + g]);
  s2[1] = exp(Rt(2) * (Rt)xs[8 * G + g]);
  s2[2] = exp(Rt(2) * (Rt)xs[9 * G + g]);
  // dR/dq_hat_k (3x3 each), row-major
  const Rt dRh[4][9] = {
      {Rt(0), -Rt(2) * c, Rt(2) * b, Rt(2) * c, Rt(0), -Rt(2) * a, -Rt(2) * b, Rt(2) * a, Rt(0)},
      {Rt(0), Rt(2) * b, Rt(2) * c, Rt(2) * b, -Rt(4) * a, -Rt(2) * w, Rt(2) * c, Rt(2) * w, -Rt(4) * a},
      {-Rt(4) * b, Rt(2) * a, Rt(2) * w, Rt(2) * a, Rt(0), Rt(2) * c, -Rt(2) * w, Rt(2) * c, -Rt(4) * b},
      {-Rt(4) * c, -Rt(2) * w, Rt(2) * a, Rt(2) * w, -Rt(4) * c, Rt(2) * b, Rt(2) * a, Rt(2) * b, Rt(0)}};
  const Rt qh[4] = {w, a, b, c};
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    const Rt S = qh[0] * dRh[0][i] + qh[1] * dRh[1][i] + qh[2] * dRh[2][i] + qh[3] * dRh[3][i];
#pragma unroll
    for (int l = 0; l < 4; ++l) Mq[l][i] = (dRh[l][i] - qh[l] * S) * iq;
  }
  const Rt o = Rt(1) / (Rt(1) + exp(-(Rt)xs[10 * G + g]));
  dopa = o * (Rt(1) - o);
}

template <int K>
static __global__ void __launch_bounds__(256) k_gauss_tab(const float* __restrict__ xs, long long G,
                                                          float* __restrict__ gtab) {
  constexpr int GT = gtab_floats(K);
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < G; g += (long long)gridDim.x * blockDim.x) {
    float Rg[9], s2[3], Mq[4][9], dopa;
    gauss_static<float>(xs, G, g, Rg, s2, Mq, dopa);
    float o[GT];
#pragma unroll
    for (int i = 0; i < 9; ++i) o[i] = Rg[i];
#pragma unroll
    for (int i = 0; i < 3; ++i) o[9 + i] = s2[i];
#pragma unroll
    for (int l = 0; l < 4; ++l)
#pragma unroll
      for (int i = 0; i < 9; ++i) o[12 + l * 9 + i] = Mq[l][i];
    o[GT_DOPA] = dopa;
#pragma unroll
    for (int i = 0; i < 3; ++i) o[GT_POS + i] = xs[i * G + g];
    // world covariance Sigma = Rg diag(s2) Rg^T (upper triangle)
    {
      int k = 0;
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = i; j < 3; ++j, ++k)
          o[GT_SIG + k] = Rg[i * 3] * s2[0] * Rg[j * 3] + Rg[i * 3 + 1] * s2[1] * Rg[j * 3 + 1] +
                          Rg[i * 3 + 2] * s2[2] * Rg[j * 3 + 2];
      o[GT_SIG + 6] = o[GT_SIG + 7] = 0.f;
    }
#pragma unroll
    for (int i = GT_SH; i < GT; ++i) o[i] = i - GT_SH < 3 * K ? xs[(long long)(11 + i - GT_SH) * G + g] : 0.f;
    float4* dst = reinterpret_cast<float4*>(gtab + (size_t)g * GT);
#pragma unroll
    for (int k = 0; k < GT / 4; ++k) dst[k] = make_float4(o[4 * k], o[4 * k + 1], o[4 * k + 2], o[4 * k + 3]);
  }
}

// 16-byte read-only load that the compiler keeps in program order relative to
// the other ordered loads: the chain kernels load each part of the gaussian's
// row right before its use, which bounds the live registers (and so keeps
// occupancy up in these latency-bound kernels)
__device__ __forceinline__ float4 ldg4_ordered(const float4* p) {
  float4 v;
  asm volatile("ld.global.nc.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}
// L1 prefetch of a row part that is loaded (ordered) later: the latency
// overlaps the work before its use without holding registers
__device__ __forceinline__ void prefetch_l1(const void* p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }

template <int N>
__device__ __forceinline__ void ldg_row(const float* __restrict__ src, float* dst) {
#pragma unroll
  for (int k = 0; k < N / 4; ++k) {
    const float4 v = ldg4_ordered(reinterpret_cast<const float4*>(src) + k);
    dst[4 * k] = v.x;
    dst[4 * k + 1] = v.y;
    dst[4 * k + 2] = v.z;
    dst[4 * k + 3] = v.w;
  }
}

template <int K, typename Rt = SLM_CHAIN_T>
__device__ __forceinline__ void pair_tab(const float* __restrict__ xs, long long G, long long g, const SlmCamera& cam,
                                         uint32_t clampbits, Tab<K>& T, const float* __restrict__ gtab) {
  constexpr int GT = gtab_floats(K);
  const float* grow = gtab + (size_t)g * GT;
  float t[GT];
  ldg_row<12>(grow, t);                 // Rg, s2
  ldg_row<4>(grow + GT_DOPA, t + GT_DOPA);  // dopa, position
  Rt Rg[9], s2[3], Mq[4][9];
#pragma unroll
  for (int i = 0; i < 9; ++i) Rg[i] = t[i];
#pragma unroll
  for (int i = 0; i < 3; ++i) s2[i] = t[9 + i];
  const Rt dopa = t[GT_DOPA];
  const Rt p0 = t[GT_POS], p1 = t[GT_POS + 1], p2 = t[GT_POS + 2];
  Rt R[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) R[i] = (Rt)cam.R[i];
  const Rt fx = (Rt)cam.fx, fy = (Rt)cam.fy;
  const Rt X = R[0] * p0 + R[1] * p1 + R[2] * p2 + (Rt)cam.t[0];
  const Rt Yc = R[3] * p0 + R[4] * p1 + R[5] * p2 + (Rt)cam.t[1];
  const Rt Z = R[6] * p0 + R[7] * p1 + R[8] * p2 + (Rt)cam.t[2];
  const Rt iz = Rt(1) / Z, iz2 = iz * iz;
  const Rt A00 = fx * iz, A02 = -fx * X * iz2, A11 = fy * iz, A12 = -fy * Yc * iz2;
  Rt U[2][3];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    U[0][j] = A00 * R[j] + A02 * R[6 + j];
    U[1][j] = A11 * R[3 + j] + A12 * R[6 + j];
    T.dmu[0][j] = U[0][j];
    T.dmu[1][j] = U[1][j];
  }
  // M = R Rg (camera-frame axes), Sc = M diag(s2) M^T
  Rt Mm[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) Mm[i * 3 + j] = R[i * 3] * Rg[j] + R[i * 3 + 1] * Rg[3 + j] + R[i * 3 + 2] * Rg[6 + j];
  Rt Sc[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int k = 0; k < 3; ++k)
      Sc[i * 3 + k] = Mm[i * 3] * s2[0] * Mm[k * 3] + Mm[i * 3 + 1] * s2[1] * Mm[k * 3 + 1] +
                      Mm[i * 3 + 2] * s2[2] * Mm[k * 3 + 2];
  // P = Sc A^T (3x2)
  Rt P[3][2];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    P[i][0] = Sc[i * 3] * A00 + Sc[i * 3 + 2] * A02;
    P[i][1] = Sc[i * 3 + 1] * A11 + Sc[i * 3 + 2] * A12;
  }
  const Rt cxx = -fx * iz2, cyy = -fy * iz2;
  const Rt kx = Rt(2) * fx * X * iz2 * iz, ky = Rt(2) * fy * Yc * iz2 * iz;
  Rt dX[3][3];
  dX[0][0] = Rt(2) * cxx * P[2][0]; dX[0][1] = cxx * P[2][1]; dX[0][2] = Rt(0);
  dX[1][0] = Rt(0); dX[1][1] = cyy * P[2][0]; dX[1][2] = Rt(2) * cyy * P[2][1];
  const Rt r00 = cxx * P[0][0] + kx * P[2][0], r01 = cxx * P[0][1] + kx * P[2][1];
  const Rt r10 = cyy * P[1][0] + ky * P[2][0], r11 = cyy * P[1][1] + ky * P[2][1];
  dX[2][0] = Rt(2) * r00; dX[2][1] = r01 + r10; dX[2][2] = Rt(2) * r11;
#pragma unroll
  for (int p = 0; p < 3; ++p)
#pragma unroll
    for (int j = 0; j < 3; ++j) T.dcov[p][j] = dX[0][p] * R[j] + dX[1][p] * R[3 + j] + dX[2][p] * R[6 + j];
  // quaternion: dcov_l = V_l W^T + W V_l^T, V_l = U Mq_l, W = U Rg diag(s2)
  Rt UR[2][3], Wm[2][3];
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      UR[r][j] = U[r][0] * Rg[j] + U[r][1] * Rg[3 + j] + U[r][2] * Rg[6 + j];
      Wm[r][j] = UR[r][j] * s2[j];
    }
  ldg_row<36>(grow + 12, t + 12);        // Mq
#pragma unroll
  for (int l = 0; l < 4; ++l)
#pragma unroll
    for (int i = 0; i < 9; ++i) Mq[l][i] = t[12 + l * 9 + i];
#pragma unroll
  for (int l = 0; l < 4; ++l) {
    Rt V[2][3];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int j = 0; j < 3; ++j) V[r][j] = U[r][0] * Mq[l][j] + U[r][1] * Mq[l][3 + j] + U[r][2] * Mq[l][6 + j];
    const Rt v0w0 = V[0][0] * Wm[0][0] + V[0][1] * Wm[0][1] + V[0][2] * Wm[0][2];
    const Rt v0w1 = V[0][0] * Wm[1][0] + V[0][1] * Wm[1][1] + V[0][2] * Wm[1][2];
    const Rt v1w0 = V[1][0] * Wm[0][0] + V[1][1] * Wm[0][1] + V[1][2] * Wm[0][2];
    const Rt v1w1 = V[1][0] * Wm[1][0] + V[1][1] * Wm[1][1] + V[1][2] * Wm[1][2];
    T.dcov[0][3 + l] = Rt(2) * v0w0;
    T.dcov[1][3 + l] = v0w1 + v1w0;
    T.dcov[2][3 + l] = Rt(2) * v1w1;
  }
  // log-scale: 2 s_i^2 (U r_i)(U r_i)^T
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    T.dcov[0][7 + i] = Rt(2) * s2[i] * UR[0][i] * UR[0][i];
    T.dcov[1][7 + i] = Rt(2) * s2[i] * UR[0][i] * UR[1][i];
    T.dcov[2][7 + i] = Rt(2) * s2[i] * UR[1][i] * UR[1][i];
  }
  // colour
  ldg_row<GT - GT_SH>(grow + GT_SH, t + GT_SH);  // SH coefficients
  const Rt v0 = p0 - (Rt)cam.C[0], v1 = p1 - (Rt)cam.C[1], v2 = p2 - (Rt)cam.C[2];
  const Rt vn = sqrt(v0 * v0 + v1 * v1 + v2 * v2), ivn = Rt(1) / vn;
  const Rt d0 = v0 * ivn, d1 = v1 * ivn, d2 = v2 * ivn;
  Rt Yr[K];
  sh_basis<Rt, K>(d0, d1, d2, Yr);
#pragma unroll
  for (int k = 0; k < K; ++k) T.Y[k] = (float)Yr[k];
  Rt dcdd[3][3];
  auto coef = [&](int ch, int k) { return (Rt)t[GT_SH + ch * K + k]; };
  sh_grad_dot<Rt, K>(d0, d1, d2, coef, dcdd);
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    T.mask[ch] = (clampbits >> ch) & 1u ? Rt(0) : Rt(1);
    const Rt dd = dcdd[ch][0] * d0 + dcdd[ch][1] * d1 + dcdd[ch][2] * d2;
    T.dcol[ch][0] = T.mask[ch] * (dcdd[ch][0] - d0 * dd) * ivn;
    T.dcol[ch][1] = T.mask[ch] * (dcdd[ch][1] - d1 * dd) * ivn;
    T.dcol[ch][2] = T.mask[ch] * (dcdd[ch][2] - d2 * dd) * ivn;
  }
  T.dopa = dopa;
}

// fp32 camera row of the per-pair chains (slm_cameras_f32): R 9 | t 3 | C 3 |
// fx | fy | pad 3 = five 16-byte loads instead of 17 fp64 loads + conversions
#define CAMF_FLOATS 20
struct CamF {
  float R[9], t[3], C[3], fx, fy;
};
__device__ __forceinline__ CamF load_camf(const float* __restrict__ camf, int v) {
  float c[CAMF_FLOATS];
  ldg_row<CAMF_FLOATS>(camf + (size_t)v * CAMF_FLOATS, c);
  CamF k;
#pragma unroll
  for (int i = 0; i < 9; ++i) k.R[i] = c[i];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    k.t[i] = c[9 + i];
    k.C[i] = c[12 + i];
  }
  k.fx = c[15];
  k.fy = c[16];
  return k;
}

// Backward row of one (gaussian, view) pair for the J^T chain (ref:
// jacobian.py:314-353) from its 9 run-partial sums a = (a_mu (2), a_cov (3,
// 1/2-scaled on 0 and 2), a_opa, a_col (3)), in the world-covariance form:
//   row[0..2]  position: U^T a_mu + dcov_pos^T a_cov + (I - d d^T)/|v| grad_d
//              (sum_k ct_k Y_k), ct_k = sum_ch mask_ch a_col,ch coef(ch, k)
//   row[3..8]  B = U^T Abar U (Abar = [[a_c0, a_c1/2], [a_c1/2, a_c2]]): the
//              gradient w.r.t. the world covariance, upper triangle; summed
//              over the gaussian's pairs and turned into the quaternion /
//              log-scale gradients once per gaussian (k_gm_to_am)
//   row[9]     opacity sigma' a_opa;  row[10 + ch K + k] SH a_col,ch mask_ch Y_k
// (P - 1 values).  The camera-frame covariance comes from the chain row's
// Sigma_world, so the per-pair work has no rotation / scale chain.
template <int K>
__device__ __forceinline__ void pair_back_row(long long g, const CamF& cam, uint32_t clampbits,
                                              const float (&a)[9], const float* __restrict__ gtab, float* row) {
  constexpr int GT = gtab_floats(K);
  const float* grow = gtab + (size_t)g * GT;
  prefetch_l1(grow + GT_SH);  // SH coefficients (used last)
  prefetch_l1(grow + GT_SH + 32);
  float t[16];
  ldg_row<4>(grow + GT_DOPA, t);       // dopa, position
  ldg_row<8>(grow + GT_SIG, t + 4);    // Sigma_world
  const float dopa = t[0], p0 = t[1], p1 = t[2], p2 = t[3];
  const float Sw[9] = {t[4], t[5], t[6], t[5], t[7], t[8], t[6], t[8], t[9]};
  float R[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) R[i] = cam.R[i];
  const float fx = cam.fx, fy = cam.fy;
  const float X = R[0] * p0 + R[1] * p1 + R[2] * p2 + cam.t[0];
  const float Yc = R[3] * p0 + R[4] * p1 + R[5] * p2 + cam.t[1];
  const float Z = R[6] * p0 + R[7] * p1 + R[8] * p2 + cam.t[2];
  const float iz = 1.f / Z, iz2 = iz * iz;
  const float A00 = fx * iz, A02 = -fx * X * iz2, A11 = fy * iz, A12 = -fy * Yc * iz2;
  float U[2][3];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    U[0][j] = A00 * R[j] + A02 * R[6 + j];
    U[1][j] = A11 * R[3 + j] + A12 * R[6 + j];
  }
  // camera-frame covariance Sc = R Sigma R^T, P = Sc A^T
  float RS[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) RS[i * 3 + j] = R[i * 3] * Sw[j] + R[i * 3 + 1] * Sw[3 + j] + R[i * 3 + 2] * Sw[6 + j];
  float Sc[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int k = 0; k < 3; ++k) Sc[i * 3 + k] = RS[i * 3] * R[k * 3] + RS[i * 3 + 1] * R[k * 3 + 1] + RS[i * 3 + 2] * R[k * 3 + 2];
  float P[3][2];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    P[i][0] = Sc[i * 3] * A00 + Sc[i * 3 + 2] * A02;
    P[i][1] = Sc[i * 3 + 1] * A11 + Sc[i * 3 + 2] * A12;
  }
  const float cxx = -fx * iz2, cyy = -fy * iz2;
  const float kx = 2.f * fx * X * iz2 * iz, ky = 2.f * fy * Yc * iz2 * iz;
  float dX[3][3];
  dX[0][0] = 2.f * cxx * P[2][0]; dX[0][1] = cxx * P[2][1]; dX[0][2] = 0.f;
  dX[1][0] = 0.f; dX[1][1] = cyy * P[2][0]; dX[1][2] = 2.f * cyy * P[2][1];
  const float r00 = cxx * P[0][0] + kx * P[2][0], r01 = cxx * P[0][1] + kx * P[2][1];
  const float r10 = cyy * P[1][0] + ky * P[2][0], r11 = cyy * P[1][1] + ky * P[2][1];
  dX[2][0] = 2.f * r00; dX[2][1] = r01 + r10; dX[2][2] = 2.f * r11;
  // a_cov through the camera-frame position: g_cam[r] = sum_p dX[r][p] a_cov[p]
  float gc[3];
#pragma unroll
  for (int r = 0; r < 3; ++r) gc[r] = dX[r][0] * a[2] + dX[r][1] * a[3] + dX[r][2] * a[4];
  float pos[3];
#pragma unroll
  for (int j = 0; j < 3; ++j)
    pos[j] = U[0][j] * a[0] + U[1][j] * a[1] + gc[0] * R[j] + gc[1] * R[3 + j] + gc[2] * R[6 + j];
  // B = U^T Abar U
  const float h = 0.5f * a[3];
  float AU[2][3];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    AU[0][j] = a[2] * U[0][j] + h * U[1][j];
    AU[1][j] = h * U[0][j] + a[4] * U[1][j];
  }
  {
    int k = 3;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = i; j < 3; ++j, ++k) row[k] = U[0][i] * AU[0][j] + U[1][i] * AU[1][j];
  }
  row[9] = dopa * a[5];
  // colour: SH block and the view-direction (position) term
  float sh[3 * K];
  ldg_row<GT - GT_SH>(grow + GT_SH, sh);
  const float v0 = p0 - cam.C[0], v1 = p1 - cam.C[1], v2 = p2 - cam.C[2];
  const float ivn = 1.f / sqrtf(v0 * v0 + v1 * v1 + v2 * v2);
  const float d0 = v0 * ivn, d1 = v1 * ivn, d2 = v2 * ivn;
  float Y[K];
  sh_basis<float, K>(d0, d1, d2, Y);
  float w[3];
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    w[ch] = (clampbits >> ch) & 1u ? 0.f : a[6 + ch];
#pragma unroll
    for (int k = 0; k < K; ++k) row[10 + ch * K + k] = w[ch] * Y[k];
  }
  float gd[1][3];
  auto ct = [&](int, int k) { return w[0] * sh[k] + w[1] * sh[K + k] + w[2] * sh[2 * K + k]; };
  sh_grad_dot1<K>(d0, d1, d2, ct, gd[0]);
  const float dd = gd[0][0] * d0 + gd[0][1] * d1 + gd[0][2] * d2;
  row[0] = pos[0] + (gd[0][0] - d0 * dd) * ivn;
  row[1] = pos[1] + (gd[0][1] - d1 * dd) * ivn;
  row[2] = pos[2] + (gd[0][2] - d2 * dd) * ivn;
}

// Forward chain m = dy/dx p of one pair from the padded gaussian-major p row
// that carries dSigma (k_pcg_p with the chain rows): the camera-dependent
// part only -- m_mu = U p_pos, m_cov = dcov_pos p_pos + U dSigma U^T, m_col =
// mask (sum_k coef_k dY_k(dd) + p_sh,k Y_k) with dd = (I - d d^T) p_pos / |v|
// the view-direction perturbation (ref: jacobian.py:434-443).
template <int K>
__device__ __forceinline__ void pair_fwd_dsig(long long g, const CamF& cam, uint32_t clampbits,
                                              const float* __restrict__ gtab, const float* __restrict__ prow,
                                              float4* __restrict__ out) {
  constexpr int GT = gtab_floats(K), P = 11 + 3 * K, DS = (P + 3) & ~3;
  const float* grow = gtab + (size_t)g * GT;
  prefetch_l1(grow + GT_SH);  // SH coefficients (used last)
  prefetch_l1(grow + GT_SH + 32);
  prefetch_l1(prow + 8);
  float t[12];
  ldg_row<4>(grow + GT_DOPA, t);       // dopa, position
  ldg_row<8>(grow + GT_SIG, t + 4);    // Sigma_world
  float pp[12];
  ldg_row<12>(prow, pp);               // p_pos 3, p_q 4, p_s 3, p_opa, p_sh[0]
  float ds[8];
  ldg_row<8>(prow + DS, ds);           // dSigma
  const float dopa = t[0], p0 = t[1], p1 = t[2], p2 = t[3];
  const float Sw[9] = {t[4], t[5], t[6], t[5], t[7], t[8], t[6], t[8], t[9]};
  float R[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) R[i] = cam.R[i];
  const float fx = cam.fx, fy = cam.fy;
  const float X = R[0] * p0 + R[1] * p1 + R[2] * p2 + cam.t[0];
  const float Yc = R[3] * p0 + R[4] * p1 + R[5] * p2 + cam.t[1];
  const float Z = R[6] * p0 + R[7] * p1 + R[8] * p2 + cam.t[2];
  const float iz = 1.f / Z, iz2 = iz * iz;
  const float A00 = fx * iz, A02 = -fx * X * iz2, A11 = fy * iz, A12 = -fy * Yc * iz2;
  float U[2][3];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    U[0][j] = A00 * R[j] + A02 * R[6 + j];
    U[1][j] = A11 * R[3 + j] + A12 * R[6 + j];
  }
  float RS[9], Sc[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) RS[i * 3 + j] = R[i * 3] * Sw[j] + R[i * 3 + 1] * Sw[3 + j] + R[i * 3 + 2] * Sw[6 + j];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int k = 0; k < 3; ++k) Sc[i * 3 + k] = RS[i * 3] * R[k * 3] + RS[i * 3 + 1] * R[k * 3 + 1] + RS[i * 3 + 2] * R[k * 3 + 2];
  float P2[3][2];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    P2[i][0] = Sc[i * 3] * A00 + Sc[i * 3 + 2] * A02;
    P2[i][1] = Sc[i * 3 + 1] * A11 + Sc[i * 3 + 2] * A12;
  }
  const float cxx = -fx * iz2, cyy = -fy * iz2;
  const float kx = 2.f * fx * X * iz2 * iz, ky = 2.f * fy * Yc * iz2 * iz;
  float dX[3][3];
  dX[0][0] = 2.f * cxx * P2[2][0]; dX[0][1] = cxx * P2[2][1]; dX[0][2] = 0.f;
  dX[1][0] = 0.f; dX[1][1] = cyy * P2[2][0]; dX[1][2] = 2.f * cyy * P2[2][1];
  const float r00 = cxx * P2[0][0] + kx * P2[2][0], r01 = cxx * P2[0][1] + kx * P2[2][1];
  const float r10 = cyy * P2[1][0] + ky * P2[2][0], r11 = cyy * P2[1][1] + ky * P2[2][1];
  dX[2][0] = 2.f * r00; dX[2][1] = r01 + r10; dX[2][2] = 2.f * r11;
  // camera-frame position perturbation R p_pos, then the position part of m_cov
  const float cp[3] = {R[0] * pp[0] + R[1] * pp[1] + R[2] * pp[2], R[3] * pp[0] + R[4] * pp[1] + R[5] * pp[2],
                       R[6] * pp[0] + R[7] * pp[1] + R[8] * pp[2]};
  float mc[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) mc[k] = dX[0][k] * cp[0] + dX[1][k] * cp[1] + dX[2][k] * cp[2];
  // + U dSigma U^T
  const float D[9] = {ds[0], ds[1], ds[2], ds[1], ds[3], ds[4], ds[2], ds[4], ds[5]};
  float UD[2][3];
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int j = 0; j < 3; ++j) UD[r][j] = U[r][0] * D[j] + U[r][1] * D[3 + j] + U[r][2] * D[6 + j];
  mc[0] += UD[0][0] * U[0][0] + UD[0][1] * U[0][1] + UD[0][2] * U[0][2];
  mc[1] += UD[0][0] * U[1][0] + UD[0][1] * U[1][1] + UD[0][2] * U[1][2];
  mc[2] += UD[1][0] * U[1][0] + UD[1][1] * U[1][1] + UD[1][2] * U[1][2];
  const float mmu0 = U[0][0] * pp[0] + U[0][1] * pp[1] + U[0][2] * pp[2];
  const float mmu1 = U[1][0] * pp[0] + U[1][1] * pp[1] + U[1][2] * pp[2];
  // colour
  const float v0 = p0 - cam.C[0], v1 = p1 - cam.C[1], v2 = p2 - cam.C[2];
  const float ivn = 1.f / sqrtf(v0 * v0 + v1 * v1 + v2 * v2);
  const float d0 = v0 * ivn, d1 = v1 * ivn, d2 = v2 * ivn;
  const float dp = d0 * pp[0] + d1 * pp[1] + d2 * pp[2];
  float Y[K], dY[K];
  sh_basis_dir<K>(d0, d1, d2, (pp[0] - d0 * dp) * ivn, (pp[1] - d1 * dp) * ivn, (pp[2] - d2 * dp) * ivn, Y, dY);
  float sh[3 * K + 4], ps[3 * K + 4];
  ldg_row<GT - GT_SH>(grow + GT_SH, sh);
  ldg_row<(P - 11 + 3 + 4) / 4 * 4>(prow + 8, ps);  // p from attribute 8 (16-byte aligned): p_sh at ps[3..]
  float mcol[3];
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    float sacc = 0.f;
#pragma unroll
    for (int k = 0; k < K; ++k) sacc = fmaf(sh[ch * K + k], dY[k], fmaf(ps[3 + ch * K + k], Y[k], sacc));
    mcol[ch] = (clampbits >> ch) & 1u ? 0.f : sacc;
  }
  out[0] = make_float4(dopa * pp[10], mmu0, mmu1, 0.5f * mc[0]);
  out[1] = make_float4(mc[1], 0.5f * mc[2], mcol[0], mcol[1]);
  out[2] = make_float4(mcol[2], 0.f, 0.f, 0.f);
}

// Forward chain of applyJ (ref: jacobian.py:434-443): thread per pair (pairs
// are (gid, view)-numbered, so neighbouring threads share the gaussian's
// parameters), m = dy/dx p packed as 3 float4 (48 B).  The product kernel's
// producer warp gathers it per run (cp.async) next to the static run records.
// p is read either attribute-major / unpadded gaussian-major (p[a sa + g sg])
// or, when sa = 1 and sg is a multiple of 4 >= P (the padded gaussian-major
// copy the PCG kernels write), as 16-byte row loads.
template <int K, bool DSIG>
__global__ void __launch_bounds__(128, DSIG ? SLM_PMD_MINB : SLM_PM_MINB) k_pair_m(SlmFwdArgs A) {
  constexpr int P = 11 + 3 * K, P4 = (P + 3) / 4;
  float4* __restrict__ pm = reinterpret_cast<float4*>(A.pm);
  const long long sa = A.sa, sg = A.sg;
  const float* __restrict__ p = A.p;
  const bool rows = sa == 1 && (sg & 3) == 0 && sg >= 4 * P4 && ((uintptr_t)p & 15) == 0;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < A.n_pairs; q += gridDim.x * blockDim.x) {
    const long long g = A.pair_gid[q];
    const uint32_t vm = A.pair_vm[q];
    if (DSIG) {  // padded gaussian-major p with dSigma: camera-dependent chain only
      pair_fwd_dsig<K>(g, load_camf(A.camf, vm & 0xffffu), vm >> 16, A.gtab, p + g * sg, pm + (size_t)q * 3);
      continue;
    }
    Tab<K> T;
    pair_tab<K>(A.xs, A.G, g, A.cams[vm & 0xffffu], vm >> 16, T, A.gtab);
    float pv[4 * P4];
    if (rows) {
      ldg_row<4 * P4>(p + g * sg, pv);
    } else {
#pragma unroll
      for (int a = 0; a < P; ++a) pv[a] = p[a * sa + g * sg];
    }
    float mmu0 = 0.f, mmu1 = 0.f, mc[3] = {0.f, 0.f, 0.f}, mcol[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      mmu0 += T.dmu[0][j] * pv[j];
      mmu1 += T.dmu[1][j] * pv[j];
    }
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
      for (int j = 0; j < 10; ++j) mc[k] += T.dcov[k][j] * pv[j];
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      float s = 0.f;
#pragma unroll
      for (int k = 0; k < K; ++k) s += T.Y[k] * pv[11 + ch * K + k];
      mcol[ch] = T.dcol[ch][0] * pv[0] + T.dcol[ch][1] * pv[1] + T.dcol[ch][2] * pv[2] + T.mask[ch] * s;
    }
    // record layout slots 5..13: inv_o * m_opa (scaled in k_run_records), m_mu0, m_mu1,
    // m_cov0/2, m_cov1, m_cov2/2, m_col0..2
    pm[(size_t)q * 3 + 0] = make_float4(T.dopa * pv[10], mmu0, mmu1, 0.5f * mc[0]);
    pm[(size_t)q * 3 + 1] = make_float4(mc[1], 0.5f * mc[2], mcol[0], mcol[1]);
    pm[(size_t)q * 3 + 2] = make_float4(mcol[2], 0.f, 0.f, 0.f);
  }
}
