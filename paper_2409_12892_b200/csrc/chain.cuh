// Per-(gaussian, view) splat -> parameter chain in fp32 (ref: jacobian.py:159-266)
// and the per-pair forward chain kernel (m = dy/dx p, ref: jacobian.py:434-443).
#pragma once
#include "slm_common.cuh"

struct PairM {  // per-pair forward chain result m = dy/dx p (J p), 48 bytes
  float4 a;     // m_mu0, m_mu1, m_cov0, m_cov1
  float4 b;     // m_cov2, m_opa, m_col0, m_col1
  float4 c;     // m_col2, -, -, -
};

template <int K>
struct Tab {
  float dmu[2][3];
  float dcov[3][10];
  float dcol[3][3];
  float Y[K];
  float dopa;
  float mask[3];
};

template <int K>
__device__ __forceinline__ void pair_tab(const float* __restrict__ xs, long long G, long long g, const SlmCamera& cam,
                                         uint32_t clampbits, Tab<K>& T) {
  const float p0 = xs[g], p1 = xs[G + g], p2 = xs[2 * G + g];
  float q[4] = {xs[3 * G + g], xs[4 * G + g], xs[5 * G + g], xs[6 * G + g]};
  const float l0 = xs[7 * G + g], l1 = xs[8 * G + g], l2 = xs[9 * G + g];
  const float logit = xs[10 * G + g];
  float R[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) R[i] = (float)cam.R[i];
  const float fx = (float)cam.fx, fy = (float)cam.fy;
  const float X = R[0] * p0 + R[1] * p1 + R[2] * p2 + (float)cam.t[0];
  const float Yc = R[3] * p0 + R[4] * p1 + R[5] * p2 + (float)cam.t[1];
  const float Z = R[6] * p0 + R[7] * p1 + R[8] * p2 + (float)cam.t[2];
  const float iz = 1.f / Z, iz2 = iz * iz;
  const float A00 = fx * iz, A02 = -fx * X * iz2, A11 = fy * iz, A12 = -fy * Yc * iz2;
  float U[2][3];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    U[0][j] = A00 * R[j] + A02 * R[6 + j];
    U[1][j] = A11 * R[3 + j] + A12 * R[6 + j];
    T.dmu[0][j] = U[0][j];
    T.dmu[1][j] = U[1][j];
  }
  // rotation of the gaussian
  const float qn = sqrtf(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
  const float iq = 1.f / qn;
  const float w = q[0] * iq, a = q[1] * iq, b = q[2] * iq, c = q[3] * iq;
  float Rg[9] = {1.f - 2.f * (b * b + c * c), 2.f * (a * b - w * c), 2.f * (a * c + w * b),
                 2.f * (a * b + w * c), 1.f - 2.f * (a * a + c * c), 2.f * (b * c - w * a),
                 2.f * (a * c - w * b), 2.f * (b * c + w * a), 1.f - 2.f * (a * a + b * b)};
  const float s2[3] = {__expf(2.f * l0), __expf(2.f * l1), __expf(2.f * l2)};
  // M = R Rg (camera-frame axes), Sc = M diag(s2) M^T
  float Mm[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) Mm[i * 3 + j] = R[i * 3] * Rg[j] + R[i * 3 + 1] * Rg[3 + j] + R[i * 3 + 2] * Rg[6 + j];
  float Sc[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int k = 0; k < 3; ++k)
      Sc[i * 3 + k] = Mm[i * 3] * s2[0] * Mm[k * 3] + Mm[i * 3 + 1] * s2[1] * Mm[k * 3 + 1] +
                      Mm[i * 3 + 2] * s2[2] * Mm[k * 3 + 2];
  // P = Sc A^T (3x2)
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
#pragma unroll
  for (int p = 0; p < 3; ++p)
#pragma unroll
    for (int j = 0; j < 3; ++j) T.dcov[p][j] = dX[0][p] * R[j] + dX[1][p] * R[3 + j] + dX[2][p] * R[6 + j];
  // quaternion: dcov_l = V_l W^T + W V_l^T, V_l = U dR/dq_l, W = U Rg diag(s2)
  float UR[2][3], Wm[2][3];
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      UR[r][j] = U[r][0] * Rg[j] + U[r][1] * Rg[3 + j] + U[r][2] * Rg[6 + j];
      Wm[r][j] = UR[r][j] * s2[j];
    }
  // dR/dq_hat_k (3x3 each), row-major
  const float dRh[4][9] = {
      {0.f, -2.f * c, 2.f * b, 2.f * c, 0.f, -2.f * a, -2.f * b, 2.f * a, 0.f},
      {0.f, 2.f * b, 2.f * c, 2.f * b, -4.f * a, -2.f * w, 2.f * c, 2.f * w, -4.f * a},
      {-4.f * b, 2.f * a, 2.f * w, 2.f * a, 0.f, 2.f * c, -2.f * w, 2.f * c, -4.f * b},
      {-4.f * c, -2.f * w, 2.f * a, 2.f * w, -4.f * c, 2.f * b, 2.f * a, 2.f * b, 0.f}};
  float Vh[4][2][3];
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int j = 0; j < 3; ++j)
        Vh[k][r][j] = U[r][0] * dRh[k][j] + U[r][1] * dRh[k][3 + j] + U[r][2] * dRh[k][6 + j];
  const float qh[4] = {w, a, b, c};
#pragma unroll
  for (int l = 0; l < 4; ++l) {
    float V[2][3];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        float s = 0.f;
#pragma unroll
        for (int k = 0; k < 4; ++k) s += ((k == l ? 1.f : 0.f) - qh[k] * qh[l]) * Vh[k][r][j];
        V[r][j] = s * iq;
      }
    const float v0w0 = V[0][0] * Wm[0][0] + V[0][1] * Wm[0][1] + V[0][2] * Wm[0][2];
    const float v0w1 = V[0][0] * Wm[1][0] + V[0][1] * Wm[1][1] + V[0][2] * Wm[1][2];
    const float v1w0 = V[1][0] * Wm[0][0] + V[1][1] * Wm[0][1] + V[1][2] * Wm[0][2];
    const float v1w1 = V[1][0] * Wm[1][0] + V[1][1] * Wm[1][1] + V[1][2] * Wm[1][2];
    T.dcov[0][3 + l] = 2.f * v0w0;
    T.dcov[1][3 + l] = v0w1 + v1w0;
    T.dcov[2][3 + l] = 2.f * v1w1;
  }
  // log-scale: 2 s_i^2 (U r_i)(U r_i)^T
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    T.dcov[0][7 + i] = 2.f * s2[i] * UR[0][i] * UR[0][i];
    T.dcov[1][7 + i] = 2.f * s2[i] * UR[0][i] * UR[1][i];
    T.dcov[2][7 + i] = 2.f * s2[i] * UR[1][i] * UR[1][i];
  }
  // colour
  const float v0 = p0 - (float)cam.C[0], v1 = p1 - (float)cam.C[1], v2 = p2 - (float)cam.C[2];
  const float vn = sqrtf(v0 * v0 + v1 * v1 + v2 * v2), ivn = 1.f / vn;
  const float d0 = v0 * ivn, d1 = v1 * ivn, d2 = v2 * ivn;
  sh_basis<float, K>(d0, d1, d2, T.Y);
  float dcdd[3][3];
  auto coef = [&](int ch, int k) { return xs[(long long)(11 + ch * K + k) * G + g]; };
  sh_grad_dot<float, K>(d0, d1, d2, coef, dcdd);
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    T.mask[ch] = (clampbits >> ch) & 1u ? 0.f : 1.f;
    const float dd = dcdd[ch][0] * d0 + dcdd[ch][1] * d1 + dcdd[ch][2] * d2;
    T.dcol[ch][0] = T.mask[ch] * (dcdd[ch][0] - d0 * dd) * ivn;
    T.dcol[ch][1] = T.mask[ch] * (dcdd[ch][1] - d1 * dd) * ivn;
    T.dcol[ch][2] = T.mask[ch] * (dcdd[ch][2] - d2 * dd) * ivn;
  }
  const float o = 1.f / (1.f + __expf(-logit));
  T.dopa = o * (1.f - o);
}

// m = dy/dx p per pair (forward chain of applyJ, ref: jacobian.py:434-443).
// p is read with strides so both layouts work: p[a * sa + g * sg].
template <int K>
__global__ void __launch_bounds__(128) k_pair_forward(const float* __restrict__ xs, long long G,
                                                      const int* __restrict__ pair_gid,
                                                      const uint32_t* __restrict__ pair_vm,
                                                      const SlmCamera* __restrict__ cams, int n_pairs,
                                                      const float* __restrict__ p, long long sa, long long sg,
                                                      PairM* __restrict__ pm) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n_pairs; q += gridDim.x * blockDim.x) {
    const long long g = pair_gid[q];
    const uint32_t vm = pair_vm[q];
    Tab<K> T;
    pair_tab<K>(xs, G, g, cams[vm & 0xffffu], vm >> 16, T);
    float pg[11];
#pragma unroll
    for (int a = 0; a < 11; ++a) pg[a] = p[a * sa + g * sg];
    float mmu0 = 0.f, mmu1 = 0.f, mc[3] = {0.f, 0.f, 0.f}, mcol[3] = {0.f, 0.f, 0.f};
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      mmu0 += T.dmu[0][j] * pg[j];
      mmu1 += T.dmu[1][j] * pg[j];
    }
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
      for (int j = 0; j < 10; ++j) mc[k] += T.dcov[k][j] * pg[j];
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      float s = 0.f;
#pragma unroll
      for (int k = 0; k < K; ++k) s += T.Y[k] * p[(11 + ch * K + k) * sa + g * sg];
      mcol[ch] = T.dcol[ch][0] * pg[0] + T.dcol[ch][1] * pg[1] + T.dcol[ch][2] * pg[2] + T.mask[ch] * s;
    }
    PairM m;
    m.a = make_float4(mmu0, mmu1, mc[0], mc[1]);
    m.b = make_float4(mc[2], T.dopa * pg[10], mcol[0], mcol[1]);
    m.c = make_float4(mcol[2], 0.f, 0.f, 0.f);
    pm[q] = m;
  }
}
