// Matrix-free Jacobian products on the gradient cache (PAPER:659-736,
// ref: jacobian.py:419-512), B200 design:
//
//   * both cache streams are read flat and coalesced, 128 entries per warp
//     chunk (4 per lane, 16-byte vector loads of every SoA field);
//   * per-segment sums (pixel for J p, (gaussian, view) pair for J^T u and
//     diag) use a warp segmented scan over HEAD flags plus a fixed-order
//     carry fix-up for segments that cross chunk boundaries -- no float
//     atomics anywhere, results are bitwise run-to-run deterministic;
//   * the splat -> parameter chain (ref: jacobian.py:192-266) is recomputed
//     per (gaussian, view) pair in fp32 from the scene, never stored per entry.
#include "slm_common.cuh"


struct RecF {
  uint32_t w;
  float ae, at, d0, d1, d2;
};

template <int D>
struct SegCarry {
  float v[D];
  int seg;
  int flags;  // 1 valid, 2 closed
};

// ---------------------------------------------------------------------------
// generic warp-chunk segmented reduction
// ---------------------------------------------------------------------------
template <int D, class Op>
__global__ void __launch_bounds__(256) k_wsr(Op op, const uint32_t* __restrict__ idx, const float* __restrict__ fae,
                                             const float* __restrict__ fat, const float* __restrict__ fd0,
                                             const float* __restrict__ fd1, const float* __restrict__ fd2,
                                             long long E, const int* __restrict__ chunk_seg,
                                             SegCarry<D>* __restrict__ head, SegCarry<D>* __restrict__ tail) {
  const int lane = threadIdx.x & 31;
  const long long n_chunks = (E + SLM_CHUNK - 1) / SLM_CHUNK;
  const long long wstride = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long c = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); c < n_chunks; c += wstride) {
    const long long e0 = c * SLM_CHUNK;
    const long long eb = e0 + lane * SLM_IPT;
    RecF r[SLM_IPT];
    int nv = (int)min((long long)SLM_IPT, max(0LL, E - eb));
    if (nv == SLM_IPT) {
      uint4 wi = __ldg(reinterpret_cast<const uint4*>(idx + eb));
      float4 a = __ldg(reinterpret_cast<const float4*>(fae + eb));
      float4 t = __ldg(reinterpret_cast<const float4*>(fat + eb));
      float4 x0 = __ldg(reinterpret_cast<const float4*>(fd0 + eb));
      float4 x1 = __ldg(reinterpret_cast<const float4*>(fd1 + eb));
      float4 x2 = __ldg(reinterpret_cast<const float4*>(fd2 + eb));
      r[0] = {wi.x, a.x, t.x, x0.x, x1.x, x2.x};
      r[1] = {wi.y, a.y, t.y, x0.y, x1.y, x2.y};
      r[2] = {wi.z, a.z, t.z, x0.z, x1.z, x2.z};
      r[3] = {wi.w, a.w, t.w, x0.w, x1.w, x2.w};
    } else {
#pragma unroll
      for (int i = 0; i < SLM_IPT; ++i) {
        if (i < nv) {
          long long e = eb + i;
          r[i] = {idx[e], fae[e], fat[e], fd0[e], fd1[e], fd2[e]};
        } else {
          r[i] = {0u, 0.f, 0.f, 0.f, 0.f, 0.f};
        }
      }
    }
    bool hh[SLM_IPT];
    int lcnt = 0;
#pragma unroll
    for (int i = 0; i < SLM_IPT; ++i) {
      hh[i] = (i < nv) && (r[i].w & SLM_HEAD) && !(lane == 0 && i == 0);
      lcnt += hh[i];
    }
    int incl = lcnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const int cs = chunk_seg[c];
    const bool head_e0 = (__shfl_sync(0xffffffffu, r[0].w, 0) & SLM_HEAD) != 0;
    const int seg_open = cs + incl - lcnt;

    float run[D], first[D];
#pragma unroll
    for (int j = 0; j < D; ++j) run[j] = 0.f;
    bool have = false;
    int cur = seg_open;
#pragma unroll
    for (int i = 0; i < SLM_IPT; ++i) {
      if (i < nv) {
        if (hh[i]) {
          if (!have) {
#pragma unroll
            for (int j = 0; j < D; ++j) first[j] = run[j];
            have = true;
          } else {
            op.emit(cur, run);
          }
#pragma unroll
          for (int j = 0; j < D; ++j) run[j] = 0.f;
          ++cur;
        }
        op.accumulate(r[i], cur, run);
      }
    }
    if (!have) {
#pragma unroll
      for (int j = 0; j < D; ++j) first[j] = 0.f;
    }
    // inclusive segmented scan over lanes of (have, run)
    bool f = have;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      bool fu = __shfl_up_sync(0xffffffffu, f, o);
      bool add = (lane >= o) && !f;
#pragma unroll
      for (int j = 0; j < D; ++j) {
        float t = __shfl_up_sync(0xffffffffu, run[j], o);
        if (add) run[j] += t;
      }
      if (add) f = fu;
    }
    // exclusive carry into this lane
    bool exf = __shfl_up_sync(0xffffffffu, f, 1);
    if (lane == 0) exf = false;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      float t = __shfl_up_sync(0xffffffffu, run[j], 1);
      if (lane > 0) first[j] += t;
    }
    const bool started_in = exf || head_e0;
    if (have) {
      if (started_in) {
        op.emit(seg_open, first);
      } else {
        SegCarry<D>& h = head[c];
#pragma unroll
        for (int j = 0; j < D; ++j) h.v[j] = first[j];
        h.seg = seg_open;
        h.flags = 3;
      }
    }
    if (lane == 31) {
      const bool started = f || head_e0;
      const int seg_last = cs + incl;
      const long long en = e0 + SLM_CHUNK;
      const bool complete = en >= E || (idx[en] & SLM_HEAD);
      if (started) {
        if (complete) {
          op.emit(seg_last, run);
          tail[c].flags = 0;
        } else {
          SegCarry<D>& t = tail[c];
#pragma unroll
          for (int j = 0; j < D; ++j) t.v[j] = run[j];
          t.seg = seg_last;
          t.flags = 1;
        }
        if (head_e0) head[c].flags = 0;
      } else {
        SegCarry<D>& h = head[c];
#pragma unroll
        for (int j = 0; j < D; ++j) h.v[j] = run[j];
        h.seg = seg_last;
        h.flags = complete ? 3 : 1;
        tail[c].flags = 0;
      }
    }
  }
}

template <int D, class Op>
__global__ void k_wsr_fix(Op op, const SegCarry<D>* __restrict__ head, const SegCarry<D>* __restrict__ tail,
                          long long n_chunks) {
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n_chunks;
       c += (long long)gridDim.x * blockDim.x) {
    if (!(tail[c].flags & 1)) continue;
    float tot[D];
#pragma unroll
    for (int j = 0; j < D; ++j) tot[j] = tail[c].v[j];
    const int seg = tail[c].seg;
    for (long long k = c + 1; k < n_chunks; ++k) {
      const SegCarry<D>& h = head[k];
#pragma unroll
      for (int j = 0; j < D; ++j) tot[j] += h.v[j];
      if (h.flags & 2) break;
    }
    op.emit(seg, tot);
  }
}

// ---------------------------------------------------------------------------
// entry ops
// ---------------------------------------------------------------------------
struct PairM {  // per-pair forward chain result m = dy/dx p (J p), 48 bytes
  float4 a;     // m_mu0, m_mu1, m_cov0, m_cov1
  float4 b;     // m_cov2, m_opa, m_col0, m_col1
  float4 c;     // m_col2, -, -, -
};

// u_hat = J p, pixel segments (ref: jacobian.py:419-455), fused residual
// weighting u = u_hat * grad_r_sq (ref: jacobian.py:458-464) when gradr != 0.
struct OpApplyJ {
  const uint2* seg_info;
  const SlmPairGeo* geo;
  const PairM* pm;
  const float4* gradr;
  float4* u;
  __device__ __forceinline__ void accumulate(const RecF& r, int seg, float (&acc)[3]) const {
    const uint32_t xy = __ldg(&seg_info[seg].y);
    const uint32_t q = r.w & SLM_IDX_MASK;
    const SlmPairGeo g = geo[q];
    const PairM m = pm[q];
    const float dx = (float)((double)(xy & 0xffffu) + 0.5 - g.mx);
    const float dy = (float)((double)(xy >> 16) + 0.5 - g.my);
    const float e1 = g.ka * dx + g.kb * dy;
    const float e2 = g.kb * dx + g.kc * dy;
    const float da = r.ae * (e1 * m.a.x + e2 * m.a.y + 0.5f * e1 * e1 * m.a.z + e1 * e2 * m.a.w +
                             0.5f * e2 * e2 * m.b.x) +
                     r.ae * g.inv_o * m.b.y;
    acc[0] += r.d0 * da + r.at * m.b.z;
    acc[1] += r.d1 * da + r.at * m.b.w;
    acc[2] += r.d2 * da + r.at * m.c.x;
  }
  __device__ __forceinline__ void emit(int seg, const float (&v)[3]) const {
    const uint32_t gp = seg_info[seg].x;
    float4 w = gradr ? gradr[gp] : make_float4(1.f, 1.f, 1.f, 0.f);
    u[gp] = make_float4(v[0] * w.x, v[1] * w.y, v[2] * w.z, 0.f);
  }
};

// J^T u partial sums per pair: 9 values (ref: jacobian.py:324-342)
struct OpApplyJT {
  const SlmPairGeo* geo;
  const uint32_t* pair_vm;
  const SlmView* views;
  const float4* u;
  float* acc_out;  // [P][9]
  __device__ __forceinline__ void accumulate(const RecF& r, int q, float (&acc)[9]) const {
    const SlmPairGeo g = geo[q];
    const SlmView vw = views[pair_vm[q] & 0xffffu];
    const uint32_t x = r.w & 0xffffu, y = (r.w >> 16) & 0x7fffu;
    const float4 uu = u[vw.pix_base + (long long)y * vw.W + x];
    const float dx = (float)((double)x + 0.5 - g.mx);
    const float dy = (float)((double)y + 0.5 - g.my);
    const float e1 = g.ka * dx + g.kb * dy;
    const float e2 = g.kb * dx + g.kc * dy;
    const float sa = r.d0 * uu.x + r.d1 * uu.y + r.d2 * uu.z;
    const float t = sa * r.ae;
    acc[0] += t * e1;
    acc[1] += t * e2;
    acc[2] += 0.5f * t * e1 * e1;
    acc[3] += t * e1 * e2;
    acc[4] += 0.5f * t * e2 * e2;
    acc[5] += t * g.inv_o;
    acc[6] += r.at * uu.x;
    acc[7] += r.at * uu.y;
    acc[8] += r.at * uu.z;
  }
  __device__ __forceinline__ void emit(int q, const float (&v)[9]) const {
    float* o = acc_out + (size_t)q * 9;
#pragma unroll
    for (int j = 0; j < 9; ++j) o[j] = v[j];
  }
};

// diag(J^T W J) moments per pair (ref: jacobian.py:486-512).  With
// w = alpha_eff [e1, e2, e1^2/2, e1 e2, e2^2/2, 1/o] the per-parameter
// derivative is dc_c/dx_k = dcda_c (w . D_k) + aT dcol_ck, so
//   M_k = D_k^T S D_k + 2 sum_c dcol_ck (T_c . D_k) + sum_c dcol_ck^2 R_c
// with S = sum s1 w w^T (21), T_c = sum gr_c dcda_c aT w (18), R_c = sum gr_c aT^2 (3).
#define DIAG_D 42
__device__ __forceinline__ int sym6(int i, int j) {  // i <= j, upper triangle row-major
  return i * 6 - (i * (i - 1)) / 2 + (j - i);
}
struct OpDiag {
  const SlmPairGeo* geo;
  const uint32_t* pair_vm;
  const SlmView* views;
  const float4* gradr;
  float* mom_out;  // [P][42]
  __device__ __forceinline__ void accumulate(const RecF& r, int q, float (&acc)[DIAG_D]) const {
    const SlmPairGeo g = geo[q];
    const SlmView vw = views[pair_vm[q] & 0xffffu];
    const uint32_t x = r.w & 0xffffu, y = (r.w >> 16) & 0x7fffu;
    const float4 gr = gradr[vw.pix_base + (long long)y * vw.W + x];
    const float dx = (float)((double)x + 0.5 - g.mx);
    const float dy = (float)((double)y + 0.5 - g.my);
    const float e1 = g.ka * dx + g.kb * dy;
    const float e2 = g.kb * dx + g.kc * dy;
    float w[6] = {r.ae * e1, r.ae * e2, 0.5f * r.ae * e1 * e1, r.ae * e1 * e2, 0.5f * r.ae * e2 * e2,
                  r.ae * g.inv_o};
    const float s1 = gr.x * r.d0 * r.d0 + gr.y * r.d1 * r.d1 + gr.z * r.d2 * r.d2;
#pragma unroll
    for (int i = 0; i < 6; ++i)
#pragma unroll
      for (int j = i; j < 6; ++j) acc[sym6(i, j)] += s1 * w[i] * w[j];
    const float t0 = gr.x * r.d0 * r.at, t1 = gr.y * r.d1 * r.at, t2 = gr.z * r.d2 * r.at;
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      acc[21 + i] += t0 * w[i];
      acc[27 + i] += t1 * w[i];
      acc[33 + i] += t2 * w[i];
    }
    const float at2 = r.at * r.at;
    acc[39] += gr.x * at2;
    acc[40] += gr.y * at2;
    acc[41] += gr.z * at2;
  }
  __device__ __forceinline__ void emit(int q, const float (&v)[DIAG_D]) const {
    float* o = mom_out + (size_t)q * DIAG_D;
#pragma unroll
    for (int j = 0; j < DIAG_D; ++j) o[j] = v[j];
  }
};

// ---------------------------------------------------------------------------
// per-(gaussian, view) chain tables in fp32 (ref: jacobian.py:159-266)
// ---------------------------------------------------------------------------
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

// per-gaussian backward chain: out = scale * sum_views tab^T acc (+ lam * Mf * p),
// attribute-major; optional p . out block partials (fp64) for PCG.
// MODE 0: acc = 9 J^T partials (apply_jt / b); MODE 1: acc = 42 diag moments.
template <int K, int MODE>
__global__ void __launch_bounds__(128) k_pair_backward(const float* __restrict__ xs, long long G,
                                                       const int* __restrict__ gpo,
                                                       const int* __restrict__ gp_list,
                                                       const uint32_t* __restrict__ pair_vm,
                                                       const SlmCamera* __restrict__ cams,
                                                       const float* __restrict__ acc, float scale,
                                                       const float* __restrict__ p, const float* __restrict__ Mdiag,
                                                       float lam, float* __restrict__ out,
                                                       double* __restrict__ dot_part) {
  __shared__ double sm[32];
  double dot = 0.0;
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < G; g += (long long)gridDim.x * blockDim.x) {
    float og[11], osh[3][K];
#pragma unroll
    for (int j = 0; j < 11; ++j) og[j] = 0.f;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch)
#pragma unroll
      for (int k = 0; k < K; ++k) osh[ch][k] = 0.f;
    const int k0 = gpo[g], k1 = gpo[g + 1];
    for (int kk = k0; kk < k1; ++kk) {  // this gaussian's pairs, in view order
      const int q = gp_list[kk];
      const uint32_t vm = pair_vm[q];
      Tab<K> T;
      pair_tab<K>(xs, G, g, cams[vm & 0xffffu], vm >> 16, T);
      if (MODE == 0) {
        const float* a = acc + (size_t)q * 9;
        const float a0 = a[0], a1 = a[1], c0 = a[2], c1 = a[3], c2 = a[4], ao = a[5];
        const float col[3] = {a[6], a[7], a[8]};
#pragma unroll
        for (int j = 0; j < 3; ++j)
          og[j] += T.dmu[0][j] * a0 + T.dmu[1][j] * a1 + T.dcol[0][j] * col[0] + T.dcol[1][j] * col[1] +
                   T.dcol[2][j] * col[2];
#pragma unroll
        for (int j = 0; j < 10; ++j) og[j] += T.dcov[0][j] * c0 + T.dcov[1][j] * c1 + T.dcov[2][j] * c2;
        og[10] += T.dopa * ao;
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
          const float s = col[ch] * T.mask[ch];
#pragma unroll
          for (int k = 0; k < K; ++k) osh[ch][k] += s * T.Y[k];
        }
      } else {
        const float* m = acc + (size_t)q * DIAG_D;
        // D_j = (dmu0, dmu1, dcov0, dcov1, dcov2, dopa) columns
#pragma unroll
        for (int j = 0; j < 11; ++j) {
          float D[6];
          D[0] = j < 3 ? T.dmu[0][j] : 0.f;
          D[1] = j < 3 ? T.dmu[1][j] : 0.f;
          D[2] = j < 10 ? T.dcov[0][j] : 0.f;
          D[3] = j < 10 ? T.dcov[1][j] : 0.f;
          D[4] = j < 10 ? T.dcov[2][j] : 0.f;
          D[5] = j == 10 ? T.dopa : 0.f;
          float quad = 0.f;
#pragma unroll
          for (int i = 0; i < 6; ++i) {
            quad += m[sym6(i, i)] * D[i] * D[i];
#pragma unroll
            for (int k = i + 1; k < 6; ++k) quad += 2.f * m[sym6(i, k)] * D[i] * D[k];
          }
          if (j < 3) {
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) {
              float td = 0.f;
#pragma unroll
              for (int i = 0; i < 6; ++i) td += m[21 + ch * 6 + i] * D[i];
              const float dc = T.dcol[ch][j];
              quad += 2.f * dc * td + dc * dc * m[39 + ch];
            }
          }
          og[j] += quad;
        }
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
          const float s = m[39 + ch] * T.mask[ch];
#pragma unroll
          for (int k = 0; k < K; ++k) osh[ch][k] += s * T.Y[k] * T.Y[k];
        }
      }
    }
    // write attribute-major
#pragma unroll
    for (int a = 0; a < 11 + 3 * K; ++a) {
      float v = scale * (a < 11 ? og[a] : osh[(a - 11) / K][(a - 11) % K]);
      const long long i = (long long)a * G + g;
      if (p) {
        const float pv = p[i];
        if (Mdiag) v += lam * fmaxf(Mdiag[i], 1e-12f) * pv;
        dot += (double)pv * (double)v;
      }
      out[i] = v;
    }
  }
  if (dot_part) {
    double t = block_sum_d(dot, sm);
    if (threadIdx.x == 0) dot_part[blockIdx.x] = t;
  }
}

// ---------------------------------------------------------------------------
// C-ABI
// ---------------------------------------------------------------------------
typedef SlmWsrStream WsrStream;

template <int D, class Op>
static int run_wsr(const Op& op, const WsrStream& s, cudaStream_t st) {
  if (s.E <= 0) return SLM_OK;
  long long n_chunks = (s.E + SLM_CHUNK - 1) / SLM_CHUNK;
  long long blocks = (n_chunks + 7) / 8;
  if (blocks > 148LL * 16) blocks = 148LL * 16;
  k_wsr<D, Op><<<(unsigned)blocks, 256, 0, st>>>(op, s.idx, s.ae, s.at, s.d0, s.d1, s.d2, s.E, s.chunk_seg,
                                                 (SegCarry<D>*)s.head, (SegCarry<D>*)s.tail);
  k_wsr_fix<D, Op><<<slm_blocks(n_chunks, 256), 256, 0, st>>>(op, (SegCarry<D>*)s.head, (SegCarry<D>*)s.tail,
                                                               n_chunks);
  return slm_cuda_status();
}

extern "C" {

int slm_wsr_stream_size() { return (int)sizeof(WsrStream); }
int slm_view_size() { return (int)sizeof(SlmView); }
long long slm_carry_bytes(int D) { return (long long)(4 * D + 8); }

// u = J p (weighted when gradr != NULL); pm must already hold the pair forward chain.
int slm_apply_j(const WsrStream* pix, const uint2* seg_info, const SlmPairGeo* geo, const void* pm,
                const float4* gradr, float4* u, cudaStream_t st) {
  OpApplyJ op{seg_info, geo, (const PairM*)pm, gradr, u};
  return run_wsr<3>(op, *pix, st);
}

int slm_apply_jt_pairs(const WsrStream* gs, const SlmPairGeo* geo, const uint32_t* pair_vm, const SlmView* views,
                       const float4* u, float* acc, cudaStream_t st) {
  OpApplyJT op{geo, pair_vm, views, u, acc};
  return run_wsr<9>(op, *gs, st);
}

int slm_diag_pairs(const WsrStream* gs, const SlmPairGeo* geo, const uint32_t* pair_vm, const SlmView* views,
                   const float4* gradr, float* mom, cudaStream_t st) {
  OpDiag op{geo, pair_vm, views, gradr, mom};
  return run_wsr<DIAG_D>(op, *gs, st);
}

int slm_pair_forward(const float* xs, long long G, int sh_degree, const int* pair_gid, const uint32_t* pair_vm,
                     const SlmCamera* cams, int n_pairs, const float* p, long long sa, long long sg, void* pm,
                     cudaStream_t st) {
  if (n_pairs <= 0) return SLM_OK;
  unsigned b = slm_blocks(n_pairs, 128, 1LL << 30);
  switch (sh_degree) {
    case 0: k_pair_forward<1><<<b, 128, 0, st>>>(xs, G, pair_gid, pair_vm, cams, n_pairs, p, sa, sg, (PairM*)pm); break;
    case 1: k_pair_forward<4><<<b, 128, 0, st>>>(xs, G, pair_gid, pair_vm, cams, n_pairs, p, sa, sg, (PairM*)pm); break;
    case 2: k_pair_forward<9><<<b, 128, 0, st>>>(xs, G, pair_gid, pair_vm, cams, n_pairs, p, sa, sg, (PairM*)pm); break;
    case 3: k_pair_forward<16><<<b, 128, 0, st>>>(xs, G, pair_gid, pair_vm, cams, n_pairs, p, sa, sg, (PairM*)pm); break;
    default: return SLM_ERR_ARG;
  }
  return slm_cuda_status();
}

// number of blocks k_pair_backward uses for G gaussians (size of dot_part)
int slm_backward_blocks(long long G) { return (int)slm_blocks(G, 128, 148LL * 16); }

int slm_pair_backward(const float* xs, long long G, int sh_degree, const int* gpo, const int* gp_list,
                      const uint32_t* pair_vm, const SlmCamera* cams, const float* acc, int mode, float scale,
                      const float* p, const float* Mdiag, float lam, float* out, double* dot_part, cudaStream_t st) {
  unsigned b = (unsigned)slm_backward_blocks(G);
#define SLM_BW(KK)                                                                                              \
  if (mode == 0)                                                                                                \
    k_pair_backward<KK, 0><<<b, 128, 0, st>>>(xs, G, gpo, gp_list, pair_vm, cams, acc, scale, p, Mdiag, lam, out, \
                                              dot_part);                                                        \
  else                                                                                                          \
    k_pair_backward<KK, 1><<<b, 128, 0, st>>>(xs, G, gpo, gp_list, pair_vm, cams, acc, scale, p, Mdiag, lam, out, \
                                              dot_part);
  switch (sh_degree) {
    case 0: SLM_BW(1) break;
    case 1: SLM_BW(4) break;
    case 2: SLM_BW(9) break;
    case 3: SLM_BW(16) break;
    default: return SLM_ERR_ARG;
  }
#undef SLM_BW
  return slm_cuda_status();
}

}  // extern "C"
