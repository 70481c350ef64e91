// diag(J^T W J), the per-pair chain kernels and the per-gaussian backward
// chain (ref: jacobian.py:159-353, 486-512).  The J / J^T entry products live
// in stream.cu.
#include "chain.cuh"

#define DIAG_M 40     // diag moment floats per run (stream.cu diag pass)

// ---------------------------------------------------------------------------
// Per-gaussian backward chain (ref: jacobian.py:314-353 / 506-510), packed:
// warp w owns the gaussians whose first pair falls in pairs [32w, 32w + 32)
// (warp_g0 from k_warp_bounds), lane = pair.  Each lane sums its pair's run
// partials (contiguous slots, 16-byte loads), applies its view's 9 -> P chain
// and writes the row to a per-warp shared tile; the lanes then sum the rows
// of each gaussian column-wise (j = lane, lane + 32), the gaussians' row
// segments found with one ballot (rows are in (gid, view) order), in fixed
// row order (deterministic), and write gaussian-major scratch rows that
// k_gm_to_am transposes.
//   MODE 0 (J^T): run partials 0-7 as 32-byte records (pacc) + partial 8 (pacc1)
//   MODE 1 (diag): 40 moment floats per run (pacc), the pair's chain applied
//                  to them once per pair; SH block via basis^2
// ---------------------------------------------------------------------------
__global__ void k_warp_bounds(const int* __restrict__ gpo, long long G, int n_warps, int* __restrict__ warp_g0) {
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g <= G; g += (long long)gridDim.x * blockDim.x) {
    const int hi = g < G ? (gpo[g] >> 5) : n_warps;
    const int lo = g == 0 ? -1 : (gpo[g - 1] >> 5);
    for (int w = lo + 1; w <= hi && w <= n_warps; ++w) warp_g0[w] = (int)g;
  }
}

#define PK_WARPS 4
template <int K, int MODE>
__global__ void __launch_bounds__(32 * PK_WARPS, MODE == 0 ? SLM_BW_MINB : SLM_BW1_MINB) k_gauss_backward_packed(SlmBackArgs A, const int* __restrict__ warp_g0,
                                                                       int n_warps) {
  constexpr int P = 11 + 3 * K;
  constexpr int PR = MODE == 0 ? P - 1 : P;  // row / scratch width (J^T: world-covariance form)
  constexpr int PP = PR | 1;  // odd row stride: conflict-free row writes and column reads
  __shared__ float s_v[PK_WARPS][32 * PP];
  const unsigned F = 0xffffffffu;
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const long long G = A.G;
  // gaussian-major scratch row (contiguous, coalesced); k_gm_to_am writes the
  // attribute-major output with the scale / lambda / dot epilogue (fusing that
  // epilogue here -- per-lane attribute-strided p / M / out accesses -- was
  // measured 1.5x slower)
  auto flush = [&](long long g, float c0, float c1) {
    float* o = A.gm + (size_t)g * PR;
    if (lane < PR) o[lane] = c0;  // PR < 32 below SH degree 2
    if (lane + 32 < PR) o[lane + 32] = c1;
  };
  for (int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < n_warps; w += (gridDim.x * blockDim.x) >> 5) {
    const int ga = warp_g0[w], gb = warp_g0[w + 1];
    if (ga >= gb) continue;
    const int q0 = A.gpo[ga], q1 = A.gpo[gb];
    long long cur = ga;  // gaussian being accumulated
    float c0 = 0.f, c1 = 0.f;
    for (int base = q0; base < q1; base += 32) {
      const int q = base + lane;
      int myg = 0x7fffffff;
      if (q < q1) {
        myg = A.pair_gid[q];
        float* row = s_v[wl] + lane * PP;
        const uint32_t vm = A.pair_vm[q];
        const int r0 = A.pair_run_off[q], r1 = A.pair_run_off[q + 1];
        if (MODE == 0) {
          float a[9];
#pragma unroll
          for (int j = 0; j < 9; ++j) a[j] = 0.f;
          const float4* p4 = reinterpret_cast<const float4*>(A.pacc);
          // two runs per step (both loads in flight; the sums keep the run order)
          for (int rr = r0; rr < r1; rr += 2) {
            const bool two = rr + 1 < r1;
            const float4 u = __ldg(p4 + 2 * (size_t)rr), v = __ldg(p4 + 2 * (size_t)rr + 1);
            const float w8 = __ldg(A.pacc1 + rr);
            float4 u2 = make_float4(0.f, 0.f, 0.f, 0.f), v2 = u2;
            float x8 = 0.f;
            if (two) {
              u2 = __ldg(p4 + 2 * (size_t)rr + 2);
              v2 = __ldg(p4 + 2 * (size_t)rr + 3);
              x8 = __ldg(A.pacc1 + rr + 1);
            }
            a[0] += u.x; a[1] += u.y; a[2] += u.z; a[3] += u.w;
            a[4] += v.x; a[5] += v.y; a[6] += v.z; a[7] += v.w;
            a[8] += w8;
            if (two) {
              a[0] += u2.x; a[1] += u2.y; a[2] += u2.z; a[3] += u2.w;
              a[4] += v2.x; a[5] += v2.y; a[6] += v2.z; a[7] += v2.w;
              a[8] += x8;
            }
          }
          pair_back_row<K>(myg, load_camf(A.camf, vm & 0xffffu), vm >> 16, a, A.gtab, row);
        } else {
          // diag from the run moments (stream.cu diag pass): S (5x5 upper
          // triangle), V_ch (3 x 5), T3_ch, O / o^2; the pair's chain applied
          // once: M_k = D^T S D + 2 sum_ch c_ch D.V_ch + sum_ch c_ch^2 T3_ch
          float mo[36];
#pragma unroll
          for (int j = 0; j < 36; ++j) mo[j] = 0.f;
          const float4* p4 = reinterpret_cast<const float4*>(A.pacc);
          for (int rr = r0; rr < r1; rr += 2) {  // two runs per step, run order kept
            const bool two = rr + 1 < r1;
            float4 v[9], w[9];
#pragma unroll
            for (int k = 0; k < 9; ++k) {
              v[k] = __ldg(p4 + (size_t)rr * (DIAG_M / 4) + k);
              w[k] = two ? __ldg(p4 + (size_t)(rr + 1) * (DIAG_M / 4) + k) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int k = 0; k < 9; ++k) {
              mo[4 * k] += v[k].x;
              mo[4 * k + 1] += v[k].y;
              mo[4 * k + 2] += v[k].z;
              mo[4 * k + 3] += v[k].w;
            }
            if (two) {
#pragma unroll
              for (int k = 0; k < 9; ++k) {
                mo[4 * k] += w[k].x;
                mo[4 * k + 1] += w[k].y;
                mo[4 * k + 2] += w[k].z;
                mo[4 * k + 3] += w[k].w;
              }
            }
          }
          Tab<K> T;
          pair_tab<K>(A.xs, G, myg, A.cams[vm & 0xffffu], vm >> 16, T, A.gtab);
          auto S = [&](int i, int j) {  // upper-triangle index of the symmetric 5x5 S
            const int a = i < j ? i : j, b = i < j ? j : i;
            return mo[a * 5 - a * (a - 1) / 2 + (b - a)];
          };
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            const float D[5] = {T.dmu[0][k], T.dmu[1][k], T.dcov[0][k], T.dcov[1][k], T.dcov[2][k]};
            float q = 0.f;
#pragma unroll
            for (int i = 0; i < 5; ++i) {
              float t = 0.f;
#pragma unroll
              for (int j = 0; j < 5; ++j) t = fmaf(S(i, j), D[j], t);
              q = fmaf(D[i], t, q);
            }
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) {
              const float c = T.dcol[ch][k];
              float dv = 0.f;
#pragma unroll
              for (int i = 0; i < 5; ++i) dv = fmaf(D[i], mo[15 + ch * 5 + i], dv);
              q = fmaf(2.f * c, dv, fmaf(c * c, mo[30 + ch], q));
            }
            row[k] = q;
          }
#pragma unroll
          for (int k = 3; k < 10; ++k) {
            const float D[3] = {T.dcov[0][k], T.dcov[1][k], T.dcov[2][k]};
            float q = 0.f;
#pragma unroll
            for (int i = 0; i < 3; ++i) {
              float t = 0.f;
#pragma unroll
              for (int j = 0; j < 3; ++j) t = fmaf(S(2 + i, 2 + j), D[j], t);
              q = fmaf(D[i], t, q);
            }
            row[k] = q;
          }
          row[10] = T.dopa * T.dopa * mo[33];
#pragma unroll
          for (int ch = 0; ch < 3; ++ch) {
            const float sc = T.mask[ch] * mo[30 + ch];
#pragma unroll
            for (int k = 0; k < K; ++k) row[11 + ch * K + k] = sc * T.Y[k] * T.Y[k];
          }
        }
      }
      __syncwarp();
      // row segments of the window's gaussians (rows are gid-sorted)
      const int nr = min(32, q1 - base);
      const int prev = __shfl_up_sync(F, myg, 1);
      unsigned starts = __ballot_sync(F, lane < nr && (lane == 0 || myg != prev));
      while (starts) {
        const int i0 = __ffs(starts) - 1;
        starts &= starts - 1;
        const int i1 = starts ? __ffs(starts) - 1 : nr;
        const int gi = __shfl_sync(F, myg, i0);
        while (cur < gi) {  // finish cur (and any pair-less gaussians before gi)
          flush(cur, c0, c1);
          c0 = c1 = 0.f;
          ++cur;
        }
        const float* r = s_v[wl] + i0 * PP + lane;
        int i = i0;
        for (; i + 4 <= i1; i += 4, r += 4 * PP) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            c0 += r[k * PP];
            if (PR > 32 && lane + 32 < PR) c1 += r[k * PP + 32];
          }
        }
        for (; i < i1; ++i, r += PP) {
          c0 += r[0];
          if (PR > 32 && lane + 32 < PR) c1 += r[32];
        }
      }
      __syncwarp();
    }
    while (cur < gb) {
      flush(cur, c0, c1);
      c0 = c1 = 0.f;
      ++cur;
    }
  }
}

// gaussian-major scratch -> attribute-major out (tiled transpose, 32 gaussians
// per tile) with out = scale * v (+ lam * max(M, 1e-12) * p) and fp64 partials
// of p.(v + lam Mf p).  MODE 0 (J^T): the scratch rows are in the
// world-covariance form (pair_back_row); each gaussian's quaternion and
// log-scale gradients are formed here from its summed B = dL/dSigma:
//   Sigma = Rg S^2 Rg^T:  dL/dq_l = 2 <B Rg S^2, Mq_l>_F,
//                          dL/dlog s_i = 2 s_i^2 r_i^T B r_i
template <int P, int MODE>
__global__ void __launch_bounds__(256) k_gm_to_am(SlmBackArgs A) {
  constexpr int PR = MODE == 0 ? P - 1 : P;
  constexpr int TS = P | 1;  // odd tile stride: conflict-free column reads
  constexpr int K = (P - 11) / 3;
  __shared__ float t[32 * TS];
  __shared__ double sm[32];
  const long long G = A.G;
  double dot = 0.0;
  for (long long g0 = (long long)blockIdx.x * 32; g0 < G; g0 += (long long)gridDim.x * 32) {
    const int ng = (int)min((long long)32, G - g0);
    __syncthreads();
    if (MODE == 0) {
      // rows land at attribute positions: pos 0-2, B -> 3-8 (temporarily),
      // opacity 9 -> 10, SH 10.. -> 11..
      for (int i = threadIdx.x; i < ng * PR; i += blockDim.x) {
        const int gl = i / PR, c = i % PR;
        t[gl * TS + (c < 9 ? c : c + 1)] = A.gm[(size_t)g0 * PR + i];
      }
      __syncthreads();
      if (threadIdx.x < ng) {
        float* r = t + threadIdx.x * TS;
        const float* gt = A.gtab + (size_t)(g0 + threadIdx.x) * gtab_floats(K);
        float Rg[9], s2[3];
#pragma unroll
        for (int i = 0; i < 9; ++i) Rg[i] = gt[i];
#pragma unroll
        for (int i = 0; i < 3; ++i) s2[i] = gt[9 + i];
        const float B[9] = {r[3], r[4], r[5], r[4], r[6], r[7], r[5], r[7], r[8]};
        float T[9];  // B Rg S^2
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int j = 0; j < 3; ++j)
            T[i * 3 + j] = (B[i * 3] * Rg[j] + B[i * 3 + 1] * Rg[3 + j] + B[i * 3 + 2] * Rg[6 + j]) * s2[j];
        float gs[3];
#pragma unroll
        for (int j = 0; j < 3; ++j) gs[j] = 2.f * (Rg[j] * T[j] + Rg[3 + j] * T[3 + j] + Rg[6 + j] * T[6 + j]);
#pragma unroll
        for (int l = 0; l < 4; ++l) {
          float q = 0.f;
#pragma unroll
          for (int i = 0; i < 9; ++i) q = fmaf(T[i], gt[12 + l * 9 + i], q);
          r[3 + l] = 2.f * q;
        }
        r[7] = gs[0];
        r[8] = gs[1];
        r[9] = gs[2];
      }
    } else if (ng == 32) {
      // full tile: 32 consecutive rows = 8 * P float4 (16-byte aligned: g0 % 32 == 0)
      const float4* src = reinterpret_cast<const float4*>(A.gm + (size_t)g0 * P);
      for (int i = threadIdx.x; i < 8 * P; i += blockDim.x) {
        const float4 v = src[i];
        const int e = 4 * i;
        t[(e / P) * TS + e % P] = v.x;
        t[((e + 1) / P) * TS + (e + 1) % P] = v.y;
        t[((e + 2) / P) * TS + (e + 2) % P] = v.z;
        t[((e + 3) / P) * TS + (e + 3) % P] = v.w;
      }
    } else {
      for (int i = threadIdx.x; i < ng * P; i += blockDim.x) t[(i / P) * TS + i % P] = A.gm[(size_t)g0 * P + i];
    }
    __syncthreads();
#pragma unroll 4
    for (int i = threadIdx.x; i < 32 * P; i += blockDim.x) {
      const int a = i >> 5, gl = i & 31;
      if (gl < ng) {
        float v = A.scale * t[gl * TS + a];
        const long long idx = (long long)a * G + g0 + gl;
        if (A.p) {
          const double pv = (double)A.p[idx];
          const double lt = A.Mdiag ? A.lam * (double)fmaxf(A.Mdiag[idx], 1e-12f) * pv : 0.0;
          dot += pv * ((double)v + lt);
          if (A.lam_out) v = (float)((double)v + lt);
        }
        A.out[idx] = v;
      }
    }
  }
  if (A.dot_part) {
    double tt = block_sum_d(dot, sm);
    if (threadIdx.x == 0) A.dot_part[blockIdx.x] = tt;
  }
}

// ---------------------------------------------------------------------------
// C-ABI
// ---------------------------------------------------------------------------
extern "C" {

__global__ void k_cameras_f32(const SlmCamera* __restrict__ cams, int V, float* __restrict__ out) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= V) return;
  const SlmCamera c = cams[v];
  float* o = out + (size_t)v * CAMF_FLOATS;
  for (int i = 0; i < 9; ++i) o[i] = (float)c.R[i];
  for (int i = 0; i < 3; ++i) {
    o[9 + i] = (float)c.t[i];
    o[12 + i] = (float)c.C[i];
  }
  o[15] = (float)c.fx;
  o[16] = (float)c.fy;
  o[17] = o[18] = o[19] = 0.f;
}

int slm_view_size() { return (int)sizeof(SlmView); }

int slm_cameras_f32(const SlmCamera* cams, int V, float* out, cudaStream_t st) {
  if (V <= 0) return SLM_OK;
  k_cameras_f32<<<(V + 127) / 128, 128, 0, st>>>(cams, V, out);
  return slm_cuda_status();
}
int slm_tile_args_size() { return (int)sizeof(SlmTileArgs); }
int slm_back_args_size() { return (int)sizeof(SlmBackArgs); }
int slm_diag_moment_floats() { return DIAG_M; }

int slm_gauss_tab(const float* xs, long long G, int sh_degree, float* gtab, cudaStream_t st) {
  if (G <= 0) return SLM_OK;
  const unsigned b = slm_blocks(G, 256, 1LL << 30);
  switch (sh_degree) {
    case 0: k_gauss_tab<1><<<b, 256, 0, st>>>(xs, G, gtab); break;
    case 1: k_gauss_tab<4><<<b, 256, 0, st>>>(xs, G, gtab); break;
    case 2: k_gauss_tab<9><<<b, 256, 0, st>>>(xs, G, gtab); break;
    case 3: k_gauss_tab<16><<<b, 256, 0, st>>>(xs, G, gtab); break;
    default: return SLM_ERR_ARG;
  }
  return slm_cuda_status();
}

int slm_gauss_tab_floats(int sh_degree) {
  return sh_degree < 0 || sh_degree > 3 ? -1 : gtab_floats((sh_degree + 1) * (sh_degree + 1));
}


int slm_fwd_args_size() { return (int)sizeof(SlmFwdArgs); }

int slm_pair_forward(const SlmFwdArgs* a, int sh_degree, cudaStream_t st) {
  if (a->n_pairs <= 0) return SLM_OK;
  if (!a->pm || !a->gtab) return SLM_ERR_ARG;
  unsigned b = slm_blocks(a->n_pairs, 128, 1LL << 30);
#define SLM_PM(KK)                                  \
  if (a->dsig)                                      \
    k_pair_m<KK, true><<<b, 128, 0, st>>>(*a);      \
  else                                              \
    k_pair_m<KK, false><<<b, 128, 0, st>>>(*a);
  switch (sh_degree) {
    case 0: SLM_PM(1) break;
    case 1: SLM_PM(4) break;
    case 2: SLM_PM(9) break;
    case 3: SLM_PM(16) break;
    default: return SLM_ERR_ARG;
  }
#undef SLM_PM
  return slm_cuda_status();
}

int slm_backward_blocks(long long G) { return (int)slm_blocks(G, 128, 148LL * 16); }

int slm_warp_bounds(const int* gpo, long long G, int n_pairs, int* warp_g0, cudaStream_t st) {
  const int n_warps = (n_pairs >> 5) + 1;
  k_warp_bounds<<<slm_blocks(G + 1, 256), 256, 0, st>>>(gpo, G, n_warps, warp_g0);
  return slm_cuda_status();
}

int slm_pair_backward(const SlmBackArgs* a, int mode, int sh_degree, cudaStream_t st) {
  if (!a->warp_g0 || !a->pair_run_off || !a->gtab || (mode == 0 && !a->pacc1)) return SLM_ERR_ARG;
  const unsigned b = (unsigned)slm_backward_blocks(a->G);
  const int nw = (int)((a->n_pairs >> 5) + 1);
#define SLM_PK(KK)                                                                         \
  if (mode == 0)                                                                           \
    k_gauss_backward_packed<KK, 0><<<b, 32 * PK_WARPS, 0, st>>>(*a, a->warp_g0, nw);       \
  else                                                                                     \
    k_gauss_backward_packed<KK, 1><<<b, 32 * PK_WARPS, 0, st>>>(*a, a->warp_g0, nw);       \
  if (mode == 0)                                                                           \
    k_gm_to_am<11 + 3 * KK, 0><<<b, 256, 0, st>>>(*a);                                     \
  else                                                                                     \
    k_gm_to_am<11 + 3 * KK, 1><<<b, 256, 0, st>>>(*a);
  switch (sh_degree) {
    case 0: SLM_PK(1) break;
    case 1: SLM_PK(4) break;
    case 2: SLM_PK(9) break;
    case 3: SLM_PK(16) break;
    default: return SLM_ERR_ARG;
  }
#undef SLM_PK
  return slm_cuda_status();
}

}  // extern "C"
