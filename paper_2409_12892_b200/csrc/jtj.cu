// diag(J^T W J), the per-pair chain kernels and the per-gaussian backward
// chain (ref: jacobian.py:159-353, 486-512).  The J / J^T entry products live
// in stream.cu.
#include "chain.cuh"

#define NW 8          // warps per CTA (diag)
#define DIAG_TAB 48   // floats per pair coefficient table (diag)
#define DIAG_RUN_D 14
#define TBD 256

__device__ __forceinline__ int view_of_tile(const int* __restrict__ vtb, int n_views, int t) {
  int v = 0;
  while (v + 1 < n_views && vtb[v + 1] <= t) ++v;
  return v;
}

__device__ __forceinline__ int rs16_slot(int lane) {
  return ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 + ((lane >> 1) & 1);
}
// reduce-scatter of 16 per-lane values in 16 shuffles; lanes 2i, 2i+1 end
// with the warp sum of value rs16_slot(lane); fixed pattern -> deterministic
__device__ __forceinline__ float warp_reduce_scatter16(const float (&v)[16], int lane) {
  const unsigned F = 0xffffffffu;
  float w8[8], w4[4], w2[2];
  const bool u16 = lane & 16, u8 = lane & 8, u4 = lane & 4, u2 = lane & 2;
#pragma unroll
  for (int j = 0; j < 8; ++j) w8[j] = (u16 ? v[j + 8] : v[j]) + __shfl_xor_sync(F, u16 ? v[j] : v[j + 8], 16);
#pragma unroll
  for (int j = 0; j < 4; ++j) w4[j] = (u8 ? w8[j + 4] : w8[j]) + __shfl_xor_sync(F, u8 ? w8[j] : w8[j + 4], 8);
#pragma unroll
  for (int j = 0; j < 2; ++j) w2[j] = (u4 ? w4[j + 2] : w4[j]) + __shfl_xor_sync(F, u4 ? w4[j] : w4[j + 2], 4);
  float w1 = (u2 ? w2[1] : w2[0]) + __shfl_xor_sync(F, u2 ? w2[0] : w2[1], 2);
  return w1 + __shfl_xor_sync(F, w1, 1);
}

// ---------------------------------------------------------------------------
// diag(J^T W J): per run, 11 geometry sums of grad_r_sq * (dc/dx_k)^2 and the
// three channel sums grad_r_sq * (alpha T)^2 that the SH block needs
// (ref: jacobian.py:496-508) -- exact squares per entry.  The per-pair
// coefficient tables come from k_pair_tables (one thread per pair).
// table layout: [0,15) k=0..2 x (dmu0, dmu1, dcov0, dcov1, dcov2);
//               [15,36) k=3..9 x (dcov0, dcov1, dcov2); [36] dopa;
//               [37,46) dcol[ch][j] (position columns)
// ---------------------------------------------------------------------------
template <int K>
__global__ void __launch_bounds__(128) k_pair_tables(const float* __restrict__ xs, long long G,
                                                     const int* __restrict__ pair_gid,
                                                     const uint32_t* __restrict__ pair_vm,
                                                     const SlmCamera* __restrict__ cams, int n_pairs,
                                                     float* __restrict__ tab, const float* __restrict__ gtab) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n_pairs; q += gridDim.x * blockDim.x) {
    const uint32_t vm = pair_vm[q];
    Tab<K> T;
    pair_tab<K>(xs, G, pair_gid[q], cams[vm & 0xffffu], vm >> 16, T, gtab);
    float o[DIAG_TAB];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      o[k * 5 + 0] = T.dmu[0][k];
      o[k * 5 + 1] = T.dmu[1][k];
      o[k * 5 + 2] = T.dcov[0][k];
      o[k * 5 + 3] = T.dcov[1][k];
      o[k * 5 + 4] = T.dcov[2][k];
    }
#pragma unroll
    for (int k = 3; k < 10; ++k) {
      o[15 + (k - 3) * 3 + 0] = T.dcov[0][k];
      o[15 + (k - 3) * 3 + 1] = T.dcov[1][k];
      o[15 + (k - 3) * 3 + 2] = T.dcov[2][k];
    }
    o[36] = T.dopa;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch)
#pragma unroll
      for (int j = 0; j < 3; ++j) o[37 + ch * 3 + j] = T.dcol[ch][j];
    o[46] = 0.f;
    o[47] = 0.f;
    float4* dst = reinterpret_cast<float4*>(tab + (size_t)q * DIAG_TAB);  // 16-byte stores
#pragma unroll
    for (int k = 0; k < DIAG_TAB / 4; ++k) dst[k] = make_float4(o[4 * k], o[4 * k + 1], o[4 * k + 2], o[4 * k + 3]);
  }
}

// ---------------------------------------------------------------------------
// per-pair sums of the run partials (fixed run order -> deterministic):
// pacc[q] = sum over the pair's runs of acc[run] (D = 9 J^T partials or 14
// diag sums); pairs are (gid, view)-numbered, so the backward chain below
// reads them contiguously
// ---------------------------------------------------------------------------
template <int D>
__global__ void k_pair_sum(const int* __restrict__ pair_run_off, const int* __restrict__ pair_runs, int n_pairs,
                           const float* __restrict__ acc, float* __restrict__ pacc) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n_pairs; q += gridDim.x * blockDim.x) {
    float a[D];
#pragma unroll
    for (int j = 0; j < D; ++j) a[j] = 0.f;
    for (int rr = pair_run_off[q]; rr < pair_run_off[q + 1]; ++rr) {
      const float* src = acc + (size_t)pair_runs[rr] * D;
#pragma unroll
      for (int j = 0; j < D; ++j) a[j] += src[j];
    }
#pragma unroll
    for (int j = 0; j < D; ++j) pacc[(size_t)q * D + j] = a[j];
  }
}

// ---------------------------------------------------------------------------
// per-gaussian backward chain (ref: jacobian.py:314-353 / 506-510):
//   MODE 0: out = scale * sum_pairs tab^T pacc   (J^T partials)
//   MODE 1: out = sum_pairs pacc, SH block via basis^2   (diag sums)
// optional fp64 partials of p.(out + lam * max(M, 1e-12) * p) (PCG), and
// out += lam * max(M, 1e-12) * p when lam_out
// ---------------------------------------------------------------------------
// sum of one pair's run partials (slot order) or its precomputed pair sum
template <int D, int J0, int J1>
__device__ __forceinline__ void pair_partials(const SlmBackArgs& A, int q, float (&a)[J1 - J0]) {
#pragma unroll
  for (int j = 0; j < J1 - J0; ++j) a[j] = 0.f;
  if (A.pair_run_off) {
    for (int rr = A.pair_run_off[q]; rr < A.pair_run_off[q + 1]; ++rr) {
#pragma unroll
      for (int j = 0; j < J1 - J0; ++j) a[j] += A.pacc[(size_t)rr * D + J0 + j];
    }
  } else {
#pragma unroll
    for (int j = 0; j < J1 - J0; ++j) a[j] = A.pacc[(size_t)q * D + J0 + j];
  }
}

// Two sweeps over the gaussian's pairs keep the live state small (geometry
// accumulators + chain, then the 3 x K SH accumulators + basis) so the kernel
// runs at 4 blocks / SM without spills.
template <int K, int MODE>
__global__ void __launch_bounds__(128, 3) k_gauss_backward(SlmBackArgs A) {
  __shared__ double sm[32];
  constexpr int D = MODE == 0 ? 9 : DIAG_RUN_D;
  const long long G = A.G;
  double dot = 0.0;
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < G; g += (long long)gridDim.x * blockDim.x) {
    const int k0 = A.gpo[g], k1 = A.gpo[g + 1];
    // ---- sweep 1: the 11 geometry parameters
    float og[11];
#pragma unroll
    for (int j = 0; j < 11; ++j) og[j] = 0.f;
    for (int q = k0; q < k1; ++q) {  // this gaussian's pairs, in view order
      if (MODE == 0) {
        float a[9];
        pair_partials<D, 0, 9>(A, q, a);
        const uint32_t vm = A.pair_vm[q];
        Tab<K> T;
        pair_tab<K>(A.xs, G, g, A.cams[vm & 0xffffu], vm >> 16, T, A.gtab);
#pragma unroll
        for (int j = 0; j < 3; ++j)
          og[j] += T.dmu[0][j] * a[0] + T.dmu[1][j] * a[1] + T.dcol[0][j] * a[6] + T.dcol[1][j] * a[7] +
                   T.dcol[2][j] * a[8];
#pragma unroll
        for (int j = 0; j < 10; ++j) og[j] += T.dcov[0][j] * a[2] + T.dcov[1][j] * a[3] + T.dcov[2][j] * a[4];
        og[10] += T.dopa * a[5];
      } else {
        float a[11];
        pair_partials<D, 0, 11>(A, q, a);
#pragma unroll
        for (int j = 0; j < 11; ++j) og[j] += a[j];
      }
    }
#pragma unroll
    for (int j = 0; j < 11; ++j) {
      float v = A.scale * og[j];
      const long long i = (long long)j * G + g;
      if (A.p) {
        const double pv = (double)A.p[i];
        const double lt = A.Mdiag ? A.lam * (double)fmaxf(A.Mdiag[i], 1e-12f) * pv : 0.0;
        dot += pv * ((double)v + lt);
        if (A.lam_out) v = (float)((double)v + lt);
      }
      A.out[i] = v;
    }
    // ---- sweep 2: the SH block, (colour partial * clamp mask) x basis (MODE 0)
    // or (colour sum * clamp mask) x basis^2 (MODE 1)
    float osh[3][K];
#pragma unroll
    for (int ch = 0; ch < 3; ++ch)
#pragma unroll
      for (int k = 0; k < K; ++k) osh[ch][k] = 0.f;
    const float px = A.xs[g], py = A.xs[G + g], pz = A.xs[2 * G + g];
    for (int q = k0; q < k1; ++q) {
      float c[3];
      if (MODE == 0) pair_partials<D, 6, 9>(A, q, c);
      else pair_partials<D, 11, 14>(A, q, c);
      const uint32_t vm = A.pair_vm[q];
      const SlmCamera& cam = A.cams[vm & 0xffffu];
      const float v0 = px - (float)cam.C[0], v1 = py - (float)cam.C[1], v2 = pz - (float)cam.C[2];
      const float ivn = 1.f / sqrtf(v0 * v0 + v1 * v1 + v2 * v2);
      float Y[K];
      sh_basis<float, K>(v0 * ivn, v1 * ivn, v2 * ivn, Y);
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) {
        const float s = ((vm >> (16 + ch)) & 1u) ? 0.f : c[ch];
#pragma unroll
        for (int k = 0; k < K; ++k) osh[ch][k] += MODE == 0 ? s * Y[k] : s * Y[k] * Y[k];
      }
    }
#pragma unroll
    for (int a = 11; a < 11 + 3 * K; ++a) {
      float v = A.scale * osh[(a - 11) / K][(a - 11) % K];
      const long long i = (long long)a * G + g;
      if (A.p) {
        const double pv = (double)A.p[i];
        const double lt = A.Mdiag ? A.lam * (double)fmaxf(A.Mdiag[i], 1e-12f) * pv : 0.0;
        dot += pv * ((double)v + lt);
        if (A.lam_out) v = (float)((double)v + lt);
      }
      A.out[i] = v;
    }
  }
  if (A.dot_part) {
    double t = block_sum_d(dot, sm);
    if (threadIdx.x == 0) A.dot_part[blockIdx.x] = t;
  }
}

// ---------------------------------------------------------------------------
// Packed per-gaussian backward: warp w owns the gaussians whose first pair
// falls in pairs [32w, 32w + 32) (warp_g0 from k_warp_bounds), lane = pair.
// Each lane sums its pair's run partials (contiguous slots), applies its
// view's 9 -> 59 chain and writes the row to a per-warp shared tile; the lanes
// then walk the rows in pair order summing columns j = lane, lane + 32 per
// gaussian (fixed order -> deterministic).  Loads are coalesced across lanes
// and there is no per-thread serial loop over a gaussian's pairs.
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
__global__ void __launch_bounds__(32 * PK_WARPS) k_gauss_backward_packed(SlmBackArgs A, const int* __restrict__ warp_g0,
                                                                       int n_warps) {
  constexpr int P = 11 + 3 * K;
  constexpr int PP = P | 1;  // odd row stride: conflict-free row writes and column reads
  constexpr int D = MODE == 0 ? 9 : DIAG_RUN_D;
  __shared__ float s_v[PK_WARPS][32 * PP];
  __shared__ int s_g[PK_WARPS][32];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const long long G = A.G;
  // gaussian-major scratch row (contiguous, coalesced); k_gm_to_am writes the
  // attribute-major output with the scale / lambda / dot epilogue
  auto flush = [&](long long g, float c0, float c1) {
    float* o = A.gm + (size_t)g * P;
    if (lane < P) o[lane] = c0;  // P < 32 below SH degree 2
    if (lane + 32 < P) o[lane + 32] = c1;
  };
  for (int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < n_warps; w += (gridDim.x * blockDim.x) >> 5) {
    const int ga = warp_g0[w], gb = warp_g0[w + 1];
    if (ga >= gb) continue;
    const int q0 = A.gpo[ga], q1 = A.gpo[gb];
    long long cur = ga;  // gaussian being accumulated
    float c0 = 0.f, c1 = 0.f;
    for (int base = q0; base < q1; base += 32) {
      const int q = base + lane;
      if (q < q1) {
        const long long g = A.pair_gid[q];
        s_g[wl][lane] = (int)g;
        float* row = s_v[wl] + lane * PP;
        float a[D];
        pair_partials<D, 0, D>(A, q, a);
        const uint32_t vm = A.pair_vm[q];
        if (MODE == 0) {
          Tab<K> T;
          pair_tab<K>(A.xs, G, g, A.cams[vm & 0xffffu], vm >> 16, T, A.gtab);
#pragma unroll
          for (int j = 0; j < 3; ++j)
            row[j] = T.dmu[0][j] * a[0] + T.dmu[1][j] * a[1] + T.dcol[0][j] * a[6] + T.dcol[1][j] * a[7] +
                     T.dcol[2][j] * a[8] + T.dcov[0][j] * a[2] + T.dcov[1][j] * a[3] + T.dcov[2][j] * a[4];
#pragma unroll
          for (int j = 3; j < 10; ++j) row[j] = T.dcov[0][j] * a[2] + T.dcov[1][j] * a[3] + T.dcov[2][j] * a[4];
          row[10] = T.dopa * a[5];
#pragma unroll
          for (int ch = 0; ch < 3; ++ch) {
            const float sc = a[6 + ch] * T.mask[ch];
#pragma unroll
            for (int k = 0; k < K; ++k) row[11 + ch * K + k] = sc * T.Y[k];
          }
        } else {
#pragma unroll
          for (int j = 0; j < 11; ++j) row[j] = a[j];
          const SlmCamera& cam = A.cams[vm & 0xffffu];
          const float v0 = A.xs[g] - (float)cam.C[0], v1 = A.xs[G + g] - (float)cam.C[1];
          const float v2 = A.xs[2 * G + g] - (float)cam.C[2];
          const float ivn = 1.f / sqrtf(v0 * v0 + v1 * v1 + v2 * v2);
          float Y[K];
          sh_basis<float, K>(v0 * ivn, v1 * ivn, v2 * ivn, Y);
#pragma unroll
          for (int ch = 0; ch < 3; ++ch) {
            const float sc = ((vm >> (16 + ch)) & 1u) ? 0.f : a[11 + ch];
#pragma unroll
            for (int k = 0; k < K; ++k) row[11 + ch * K + k] = sc * Y[k] * Y[k];
          }
        }
      }
      __syncwarp();
      const int nr = min(32, q1 - base);
      for (int i = 0; i < nr; ++i) {  // rows in pair order
        const int gi = s_g[wl][i];
        while (cur < gi) {  // finish cur (and any pair-less gaussians before gi)
          flush(cur, c0, c1);
          c0 = c1 = 0.f;
          ++cur;
        }
        const float* r = s_v[wl] + i * PP;
        c0 += r[lane];
        if (lane + 32 < P) c1 += r[lane + 32];
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
// of p.(v + lam Mf p)
template <int P>
__global__ void __launch_bounds__(256) k_gm_to_am(SlmBackArgs A) {
  __shared__ float t[32][P + 1];
  __shared__ double sm[32];
  const long long G = A.G;
  double dot = 0.0;
  for (long long g0 = (long long)blockIdx.x * 32; g0 < G; g0 += (long long)gridDim.x * 32) {
    const int ng = (int)min((long long)32, G - g0);
    __syncthreads();
    for (int i = threadIdx.x; i < ng * P; i += blockDim.x) t[i / P][i % P] = A.gm[(size_t)g0 * P + i];
    __syncthreads();
    for (int i = threadIdx.x; i < 32 * P; i += blockDim.x) {
      const int a = i >> 5, gl = i & 31;
      if (gl >= ng) continue;
      float v = A.scale * t[gl][a];
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
  if (A.dot_part) {
    double tt = block_sum_d(dot, sm);
    if (threadIdx.x == 0) A.dot_part[blockIdx.x] = tt;
  }
}

// ---------------------------------------------------------------------------
// C-ABI
// ---------------------------------------------------------------------------
extern "C" {

int slm_view_size() { return (int)sizeof(SlmView); }
int slm_tile_args_size() { return (int)sizeof(SlmTileArgs); }
int slm_back_args_size() { return (int)sizeof(SlmBackArgs); }
int slm_diag_tab_floats() { return DIAG_TAB; }

int slm_gauss_tab(const float* xs, long long G, float* gtab, cudaStream_t st) {
  if (G <= 0) return SLM_OK;
  k_gauss_tab<<<slm_blocks(G, 256, 1LL << 30), 256, 0, st>>>(xs, G, gtab);
  return slm_cuda_status();
}

int slm_gauss_tab_floats(void) { return GTAB; }

int slm_pair_tables(const float* xs, long long G, int sh_degree, const int* pair_gid, const uint32_t* pair_vm,
                    const SlmCamera* cams, int n_pairs, float* tab, const float* gtab, cudaStream_t st) {
  if (n_pairs <= 0) return SLM_OK;
  unsigned b = slm_blocks(n_pairs, 128, 1LL << 30);
  switch (sh_degree) {
    case 0: k_pair_tables<1><<<b, 128, 0, st>>>(xs, G, pair_gid, pair_vm, cams, n_pairs, tab, gtab); break;
    case 1: k_pair_tables<4><<<b, 128, 0, st>>>(xs, G, pair_gid, pair_vm, cams, n_pairs, tab, gtab); break;
    case 2: k_pair_tables<9><<<b, 128, 0, st>>>(xs, G, pair_gid, pair_vm, cams, n_pairs, tab, gtab); break;
    case 3: k_pair_tables<16><<<b, 128, 0, st>>>(xs, G, pair_gid, pair_vm, cams, n_pairs, tab, gtab); break;
    default: return SLM_ERR_ARG;
  }
  return slm_cuda_status();
}

int slm_fwd_args_size() { return (int)sizeof(SlmFwdArgs); }

int slm_pair_forward(const SlmFwdArgs* a, int sh_degree, cudaStream_t st) {
  if (a->n_pairs <= 0) return SLM_OK;
  if (!a->pm) return SLM_ERR_ARG;
  unsigned b = slm_blocks(a->n_pairs, 128, 1LL << 30);
  switch (sh_degree) {
    case 0: k_pair_m<1><<<b, 128, 0, st>>>(*a); break;
    case 1: k_pair_m<4><<<b, 128, 0, st>>>(*a); break;
    case 2: k_pair_m<9><<<b, 128, 0, st>>>(*a); break;
    case 3: k_pair_m<16><<<b, 128, 0, st>>>(*a); break;
    default: return SLM_ERR_ARG;
  }
  return slm_cuda_status();
}

int slm_pair_sum(const int* pair_run_off, const int* pair_runs, int n_pairs, const float* run_acc, int d,
                 float* pacc, cudaStream_t st) {
  if (n_pairs <= 0) return SLM_OK;
  unsigned b = slm_blocks(n_pairs, 256, 1LL << 30);
  if (d == 9) k_pair_sum<9><<<b, 256, 0, st>>>(pair_run_off, pair_runs, n_pairs, run_acc, pacc);
  else if (d == DIAG_RUN_D) k_pair_sum<DIAG_RUN_D><<<b, 256, 0, st>>>(pair_run_off, pair_runs, n_pairs, run_acc, pacc);
  else return SLM_ERR_ARG;
  return slm_cuda_status();
}

int slm_backward_blocks(long long G) { return (int)slm_blocks(G, 128, 148LL * 16); }

int slm_warp_bounds(const int* gpo, long long G, int n_pairs, int* warp_g0, cudaStream_t st) {
  const int n_warps = (n_pairs >> 5) + 1;
  k_warp_bounds<<<slm_blocks(G + 1, 256), 256, 0, st>>>(gpo, G, n_warps, warp_g0);
  return slm_cuda_status();
}

int slm_pair_backward(const SlmBackArgs* a, int mode, int sh_degree, cudaStream_t st) {
  unsigned b = (unsigned)slm_backward_blocks(a->G);
  if (a->warp_g0) {  // packed: warp per 32-pair window of gaussians
    const int nw = (int)((a->n_pairs >> 5) + 1);
#define SLM_PK(KK)                                                                         \
  if (mode == 0)                                                                           \
    k_gauss_backward_packed<KK, 0><<<b, 32 * PK_WARPS, 0, st>>>(*a, a->warp_g0, nw);       \
  else                                                                                     \
    k_gauss_backward_packed<KK, 1><<<b, 32 * PK_WARPS, 0, st>>>(*a, a->warp_g0, nw);       \
  k_gm_to_am<11 + 3 * KK><<<b, 256, 0, st>>>(*a);
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
#define SLM_BW(KK)                                  \
  if (mode == 0)                                    \
    k_gauss_backward<KK, 0><<<b, 128, 0, st>>>(*a); \
  else                                              \
    k_gauss_backward<KK, 1><<<b, 128, 0, st>>>(*a);
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
