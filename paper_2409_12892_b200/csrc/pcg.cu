// PCG vector kernels (Alg. 1), the Eq. 7
// weighted-mean combine and the sortX layout
// permutation (ref: scene.py:79-92).
//
// Scalars (r^T z, p^T g, alpha, beta, ...) live in a device fp64 state block;
// every reduction is a fixed-shape fp64 tree, so the solver is bitwise
// deterministic and needs one 8-byte host read per iteration (exit test).
#include "slm_common.cuh"

#include <algorithm>

// state layout (double[16])
#define ST_RZ 0
#define ST_PG 2
#define ST_BB 3
#define ST_RR 4
#define ST_ALPHA 5
#define ST_BETA 6
#define ST_FLAGS 7   // bit0 non-SPD (p^T g <= 0), bit1 converged
#define ST_ITERS 8
#define ST_STOP 9    // sticky: the solve has ended (b = 0, converged or non-SPD); the
                     // iteration kernels become no-ops, so the host can queue
                     // iterations ahead without a per-iteration sync

#define VEC_BLOCKS 1184  // 148 SMs x 8, fixed -> deterministic partial shapes
#define VEC_THREADS 256

__device__ __forceinline__ float mfloor(float m) { return fmaxf(m, 1e-12f); }

#ifndef SLM_P_UNROLL
#define SLM_P_UNROLL 3
#endif
#ifndef SLM_UPD_UNROLL
#define SLM_UPD_UNROLL 1
#endif
// loop unrolls of the tile loops of k_pcg_p (more independent loads in
// flight: 0.557 -> 0.453 ms per launch at C3 with 3) and of k_pcg_update
constexpr int kPUnroll = SLM_P_UNROLL, kUpdUnroll = SLM_UPD_UNROLL;

// padded gaussian-major stride of the forward chain's copy of p (16-byte
// rows): P values, pad, then (with the chain rows) the 6 entries of the
// world-covariance perturbation dSigma at GM_DSIG
__host__ __device__ constexpr int gm_stride(int P) { return ((P + 3) & ~3) + 8; }
#define GM_DSIG(P) (((P) + 3) & ~3)

// p = r / Mf + beta * p  (INIT: p = x0 = b / Mf, Alg. 1 line 4), r fp64; p is
// stored fp32 and used consistently as the search direction by the product,
// x += alpha p and r -= alpha A p.  Tiles of 32 gaussians: attribute-major
// reads / writes coalesced over gaussians, and (p_gm != NULL) the tile is
// transposed in shared memory to the padded gaussian-major rows the forward
// chain loads with 16-byte loads.
//
// With the cache's per-gaussian chain rows (gtab, stride gts: Rg 9 | s2 3 |
// Mq 36 at 0 / 9 / 12) each gaussian's row also gets the world-covariance
// perturbation of p's rotation / scale block,
//   dSigma = sum_l p_q,l (Mq_l S^2 Rg^T + (.)^T) + sum_i 2 s_i^2 p_s,i r_i r_i^T
// (upper triangle), so the per-pair forward chain only maps it to the image
// plane (U dSigma U^T) instead of chaining every rotation / scale column.
#define P_INIT 0
#define P_UPDATE 1
#define P_COPY 2   // p_gm (+ dSigma) of a given attribute-major p, p untouched
template <int MODE>
__global__ void __launch_bounds__(256) k_pcg_p(float* __restrict__ p, float* __restrict__ p_gm,
                                               const double* __restrict__ r, const float* __restrict__ b,
                                               const float* __restrict__ M, const double* __restrict__ st,
                                               long long G, int P, const float* __restrict__ gtab, int gts) {
  if (MODE == P_UPDATE && st[ST_STOP] != 0.0) return;
  extern __shared__ float tile[];  // [32][PG + 1]
  const double beta = MODE == P_UPDATE ? st[ST_BETA] : 0.0;
  const int PG = gm_stride(P), TS = PG + 1;
  for (long long g0 = (long long)blockIdx.x * 32; g0 < G; g0 += (long long)gridDim.x * 32) {
    const int ng = (int)min((long long)32, G - g0);
    __syncthreads();
#pragma unroll(kPUnroll)
    for (int i = threadIdx.x; i < 32 * PG; i += blockDim.x) {
      const int a = i >> 5, gl = i & 31;
      float v = 0.f;
      if (a < P && gl < ng) {
        const long long idx = (long long)a * G + g0 + gl;
        if (MODE == P_COPY) {
          v = p[idx];
        } else {
          v = MODE == P_INIT ? (float)((double)b[idx] / (double)mfloor(M[idx]))
                             : (float)(r[idx] / (double)mfloor(M[idx]) + beta * (double)p[idx]);
          p[idx] = v;
        }
      }
      tile[gl * TS + a] = v;
    }
    if (!p_gm) continue;
    __syncthreads();
    if (gtab && (int)threadIdx.x < ng) {
      float* row = tile + threadIdx.x * TS;
      // the chain row's first 48 floats (Rg | s2 | Mq) as 12 16-byte loads
      const float4* gt4 = reinterpret_cast<const float4*>(gtab + (size_t)(g0 + threadIdx.x) * gts);
      float gt[48];
#pragma unroll
      for (int k = 0; k < 12; ++k) {
        const float4 v = __ldg(gt4 + k);
        gt[4 * k] = v.x;
        gt[4 * k + 1] = v.y;
        gt[4 * k + 2] = v.z;
        gt[4 * k + 3] = v.w;
      }
      float Rg[9], s2[3], Mp[9];
#pragma unroll
      for (int i = 0; i < 9; ++i) Rg[i] = gt[i];
#pragma unroll
      for (int i = 0; i < 3; ++i) s2[i] = gt[9 + i];
#pragma unroll
      for (int i = 0; i < 9; ++i)
        Mp[i] = row[3] * gt[12 + i] + row[4] * gt[21 + i] + row[5] * gt[30 + i] + row[6] * gt[39 + i];
      float W[9];  // Mp S^2 Rg^T
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
          W[i * 3 + j] = Mp[i * 3] * s2[0] * Rg[j * 3] + Mp[i * 3 + 1] * s2[1] * Rg[j * 3 + 1] +
                         Mp[i * 3 + 2] * s2[2] * Rg[j * 3 + 2];
      const float cs[3] = {2.f * s2[0] * row[7], 2.f * s2[1] * row[8], 2.f * s2[2] * row[9]};
      int k = 0;
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = i; j < 3; ++j, ++k)
          row[GM_DSIG(P) + k] = W[i * 3 + j] + W[j * 3 + i] + cs[0] * Rg[i * 3] * Rg[j * 3] +
                                cs[1] * Rg[i * 3 + 1] * Rg[j * 3 + 1] + cs[2] * Rg[i * 3 + 2] * Rg[j * 3 + 2];
    }
    __syncthreads();
#pragma unroll(kPUnroll)
    for (int i = threadIdx.x; i < ng * PG; i += blockDim.x) p_gm[g0 * PG + i] = tile[(i / PG) * TS + i % PG];
  }
}

// sum of a block-partials array in a fixed order (every block gets the same bits)
__device__ double sum_parts(const double* __restrict__ part, int n, double* sm) {
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += part[i];
  double t = block_sum_d(s, sm);
  __shared__ double bc;
  if (threadIdx.x == 0) bc = t;
  __syncthreads();
  return bc;
}

// A p = g + lam * Mf * p with g = J^T W J p from the product kernels; the
// lam term is added here in fp64 because x0 = b / Mf makes |A x0| >> |b| and
// the residual recurrence would otherwise cancel in fp32 (large lam).
// INIT (mode 0): x = p (= x0), r = b - A p;   partials: r.r/Mf, r.r, b.b
// STEP (mode 1): alpha = rz / pg; x += alpha p; r -= alpha A p; partials r.r/Mf, r.r
__global__ void k_pcg_update(int mode, double* __restrict__ x, double* __restrict__ r, const float* __restrict__ p,
                             const float* __restrict__ g, const float* __restrict__ b, const float* __restrict__ M,
                             double lam, double* __restrict__ st, const double* __restrict__ dot_part, int n_dot,
                             double* __restrict__ part /*[3][VEC_BLOCKS]*/, long long n) {
  __shared__ double sm[32];
  if (mode == 1 && st[ST_STOP] != 0.0) return;
  double alpha = 0.0;
  if (mode == 1) {
    double pg = sum_parts(dot_part, n_dot, sm);
    alpha = st[ST_RZ] / pg;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      st[ST_PG] = pg;
      st[ST_ALPHA] = alpha;
    }
  }
  double s_rz = 0.0, s_rr = 0.0, s_bb = 0.0;
#pragma unroll(kUpdUnroll)
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double mf = (double)mfloor(M[i]);
    const double pi = (double)p[i];
    const double ap = (double)g[i] + lam * mf * pi;
    double ri;
    if (mode == 0) {
      x[i] = pi;
      const double bi = (double)b[i];
      ri = bi - ap;
      s_bb += bi * bi;
    } else {
      x[i] += alpha * pi;
      ri = r[i] - alpha * ap;
    }
    r[i] = ri;
    s_rz += ri * ri / mf;
    s_rr += ri * ri;
  }
  double t;
  t = block_sum_d(s_rz, sm);
  if (threadIdx.x == 0) part[blockIdx.x] = t;
  t = block_sum_d(s_rr, sm);
  if (threadIdx.x == 0) part[VEC_BLOCKS + blockIdx.x] = t;
  if (mode == 0) {
    t = block_sum_d(s_bb, sm);
    if (threadIdx.x == 0) part[2 * VEC_BLOCKS + blockIdx.x] = t;
  }
}

// single block: beta = rz_new / rz, exit flags
__global__ void k_pcg_finalize(int mode, double* __restrict__ st, const double* __restrict__ part, int nb) {
  __shared__ double sm[32];
  if (mode == 1 && st[ST_STOP] != 0.0) return;
  double rz = sum_parts(part, nb, sm);
  double rr = sum_parts(part + VEC_BLOCKS, nb, sm);
  double bb = mode == 0 ? sum_parts(part + 2 * VEC_BLOCKS, nb, sm) : 0.0;
  if (threadIdx.x == 0) {
    double flags = 0.0;
    if (mode == 0) {
      st[ST_BB] = bb;
      st[ST_BETA] = 0.0;
      st[ST_ITERS] = 0.0;
      st[ST_STOP] = bb > 0.0 ? 0.0 : 1.0;  // b = 0: x = x0
    } else {
      double pg = st[ST_PG];
      if (!(pg > 0.0)) flags = 1.0;
      st[ST_BETA] = rz / st[ST_RZ];
      st[ST_ITERS] += 1.0;
      if (flags == 0.0 && rr < 0.01 * st[ST_BB]) flags = 2.0;
    }
    st[ST_RZ] = rz;
    st[ST_RR] = rr;
    st[ST_FLAGS] = flags;
    if (flags != 0.0) st[ST_STOP] = 1.0;
  }
}

// Eq. 7 in fp64: num += M * delta, den += M;  finalize delta = num / max(den, 1e-12)
__global__ void k_combine_acc(double* __restrict__ num, double* __restrict__ den, const double* __restrict__ delta,
                              const float* __restrict__ M, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double m = (double)M[i];
    num[i] += m * delta[i];
    den[i] += m;
  }
}

__global__ void k_combine_fin(float* __restrict__ out, const double* __restrict__ num, const double* __restrict__ den,
                              long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = (float)(num[i] / fmax(den[i], 1e-12));
}

// (rows x cols) -> (cols x rows) tiled transpose; sortX is the transpose of
// the P x G attribute-major matrix (ref: scene.py:79-92)
template <typename T>
__global__ void k_transpose(const T* __restrict__ in, T* __restrict__ out, long long rows, long long cols) {
  __shared__ T tile[32][33];
  long long c0 = (long long)blockIdx.x * 32, r0 = (long long)blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    long long r = r0 + k, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[k][threadIdx.x] = in[r * cols + c];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    long long c = c0 + k, r = r0 + threadIdx.x;
    if (r < rows && c < cols) out[c * rows + r] = tile[threadIdx.x][k];
  }
}

__global__ void k_f64_to_f32(const double* __restrict__ in, float* __restrict__ out, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = (float)in[i];
}

// x_out = x + gamma * delta (fp64 scene, fp32 direction) -- line search / step
__global__ void k_axpy_scene(const double* __restrict__ x, const float* __restrict__ d, double gamma,
                             double* __restrict__ out, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = x[i] + gamma * (double)d[i];
}

extern "C" {

int slm_vec_blocks() { return VEC_BLOCKS; }

int slm_gm_stride(int P) { return gm_stride(P); }

static unsigned p_blocks(long long G) { return (unsigned)std::min<long long>((G + 31) / 32, 1LL << 30); }  // one 32-gaussian tile per block

int slm_pcg_pinit(float* p, float* p_gm, const float* b, const float* M, long long G, int P, const float* gtab,
                  int gtab_stride, cudaStream_t s) {
  if (G <= 0) return SLM_OK;
  if (gtab && gtab_stride % 4) return SLM_ERR_ARG;  // 16-byte chain-row loads
  const size_t sm = (size_t)32 * (gm_stride(P) + 1) * sizeof(float);
  k_pcg_p<P_INIT><<<p_blocks(G), 256, sm, s>>>(p, p_gm, nullptr, b, M, nullptr, G, P, gtab, gtab_stride);
  return slm_cuda_status();
}

int slm_pcg_pupdate(float* p, float* p_gm, const double* r, const float* M, const double* st, long long G, int P,
                    const float* gtab, int gtab_stride, cudaStream_t s) {
  if (G <= 0) return SLM_OK;
  if (gtab && gtab_stride % 4) return SLM_ERR_ARG;  // 16-byte chain-row loads
  const size_t sm = (size_t)32 * (gm_stride(P) + 1) * sizeof(float);
  k_pcg_p<P_UPDATE><<<p_blocks(G), 256, sm, s>>>(p, p_gm, r, nullptr, M, st, G, P, gtab, gtab_stride);
  return slm_cuda_status();
}

int slm_gm_pack(const float* p, float* p_gm, long long G, int P, const float* gtab, int gtab_stride, cudaStream_t s) {
  if (G <= 0) return SLM_OK;
  if (gtab && gtab_stride % 4) return SLM_ERR_ARG;  // 16-byte chain-row loads
  const size_t sm = (size_t)32 * (gm_stride(P) + 1) * sizeof(float);
  k_pcg_p<P_COPY><<<p_blocks(G), 256, sm, s>>>(const_cast<float*>(p), p_gm, nullptr, nullptr, nullptr, nullptr, G, P,
                                               gtab, gtab_stride);
  return slm_cuda_status();
}

int slm_pcg_update(int mode, double* x, double* r, const float* p, const float* g, const float* b, const float* M,
                   double lam, double* st, const double* dot_part, int n_dot, double* part, long long n,
                   cudaStream_t s) {
  k_pcg_update<<<VEC_BLOCKS, VEC_THREADS, 0, s>>>(mode, x, r, p, g, b, M, lam, st, dot_part, n_dot, part, n);
  return slm_cuda_status();
}

int slm_pcg_finalize(int mode, double* st, const double* part, cudaStream_t s) {
  k_pcg_finalize<<<1, 1024, 0, s>>>(mode, st, part, VEC_BLOCKS);
  return slm_cuda_status();
}

int slm_combine_acc(double* num, double* den, const double* delta, const float* M, long long n, cudaStream_t s) {
  k_combine_acc<<<VEC_BLOCKS, VEC_THREADS, 0, s>>>(num, den, delta, M, n);
  return slm_cuda_status();
}

int slm_combine_fin(float* out, const double* num, const double* den, long long n, cudaStream_t s) {
  k_combine_fin<<<VEC_BLOCKS, VEC_THREADS, 0, s>>>(out, num, den, n);
  return slm_cuda_status();
}

int slm_transpose_f32(const float* in, float* out, long long rows, long long cols, cudaStream_t s) {
  if (rows <= 0 || cols <= 0) return SLM_OK;
  dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
  if (grid.y > 65535) return SLM_ERR_SIZE;
  k_transpose<float><<<grid, dim3(32, 8), 0, s>>>(in, out, rows, cols);
  return slm_cuda_status();
}

int slm_transpose_f64(const double* in, double* out, long long rows, long long cols, cudaStream_t s) {
  if (rows <= 0 || cols <= 0) return SLM_OK;
  dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
  if (grid.y > 65535) return SLM_ERR_SIZE;
  k_transpose<double><<<grid, dim3(32, 8), 0, s>>>(in, out, rows, cols);
  return slm_cuda_status();
}

int slm_f64_to_f32(const double* in, float* out, long long n, cudaStream_t s) {
  k_f64_to_f32<<<VEC_BLOCKS, VEC_THREADS, 0, s>>>(in, out, n);
  return slm_cuda_status();
}

int slm_axpy_scene(const double* x, const float* d, double gamma, double* out, long long n, cudaStream_t s) {
  k_axpy_scene<<<VEC_BLOCKS, VEC_THREADS, 0, s>>>(x, d, gamma, out, n);
  return slm_cuda_status();
}

}  // extern "C"
