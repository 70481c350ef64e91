// Residual weights for one view: sqrt-L1 + sqrt-(1-SSIM) residuals, the
// per-slot weight grad_r_sq = (dr/dc)^2 summed over both terms, and
// color_grad = sum_terms r * dr/dc (ref: residuals.py:249-296, center-pixel
// SSIM gradient ref: residuals.py:143-159, reflect padding ref: 58-91).
//
// fp64 throughout; separable 2-D window over five statistics x 3 channels,
// fused into one tiled kernel (no global scratch).
#include "slm_common.cuh"

#define SSIM_WIN_MAX 31

typedef SlmResidArgs ResidArgs;

__device__ __forceinline__ int reflect_idx(int i, int n) {
  int p = 2 * n;
  i %= p;
  if (i < 0) i += p;
  return i >= n ? p - 1 - i : i;
}

__device__ __forceinline__ double gt_at(const ResidArgs& A, size_t i) {
  return A.gt_f32 ? (double)((const float*)A.gt)[i] : ((const double*)A.gt)[i];
}

// One kernel, 16x16 output pixels per CTA (grid-stride over tiles).  Per
// tile the (16 + win - 1)^2 reflect-padded window of the rendered and the
// ground-truth image (3 channels) is staged in shared memory; per channel the
// horizontal pass writes five statistics per (window row, output column) to
// shared memory and each thread finishes its pixel's vertical pass.  Taps are summed in
// ascending order in both passes (the order of the reference's separable
// correlate1d, residuals.py:58-91).
#define RT 16

// WIN > 0: the window size as a compile-time constant (the tap loops unroll;
// 11 is the reference's default, residuals.py); WIN = 0: A.win at run time
template <int WIN>
__global__ void __launch_bounds__(256, 4) k_residuals(ResidArgs A) {
  extern __shared__ double sm[];
  __shared__ double red[32];
  __shared__ double taps[SSIM_WIN_MAX];
  const int win = WIN > 0 ? WIN : A.win;
  const int half = win / 2, IW = RT + 2 * half;
  double* s_a = sm;
  double* s_b = s_a + 3 * IW * IW;
  double* s_h = s_b + 3 * IW * IW;
  const bool ssim = A.mode == 0 && A.lambda2 > 0.0;
  if (threadIdx.x < win) taps[threadIdx.x] = A.taps[threadIdx.x];
  const int tx = threadIdx.x & (RT - 1), ty = threadIdx.x / RT;
  const int ntx = (A.W + RT - 1) / RT, nty = (A.H + RT - 1) / RT;
  double e_acc = 0.0;
  for (int t = blockIdx.x; t < ntx * nty; t += gridDim.x) {
    const int x0 = (t % ntx) * RT, y0 = (t / ntx) * RT;
    const int x = x0 + tx, y = y0 + ty;
    const bool inside = x < A.W && y < A.H;
    const size_t p = inside ? (size_t)y * A.W + x : 0;
    const double cw = inside ? A.cw_y[y] * A.cw_x[x] : 0.0;
    float gr[3], cg[3];
    if (ssim) {
      __syncthreads();  // previous tile done with the buffers
      for (int i = threadIdx.x; i < IW * IW; i += blockDim.x) {
        const int iy = i / IW, ix = i - iy * IW;
        const int gy = reflect_idx(y0 + iy - half, A.H), gx = reflect_idx(x0 + ix - half, A.W);
        const size_t q = ((size_t)gy * A.W + gx) * 3;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          s_a[c * IW * IW + i] = A.img[q + c];
          s_b[c * IW * IW + i] = gt_at(A, q + c);
        }
      }
    }
#pragma unroll 1
    for (int c = 0; c < 3; ++c) {
      double st[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
      if (ssim) {
        __syncthreads();  // window staged / previous channel's s_h consumed
        for (int i = threadIdx.x; i < IW * RT; i += blockDim.x) {
          const int iy = i / RT, ix = i - iy * RT;
          const double* ra = s_a + c * IW * IW + iy * IW + ix;
          const double* rb = s_b + c * IW * IW + iy * IW + ix;
          double h0 = 0.0, h1 = 0.0, h2 = 0.0, h3 = 0.0, h4 = 0.0;
#pragma unroll
          for (int j = 0; j < win; ++j) {
            const double w = taps[j], a = ra[j], b = rb[j];
            h0 += w * a;
            h1 += w * b;
            h2 += w * (a * a);
            h3 += w * (b * b);
            h4 += w * (a * b);
          }
          double* o = s_h + (size_t)i * 5;
          o[0] = h0; o[1] = h1; o[2] = h2; o[3] = h3; o[4] = h4;
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < win; ++j) {
          const double w = taps[j];
          const double* hh = s_h + ((ty + j) * RT + tx) * 5;
#pragma unroll
          for (int k = 0; k < 5; ++k) st[k] += w * hh[k];
        }
      }
      if (!inside) continue;
      const size_t i = p * 3 + c;
      const double im = A.img[i], g = gt_at(A, i);
      const double e = im - g;
      double grad, cgrad, rabs, rssim = 0.0, drabs, drssim = 0.0;
      if (A.mode == 1) {
        grad = 1.0; cgrad = e; rabs = e; drabs = 1.0;
        e_acc += e * e;
      } else {
        const double ae = fabs(e);
        rabs = sqrt(A.lambda1 * ae);
        double w1 = 0.0;
        drabs = 0.0;
        if (A.lambda1 > 0.0) {
          const double ge = ae > A.eps_den ? ae : A.eps_den;
          const double sg = e > 0.0 ? 1.0 : (e < 0.0 ? -1.0 : 0.0);
          drabs = A.lambda1 * sg / (2.0 * sqrt(A.lambda1 * ge));
          w1 = A.lambda1 / (4.0 * ge);
        }
        double w2 = 0.0;
        if (ssim) {
          const double mx = st[0], my = st[1];
          const double sxx = st[2] - mx * mx, syy = st[3] - my * my, sxy = st[4] - mx * my;
          const double a1 = 2.0 * mx * my + A.ssim_c1, a2 = 2.0 * sxy + A.ssim_c2;
          const double b1 = mx * mx + my * my + A.ssim_c1, b2 = sxx + syy + A.ssim_c2;
          const double score = (a1 * a2) / (b1 * b2);
          const double dsc = (2.0 * cw / (b1 * b2)) * (my * a2 + a1 * (g - my)) -
                             score * 2.0 * cw * (mx / b1 + (im - mx) / b2);
          double om = 1.0 - score;
          om = om > 0.0 ? om : 0.0;
          rssim = sqrt(A.lambda2 * om);
          const double go = om > A.eps_den ? om : A.eps_den;
          drssim = -A.lambda2 * dsc / (2.0 * sqrt(A.lambda2 * go));
          w2 = A.lambda2 * dsc * dsc / (4.0 * go);
        }
        grad = w1 + w2;
        cgrad = drabs * rabs + drssim * rssim;
        e_acc += rabs * rabs + rssim * rssim;
      }
      gr[c] = (float)grad;
      cg[c] = (float)cgrad;
      if (A.o_gradr) {
        A.o_gradr[i] = grad; A.o_cgrad[i] = cgrad; A.o_rabs[i] = rabs; A.o_drabs[i] = drabs;
        if (A.o_rssim) { A.o_rssim[i] = rssim; A.o_drssim[i] = drssim; }
      }
    }
    if (inside) {
      A.gradr[p] = make_float4(gr[0], gr[1], gr[2], 0.f);
      A.cgrad[p] = make_float4(cg[0], cg[1], cg[2], 0.f);
    }
  }
  const double tot = block_sum_d(e_acc, red);
  if (threadIdx.x == 0) A.energy_part[blockIdx.x] = tot;
}

extern "C" {

int slm_resid_args_size() { return (int)sizeof(ResidArgs); }

// Runs both passes; energy_part must hold `blocks` doubles where blocks is
// returned through *n_blocks (caller sums them on device or host).
int slm_residuals(const ResidArgs* a, int blocks, cudaStream_t stream) {
  if (a->win > SSIM_WIN_MAX || a->win % 2 != 1 || blocks <= 0) return SLM_ERR_ARG;
  const int IW = RT + 2 * (a->win / 2);
  const size_t smem = (a->mode == 0 && a->lambda2 > 0.0) ? ((size_t)6 * IW * IW + (size_t)IW * RT * 5) * 8 : 0;
  // opt-in above the 48 KB default (static + dynamic), per device and kernel
  constexpr int kMaxDev = 64;
  static size_t smem_set[kMaxDev][2] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  const int w = a->win == 11 ? 1 : 0;
  if (dev < kMaxDev && smem > smem_set[dev][w]) {
    if (w) cudaFuncSetAttribute(k_residuals<11>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    else cudaFuncSetAttribute(k_residuals<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    smem_set[dev][w] = smem;
  }
  if (w) k_residuals<11><<<blocks, 256, smem, stream>>>(*a);
  else k_residuals<0><<<blocks, 256, smem, stream>>>(*a);
  return slm_cuda_status();
}

}  // extern "C"
