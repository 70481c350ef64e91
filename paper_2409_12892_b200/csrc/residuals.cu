// Residual weights for one view: sqrt-L1 + sqrt-(1-SSIM) residuals, the
// per-slot weight grad_r_sq = (dr/dc)^2 summed over both terms, and
// color_grad = sum_terms r * dr/dc (ref: residuals.py:249-296, center-pixel
// SSIM gradient ref: residuals.py:143-159, reflect padding ref: 58-91).
//
// fp64 throughout; two separable passes over five statistics x 3 channels.
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

// horizontal pass: tmp[p*15 + s*3 + c] for statistics s = x, y, xx, yy, xy
__global__ void k_ssim_h(ResidArgs A) {
  long long n = (long long)A.W * A.H;
  int half = A.win / 2;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
    int y = (int)(p / A.W), x = (int)(p % A.W);
    double acc[15];
#pragma unroll
    for (int s = 0; s < 15; ++s) acc[s] = 0.0;
    for (int j = 0; j < A.win; ++j) {
      int xx = reflect_idx(x + j - half, A.W);
      size_t q = ((size_t)y * A.W + xx) * 3;
      double w = A.taps[j];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double a = A.img[q + c], b = gt_at(A, q + c);
        acc[0 + c] += w * a;
        acc[3 + c] += w * b;
        acc[6 + c] += w * (a * a);
        acc[9 + c] += w * (b * b);
        acc[12 + c] += w * (a * b);
      }
    }
#pragma unroll
    for (int s = 0; s < 15; ++s) A.tmp[(size_t)p * 15 + s] = acc[s];
  }
}

__global__ void k_ssim_v(ResidArgs A) {
  __shared__ double sm[32];
  long long n = (long long)A.W * A.H;
  int half = A.win / 2;
  double e_acc = 0.0;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
    int y = (int)(p / A.W), x = (int)(p % A.W);
    double st[15];
#pragma unroll
    for (int s = 0; s < 15; ++s) st[s] = 0.0;
    if (A.mode == 0 && A.lambda2 > 0.0) {
      for (int j = 0; j < A.win; ++j) {
        int yy = reflect_idx(y + j - half, A.H);
        const double* t = A.tmp + ((size_t)yy * A.W + x) * 15;
        double w = A.taps[j];
#pragma unroll
        for (int s = 0; s < 15; ++s) st[s] += w * t[s];
      }
    }
    double cw = A.cw_y[y] * A.cw_x[x];
    float gr[3], cg[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      size_t i = (size_t)p * 3 + c;
      double im = A.img[i], g = gt_at(A, i);
      double e = im - g;
      double grad, cgrad, rabs, rssim = 0.0, drabs, drssim = 0.0;
      if (A.mode == 1) {
        grad = 1.0; cgrad = e; rabs = e; drabs = 1.0;
        e_acc += e * e;
      } else {
        double ae = fabs(e);
        rabs = sqrt(A.lambda1 * ae);
        double w1 = 0.0;
        drabs = 0.0;
        if (A.lambda1 > 0.0) {
          double ge = ae > A.eps_den ? ae : A.eps_den;
          double sg = e > 0.0 ? 1.0 : (e < 0.0 ? -1.0 : 0.0);
          drabs = A.lambda1 * sg / (2.0 * sqrt(A.lambda1 * ge));
          w1 = A.lambda1 / (4.0 * ge);
        }
        double w2 = 0.0;
        if (A.lambda2 > 0.0) {
          double mx = st[0 + c], my = st[3 + c];
          double sxx = st[6 + c] - mx * mx, syy = st[9 + c] - my * my, sxy = st[12 + c] - mx * my;
          double a1 = 2.0 * mx * my + A.ssim_c1, a2 = 2.0 * sxy + A.ssim_c2;
          double b1 = mx * mx + my * my + A.ssim_c1, b2 = sxx + syy + A.ssim_c2;
          double score = (a1 * a2) / (b1 * b2);
          double dsc = (2.0 * cw / (b1 * b2)) * (my * a2 + a1 * (g - my)) -
                       score * 2.0 * cw * (mx / b1 + (im - mx) / b2);
          double om = 1.0 - score;
          om = om > 0.0 ? om : 0.0;
          rssim = sqrt(A.lambda2 * om);
          double go = om > A.eps_den ? om : A.eps_den;
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
    A.gradr[p] = make_float4(gr[0], gr[1], gr[2], 0.f);
    A.cgrad[p] = make_float4(cg[0], cg[1], cg[2], 0.f);
  }
  double tot = block_sum_d(e_acc, sm);
  if (threadIdx.x == 0) A.energy_part[blockIdx.x] = tot;
}

extern "C" {

int slm_resid_args_size() { return (int)sizeof(ResidArgs); }

// Runs both passes; energy_part must hold `blocks` doubles where blocks is
// returned through *n_blocks (caller sums them on device or host).
int slm_residuals(const ResidArgs* a, int blocks, cudaStream_t stream) {
  if (a->win > SSIM_WIN_MAX || a->win % 2 != 1) return SLM_ERR_ARG;
  long long n = (long long)a->W * a->H;
  if (a->mode == 0 && a->lambda2 > 0.0) k_ssim_h<<<slm_blocks(n, 256), 256, 0, stream>>>(*a);
  k_ssim_v<<<blocks, 256, 0, stream>>>(*a);
  return slm_cuda_status();
}

}  // extern "C"
