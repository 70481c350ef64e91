// fp64 projection, depth order, tile binning and the two-pass tile rasteriser
// that emits the gradient cache (the forward half of buildCache_p1).
//
// Parity contract: every discrete decision (valid mask, bbox, (depth, gid)
// order, alpha >= alpha_min, T >= t_stop, alpha clamp) is taken in fp64 with
// the reference's operation order (ref: rasterizer.py:116-165, 253-316), so
// cache indexing matches the CPU reference bit for bit.
#include "slm_common.cuh"

#include <cub/cub.cuh>

// ---------------------------------------------------------------------------
// projection (ref: rasterizer.py:78-165)
// ---------------------------------------------------------------------------
// view-independent part of the projection of one gaussian (finiteness, the
// world covariance R diag(s^2) R^T and the opacity), computed once per
// gaussian and reused for every view of a subset (same fp64 operations, so
// the per-view results are bit-identical to computing it per view)
struct GaussPre {
  double p0, p1, p2;
  double Sw[9];
  double o;
  bool finite;
};

template <int K>
__device__ __forceinline__ GaussPre gauss_pre(const double* __restrict__ x, long long G, long long g,
                                              int* __restrict__ err) {
  GaussPre P;
  P.p0 = x[g];
  P.p1 = x[G + g];
  P.p2 = x[2 * G + g];
  double qw = x[3 * G + g], qx = x[4 * G + g], qy = x[5 * G + g], qz = x[6 * G + g];
  double l0 = x[7 * G + g], l1 = x[8 * G + g], l2 = x[9 * G + g];
  double logit = x[10 * G + g];
  bool finite = isfinite(P.p0) && isfinite(P.p1) && isfinite(P.p2) && isfinite(qw) && isfinite(qx) &&
                isfinite(qy) && isfinite(qz) && isfinite(l0) && isfinite(l1) && isfinite(l2) && isfinite(logit);
  for (int a = 11; a < 11 + 3 * K; ++a) finite = finite && isfinite(x[(long long)a * G + g]);
  if (!finite) atomicOr(err, 1);
  P.finite = finite;
  double qn = sqrt(qw * qw + qx * qx + qy * qy + qz * qz);
  if (qn < 1e-12) atomicOr(err, 2);
  double w = qw / qn, a = qx / qn, b = qy / qn, c = qz / qn;
  double Rg[9] = {1 - 2 * (b * b + c * c), 2 * (a * b - w * c), 2 * (a * c + w * b),
                  2 * (a * b + w * c), 1 - 2 * (a * a + c * c), 2 * (b * c - w * a),
                  2 * (a * c - w * b), 2 * (b * c + w * a), 1 - 2 * (a * a + b * b)};
  double s2[3] = {exp(2.0 * l0), exp(2.0 * l1), exp(2.0 * l2)};
  // world covariance R diag(s^2) R^T
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int k = 0; k < 3; ++k)
      P.Sw[i * 3 + k] = Rg[i * 3 + 0] * s2[0] * Rg[k * 3 + 0] + Rg[i * 3 + 1] * s2[1] * Rg[k * 3 + 1] +
                        Rg[i * 3 + 2] * s2[2] * Rg[k * 3 + 2];
  P.o = 1.0 / (1.0 + exp(-logit));
  return P;
}

// the per-view part (ref: rasterizer.py:116-165)
template <int K>
__device__ __forceinline__ void preprocess_view(const GaussPre& P, const double* __restrict__ x, long long G,
                                                long long g, const SlmCamera& cam, const SlmRastCfg& cfg,
                                                SlmSplat& s_out, unsigned long long& key_out) {
  const double p0 = P.p0, p1 = P.p1, p2 = P.p2;
  const double* Sw = P.Sw;
  const double* R = cam.R;
  // cam_points = positions @ R^T + t
  double X0 = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(p0, R[0]), __dmul_rn(p1, R[1])), __dmul_rn(p2, R[2])), cam.t[0]);
  double X1 = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(p0, R[3]), __dmul_rn(p1, R[4])), __dmul_rn(p2, R[5])), cam.t[1]);
  double X2 = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(p0, R[6]), __dmul_rn(p1, R[7])), __dmul_rn(p2, R[8])), cam.t[2]);
  bool valid = X2 > cfg.z_near;
  double zz = valid ? X2 : 1.0;
  double mx = __dadd_rn(__ddiv_rn(__dmul_rn(cam.fx, X0), zz), cam.cx);
  double my = __dadd_rn(__ddiv_rn(__dmul_rn(cam.fy, X1), zz), cam.cy);
  // camera covariance R Sw R^T
  double T1[9], Sc[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int k = 0; k < 3; ++k)
      T1[i * 3 + k] = R[i * 3 + 0] * Sw[0 * 3 + k] + R[i * 3 + 1] * Sw[1 * 3 + k] + R[i * 3 + 2] * Sw[2 * 3 + k];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int k = 0; k < 3; ++k)
      Sc[i * 3 + k] = T1[i * 3 + 0] * R[k * 3 + 0] + T1[i * 3 + 1] * R[k * 3 + 1] + T1[i * 3 + 2] * R[k * 3 + 2];
  double Xs0 = valid ? X0 : 0.0, Xs1 = valid ? X1 : 0.0, Xs2 = valid ? X2 : 1.0;
  double iz = 1.0 / Xs2;
  double A00 = cam.fx * iz, A02 = -cam.fx * Xs0 * iz * iz;
  double A11 = cam.fy * iz, A12 = -cam.fy * Xs1 * iz * iz;
  // cov2 = A Sc A^T (A has zeros at (0,1), (1,0))
  double r00 = A00 * Sc[0] + A02 * Sc[6], r01 = A00 * Sc[1] + A02 * Sc[7], r02 = A00 * Sc[2] + A02 * Sc[8];
  double r11 = A11 * Sc[4] + A12 * Sc[7], r12 = A11 * Sc[5] + A12 * Sc[8];
  double c00 = r00 * A00 + r02 * A02;
  double c01 = r01 * A11 + r02 * A12;
  double c11 = r11 * A11 + r12 * A12;
  double va = c00 + cfg.cov_eps, vb = c01, vc = c11 + cfg.cov_eps;
  double det = va * vc - vb * vb;
  valid = valid && (det > 0.0);
  double detu = det > 0.0 ? det : 1.0;
  double ca = vc / detu, cb = -vb / detu, cc = va / detu;

  // view-dependent colour
  double v0 = p0 - cam.C[0], v1 = p1 - cam.C[1], v2 = p2 - cam.C[2];
  double vn = sqrt(v0 * v0 + v1 * v1 + v2 * v2);
  double d0 = v0 / vn, d1 = v1 / vn, d2 = v2 / vn;
  double Y[16];
  sh_basis<double, K>(d0, d1, d2, Y);
  double col[3];
  unsigned clampbits = 0;
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    double raw = 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k) raw += x[(long long)(11 + ch * K + k) * G + g] * Y[k];
    raw += 0.5;
    col[ch] = raw > 0.0 ? raw : 0.0;
    if (raw <= 0.0) clampbits |= (1u << (1 + ch));
  }
  double lam = 0.5 * (va + vc) + sqrt(0.25 * (va - vc) * (va - vc) + vb * vb);
  if (cfg.cull_sigma > 0.0) {
    double rad = cfg.cull_sigma * sqrt(lam);
    valid = valid && (mx + rad > 0.0) && (mx - rad < (double)cam.W) && (my + rad > 0.0) &&
            (my - rad < (double)cam.H);
  }
  int x0 = 0, x1 = cam.W - 1, y0 = 0, y1 = cam.H - 1;
  if (cfg.reach_fac > 0.0) {
    double reach = cfg.reach_fac * sqrt(lam);
    double fx0 = ceil(mx - reach - 0.5), fx1 = floor(mx + reach - 0.5);
    double fy0 = ceil(my - reach - 0.5), fy1 = floor(my + reach - 0.5);
    x0 = fx0 > 0.0 ? (fx0 < 1e9 ? (int)fx0 : 1000000000) : 0;
    y0 = fy0 > 0.0 ? (fy0 < 1e9 ? (int)fy0 : 1000000000) : 0;
    x1 = fx1 < (double)(cam.W - 1) ? (fx1 > -1e9 ? (int)fx1 : -1000000000) : cam.W - 1;
    y1 = fy1 < (double)(cam.H - 1) ? (fy1 > -1e9 ? (int)fy1 : -1000000000) : cam.H - 1;
  }
  if (!P.finite) valid = false;
  SlmSplat s;
  s.mx = mx; s.my = my; s.ca = ca; s.cb = cb; s.cc = cc; s.o = P.o;
  s.c0 = col[0]; s.c1 = col[1]; s.c2 = col[2];
  s.x0 = x0; s.x1 = x1; s.y0 = y0; s.y1 = y1;
  s.flags = (valid ? SLM_FLAG_VALID : 0u) | clampbits;
  s.pad = 0;
  s_out = s;
  key_out = valid ? (unsigned long long)__double_as_longlong(X2) : ~0ull;
}

template <int K>
__global__ void k_preprocess(const double* __restrict__ x, long long G, SlmCamera cam, SlmRastCfg cfg,
                             SlmSplat* __restrict__ out, unsigned long long* __restrict__ depth_key,
                             uint32_t* __restrict__ order_val, int* __restrict__ err) {
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < G; g += (long long)gridDim.x * blockDim.x) {
    const GaussPre P = gauss_pre<K>(x, G, g, err);
    preprocess_view<K>(P, x, G, g, cam, cfg, out[g], depth_key[g]);
    order_val[g] = (uint32_t)g;
  }
}

// all views of a subset in one launch: thread per gaussian, the
// view-independent part once, then a loop over the views (the SH coefficients
// stay in L1 across views), element i = v * G + g, value (v << 24) | g
#ifndef SLM_PRE_MINB
#define SLM_PRE_MINB 4  // 128 registers: 2.71 -> 1.67 ms at C3 despite a small spill
#endif
template <int K>
__global__ void __launch_bounds__(128, SLM_PRE_MINB) k_preprocess_views(const double* __restrict__ x, long long G, const SlmCamera* __restrict__ cams,
                                   int V, SlmRastCfg cfg, SlmSplat* __restrict__ out,
                                   unsigned long long* __restrict__ depth_key, uint32_t* __restrict__ order_val,
                                   int* __restrict__ err) {
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < G; g += (long long)gridDim.x * blockDim.x) {
    const GaussPre P = gauss_pre<K>(x, G, g, err);  // once per gaussian
    for (int v = 0; v < V; ++v) {
      const long long i = (long long)v * G + g;
      preprocess_view<K>(P, x, G, g, cams[v], cfg, out[i], depth_key[i]);
      order_val[i] = ((uint32_t)v << 24) | (uint32_t)g;
    }
  }
}

// ---------------------------------------------------------------------------
// tile binning: instances (tile, depth rank) -> gid, sorted by tile then rank
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool splat_tiles(const SlmSplat& s, int tiles_x, int tiles_y, int& tx0, int& tx1,
                                            int& ty0, int& ty1) {
  if (!(s.flags & SLM_FLAG_VALID) || s.x0 > s.x1 || s.y0 > s.y1) return false;
  tx0 = s.x0 / SLM_TILE; tx1 = s.x1 / SLM_TILE;
  ty0 = s.y0 / SLM_TILE; ty1 = s.y1 / SLM_TILE;
  if (tx1 >= tiles_x) tx1 = tiles_x - 1;
  if (ty1 >= tiles_y) ty1 = tiles_y - 1;
  return tx0 <= tx1 && ty0 <= ty1;
}

__global__ void k_tile_count(const uint32_t* __restrict__ sorted_gid, const unsigned long long* __restrict__ sorted_key,
                             long long G, const SlmSplat* __restrict__ splats, int tiles_x, int tiles_y,
                             unsigned long long* __restrict__ n_inst) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (; i < G; i += (long long)gridDim.x * blockDim.x) {
    unsigned long long n = 0;
    if (sorted_key[i] != ~0ull) {
      int tx0, tx1, ty0, ty1;
      if (splat_tiles(splats[sorted_gid[i]], tiles_x, tiles_y, tx0, tx1, ty0, ty1))
        n = (unsigned long long)(tx1 - tx0 + 1) * (ty1 - ty0 + 1);
    }
    n_inst[i] = n;
  }
}

// instances are emitted per splat in (tile row, tile column) order with the
// key (tile, depth rank) -- unique per instance -- and the splat as the value,
// so after the key sort the values are each tile's splats in depth order
// Instances are emitted in depth-rank order (inst_off is the scan over the
// depth-sorted splats), so their key is the tile alone: a STABLE radix sort
// by tile leaves every tile's splats in depth order (17 key bits at C3
// instead of tile | rank = 37: 3 radix passes instead of 5, and 4-byte keys)
__global__ void k_tile_emit(const uint32_t* __restrict__ sorted_gid, const unsigned long long* __restrict__ inst_off,
                            long long G, const SlmSplat* __restrict__ splats, int tiles_x, int tiles_y,
                            uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (; i < G; i += (long long)gridDim.x * blockDim.x) {
    unsigned long long beg = inst_off[i], end = inst_off[i + 1];
    if (beg == end) continue;
    uint32_t g = sorted_gid[i];
    int tx0, tx1, ty0, ty1;
    splat_tiles(splats[g], tiles_x, tiles_y, tx0, tx1, ty0, ty1);
    unsigned long long k = beg;
    for (int ty = ty0; ty <= ty1; ++ty)
      for (int tx = tx0; tx <= tx1; ++tx) {
        keys[k] = (uint32_t)(ty * tiles_x + tx);
        vals[k] = g;  // the sort carries the splat itself
        ++k;
      }
  }
}

// ---- subset-batched binning (all views in one launch each) -----------------
// sorted element i (view-major, depth order within the view) carries
// sv = (v << 24) | g; its global splat index is v * G + g; tiles are numbered
// globally (view_tile_base[v] + ty * tiles_x + tx)
__device__ __forceinline__ int tiles_x_of(const SlmView& vw) { return (vw.W + SLM_TILE - 1) / SLM_TILE; }
__device__ __forceinline__ int tiles_y_of(const SlmView& vw) { return (vw.H + SLM_TILE - 1) / SLM_TILE; }

__global__ void k_tile_count_v(const uint32_t* __restrict__ sv, long long n, long long G,
                               const SlmSplat* __restrict__ splats, const SlmView* __restrict__ views,
                               unsigned long long* __restrict__ n_inst) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const uint32_t e = sv[i];
    const int v = (int)(e >> 24);
    const SlmView vw = views[v];
    unsigned long long c = 0;
    int tx0, tx1, ty0, ty1;
    if (splat_tiles(splats[(long long)v * G + (e & 0xffffffu)], tiles_x_of(vw), tiles_y_of(vw), tx0, tx1, ty0, ty1))
      c = (unsigned long long)(tx1 - tx0 + 1) * (ty1 - ty0 + 1);
    n_inst[i] = c;
  }
}

__global__ void k_tile_emit_v(const uint32_t* __restrict__ sv, const unsigned long long* __restrict__ inst_off,
                              long long n, long long G, const SlmSplat* __restrict__ splats,
                              const SlmView* __restrict__ views, const int* __restrict__ view_tile_base,
                              uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const unsigned long long beg = inst_off[i], end = inst_off[i + 1];
    if (beg == end) continue;
    const uint32_t e = sv[i];
    const int v = (int)(e >> 24);
    const long long gs = (long long)v * G + (e & 0xffffffu);
    const SlmView vw = views[v];
    const int tiles_x = tiles_x_of(vw);
    int tx0, tx1, ty0, ty1;
    splat_tiles(splats[gs], tiles_x, tiles_y_of(vw), tx0, tx1, ty0, ty1);
    unsigned long long k = beg;
    for (int ty = ty0; ty <= ty1; ++ty)
      for (int tx = tx0; tx <= tx1; ++tx) {
        keys[k] = (uint32_t)(view_tile_base[v] + ty * tiles_x + tx);  // (view, depth) emission order, see k_tile_emit
        vals[k] = (uint32_t)gs;  // the sort carries the global splat
        ++k;
      }
  }
}

// ---------------------------------------------------------------------------
// runs: a (tile, splat) instance with >= 1 kept pixel.  The COUNT pass leaves
// a 256-bit keep mask per instance (one ballot word per warp of the tile);
// here instances become runs, numbered in (view, tile, depth) order -- the
// order the rasteriser produces entries -- so the FILL pass writes each run's
// entries contiguously.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int mask_popc(const uint32_t* m) {
  int c = 0;
#pragma unroll
  for (int w = 0; w < SLM_TILE * SLM_TILE / 32; ++w) c += __popc(m[w]);
  return c;
}

// per instance of one view: entry count, used flag, and the per-(view,
// gaussian) entry count (integer atomics: deterministic)
__global__ void k_inst_count(const uint32_t* __restrict__ mask, const uint32_t* __restrict__ inst_gid, long long n,
                             long long* __restrict__ cnt, int* __restrict__ used, int* __restrict__ pair_cnt) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n; j += (long long)gridDim.x * blockDim.x) {
    const int c = mask_popc(mask + (size_t)j * 8);
    cnt[j] = c;
    used[j] = c > 0;
    if (c > 0) atomicAdd(&pair_cnt[inst_gid[j]], c);
  }
}

// run table of one view: instance j -> run r = run_of[j] (exclusive scan of
// used), entry start (exclusive scan of counts), pair, tile and mask; plus
// each pair's run count
// run_of / ent_of are exclusive scans over the SUBSET's concatenated
// instances; `ibase` is this view's first instance in that concatenation
__global__ void k_runs_emit(const uint32_t* __restrict__ mask, const uint32_t* __restrict__ inst_gid,
                            const int* __restrict__ used, const int* __restrict__ run_of,
                            const long long* __restrict__ ent_of, long long ibase, long long n,
                            const int* __restrict__ pidx, long long* __restrict__ run_start, int* __restrict__ run_q,
                            uint32_t* __restrict__ run_mask, int* __restrict__ pair_nruns,
                            long long* __restrict__ inst_start) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n; j += (long long)gridDim.x * blockDim.x) {
    const long long jg = ibase + j;
    inst_start[j] = ent_of[jg];
    if (!used[jg]) continue;
    const int r = run_of[jg];
    const int q = pidx[inst_gid[j]];
    run_start[r] = ent_of[jg];
    run_q[r] = q;
    if (run_mask) {  // optional per-run keep mask (not needed by the product path)
#pragma unroll
      for (int w = 0; w < 8; ++w) run_mask[(size_t)r * 8 + w] = mask[(size_t)j * 8 + w];
    }
    atomicAdd(&pair_nruns[q], 1);
  }
}

// per tile: its run count and each run's (view, tile) tag; one warp per tile
// (the tile's instances are contiguous).  Tiles are global when
// view_tile_base != NULL (subset-batched), else local to `view`.
__global__ void k_tile_runs(const slm_u2* __restrict__ ranges, int n_tiles, const int* __restrict__ used,
                            const int* __restrict__ run_of, long long ibase, int view, int* __restrict__ tile_nruns,
                            uint32_t* __restrict__ run_tile, const int* __restrict__ view_tile_base, int n_views) {
  const int lane = threadIdx.x & 31;
  for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < n_tiles; t += (gridDim.x * blockDim.x) >> 5) {
    const slm_u2 rg = ranges[t];
    int vv = view, lt = t;
    if (view_tile_base) {
      vv = 0;
      while (vv + 1 < n_views && view_tile_base[vv + 1] <= t) ++vv;
      lt = t - view_tile_base[vv];
    }
    int c = 0;
    for (uint32_t j0 = rg.x; j0 < rg.y; j0 += 32) {
      const uint32_t j = j0 + lane;
      const bool u = j < rg.y && used[ibase + j];
      if (u) run_tile[run_of[ibase + j]] = ((uint32_t)vv << 24) | (uint32_t)lt;
      c += __popc(__ballot_sync(0xffffffffu, u));
    }
    if (lane == 0) tile_nruns[t] = c;
  }
}

__global__ void k_tile_ranges(const uint32_t* __restrict__ keys, long long n, uint2* __restrict__ ranges) {
  long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (; j < n; j += (long long)gridDim.x * blockDim.x) {
    const uint32_t t = keys[j];
    if (j == 0 || keys[j - 1] != t) ranges[t].x = (unsigned)j;
    if (j == n - 1 || keys[j + 1] != t) ranges[t].y = (unsigned)(j + 1);
  }
}

// ---------------------------------------------------------------------------
// tile rasteriser (ref: rasterizer.py:264-316), one 16x16 tile per CTA,
// one pixel per thread, splats staged in shared memory in batches.
//   COUNT pass: per-pixel entry count, rendered colour, T_final and, per
//               tile instance, the 256-bit keep mask (one ballot word per warp).
//   FILL pass : writes the cache records in run order: entry of (instance,
//               pixel) at inst_start[instance] + (number of keepers of the
//               instance at lower tile-local pixel indices) -- one contiguous
//               chunk per (instance, warp).  dc/dalpha uses the per-pixel
//               colour total of the COUNT pass (ref: jacobian.py:391-399).
//               Optionally also the pixel-order Traversals export.
// ---------------------------------------------------------------------------
typedef SlmRasterArgs RasterArgs;

// 32x32 bit-matrix transpose across a warp: lane i holds row i on entry and
// column i on exit (bit j of lane i's result = bit i of lane j's input);
// five butterfly rounds swapping the off-diagonal blocks
__device__ __forceinline__ unsigned transpose32(unsigned x, int lane) {
  const unsigned lo[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
  for (int r = 0; r < 5; ++r) {
    const int j = 16 >> r;
    const unsigned y = __shfl_xor_sync(0xffffffffu, x, j);
    x = (lane & j) ? ((x & ~lo[r]) | ((y >> j) & lo[r])) : ((x & lo[r]) | ((y & lo[r]) << j));
  }
  return x;
}

#define RB 256
#define RW (RB / 32)

// 16-byte shared load at a 32-bit shared-window address (one IMAD per
// instance instead of re-forming the generic window address per access)
__device__ __forceinline__ double2 lds2(unsigned a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ double lds1(unsigned a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
// register budgets of the two passes (resident blocks per SM), measured at C3:
// COUNT 4 blocks (64 registers) 13.98 -> 13.72 ms against the compiler's
// default 5; FILL 1 (79 registers, 3 blocks resident) 15.01 -> 14.87 ms
// against 4; higher occupancy (5 / 6) is slower for both
#ifndef SLM_COUNT_MINB
#define SLM_COUNT_MINB 4
#endif
#ifndef SLM_FILL_MINB
#define SLM_FILL_MINB 1
#endif
template <bool FILL>
__global__ void __launch_bounds__(RB, FILL ? SLM_FILL_MINB : SLM_COUNT_MINB) k_raster(RasterArgs A) {
  // per-instance fp64 staging, one array each so that every access is one
  // base + k * 16 (or 8) with immediate offsets: (mx, my), (ca, 2 cb), (cc, o)
  // and the colour (c0, c1, c2); 2 cb is exact, so q is bit-identical
  __shared__ double2 s_geo[3 * RB];
  __shared__ double s_col[3 * RB];
  unsigned a_geo = (unsigned)__cvta_generic_to_shared(s_geo), a_col = (unsigned)__cvta_generic_to_shared(s_col);
  asm volatile("" : "+r"(a_geo), "+r"(a_col));  // opaque: kept in registers, not re-formed per access
  __shared__ int4 s_box[RB];
  __shared__ uint32_t s_gid[RB];
  __shared__ uint32_t s_mask[RB * RW];              // keep masks of the batch (COUNT out, FILL in)
  __shared__ long long s_start[FILL ? RB : 1];      // FILL: first entry of each instance's run
  __shared__ uint8_t s_pre[FILL ? RB * RW : 1];     // FILL: keepers in lower warps, per instance
  __shared__ uint8_t s_list[RW][RB];                // per warp: batch instances that concern it

  // batched (A.views != NULL): one launch over the tiles of all the subset's
  // views; pixel buffers are subset-global (pix_base + y * W + x)
  int W = A.W, H = A.H, tiles_x = A.tiles_x, tile = blockIdx.x;
  long long pb = 0;
  if (A.views) {
    int v = 0;
    while (v + 1 < A.n_views && A.view_tile_base[v + 1] <= tile) ++v;
    const SlmView vw = A.views[v];
    W = vw.W;
    H = vw.H;
    tiles_x = (W + SLM_TILE - 1) / SLM_TILE;
    tile -= A.view_tile_base[v];
    pb = vw.pix_base;
  }
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const int lx = threadIdx.x % SLM_TILE, ly = threadIdx.x / SLM_TILE;
  const int px = tx * SLM_TILE + lx, py = ty * SLM_TILE + ly;
  const bool inside = px < W && py < H;
  const long long pix = pb + (long long)py * W + px;
  const uint2 rng = A.tile_range[blockIdx.x];
  const double dxp = (double)px + 0.5, dyp = (double)py + 0.5;
  const double amin = A.cfg.alpha_min, tstop = A.cfg.t_stop, aclamp = A.cfg.alpha_clamp;
  // o * exp(-40) < 4.3e-18: below any alpha_min > 1e-17 the tail can never be
  // kept and is mapped to alpha = 0; with alpha_min = 0 (RenderConfig.smooth,
  // ref rasterizer.py:42-45, 292-296) every alpha > 0 counts, so the tail is
  // evaluated with the full-range exp down to its underflow
  const bool tail = !(amin > 1e-17);
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const unsigned lanes_below = (1u << lane) - 1u;
  const int row0 = ty * SLM_TILE + 2 * warp;  // the warp's two pixel rows

  double T = 1.0, C0 = 0.0, C1 = 0.0, C2 = 0.0;
  uint32_t cnt = 0;
  bool done = !inside;
  long long e = 0;  // pixel-order position (Traversals export only)
  double tot0 = 0, tot1 = 0, tot2 = 0;
  if (FILL && inside) {
    tot0 = A.rgb[(size_t)pix * 3 + 0];
    tot1 = A.rgb[(size_t)pix * 3 + 1];
    tot2 = A.rgb[(size_t)pix * 3 + 2];
    if (A.trav_gid) e = A.pix_off[A.pix_base + pix];  // single-view export only (pb = 0)
  }

  for (unsigned base = rng.x; base < rng.y; base += RB) {
    if (__syncthreads_and(done)) break;
    unsigned j = base + threadIdx.x;
    if (j < rng.y) {
      uint32_t g = A.inst_gid[j];
      const SlmSplat s = A.splats[g];
      s_geo[threadIdx.x] = make_double2(s.mx, s.my);
      s_geo[RB + threadIdx.x] = make_double2(s.ca, 2.0 * s.cb);
      s_geo[2 * RB + threadIdx.x] = make_double2(s.cc, s.o);
      s_col[threadIdx.x] = s.c0;
      s_col[RB + threadIdx.x] = s.c1;
      s_col[2 * RB + threadIdx.x] = s.c2;
      s_box[threadIdx.x] = make_int4(s.x0, s.x1, s.y0, s.y1);
      s_gid[threadIdx.x] = g;
      if (FILL) {
        const uint32_t* mk = A.inst_mask + (size_t)j * RW;
        int acc = 0;
#pragma unroll
        for (int w = 0; w < RW; ++w) {
          const uint32_t mw = mk[w];
          s_mask[threadIdx.x * RW + w] = mw;
          s_pre[threadIdx.x * RW + w] = (uint8_t)acc;
          acc += __popc(mw);
        }
        if (A.rec4) s_start[threadIdx.x] = A.inst_start[j];
      }
    }
    __syncthreads();
    const int nb = min((unsigned)RB, rng.y - base);
    // each warp compacts the batch's instances that concern its two pixel rows:
    // COUNT -- bbox meets the rows (the others get an empty keep mask);
    // FILL  -- the COUNT pass kept at least one of the warp's pixels
    int nrel = 0;
    for (int k0 = 0; k0 < nb; k0 += 32) {
      const int k = k0 + lane;
      bool rel = false;
      if (k < nb) {
        if (FILL) {
          rel = s_mask[k * RW + warp] != 0u;
        } else {
          const int4 bx = s_box[k];
          rel = !(bx.w < row0 || bx.z > row0 + 1);
          if (!rel) s_mask[k * RW + warp] = 0u;
        }
      }
      const unsigned bal = __ballot_sync(0xffffffffu, rel);
      if (rel) s_list[warp][nrel + __popc(bal & lanes_below)] = (uint8_t)k;
      nrel += __popc(bal);
    }
    __syncwarp();
    if (!FILL) {
      // COUNT, lane queues: per block of 32 relevant instances each lane
      // collects the ones whose bbox holds its pixel (a 32-bit word) and
      // walks its own set bits in order, so a step evaluates one (instance,
      // pixel) pair on every busy lane instead of idling the lanes outside
      // the bbox; per-pixel depth order is kept.  The keep masks come back
      // through the inverse transpose of the lanes' kept-bit words.
      for (int b0 = 0; b0 < nrel; b0 += 32) {
        const int nbk = min(32, nrel - b0);
        // lane i: the warp-pixel mask of instance b0 + i (its bbox clipped to
        // the warp's two rows), then a 32x32 bit transpose gives every lane
        // its word (bit i: instance b0 + i may touch the lane's pixel)
        unsigned m = 0u;
        if (lane < nbk) {
          const int4 bx = s_box[s_list[warp][b0 + lane]];
          const int cx0 = max(bx.x - tx * SLM_TILE, 0), cx1 = min(bx.y - tx * SLM_TILE, SLM_TILE - 1);
          if (cx0 <= cx1) {
            const unsigned rm = (2u << cx1) - (1u << cx0);
            if (bx.z <= row0 && row0 <= bx.w) m |= rm;
            if (bx.z <= row0 + 1 && row0 + 1 <= bx.w) m |= rm << 16;
          }
        }
        unsigned wq = transpose32(m, lane);
        if (done) wq = 0u;
        unsigned kw = 0u;  // bit i: this lane's pixel keeps instance b0 + i
        while (__any_sync(0xffffffffu, wq != 0u)) {
          if (wq == 0u) continue;
          const int i = __ffs(wq) - 1;
          const int k = s_list[warp][b0 + i];
          wq &= wq - 1u;
          const unsigned ag = a_geo + 16u * k;
          const double2 g0 = lds2(ag), g1 = lds2(ag + 16u * RB), g2 = lds2(ag + 32u * RB);
          const double dx = __dsub_rn(dxp, g0.x);
          const double dy = __dsub_rn(dyp, g0.y);
          const double q = __dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(g1.x, dx), dx), __dmul_rn(g2.x, __dmul_rn(dy, dy))),
                                     __dmul_rn(__dmul_rn(g1.y, dy), dx));
          const double ex = __dmul_rn(-0.5, q);
          double a = ex >= -40.0 ? __dmul_rn(g2.y, slm_exp_neg(ex)) : (tail ? __dmul_rn(g2.y, exp(ex)) : 0.0);
          a = a < aclamp ? a : aclamp;
          if ((a >= amin) && (a > 0.0)) {  // T >= t_stop holds while the lane is not done
            kw |= 1u << i;
            const double wgt = __dmul_rn(a, T);
            const unsigned ac = a_col + 8u * k;
            C0 = __dadd_rn(C0, __dmul_rn(wgt, lds1(ac)));
            C1 = __dadd_rn(C1, __dmul_rn(wgt, lds1(ac + 8u * RB)));
            C2 = __dadd_rn(C2, __dmul_rn(wgt, lds1(ac + 16u * RB)));
            T = __dmul_rn(T, 1.0 - a);
            ++cnt;
            if (T < tstop) {
              done = true;
              wq = 0u;
            }
          }
        }
        // the transpose back gives lane i instance b0 + i's keep mask
        const unsigned km = transpose32(kw, lane);
        if (lane < nbk) s_mask[s_list[warp][b0 + lane] * RW + warp] = km;
      }
    }
    if (FILL) {
      // FILL, lane queues over the COUNT keep masks: per block of 32 relevant
      // instances each lane walks the ones that kept its pixel, in depth
      // order, and writes their records (every step is a cache entry)
      for (int b0 = 0; b0 < nrel; b0 += 32) {
        const int nbk = min(32, nrel - b0);
        unsigned wq = transpose32(lane < nbk ? s_mask[s_list[warp][b0 + lane] * RW + warp] : 0u, lane);
        while (__any_sync(0xffffffffu, wq != 0u)) {
          if (wq == 0u) continue;
          const int k = s_list[warp][b0 + __ffs(wq) - 1];
          wq &= wq - 1u;
          const unsigned ag = a_geo + 16u * k;
          const double2 g0 = lds2(ag), g1 = lds2(ag + 16u * RB), g2 = lds2(ag + 32u * RB);
          const double dx = __dsub_rn(dxp, g0.x);
          const double dy = __dsub_rn(dyp, g0.y);
          const double q = __dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(g1.x, dx), dx), __dmul_rn(g2.x, __dmul_rn(dy, dy))),
                                     __dmul_rn(__dmul_rn(g1.y, dy), dx));
          const double ex = __dmul_rn(-0.5, q);
          double a = ex >= -40.0 ? __dmul_rn(g2.y, slm_exp_neg(ex)) : (tail ? __dmul_rn(g2.y, exp(ex)) : 0.0);
          a = a < aclamp ? a : aclamp;
          const double wgt = __dmul_rn(a, T);
          const unsigned ac = a_col + 8u * k;
          const double c0 = lds1(ac), c1 = lds1(ac + 8u * RB), c2 = lds1(ac + 16u * RB);
          C0 = __dadd_rn(C0, __dmul_rn(wgt, c0));
          C1 = __dadd_rn(C1, __dmul_rn(wgt, c1));
          C2 = __dadd_rn(C2, __dmul_rn(wgt, c2));
          if (A.rec4) {
            const unsigned m = s_mask[k * RW + warp];
            // stored values are fp32: an fp32 reciprocal (1 ulp) suffices (a <= alpha_clamp = 0.99)
            const double iom = (double)__frcp_rn((float)(1.0 - a));
            long long dest = s_start[k] + s_pre[k * RW + warp] + __popc(m & lanes_below);
            slm_f4* r4 = A.rec4;
            float* rd2 = A.rec_d2;
            uint8_t* rpx = A.rec_pix;
            if (A.rec4_h && dest >= A.e_split) {  // offloaded tail (host-mapped streams)
              r4 = A.rec4_h;
              rd2 = A.rec_d2_h;
              rpx = A.rec_pix_h;
              dest -= A.e_hbase;
            }
            r4[dest] = make_float4(a < aclamp ? (float)a : 0.0f, (float)wgt,
                                   (float)(c0 * T - (tot0 - C0) * iom),
                                   (float)(c1 * T - (tot1 - C1) * iom));
            rd2[dest] = (float)(c2 * T - (tot2 - C2) * iom);
            rpx[dest] = (uint8_t)threadIdx.x;
          }
          if (A.trav_gid) {
            const long long le = e - A.view_entry_base;
            A.trav_gid[le] = s_gid[k];
            A.trav_alpha[le] = a;
            A.trav_T[le] = T;
          }
          ++e;
          T = __dmul_rn(T, 1.0 - a);
        }
      }
      done = done || T < tstop;
    }
    __syncthreads();
    if (!FILL && A.inst_mask) {
      uint32_t* dst = A.inst_mask + (size_t)base * RW;
      for (int w = threadIdx.x; w < nb * RW; w += RB) dst[w] = s_mask[w];
    }
  }
  if (!FILL && inside) {
    A.px_count[pix] = cnt;
    A.rgb[(size_t)pix * 3 + 0] = __dadd_rn(C0, __dmul_rn(A.cfg.bg[0], T));
    A.rgb[(size_t)pix * 3 + 1] = __dadd_rn(C1, __dmul_rn(A.cfg.bg[1], T));
    A.rgb[(size_t)pix * 3 + 2] = __dadd_rn(C2, __dmul_rn(A.cfg.bg[2], T));
    A.t_final[pix] = T;
  }
}

// ---------------------------------------------------------------------------
// C-ABI entry points
// ---------------------------------------------------------------------------
extern "C" {

int slm_preprocess(const double* x, long long G, int sh_degree, const SlmCamera* cam, const SlmRastCfg* cfg,
                   SlmSplat* out, unsigned long long* depth_key, uint32_t* order_val, int* err,
                   cudaStream_t stream) {
  if (G <= 0 || !x || !cam || !cfg || !out) return SLM_ERR_ARG;
  unsigned blocks = slm_blocks(G, 256);
  switch (sh_degree) {
    case 0: k_preprocess<1><<<blocks, 256, 0, stream>>>(x, G, *cam, *cfg, out, depth_key, order_val, err); break;
    case 1: k_preprocess<4><<<blocks, 256, 0, stream>>>(x, G, *cam, *cfg, out, depth_key, order_val, err); break;
    case 2: k_preprocess<9><<<blocks, 256, 0, stream>>>(x, G, *cam, *cfg, out, depth_key, order_val, err); break;
    case 3: k_preprocess<16><<<blocks, 256, 0, stream>>>(x, G, *cam, *cfg, out, depth_key, order_val, err); break;
    default: return SLM_ERR_ARG;
  }
  return slm_cuda_status();
}

int slm_preprocess_views(const double* x, long long G, int sh_degree, const SlmCamera* cams_dev, int V,
                         const SlmRastCfg* cfg, SlmSplat* out, unsigned long long* depth_key, uint32_t* order_val,
                         int* err, cudaStream_t stream) {
  if (G <= 0 || V <= 0 || G >= (1LL << 24) || V > 255) return SLM_ERR_ARG;
  unsigned blocks = slm_blocks(G, 128, 1LL << 30);
  switch (sh_degree) {
    case 0: k_preprocess_views<1><<<blocks, 128, 0, stream>>>(x, G, cams_dev, V, *cfg, out, depth_key, order_val, err); break;
    case 1: k_preprocess_views<4><<<blocks, 128, 0, stream>>>(x, G, cams_dev, V, *cfg, out, depth_key, order_val, err); break;
    case 2: k_preprocess_views<9><<<blocks, 128, 0, stream>>>(x, G, cams_dev, V, *cfg, out, depth_key, order_val, err); break;
    case 3: k_preprocess_views<16><<<blocks, 128, 0, stream>>>(x, G, cams_dev, V, *cfg, out, depth_key, order_val, err); break;
    default: return SLM_ERR_ARG;
  }
  return slm_cuda_status();
}

int slm_tile_count_v(const uint32_t* sv, long long n, long long G, const SlmSplat* splats, const SlmView* views,
                     unsigned long long* n_inst, cudaStream_t stream) {
  if (n <= 0) return SLM_OK;
  k_tile_count_v<<<slm_blocks(n, 256), 256, 0, stream>>>(sv, n, G, splats, views, n_inst);
  return slm_cuda_status();
}

int slm_tile_emit_v(const uint32_t* sv, const unsigned long long* inst_off, long long n, long long G,
                    const SlmSplat* splats, const SlmView* views, const int* view_tile_base, uint32_t* keys,
                    uint32_t* vals, cudaStream_t stream) {
  if (n <= 0) return SLM_OK;
  k_tile_emit_v<<<slm_blocks(n, 256), 256, 0, stream>>>(sv, inst_off, n, G, splats, views, view_tile_base, keys,
                                                         vals);
  return slm_cuda_status();
}

// radix sort of u32 keys on bits [begin_bit, end_bit) (stable): the per-view
// grouping pass after the subset-wide depth sort
long long slm_sort_keys_u32_workspace(long long n) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)n);
  return (long long)bytes;
}

int slm_sort_keys_u32(void* ws, long long ws_bytes, const uint32_t* kin, uint32_t* kout, long long n, int begin_bit,
                      int end_bit, cudaStream_t stream) {
  if (n <= 0) return SLM_OK;
  if (n > 0x7fffffffLL) return SLM_ERR_SIZE;
  size_t bytes = (size_t)ws_bytes;
  cudaError_t e = cub::DeviceRadixSort::SortKeys(ws, bytes, kin, kout, (int)n, begin_bit, end_bit, stream);
  return e == cudaSuccess ? SLM_OK : SLM_ERR_CUDA;
}

// stable (depth, gid) order of the valid splats: CUB radix sort over the
// fp64 depth bit patterns (positive doubles order like their bits)
long long slm_sort_pairs_u64_workspace(long long n) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const unsigned long long*)nullptr,
                                  (unsigned long long*)nullptr, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (int)n);
  return (long long)bytes;
}

int slm_sort_pairs_u64(void* ws, long long ws_bytes, const unsigned long long* keys_in, unsigned long long* keys_out,
                       const uint32_t* vals_in, uint32_t* vals_out, long long n, int begin_bit, int end_bit,
                       cudaStream_t stream) {
  if (n <= 0) return SLM_OK;
  if (n > 0x7fffffffLL) return SLM_ERR_SIZE;
  size_t bytes = (size_t)ws_bytes;
  cudaError_t e = cub::DeviceRadixSort::SortPairs(ws, bytes, keys_in, keys_out, vals_in, vals_out, (int)n,
                                                  begin_bit, end_bit, stream);
  return e == cudaSuccess ? SLM_OK : SLM_ERR_CUDA;
}

int slm_tile_count(const uint32_t* sorted_gid, const unsigned long long* sorted_key, long long G,
                   const SlmSplat* splats, int tiles_x, int tiles_y, unsigned long long* n_inst,
                   cudaStream_t stream) {
  k_tile_count<<<slm_blocks(G, 256), 256, 0, stream>>>(sorted_gid, sorted_key, G, splats, tiles_x, tiles_y, n_inst);
  return slm_cuda_status();
}

int slm_tile_emit(const uint32_t* sorted_gid, const unsigned long long* inst_off, long long G, const SlmSplat* splats,
                  int tiles_x, int tiles_y, uint32_t* keys, uint32_t* vals, cudaStream_t stream) {
  k_tile_emit<<<slm_blocks(G, 256), 256, 0, stream>>>(sorted_gid, inst_off, G, splats, tiles_x, tiles_y, keys, vals);
  return slm_cuda_status();
}


int slm_inst_count(const uint32_t* mask, const uint32_t* inst_gid, long long n, long long* cnt, int* used,
                   int* pair_cnt, cudaStream_t stream) {
  if (n <= 0) return SLM_OK;
  k_inst_count<<<slm_blocks(n, 256), 256, 0, stream>>>(mask, inst_gid, n, cnt, used, pair_cnt);
  return slm_cuda_status();
}

int slm_runs_emit(const uint32_t* mask, const uint32_t* inst_gid, const int* used, const int* run_of,
                  const long long* ent_of, long long ibase, long long n, const int* pidx, long long* run_start,
                  int* run_q, uint32_t* run_mask, int* pair_nruns, long long* inst_start, cudaStream_t stream) {
  if (n <= 0) return SLM_OK;
  k_runs_emit<<<slm_blocks(n, 256), 256, 0, stream>>>(mask, inst_gid, used, run_of, ent_of, ibase, n, pidx,
                                                       run_start, run_q, run_mask, pair_nruns, inst_start);
  return slm_cuda_status();
}

int slm_tile_runs(const slm_u2* ranges, int n_tiles, const int* used, const int* run_of, long long ibase, int view,
                  int* tile_nruns, uint32_t* run_tile, const int* view_tile_base, int n_views, cudaStream_t stream) {
  k_tile_runs<<<slm_blocks((long long)n_tiles * 32, 256), 256, 0, stream>>>(ranges, n_tiles, used, run_of, ibase, view,
                                                                             tile_nruns, run_tile, view_tile_base,
                                                                             n_views);
  return slm_cuda_status();
}

int slm_tile_ranges(const uint32_t* keys, long long n, uint2* ranges, int n_tiles, cudaStream_t stream) {
  cudaMemsetAsync(ranges, 0, sizeof(uint2) * (size_t)n_tiles, stream);
  if (n > 0) k_tile_ranges<<<slm_blocks(n, 256), 256, 0, stream>>>(keys, n, ranges);
  return slm_cuda_status();
}

static int raster_grid(const RasterArgs* a) {
  if (a->views) return a->n_tiles;
  return a->tiles_x * ((a->H + SLM_TILE - 1) / SLM_TILE);
}

int slm_raster_count(const RasterArgs* a, cudaStream_t stream) {
  k_raster<false><<<raster_grid(a), RB, 0, stream>>>(*a);
  return slm_cuda_status();
}

int slm_raster_fill(const RasterArgs* a, cudaStream_t stream) {
  if (!a->inst_mask) return SLM_ERR_ARG;  // FILL replays the COUNT pass's keep masks
  k_raster<true><<<raster_grid(a), RB, 0, stream>>>(*a);
  return slm_cuda_status();
}

int slm_raster_args_size() { return (int)sizeof(RasterArgs); }
int slm_camera_size() { return (int)sizeof(SlmCamera); }
int slm_rastcfg_size() { return (int)sizeof(SlmRastCfg); }
int slm_splat_size() { return (int)sizeof(SlmSplat); }

}  // extern "C"
