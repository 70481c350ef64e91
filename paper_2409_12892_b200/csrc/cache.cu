// Gradient-cache assembly: pixel segments, (gaussian, view) pairs, and the
// gaussian-order record stream (sortCacheByGaussians).
//
// Gaussian order = (gid, view, pixel row-major); restricted to one view it is
// exactly the reference's np.lexsort((pixel_ids, gaussian_ids))
// (ref: jacobian.py:93-105), produced by a stable radix sort of each view's
// pixel-order entries by gid followed by a scatter into pair blocks.
#include "slm_common.cuh"

#include <cub/cub.cuh>

// ---------------------------------------------------------------------------
// scans / sorts (CUB) -- workspace sizes are queried by the host
// ---------------------------------------------------------------------------
extern "C" {

long long slm_scan_i64_workspace(long long n) {
  size_t b = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, b, (const long long*)nullptr, (long long*)nullptr, (int)n);
  return (long long)b;
}
int slm_scan_i64(void* ws, long long wsb, const long long* in, long long* out, long long n, cudaStream_t s) {
  if (n <= 0) return SLM_OK;
  if (n > 0x7fffffffLL) return SLM_ERR_SIZE;
  size_t b = (size_t)wsb;
  return cub::DeviceScan::ExclusiveSum(ws, b, in, out, (int)n, s) == cudaSuccess ? SLM_OK : SLM_ERR_CUDA;
}
long long slm_scan_i32_workspace(long long n) {
  size_t b = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, b, (const int*)nullptr, (int*)nullptr, (int)n);
  return (long long)b;
}
int slm_scan_i32(void* ws, long long wsb, const int* in, int* out, long long n, cudaStream_t s) {
  if (n <= 0) return SLM_OK;
  if (n > 0x7fffffffLL) return SLM_ERR_SIZE;
  size_t b = (size_t)wsb;
  return cub::DeviceScan::ExclusiveSum(ws, b, in, out, (int)n, s) == cudaSuccess ? SLM_OK : SLM_ERR_CUDA;
}
long long slm_sort_pairs_u32_workspace(long long n) {
  size_t b = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, b, (const uint32_t*)nullptr, (uint32_t*)nullptr, (const uint32_t*)nullptr,
                                  (uint32_t*)nullptr, (int)n);
  return (long long)b;
}
int slm_sort_pairs_u32(void* ws, long long wsb, const uint32_t* kin, uint32_t* kout, const uint32_t* vin,
                       uint32_t* vout, long long n, int begin_bit, int end_bit, cudaStream_t s) {
  if (n <= 0) return SLM_OK;
  if (n > 0x7fffffffLL) return SLM_ERR_SIZE;
  size_t b = (size_t)wsb;
  return cub::DeviceRadixSort::SortPairs(ws, b, kin, kout, vin, vout, (int)n, begin_bit, end_bit, s) == cudaSuccess
             ? SLM_OK
             : SLM_ERR_CUDA;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// pixel segments
// ---------------------------------------------------------------------------
__global__ void k_px_prepare(const uint32_t* __restrict__ cnt, long long n, long long* __restrict__ cnt64,
                             int* __restrict__ nonempty) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    uint32_t c = cnt[i];
    cnt64[i] = c;
    nonempty[i] = c > 0;
  }
}

// seg_info[seg] = {gp, (y << 16) | x}; views are given by a gp -> view table
__global__ void k_px_segments(const uint32_t* __restrict__ cnt, const int* __restrict__ seg_idx, long long n,
                              const SlmCamera* __restrict__ cams, int n_views, uint2* __restrict__ seg_info) {
  for (long long gp = blockIdx.x * (long long)blockDim.x + threadIdx.x; gp < n; gp += (long long)gridDim.x * blockDim.x) {
    if (cnt[gp] == 0) continue;
    int v = 0;
    while (v + 1 < n_views && cams[v + 1].pix_base <= gp) ++v;
    long long p = gp - cams[v].pix_base;
    int y = (int)(p / cams[v].W), x = (int)(p % cams[v].W);
    seg_info[seg_idx[gp]] = make_uint2((uint32_t)gp, ((uint32_t)y << 16) | (uint32_t)x);
  }
}

// ---------------------------------------------------------------------------
// pairs: (gaussian, view) with >= 1 entry, numbered in (gid, view) order
// ---------------------------------------------------------------------------
__global__ void k_pairs_prepare(const int* __restrict__ cnt /*[V][G]*/, int V, long long G,
                                long long* __restrict__ cntT /*[G*V]*/, int* __restrict__ flagT,
                                long long* __restrict__ cntV /*[V*G] view-major int64*/) {
  long long n = (long long)V * G;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    long long g = i / V;
    int v = (int)(i % V);
    int c = cnt[(long long)v * G + g];
    cntT[i] = c;
    flagT[i] = c > 0;
    cntV[(long long)v * G + g] = c;
  }
}

__global__ void k_pairs_emit(const int* __restrict__ cnt, int V, long long G, const int* __restrict__ pair_of,
                             const long long* __restrict__ off_of, const SlmSplat* __restrict__ splats /*[V][G]*/,
                             long long* __restrict__ pair_off, int* __restrict__ pair_gid,
                             uint32_t* __restrict__ pair_vm, SlmPairGeo* __restrict__ geo, int* __restrict__ pidx,
                             int* __restrict__ gpo /*[G+1]*/, int n_pairs, long long n_entries) {
  long long n = (long long)V * G;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    long long g = i / V;
    int v = (int)(i % V);
    if (v == 0) gpo[g] = pair_of[i];
    long long vg = (long long)v * G + g;
    int c = cnt[vg];
    if (c <= 0) {
      pidx[vg] = -1;
      continue;
    }
    int q = pair_of[i];
    pair_off[q] = off_of[i];
    pair_gid[q] = (int)g;
    const SlmSplat s = splats[vg];
    pair_vm[q] = (uint32_t)v | (((s.flags >> 1) & 7u) << 16);
    SlmPairGeo pg;
    pg.mx = s.mx; pg.my = s.my;
    pg.ka = (float)s.ca; pg.kb = (float)s.cb; pg.kc = (float)s.cc;
    pg.inv_o = (float)(1.0 / s.o);
    geo[q] = pg;
    pidx[vg] = q;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    gpo[G] = n_pairs;
    pair_off[n_pairs] = n_entries;
  }
}

// ---------------------------------------------------------------------------
// gaussian-order stream for one view: scatter the gid-sorted entries into
// their pair blocks
// ---------------------------------------------------------------------------
typedef SlmGaussOrderArgs GaussOrderArgs;

__global__ void k_gauss_scatter(GaussOrderArgs A) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < A.Ev; j += (long long)gridDim.x * blockDim.x) {
    uint32_t g = A.sorted_gid[j];
    uint32_t sl = A.sorted_src[j];
    long long vg = (long long)A.v * A.G + g;
    int q = A.pidx[vg];
    long long base = A.pair_off[q];
    long long dest = base + (A.view_base + j - A.vscan[vg]);
    long long src = A.view_base + sl;
    A.g_idx[dest] = A.ent_xy[sl] | (dest == base ? SLM_HEAD : 0u);
    A.g_ae[dest] = A.ae[src];
    A.g_at[dest] = A.at[src];
    A.g_d0[dest] = A.d0[src];
    A.g_d1[dest] = A.d1[src];
    A.g_d2[dest] = A.d2[src];
    if ((dest & (SLM_CHUNK - 1)) == 0) A.chunk_seg[dest / SLM_CHUNK] = q;
    if (A.g_src) A.g_src[dest] = (int)sl;
  }
}

__global__ void k_iota_u32(uint32_t* out, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = (uint32_t)i;
}

extern "C" {

int slm_px_prepare(const uint32_t* cnt, long long n, long long* cnt64, int* nonempty, cudaStream_t s) {
  k_px_prepare<<<slm_blocks(n, 256), 256, 0, s>>>(cnt, n, cnt64, nonempty);
  return slm_cuda_status();
}

int slm_px_segments(const uint32_t* cnt, const int* seg_idx, long long n, const SlmCamera* cams_dev, int n_views,
                    uint2* seg_info, cudaStream_t s) {
  k_px_segments<<<slm_blocks(n, 256), 256, 0, s>>>(cnt, seg_idx, n, cams_dev, n_views, seg_info);
  return slm_cuda_status();
}

int slm_pairs_prepare(const int* cnt, int V, long long G, long long* cntT, int* flagT, long long* cntV,
                      cudaStream_t s) {
  k_pairs_prepare<<<slm_blocks((long long)V * G, 256), 256, 0, s>>>(cnt, V, G, cntT, flagT, cntV);
  return slm_cuda_status();
}

int slm_pairs_emit(const int* cnt, int V, long long G, const int* pair_of, const long long* off_of,
                   const SlmSplat* splats, long long* pair_off, int* pair_gid, uint32_t* pair_vm, SlmPairGeo* geo,
                   int* pidx, int* gpo, int n_pairs, long long n_entries, cudaStream_t s) {
  k_pairs_emit<<<slm_blocks((long long)V * G, 256), 256, 0, s>>>(cnt, V, G, pair_of, off_of, splats, pair_off,
                                                                  pair_gid, pair_vm, geo, pidx, gpo, n_pairs,
                                                                  n_entries);
  return slm_cuda_status();
}

int slm_gauss_order_args_size() { return (int)sizeof(GaussOrderArgs); }

int slm_gauss_scatter(const GaussOrderArgs* a, cudaStream_t s) {
  if (a->Ev <= 0) return SLM_OK;
  k_gauss_scatter<<<slm_blocks(a->Ev, 256), 256, 0, s>>>(*a);
  return slm_cuda_status();
}

int slm_iota_u32(uint32_t* out, long long n, cudaStream_t s) {
  if (n <= 0) return SLM_OK;
  k_iota_u32<<<slm_blocks(n, 256), 256, 0, s>>>(out, n);
  return slm_cuda_status();
}

int slm_pair_geo_size() { return (int)sizeof(SlmPairGeo); }

}  // extern "C"
