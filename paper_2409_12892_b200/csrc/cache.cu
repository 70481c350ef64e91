// Gradient-cache assembly: pixel segments and (gaussian, view) pairs.
//
// There is no second (gaussian-order) record stream: the FILL raster pass
// writes one run-ordered stream whose runs are reachable per tile (J) and per
// (gaussian, view) pair through the pair -> runs CSR (J^T, backward), and the
// reference's pixel- and gaussian-sorted orders (ref: jacobian.py:93-121) are
// exported from it on demand (slm_export_view, parity / interop only).
#include "slm_common.cuh"

#include <cub/cub.cuh>

#include <algorithm>

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
// ---------------------------------------------------------------------------
// pairs: (gaussian, view) with >= 1 entry, numbered in (gid, view) order:
// the pairs of one gaussian are contiguous (gpo CSR), so the per-pair chain
// kernels read each gaussian's parameters once and the per-gaussian backward
// chain reads its pairs' sums contiguously.
// ---------------------------------------------------------------------------
__global__ void k_pairs_prepare(const int* __restrict__ cnt /*[V][G]*/, int V, long long G,
                                long long* __restrict__ cntV /*[V*G] view-major*/, int* __restrict__ flagV,
                                int* __restrict__ flagT /*[G*V] gid-major*/) {
  long long n = (long long)V * G;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int c = cnt[i];
    cntV[i] = c;
    flagV[i] = c > 0;
    const long long v = i / G, g = i % G;
    flagT[g * V + v] = c > 0;
  }
}

// Tiled transpose: a block owns PE_SLOTS / V gaussians x all V views.  The
// view-major inputs (counts, entry scan) are read coalesced and staged in
// shared memory, the pair outputs are written in (gid, view) order (their q
// indices are consecutive) and pidx goes back out view-major -- instead of
// scattering every pair record from a view-major sweep.
#define PE_SLOTS 1024
__global__ void __launch_bounds__(256) k_pairs_emit(const int* __restrict__ cnt, int V, long long G,
                                                    const int* __restrict__ pair_of,
                                                    const long long* __restrict__ vscan, const int* __restrict__ tscan,
                                                    const SlmSplat* __restrict__ splats /*[V][G]*/,
                                                    long long* __restrict__ pair_off, int* __restrict__ pair_gid,
                                                    uint32_t* __restrict__ pair_vm, SlmPairGeo* __restrict__ geo,
                                                    int* __restrict__ pidx, int* __restrict__ gpo /*[G+1]*/,
                                                    int n_pairs, long long n_entries) {
  __shared__ int s_c[PE_SLOTS], s_q[PE_SLOTS];
  __shared__ long long s_vs[PE_SLOTS];
  (void)pair_of;
  const int GB = PE_SLOTS / V;  // gaussians per block (V <= 255 -> >= 4)
  const int ns = GB * V;
  for (long long g0 = (long long)blockIdx.x * GB; g0 < G; g0 += (long long)gridDim.x * GB) {
    const int gb = (int)min((long long)GB, G - g0);
    // 1: view-major reads (consecutive threads = consecutive gaussians of a view)
    for (int k = threadIdx.x; k < ns; k += blockDim.x) {
      const int v = k / GB, gl = k - v * GB;
      if (gl < gb) {
        const long long i = (long long)v * G + g0 + gl;
        const int c = cnt[i];
        s_c[gl * V + v] = c;
        s_vs[gl * V + v] = c > 0 ? vscan[i] : 0;
      }
    }
    __syncthreads();
    // 2: (gid, view) order: q = tscan is consecutive over the pairs
    for (int k = threadIdx.x; k < gb * V; k += blockDim.x) {
      const int gl = k / V, v = k - gl * V;
      const long long g = g0 + gl;
      const int q = tscan[g * V + v];
      if (v == 0) gpo[g] = q;
      const int c = s_c[k];
      s_q[k] = c > 0 ? q : -1;
      if (c > 0) {
        const SlmSplat sp = splats[(long long)v * G + g];
        pair_off[q] = s_vs[k];
        pair_gid[q] = (int)g;
        pair_vm[q] = (uint32_t)v | (((sp.flags >> 1) & 7u) << 16);
        SlmPairGeo pg;
        pg.mx = sp.mx; pg.my = sp.my;
        pg.ka = (float)sp.ca; pg.kb = (float)sp.cb; pg.kc = (float)sp.cc;
        pg.inv_o = (float)(1.0 / sp.o);
        geo[q] = pg;
      }
    }
    __syncthreads();
    // 3: pidx back in view-major order
    for (int k = threadIdx.x; k < ns; k += blockDim.x) {
      const int v = k / GB, gl = k - v * GB;
      if (gl < gb) pidx[(long long)v * G + g0 + gl] = s_q[gl * V + v];
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    gpo[G] = n_pairs;
    pair_off[n_pairs] = n_entries;
  }
}

// inverse of a permutation of [0, n): inv[perm[k]] = k
__global__ void k_invert_perm(const int* __restrict__ perm, long long n, int* __restrict__ inv) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
    inv[perm[k]] = (int)k;
}

__global__ void k_iota_u32(uint32_t* out, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = (uint32_t)i;
}


// ---------------------------------------------------------------------------
// Reference-order export of one view (parity / interop only, not on the
// solve path), computed on the device from the run order:
//   pixel order    (ref: jacobian.py:401-409; entries pixel-major, blending
//                   (depth) order within a pixel)
//   gaussian order (ref: jacobian.py:93-105, np.lexsort((pixel_ids,
//                   gaussian_ids)): gid-major, pixel id within a gaussian)
// k_export_pixel: block per tile, a shared counter per tile pixel; runs are
//   taken in depth order and a run never repeats a pixel, so an entry's rank
//   at its pixel is the counter value when its run is reached:
//   pos_pix[e] = px_off[pixel] + rank.
// k_export_gauss: thread per pair of the view.  The pair's runs are in tile
//   row-major order (pair_runs CSR) and each run's entries in tile-local
//   row-major order, so within one tile row of the pair the entries of local
//   row ly follow run by run in tile-column order; 16 row counters (pass 1)
//   give each row's first rank and pass 2 hands out consecutive ranks:
//   pos_g[e] = g_off[gid] + rank by pixel id among the pair's entries.
// Outputs are the reference's index arrays: pixel_ids / gaussian_ids (pixel
// order), g_pixel_ids / g_gaussian_ids / source_index (gaussian order).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_export_pixel(const int* __restrict__ tile_run_off, int t0, int n_tiles,
                                                      int tiles_x, int W, const long long* __restrict__ run_start,
                                                      const int* __restrict__ run_q, const int* __restrict__ pair_gid,
                                                      const uint8_t* __restrict__ pix,
                                                      const long long* __restrict__ px_off, long long e_base,
                                                      long long* __restrict__ pos_pix, long long* __restrict__ pixel_ids,
                                                      long long* __restrict__ gaussian_ids) {
  __shared__ int cnt[256];
  for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    cnt[threadIdx.x] = 0;
    __syncthreads();
    const long long ox = (long long)(t % tiles_x) * SLM_TILE, oy = (long long)(t / tiles_x) * SLM_TILE;
    const int r0 = tile_run_off[t0 + t], r1 = tile_run_off[t0 + t + 1];
    for (int r = r0; r < r1; ++r) {
      const long long s = run_start[r];
      const int n = (int)(run_start[r + 1] - s);
      if ((int)threadIdx.x < n) {
        const int pl = pix[s + threadIdx.x];
        const long long px = (oy + (pl >> 4)) * W + ox + (pl & 15);
        const int k = cnt[pl];
        cnt[pl] = k + 1;
        const long long pp = px_off[px] + k;
        pos_pix[s + threadIdx.x - e_base] = pp;
        pixel_ids[pp] = px;
        gaussian_ids[pp] = pair_gid[run_q[r]];
      }
      __syncthreads();
    }
  }
}

__global__ void k_export_gauss(int n_pairs, int view, int tiles_x, int W, const uint32_t* __restrict__ pair_vm,
                               const int* __restrict__ pair_gid, const int* __restrict__ pair_run_off,
                               const int* __restrict__ pair_runs, const uint32_t* __restrict__ run_tile,
                               const long long* __restrict__ run_start, const uint8_t* __restrict__ pix,
                               const long long* __restrict__ g_off, long long e_base,
                               const long long* __restrict__ pos_pix, long long* __restrict__ g_pixel_ids,
                               long long* __restrict__ g_gaussian_ids, long long* __restrict__ g_source_index) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n_pairs; q += gridDim.x * blockDim.x) {
    if ((int)(pair_vm[q] & 0xffffu) != view) continue;
    const int gid = pair_gid[q];
    long long rank = g_off[gid];
    const int a = pair_run_off[q], b = pair_run_off[q + 1];
    for (int k = a; k < b;) {
      const int ty = (int)(run_tile[pair_runs[k]] & 0xffffffu) / tiles_x;
      int k2 = k + 1;
      while (k2 < b && (int)(run_tile[pair_runs[k2]] & 0xffffffu) / tiles_x == ty) ++k2;
      long long cur[16];
      int rc[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) rc[i] = 0;
      for (int kk = k; kk < k2; ++kk) {  // pass 1: entries per local row of this tile row
        const int r = pair_runs[kk];
        for (long long e = run_start[r]; e < run_start[r + 1]; ++e) ++rc[pix[e] >> 4];
      }
      long long acc = rank;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        cur[i] = acc;
        acc += rc[i];
      }
      for (int kk = k; kk < k2; ++kk) {  // pass 2: ranks by pixel id
        const int r = pair_runs[kk];
        const int lt = (int)(run_tile[r] & 0xffffffu);
        const long long ox = (long long)(lt % tiles_x) * SLM_TILE, oy = (long long)ty * SLM_TILE;
        for (long long e = run_start[r]; e < run_start[r + 1]; ++e) {
          const int pl = pix[e];
          const long long pos = cur[pl >> 4]++;
          g_pixel_ids[pos] = (oy + (pl >> 4)) * W + ox + (pl & 15);
          g_gaussian_ids[pos] = gid;
          g_source_index[pos] = pos_pix[e - e_base];
        }
      }
      rank = acc;
      k = k2;
    }
  }
}

extern "C" {

int slm_pairs_prepare(const int* cnt, int V, long long G, long long* cntV, int* flagV, int* flagT, cudaStream_t s) {
  k_pairs_prepare<<<slm_blocks((long long)V * G, 256), 256, 0, s>>>(cnt, V, G, cntV, flagV, flagT);
  return slm_cuda_status();
}

int slm_pairs_emit(const int* cnt, int V, long long G, const int* pair_of, const long long* vscan, const int* tscan,
                   const SlmSplat* splats, long long* pair_off, int* pair_gid, uint32_t* pair_vm, SlmPairGeo* geo,
                   int* pidx, int* gpo, int n_pairs, long long n_entries, cudaStream_t s) {
  if (V <= 0 || V > 255) return SLM_ERR_ARG;
  const long long GB = PE_SLOTS / V;
  k_pairs_emit<<<slm_blocks((G + GB - 1) / GB, 1, 1LL << 30), 256, 0, s>>>(cnt, V, G, pair_of, vscan, tscan, splats, pair_off,
                                                                  pair_gid, pair_vm, geo, pidx, gpo, n_pairs, n_entries);
  return slm_cuda_status();
}

int slm_invert_perm(const int* perm, long long n, int* inv, cudaStream_t s) {
  if (n <= 0) return SLM_OK;
  k_invert_perm<<<slm_blocks(n, 256), 256, 0, s>>>(perm, n, inv);
  return slm_cuda_status();
}

int slm_iota_u32(uint32_t* out, long long n, cudaStream_t s) {
  if (n <= 0) return SLM_OK;
  k_iota_u32<<<slm_blocks(n, 256), 256, 0, s>>>(out, n);
  return slm_cuda_status();
}

int slm_export_view(const int* tile_run_off, int t0, int n_tiles, int tiles_x, int W, const long long* run_start,
                    const int* run_q, const uint32_t* run_tile, const int* pair_gid, const uint32_t* pair_vm,
                    const int* pair_run_off, const int* pair_runs, int n_pairs, int view, const uint8_t* pix,
                    const long long* px_off, const long long* g_off, long long e_base, long long* pos_pix,
                    long long* pixel_ids, long long* gaussian_ids, long long* g_pixel_ids, long long* g_gaussian_ids,
                    long long* g_source_index, cudaStream_t s) {
  if (n_tiles <= 0) return SLM_OK;
  k_export_pixel<<<(unsigned)std::min(n_tiles, 148 * 16), 256, 0, s>>>(tile_run_off, t0, n_tiles, tiles_x, W, run_start,
                                                                     run_q, pair_gid, pix, px_off, e_base, pos_pix,
                                                                     pixel_ids, gaussian_ids);
  if (n_pairs > 0)
    k_export_gauss<<<slm_blocks(n_pairs, 128, 1LL << 30), 128, 0, s>>>(
        n_pairs, view, tiles_x, W, pair_vm, pair_gid, pair_run_off, pair_runs, run_tile, run_start, pix, g_off, e_base,
        pos_pix, g_pixel_ids, g_gaussian_ids, g_source_index);
  return slm_cuda_status();
}

int slm_pair_geo_size() { return (int)sizeof(SlmPairGeo); }

}  // extern "C"
