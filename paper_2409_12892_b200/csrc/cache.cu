// Gradient-cache assembly: pixel segments and (gaussian, view) pairs.
//
// The gaussian-order record stream itself (sortCacheByGaussians, PAPER:273,
// 305-306) is written directly by the FILL raster pass (raster.cu): pairs are
// numbered in (view, gid) order and each pair's block is filled in pixel
// row-major order, so one view's gaussian-order sequence equals the
// reference's np.lexsort((pixel_ids, gaussian_ids)) (ref: jacobian.py:93-105)
// with no sort at all.
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

int slm_pair_geo_size() { return (int)sizeof(SlmPairGeo); }

}  // extern "C"
