// Persistent, warp-specialised J / J^T / fused J^T W J product kernel over the
// run-ordered gradient cache (ref: jacobian.py:419-483).
//
// Why fused: u at a tile's pixels depends only on that tile's runs and J^T(W u)
// for those runs needs u only at that tile's pixels, so J^T W J p is computed
// tile by tile with u kept in shared memory; the cache is read from HBM once
// per product (the J^T pass re-reads the tile's entries from L2).
//
// Structure (one CTA per SM slot, looping over tiles):
//   producer warp : for every chunk (<= 32 runs, <= 512 entries, cut at run
//                   boundaries; table built once per cache) of every tile and
//                   pass, wait for a free ring stage and issue TMA bulk copies
//                   (cp.async.bulk) of the chunk's entries (5 x f32 + u8), its
//                   runs' 64-byte parameter records and run starts; completion
//                   is signalled on the stage's full mbarrier.
//   8 consumer warps: wait full, take the chunk's runs round-robin with lanes
//                   over each run's entries (all reads from shared memory),
//                   arrive on the stage's empty mbarrier.  A named barrier among
//                   the consumers only separates pass J, the per-tile u
//                   reduction and pass J^T.
//   pass J  : per-warp shared pixel accumulators (a run never repeats a pixel),
//             summed in fixed warp order -> deterministic, no atomics.
//   pass J^T: 9 partials per run, 16-shuffle reduce-scatter, one store per run.
#include "chain.cuh"

#define NW 8
#define NT (32 * (NW + 1))
#define CH 512           // max entries per chunk
#define CR 32            // max runs per chunk
#define CHF (CH + 8)     // f32 stage slots (start aligned down to 4 entries)
#define CHB (CH + 32)    // u8 stage slots (start aligned down to 16 entries)
#define NS 6             // ring stages
#define PAR 16           // floats per run parameter record
#define TMETA 128        // producer chunk-metadata window

#define MODE_J 1
#define MODE_WRITEU 2
#define MODE_JT 4

#define ST_F (5 * CHF * 4)
#define ST_PIX CHB
#define ST_PAR (CR * PAR * 4)
#define ST_RS ((CR + 4) * 8)
#define ST_HDR 16
#define ST_BYTES (ST_F + ST_PIX + ST_PAR + ST_RS + ST_HDR)
static_assert(ST_F % 16 == 0 && (ST_F + ST_PIX) % 16 == 0 && ST_PAR % 16 == 0 && ST_RS % 16 == 0 &&
                  ST_BYTES % 16 == 0,
              "stage sections must stay 16-byte aligned for cp.async.bulk");

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(NW * 32) : "memory"); }

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

__device__ __forceinline__ int view_of_tile(const int* __restrict__ vtb, int n_views, int t) {
  int v = 0;
  while (v + 1 < n_views && vtb[v + 1] <= t) ++v;
  return v;
}

// ---------------------------------------------------------------------------
// per-product run parameter records (64 B, contiguous per chunk)
//   P[0..1] splat centre minus tile pixel-centre origin, P[2..4] conic,
//   P[5] inv_o * m_opa, P[6..10] m_mu0, m_mu1, m_cov0/2, m_cov1, m_cov2/2,
//   P[11..13] m_col, P[14] inv_o
// ---------------------------------------------------------------------------
template <bool WITH_M>
__global__ void k_run_params(SlmTileArgs A, long long n_runs, float* __restrict__ out) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n_runs;
       r += (long long)gridDim.x * blockDim.x) {
    const uint32_t tg = A.run_tile[r];
    const SlmView vw = A.views[tg >> 24];
    const int lt = (int)(tg & 0xffffffu);
    const int tiles_x = (vw.W + SLM_TILE - 1) / SLM_TILE;
    const double ox = (double)((lt % tiles_x) * SLM_TILE) + 0.5, oy = (double)((lt / tiles_x) * SLM_TILE) + 0.5;
    const int q = A.run_q[r];
    const SlmPairGeo g = A.geo[q];
    float P[16];
    P[0] = (float)(g.mx - ox);
    P[1] = (float)(g.my - oy);
    P[2] = g.ka; P[3] = g.kb; P[4] = g.kc;
    P[14] = g.inv_o;
    P[15] = 0.f;
    if (WITH_M) {
      const PairM m = reinterpret_cast<const PairM*>(A.pm)[q];
      P[5] = g.inv_o * m.b.y;
      P[6] = m.a.x; P[7] = m.a.y; P[8] = 0.5f * m.a.z; P[9] = m.a.w; P[10] = 0.5f * m.b.x;
      P[11] = m.b.z; P[12] = m.b.w; P[13] = m.c.x;
    } else {
#pragma unroll
      for (int i = 5; i < 14; ++i) P[i] = 0.f;
    }
    float4* o = reinterpret_cast<float4*>(out + r * PAR);
    o[0] = make_float4(P[0], P[1], P[2], P[3]);
    o[1] = make_float4(P[4], P[5], P[6], P[7]);
    o[2] = make_float4(P[8], P[9], P[10], P[11]);
    o[3] = make_float4(P[12], P[13], P[14], P[15]);
  }
}

// ---------------------------------------------------------------------------
// chunk table: per tile, run-aligned chunks of <= CR runs and <= CH entries
// ---------------------------------------------------------------------------
template <bool FILL>
__global__ void k_tile_chunks(const int* __restrict__ tile_run_off, int n_tiles,
                              const long long* __restrict__ run_start, const int* __restrict__ tile_chunk_off,
                              int* __restrict__ out /* count per tile or chunk_run */) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n_tiles; t += gridDim.x * blockDim.x) {
    const int r0 = tile_run_off[t], r1 = tile_run_off[t + 1];
    int nc = 0, k0 = r0;
    long long acc = 0;
    for (int r = r0; r < r1; ++r) {
      const long long n = run_start[r + 1] - run_start[r];
      if (r > k0 && (acc + n > CH || r - k0 >= CR)) {
        if (FILL) out[tile_chunk_off[t] + nc] = k0;
        ++nc;
        k0 = r;
        acc = 0;
      }
      acc += n;
    }
    if (r1 > r0) {
      if (FILL) out[tile_chunk_off[t] + nc] = k0;
      ++nc;
    }
    if (!FILL) out[t] = nc;
  }
}

// ---------------------------------------------------------------------------
// the product kernel
// ---------------------------------------------------------------------------
struct Ent {
  float ae, at, d0, d1, d2;
  int pl;
};

__device__ __forceinline__ uint8_t* stage_ptr(uint8_t* ring, int s) { return ring + (size_t)s * ST_BYTES; }

__host__ __device__ constexpr size_t stream_smem_bytes(int mode) {
  return 256 * 16 + ((mode & MODE_J) ? 3 * NW * 256 * 4 : 0) + (size_t)NS * ST_BYTES + TMETA * 32;
}

struct ChunkMeta {
  int k0, k1;
  long long e0, e1;
};

template <int MODE>
__global__ void __launch_bounds__(NT) k_stream(SlmTileArgs A) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t full[NS], empty[NS];
  unsigned char* sp = smem;
  float4* s_u = reinterpret_cast<float4*>(sp);
  sp += 256 * 16;
  float* s_acc = reinterpret_cast<float*>(sp);
  sp += (MODE & MODE_J) ? 3 * NW * 256 * 4 : 0;
  uint8_t* ring = sp;
  sp += (size_t)NS * ST_BYTES;
  ChunkMeta* tmeta = reinterpret_cast<ChunkMeta*>(sp);

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int n_pass = ((MODE & MODE_J) ? 1 : 0) + ((MODE & MODE_JT) ? 1 : 0);

  if (warp == NW) {
    // ------------------------------ producer ------------------------------
    unsigned g = 0;
    for (int t = blockIdx.x; t < A.n_tiles; t += gridDim.x) {
      const int c0 = A.tile_chunk_off[t], c1 = A.tile_chunk_off[t + 1];
      for (int pass = 0; pass < n_pass; ++pass) {
        for (int w0 = c0; w0 < c1; w0 += TMETA) {
          const int wn = min(TMETA, c1 - w0);
          __syncwarp();
          for (int i = lane; i < wn; i += 32) {
            ChunkMeta m;
            m.k0 = A.chunk_run[w0 + i];
            m.k1 = A.chunk_run[w0 + i + 1];
            m.e0 = A.run_start[m.k0];
            m.e1 = A.run_start[m.k1];
            tmeta[i] = m;
          }
          __syncwarp();
          if (lane == 0) {
            for (int i = 0; i < wn; ++i, ++g) {
              const int s = (int)(g % NS);
              if (g >= NS) mbar_wait(&empty[s], ((g / NS) - 1) & 1u);
              const ChunkMeta m = tmeta[i];
              uint8_t* st = stage_ptr(ring, s);
              const long long a4 = m.e0 & ~3LL, z4 = (m.e1 + 3) & ~3LL;
              const long long a16 = m.e0 & ~15LL, z16 = (m.e1 + 15) & ~15LL;
              const long long a2 = m.k0 & ~1LL, z2 = (m.k1 + 2) & ~1LL;
              const unsigned bf = (unsigned)(z4 - a4) * 4u, bb = (unsigned)(z16 - a16);
              const unsigned bp = (unsigned)(m.k1 - m.k0) * PAR * 4u, br = (unsigned)(z2 - a2) * 8u;
              int* hdr = reinterpret_cast<int*>(st + ST_F + ST_PIX + ST_PAR + ST_RS);
              hdr[0] = m.k1 - m.k0;
              hdr[1] = (int)(m.k0 - a2);
              hdr[2] = m.k0;
              asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
              mbar_arrive_tx(&full[s], 5u * bf + bb + bp + br);
              float* sf = reinterpret_cast<float*>(st);
              bulk_g2s(sf + 0 * CHF, A.ae + a4, bf, &full[s]);
              bulk_g2s(sf + 1 * CHF, A.at + a4, bf, &full[s]);
              bulk_g2s(sf + 2 * CHF, A.d0 + a4, bf, &full[s]);
              bulk_g2s(sf + 3 * CHF, A.d1 + a4, bf, &full[s]);
              bulk_g2s(sf + 4 * CHF, A.d2 + a4, bf, &full[s]);
              bulk_g2s(st + ST_F, A.pix + a16, bb, &full[s]);
              bulk_g2s(st + ST_F + ST_PIX, A.run_par + (size_t)m.k0 * PAR, bp, &full[s]);
              bulk_g2s(st + ST_F + ST_PIX + ST_PAR, A.run_start + a2, br, &full[s]);
            }
          }
        }
      }
    }
    return;
  }

  // ------------------------------ consumers -------------------------------
  unsigned g = 0;
  float* acc0 = s_acc + (0 * NW + warp) * 256;
  float* acc1 = s_acc + (1 * NW + warp) * 256;
  float* acc2 = s_acc + (2 * NW + warp) * 256;
  const int p = threadIdx.x;
  for (int t = blockIdx.x; t < A.n_tiles; t += gridDim.x) {
    const int v = view_of_tile(A.view_tile_base, A.n_views, t);
    const SlmView vw = A.views[v];
    const int tiles_x = (vw.W + SLM_TILE - 1) / SLM_TILE;
    const int lt = t - A.view_tile_base[v];
    const int px = (lt % tiles_x) * SLM_TILE + (p & 15), py = (lt / tiles_x) * SLM_TILE + (p >> 4);
    const bool inside = px < vw.W && py < vw.H;
    const long long gp = vw.pix_base + (long long)py * vw.W + px;
    const int c0 = A.tile_chunk_off[t], c1 = A.tile_chunk_off[t + 1];

    if (MODE & MODE_J) {
      for (int i = lane; i < 256; i += 32) acc0[i] = acc1[i] = acc2[i] = 0.f;
      for (int ci = c0; ci < c1; ++ci, ++g) {
        const int s = (int)(g % NS);
        mbar_wait(&full[s], (g / NS) & 1u);
        const uint8_t* st = stage_ptr(ring, s);
        const int* hdr = reinterpret_cast<const int*>(st + ST_F + ST_PIX + ST_PAR + ST_RS);
        const int nr = hdr[0];
        const long long* rs = reinterpret_cast<const long long*>(st + ST_F + ST_PIX + ST_PAR) + hdr[1];
        const float* sf = reinterpret_cast<const float*>(st);
        const uint8_t* spx = st + ST_F;
        const long long b4 = rs[0] & ~3LL, b16 = rs[0] & ~15LL;
        for (int i = warp; i < nr; i += NW) {
          const float* P = reinterpret_cast<const float*>(st + ST_F + ST_PIX) + i * PAR;
          const float p0 = P[0], p1 = P[1], ka = P[2], kb = P[3], kc = P[4], a0 = P[5], m0 = P[6], m1 = P[7];
          const float m2 = P[8], m3 = P[9], m4 = P[10], q0 = P[11], q1 = P[12], q2 = P[13];
          const int f0 = (int)(rs[i] - b4), n = (int)(rs[i + 1] - rs[i]);
          const int x0 = (int)(rs[i] - b16);
          for (int j = lane; j < n; j += 32) {
            const float ae = sf[0 * CHF + f0 + j], at = sf[1 * CHF + f0 + j];
            const float d0 = sf[2 * CHF + f0 + j], d1 = sf[3 * CHF + f0 + j], d2 = sf[4 * CHF + f0 + j];
            const int pl = spx[x0 + j];
            const float dx = (float)(pl & 15) - p0, dy = (float)(pl >> 4) - p1;
            const float e1 = ka * dx + kb * dy, e2 = kb * dx + kc * dy;
            const float da = ae * (a0 + e1 * m0 + e2 * m1 + e1 * e1 * m2 + e1 * e2 * m3 + e2 * e2 * m4);
            acc0[pl] += d0 * da + at * q0;
            acc1[pl] += d1 * da + at * q1;
            acc2[pl] += d2 * da + at * q2;
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
      consumer_sync();
      float u0 = 0.f, u1 = 0.f, u2 = 0.f;
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        u0 += s_acc[(0 * NW + w) * 256 + p];
        u1 += s_acc[(1 * NW + w) * 256 + p];
        u2 += s_acc[(2 * NW + w) * 256 + p];
      }
      float4 uw = make_float4(0.f, 0.f, 0.f, 0.f);
      if (inside) {
        const float4 wt = A.gradr ? A.gradr[gp] : make_float4(1.f, 1.f, 1.f, 0.f);
        uw = make_float4(u0 * wt.x, u1 * wt.y, u2 * wt.z, 0.f);
        if (MODE & MODE_WRITEU) A.u_out[gp] = uw;
      }
      s_u[p] = uw;
    } else {
      s_u[p] = inside ? A.u[gp] : make_float4(0.f, 0.f, 0.f, 0.f);
    }

    if (MODE & MODE_JT) {
      consumer_sync();
      for (int ci = c0; ci < c1; ++ci, ++g) {
        const int s = (int)(g % NS);
        mbar_wait(&full[s], (g / NS) & 1u);
        const uint8_t* st = stage_ptr(ring, s);
        const int* hdr = reinterpret_cast<const int*>(st + ST_F + ST_PIX + ST_PAR + ST_RS);
        const int nr = hdr[0], kg = hdr[2];
        const long long* rs = reinterpret_cast<const long long*>(st + ST_F + ST_PIX + ST_PAR) + hdr[1];
        const float* sf = reinterpret_cast<const float*>(st);
        const uint8_t* spx = st + ST_F;
        const long long b4 = rs[0] & ~3LL, b16 = rs[0] & ~15LL;
        for (int i = warp; i < nr; i += NW) {
          const float* P = reinterpret_cast<const float*>(st + ST_F + ST_PIX) + i * PAR;
          const float p0 = P[0], p1 = P[1], ka = P[2], kb = P[3], kc = P[4], io = P[14];
          const int f0 = (int)(rs[i] - b4), n = (int)(rs[i + 1] - rs[i]);
          const int x0 = (int)(rs[i] - b16);
          float a[16];
#pragma unroll
          for (int k = 0; k < 16; ++k) a[k] = 0.f;
          for (int j = lane; j < n; j += 32) {
            const float ae = sf[0 * CHF + f0 + j], at = sf[1 * CHF + f0 + j];
            const float d0 = sf[2 * CHF + f0 + j], d1 = sf[3 * CHF + f0 + j], d2 = sf[4 * CHF + f0 + j];
            const int pl = spx[x0 + j];
            const float4 uu = s_u[pl];
            const float dx = (float)(pl & 15) - p0, dy = (float)(pl >> 4) - p1;
            const float e1 = ka * dx + kb * dy, e2 = kb * dx + kc * dy;
            const float sa = d0 * uu.x + d1 * uu.y + d2 * uu.z;
            const float tt = sa * ae;
            a[0] += tt * e1;
            a[1] += tt * e2;
            a[2] += 0.5f * tt * e1 * e1;
            a[3] += tt * e1 * e2;
            a[4] += 0.5f * tt * e2 * e2;
            a[5] += tt;
            a[6] += at * uu.x;
            a[7] += at * uu.y;
            a[8] += at * uu.z;
          }
          const float sum = warp_reduce_scatter16(a, lane);
          const int slot = rs16_slot(lane);
          if (!(lane & 1) && slot < 9) A.out[(size_t)(kg + i) * 9 + slot] = slot == 5 ? sum * io : sum;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
    }
    consumer_sync();  // s_u / s_acc are reused by the next tile
  }
}

template <int MODE>
static int launch_stream(const SlmTileArgs* a, cudaStream_t st) {
  if (a->n_tiles <= 0) return SLM_OK;
  const size_t bytes = stream_smem_bytes(MODE);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_stream<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    configured = true;
  }
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_stream<MODE>, NT, bytes);
  if (per_sm < 1) per_sm = 1;
  const int grid = (int)std::min<long long>((long long)a->n_tiles, (long long)sms * per_sm);
  k_stream<MODE><<<grid, NT, bytes, st>>>(*a);
  return slm_cuda_status();
}

extern "C" {

int slm_run_params(const SlmTileArgs* a, long long n_runs, int with_m, float* out, cudaStream_t st) {
  if (n_runs <= 0) return SLM_OK;
  const unsigned b = slm_blocks(n_runs, 256, 1LL << 30);
  if (with_m) k_run_params<true><<<b, 256, 0, st>>>(*a, n_runs, out);
  else k_run_params<false><<<b, 256, 0, st>>>(*a, n_runs, out);
  return slm_cuda_status();
}

int slm_tile_chunks(const int* tile_run_off, int n_tiles, const long long* run_start, const int* tile_chunk_off,
                    int* out, int fill, cudaStream_t st) {
  if (n_tiles <= 0) return SLM_OK;
  const unsigned b = slm_blocks(n_tiles, 128, 1LL << 30);
  if (fill) k_tile_chunks<true><<<b, 128, 0, st>>>(tile_run_off, n_tiles, run_start, tile_chunk_off, out);
  else k_tile_chunks<false><<<b, 128, 0, st>>>(tile_run_off, n_tiles, run_start, tile_chunk_off, out);
  return slm_cuda_status();
}

// u = J p (a->gradr weights it) written to a->u_out
int slm_apply_j(const SlmTileArgs* a, cudaStream_t st) { return launch_stream<MODE_J | MODE_WRITEU>(a, st); }

// J^T partials per run from the per-pixel a->u
int slm_apply_jt_runs(const SlmTileArgs* a, cudaStream_t st) { return launch_stream<MODE_JT>(a, st); }

// fused: J^T partials of (grad_r_sq * J p) per run; u never leaves the SM
int slm_jtwj_runs(const SlmTileArgs* a, cudaStream_t st) { return launch_stream<MODE_J | MODE_JT>(a, st); }

}  // extern "C"
