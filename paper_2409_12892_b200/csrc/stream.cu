// Persistent, warp-specialised J / J^T / fused J^T W J product kernel over the
// run-ordered gradient cache (ref: jacobian.py:419-483).
//
// Why fused: u at a tile's pixels depends only on that tile's runs and J^T(W u)
// for those runs needs u only at that tile's pixels, so J^T W J p is computed
// tile by tile with u kept in shared memory; the cache is read from HBM once
// per product (the J^T pass re-reads the tile's entries from L2).
//
// Structure (2 persistent CTAs per SM, tiles claimed from a global counter):
//   producer warp : for every chunk (<= 64 runs whose packed image fits one
//                   25 KB ring stage, cut at run boundaries; table built once
//                   per cache) of every tile and pass, wait for a free stage
//                   and issue TMA bulk copies (cp.async.bulk) of the chunk's
//                   records (float4 + float + u8 = 21 B per entry), its runs'
//                   32-byte static records and (offset | length) words and the
//                   J^T schedule, plus cp.async gathers of the runs' 48-byte
//                   pair forward chain m (J pass); completion is signalled on
//                   the stage's full mbarrier.
//   8 consumer warps: wait full, work from shared memory only, arrive on the
//                   stage's empty mbarrier.  A named barrier among the
//                   consumers only separates pass J, the per-tile u reduction
//                   and pass J^T.
//   pass J  : one run per warp, lanes over its entries, per-warp shared pixel
//             accumulators (a run never repeats a pixel), summed in fixed warp
//             order -> deterministic, no atomics.
//   pass J^T: GL-lane groups (8) on the chunk's length-sorted schedule, 9
//             partials per run, GL-lane reduce-scatter, one 32-byte record per run.
#include "chain.cuh"

#define NW 8
#define NT (32 * (NW + 1))
#ifndef SLM_NS
#define SLM_NS 3
#endif
#define CR SLM_CHUNK_RUNS  // max runs per chunk (64)
static_assert(CR % 32 == 0 && CR <= 255, "run slots are bytes, 32 per J^T round");
#define NS SLM_NS        // ring stages
#ifndef SLM_JT_UNROLL
#define SLM_JT_UNROLL 2
#endif
constexpr int kJtUnroll = SLM_JT_UNROLL;  // J^T entry-loop unroll (tuning)
#ifndef SLM_JT_GL
#define SLM_JT_GL 8
#endif
#ifndef SLM_DG_GL
#define SLM_DG_GL 4
#endif
// lanes per run in the J^T and diag passes (groups of GL lanes, 32 / GL runs
// per warp at a time): the per-run reduce-scatter costs log2(GL) shuffle
// levels per GL values, so narrower groups spend fewer shuffles per run but
// walk each run longer.  Measured at C3: diag 4 lanes 14.84 -> 14.56 ms
// (40 values to reduce per run); J^T 8 lanes 9.93 vs 10.21 ms with 4 (9 values)
constexpr int kJtGL = SLM_JT_GL, kDgGL = SLM_DG_GL;
static_assert((kJtGL == 4 || kJtGL == 8) && (kDgGL == 4 || kDgGL == 8), "group width");
static_assert(CR % (NW * 32 / 8) == 0, "J^T rounds");

// GL-lane reduce-scatter of NB blocks of GL values: lane lg ends with the
// group total of value b * GL + lg in res[b]; a fixed pattern, so the sums
// are deterministic
template <int GL, int NB>
__device__ __forceinline__ void group_rs(const float* a, float* res, int lg) {
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    float v[GL];
#pragma unroll
    for (int k = 0; k < GL; ++k) v[k] = a[b * GL + k];
#pragma unroll
    for (int h = GL / 2; h >= 1; h >>= 1) {
      const bool up = lg & h;
#pragma unroll
      for (int k = 0; k < h; ++k) v[k] = (up ? v[k + h] : v[k]) + __shfl_xor_sync(0xffffffffu, up ? v[k] : v[k + h], h);
    }
    res[b] = v[0];
  }
}

template <int GL>
__device__ __forceinline__ float group_sum(float v) {
#pragma unroll
  for (int h = GL / 2; h >= 1; h >>= 1) v += __shfl_xor_sync(0xffffffffu, v, h);
  return v;
}

// the 8 J^T partials as stored: a[2] and a[4] carry 1/2, a[5] the 1/o factor
__device__ __forceinline__ float jt_scale(int vi, float v, float io) {
  return vi == 5 ? v * io : ((vi == 2 || vi == 4) ? 0.5f * v : v);
}
__device__ __forceinline__ float jt_scl(int vi) { return (vi == 2 || vi == 4) ? 0.5f : 1.f; }
#define PAR 16           // floats per run parameter record
#define TMETA 64         // producer chunk-metadata window
#define TQ 4             // tile queue depth (producer -> consumers)

#define MODE_J 1
#define MODE_WRITEU 2
#define MODE_JT 4
#define MODE_DIAG 8
#define DIAG_M 40        // diag moment floats per run (34 used, see the diag pass)

// one ring stage (ST_BYTES): a packed per-chunk region
//   rec4 | d2 | pix | static run records | pair m | run starts
// whose section offsets follow from the chunk's entries and runs (so a chunk
// of long runs carries more entries and a chunk of short runs more runs),
// then the J^T schedule and the header at fixed offsets
#ifndef SLM_STAGE
#define SLM_STAGE 25680  // the largest stage that keeps 2 CTAs / SM (static_assert below)
#endif
#define ST_BYTES SLM_STAGE
#define ST_HDR 32
#define ST_PERM CR
#define OFF_HDR (ST_BYTES - ST_HDR)
#define OFF_PERM (OFF_HDR - ST_PERM)
#define ST_DYN OFF_PERM  // capacity of the packed region
static_assert(OFF_PERM % 16 == 0 && OFF_HDR % 16 == 0 && ST_BYTES % 16 == 0,
              "stage sections must stay 16-byte aligned for cp.async.bulk");

struct StageLayout {
  int d2, pix, pst, pdy, rf, end;  // byte offsets of the sections, end of the packed region
};
__host__ __device__ __forceinline__ int al16(int x) { return (x + 15) & ~15; }
// e entries, r runs; the d2 / pix / run-word copies are widened to 16-byte
// aligned global ranges (<= e + 6 floats, <= e + 30 bytes, <= r + 6 words)
__host__ __device__ __forceinline__ StageLayout stage_layout(int e, int r) {
  StageLayout L;
  L.d2 = e * 16;
  L.pix = L.d2 + al16((e + 8) * 4);
  L.pst = L.pix + al16(e + 32);
  L.pdy = L.pst + r * 32;
  L.rf = L.pdy + r * 48;
  L.end = L.rf + al16((r + 6) * 4);
  return L;
}

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
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000000;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// global -> shared bulk copy, completion on an mbarrier, with an L2 eviction policy
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
// arrive on the mbarrier once this thread's prior cp.async copies have landed
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(NW * 32) : "memory"); }

// view of global tile t: the number of views after the first whose first
// tile is <= t, counted 32 views per ballot (vtb ascending)
__device__ __forceinline__ int view_of_tile_warp(const int* __restrict__ vtb, int n_views, int t, int lane) {
  int v = 0;
  for (int b = 1; b < n_views; b += 32) {
    const int i = b + lane;
    const unsigned m = __ballot_sync(0xffffffffu, i < n_views && __ldg(vtb + i) <= t);
    v += __popc(m);
    if (m != 0xffffffffu) break;
  }
  return v;
}

// ---------------------------------------------------------------------------
// static run records (once per cache; the scene is fixed during a solve):
//   (c1, c2, ka, kb), (kb, kc, inv_o, slot): the conic (ka, kb, kc) and
//   e = conic (px - mu) at the tile's first pixel centre, so that at tile-local
//   pixel (x, y) e1 = ka x + kb y + c1, e2 = kb x + kc y + c2 (two FFMA2 per
//   entry; c1, c2 formed in fp64); slot = the run's position in pair_runs
//   (J^T / diag outputs go there).  The two float4 halves load as the
//   register pairs (c1, c2), (ka, kb), (kb, kc) the packed FMAs use.
// The per-product forward chain m of the run's pair is gathered per chunk by
// the producer warp (cp.async from the per-pair m of slm_pair_forward).
// ---------------------------------------------------------------------------
__global__ void k_run_static(SlmTileArgs A, long long n_runs, const int* __restrict__ run_slot,
                             float* __restrict__ out) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n_runs;
       r += (long long)gridDim.x * blockDim.x) {
    const uint32_t tg = A.run_tile[r];
    const SlmView vw = A.views[tg >> 24];
    const int lt = (int)(tg & 0xffffffu);
    const int tiles_x = (vw.W + SLM_TILE - 1) / SLM_TILE;
    const double ox = (double)((lt % tiles_x) * SLM_TILE) + 0.5, oy = (double)((lt / tiles_x) * SLM_TILE) + 0.5;
    const int q = A.run_q[r];
    const SlmPairGeo g = A.geo[q];
    const double dx = ox - g.mx, dy = oy - g.my;
    const double c1 = (double)g.ka * dx + (double)g.kb * dy, c2 = (double)g.kb * dx + (double)g.kc * dy;
    float4* o = reinterpret_cast<float4*>(out + r * 8);
    o[0] = make_float4((float)c1, (float)c2, g.ka, g.kb);
    o[1] = make_float4(g.kb, g.kc, g.inv_o, __int_as_float(run_slot[r]));
  }
}

// e = (e1, e2) = conic (px - mu) at tile-local pixel pl of a run: two packed
// FMAs on the run's (ka, kb), (kb, kc), (c1, c2) (RunE, formed once per run)
// (packed 64-bit operands, so the pairs stay in fixed register pairs)
struct RunE {
  uint64_t kab, kbc, c;
};
__device__ __forceinline__ uint64_t pack2(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ RunE run_e_of(const float4& q0, const float4& s1) {
  return RunE{pack2(q0.z, q0.w), pack2(s1.x, s1.y), pack2(q0.x, q0.y)};
}
__device__ __forceinline__ float2 run_e(const RunE& k, int pl) {
  const float x = (float)(pl & 15), y = (float)(pl >> 4);
  uint64_t t, e;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(t) : "l"(k.kbc), "l"(pack2(y, y)), "l"(k.c));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(e) : "l"(k.kab), "l"(pack2(x, x)), "l"(t));
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(e));
  return r;
}

// ---------------------------------------------------------------------------
// chunk table: per tile, run-aligned chunks of <= CR runs whose packed stage
// region (stage_layout) fits ST_DYN bytes
// (FILL=false: chunks per tile; FILL=true: first run of each chunk)
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
      if (r > k0 && (r - k0 >= CR || stage_layout((int)(acc + n), r - k0 + 1).end > ST_DYN)) {
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

// each chunk's group schedule: its runs by decreasing length (ties by index),
// 0xff-padded to 32 slots; one warp per chunk, lane = run
__global__ void k_chunk_perm(const int* __restrict__ chunk_run, long long n_chunks,
                             const long long* __restrict__ run_start, uint8_t* __restrict__ perm,
                             uint32_t* __restrict__ run_fn) {
  constexpr int RL = CR / 32;  // runs per lane
  const int lane = threadIdx.x & 31;
  for (long long c = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; c < n_chunks;
       c += ((long long)gridDim.x * blockDim.x) >> 5) {
    const int k0 = chunk_run[c], n = chunk_run[c + 1] - k0;
    const long long e0 = run_start[k0];
    int len[RL], rank[RL];  // run lengths <= 256: one 32-bit shuffle per comparison
#pragma unroll
    for (int h = 0; h < RL; ++h) {
      const int r = lane + 32 * h;
      const long long s0 = r < n ? run_start[k0 + r] : 0;
      len[h] = r < n ? (int)(run_start[k0 + r + 1] - s0) : -1;
      rank[h] = 0;
      // the run's word: chunk-local first entry | length << 16
      if (r < n) run_fn[k0 + r] = (uint32_t)(s0 - e0) | ((uint32_t)len[h] << 16);
    }
#pragma unroll
    for (int hj = 0; hj < RL; ++hj) {
      if (32 * hj >= n) break;  // warp-uniform
#pragma unroll 8
      for (int j = 0; j < 32; ++j) {
        const int lj = __shfl_sync(0xffffffffu, len[hj], j);
        const int rj = j + 32 * hj;
#pragma unroll
        for (int h = 0; h < RL; ++h) rank[h] += (lj > len[h]) || (lj == len[h] && rj < lane + 32 * h);
      }
    }
    uint8_t* pc = perm + c * CR;
#pragma unroll
    for (int h = 0; h < RL; ++h) pc[lane + 32 * h] = 0xff;
    __syncwarp();
#pragma unroll
    for (int h = 0; h < RL; ++h)
      if (lane + 32 * h < n) pc[rank[h]] = (uint8_t)(lane + 32 * h);
  }
}

// ---------------------------------------------------------------------------
// the product kernel
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint8_t* stage_ptr(uint8_t* ring, int s) { return ring + (size_t)s * ST_BYTES; }

// ring depth: the J modes spend 32 KB on per-warp pixel accumulators; the
// J^T-only and diag modes use that room for one more stage
__host__ __device__ constexpr int ns_of(int mode) { return (mode & MODE_J) ? NS : NS + 1; }

__host__ __device__ constexpr size_t stream_smem_bytes(int mode) {
  return 256 * 16 + ((mode & MODE_J) ? (size_t)NW * 256 * 16 : 0) + ((mode & MODE_DIAG) ? 256 * 16 : 0) +
         (size_t)ns_of(mode) * ST_BYTES + TMETA * 24;
}

// 2 CTAs / SM: 228 KB of shared memory per SM, 1 KB reserved per CTA, and a
// few hundred bytes of static barriers / tile queue per CTA
static_assert(stream_smem_bytes(MODE_J | MODE_JT) + 256 <= 228 * 1024 / 2 - 1024 &&
                  stream_smem_bytes(MODE_JT) + 256 <= 228 * 1024 / 2 - 1024 &&
                  stream_smem_bytes(MODE_DIAG) + 256 <= 228 * 1024 / 2 - 1024,
              "the streaming kernels must keep 2 CTAs per SM");

struct ChunkMeta {
  int k0, k1;
  long long e0, e1;
};

// stage header: [0] runs, [1] run-start offset (k0 - a2), [2] k0 (global run),
// [3] d2 offset (e0 - a4), [4] pix offset (e0 - a16)
template <int MODE, int JGL = kJtGL>
__global__ void __launch_bounds__(NT, 2) k_stream(SlmTileArgs A) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int NSM = ns_of(MODE);
  __shared__ uint64_t full[NSM], empty[NSM];
  // tile queue: the producer claims tiles from a global counter (dynamic
  // load balance over tiles of very different sizes; results do not depend
  // on which CTA runs a tile) and hands them to the consumers in order
  __shared__ uint64_t tq_full[TQ], tq_empty[TQ];
  __shared__ int tq[TQ];
  // per queued tile, resolved once by the producer: (first pixel lo, hi, view
  // width, valid columns | valid rows << 8) and the tile's chunk range -- the
  // consumers start a tile with shared-memory reads instead of a chain of
  // dependent global loads (view search, view record, chunk offsets)
  __shared__ int4 tqi[TQ];
  __shared__ int2 tqc[TQ];
  unsigned char* sp = smem;
  float4* s_u = reinterpret_cast<float4*>(sp);
  sp += 256 * 16;
  float4* s_acc = reinterpret_cast<float4*>(sp);
  sp += (MODE & MODE_J) ? (size_t)NW * 256 * 16 : 0;
  float4* s_c = reinterpret_cast<float4*>(sp);  // diag: the rhs colour gradient per pixel
  sp += (MODE & MODE_DIAG) ? 256 * 16 : 0;
  uint8_t* ring = sp;
  sp += (size_t)NSM * ST_BYTES;
  ChunkMeta* tmeta = reinterpret_cast<ChunkMeta*>(sp);

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NSM; ++s) {
      mbar_init(&full[s], 1 + 32);  // producer lane 0 (expect_tx) + 32 cp.async arrivals
      mbar_init(&empty[s], NW);
    }
    for (int s = 0; s < TQ; ++s) {
      mbar_init(&tq_full[s], 1);
      mbar_init(&tq_empty[s], NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int n_pass = ((MODE & MODE_J) ? 1 : 0) + ((MODE & (MODE_JT | MODE_DIAG)) ? 1 : 0);

  if (warp == NW) {
    // ------------------------------ producer ------------------------------
    const uint64_t keep = policy_evict_last(), drop = policy_evict_first();
    unsigned g = 0;
    for (unsigned tk = 0;; ++tk) {
      int t = 0;
      if (lane == 0) t = A.tile_counter ? atomicAdd(A.tile_counter, 1) : (int)(blockIdx.x + tk * gridDim.x);
      t = __shfl_sync(0xffffffffu, t, 0);
      int c0 = 0, c1 = 0;
      int4 ti = make_int4(0, 0, 0, 0);
      if (t < A.n_tiles) {
        const int v = view_of_tile_warp(A.view_tile_base, A.n_views, t, lane);
        const SlmView vw = A.views[v];
        const int tiles_x = (vw.W + SLM_TILE - 1) / SLM_TILE;
        const int lt = t - A.view_tile_base[v];
        const int x0 = (lt % tiles_x) * SLM_TILE, y0 = (lt / tiles_x) * SLM_TILE;
        const long long gp0 = vw.pix_base + (long long)y0 * vw.W + x0;
        ti = make_int4((int)(unsigned)(gp0 & 0xffffffffLL), (int)(gp0 >> 32), vw.W,
                       min(SLM_TILE, vw.W - x0) | (min(SLM_TILE, vw.H - y0) << 8));
        c0 = A.tile_chunk_off[t];
        c1 = A.tile_chunk_off[t + 1];
      }
      if (lane == 0) {
        const unsigned qs = tk % TQ;
        if (tk >= TQ) mbar_wait(&tq_empty[qs], ((tk / TQ) - 1) & 1u);
        tq[qs] = t < A.n_tiles ? t : -1;
        tqi[qs] = ti;
        tqc[qs] = make_int2(c0, c1);
        mbar_arrive(&tq_full[qs]);
      }
      if (t >= A.n_tiles) break;
      for (int pass = 0; pass < n_pass; ++pass) {
        // the cache of a tile is read twice in the fused mode: keep it in L2
        // for the J^T pass, then let it go
        const uint64_t pol = (n_pass == 2 && pass == 0) ? keep : drop;
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
          const bool gather = (MODE & MODE_J) && pass == 0 && A.pm;
          constexpr int RL = CR / 32;  // runs per producer lane
          int qn[RL];                  // pairs of this lane's runs in the next chunk (prefetched)
#pragma unroll
          for (int h = 0; h < RL; ++h)
            qn[h] = gather && lane + 32 * h < tmeta[0].k1 - tmeta[0].k0 ? A.run_q[tmeta[0].k0 + lane + 32 * h] : 0;
          for (int i = 0; i < wn; ++i, ++g) {
            const int s = (int)(g % NSM);
            int q[RL];
#pragma unroll
            for (int h = 0; h < RL; ++h) {
              q[h] = qn[h];
              if (gather && i + 1 < wn && lane + 32 * h < tmeta[i + 1].k1 - tmeta[i + 1].k0)
                qn[h] = A.run_q[tmeta[i + 1].k0 + lane + 32 * h];
            }
            if (g >= NSM) mbar_wait(&empty[s], ((g / NSM) - 1) & 1u);
            const ChunkMeta m = tmeta[i];
            uint8_t* st = stage_ptr(ring, s);
            const StageLayout L = stage_layout((int)(m.e1 - m.e0), m.k1 - m.k0);
            // per-run forward-chain m of the run's pair (J pass only): lane per run
#pragma unroll
            for (int h = 0; h < RL; ++h) {
              const int r = lane + 32 * h;
              if (gather && r < m.k1 - m.k0) {
                const uint8_t* src = reinterpret_cast<const uint8_t*>(A.pm) + (size_t)q[h] * 48;
                uint8_t* dst = st + L.pdy + r * 48;
                cp_async16(dst, src);
                cp_async16(dst + 16, src + 16);
                cp_async16(dst + 32, src + 32);
              }
            }
            cp_async_mbar_arrive(&full[s]);
            __syncwarp();
            if (lane == 0) {
              const long long a4 = m.e0 & ~3LL, z4 = (m.e1 + 3) & ~3LL;
              const long long a16 = m.e0 & ~15LL, z16 = (m.e1 + 15) & ~15LL;
              const long long aq = m.k0 & ~3LL, zq = (m.k1 + 3) & ~3LL;
              const unsigned b4 = (unsigned)(m.e1 - m.e0) * 16u, bd = (unsigned)(z4 - a4) * 4u;
              const unsigned bx = (unsigned)(z16 - a16), bp = (unsigned)(m.k1 - m.k0) * 32u;
              const unsigned br = (unsigned)(zq - aq) * 4u;
              int* hdr = reinterpret_cast<int*>(st + OFF_HDR);
              hdr[0] = m.k1 - m.k0;
              hdr[1] = (int)(m.k0 - aq);                // first run word / pair index
              hdr[2] = m.k0;
              hdr[3] = 0;
              hdr[4] = L.d2 + (int)(m.e0 - a4) * 4;     // the chunk's first d2
              hdr[5] = L.pix + (int)(m.e0 - a16);       // the chunk's first pixel byte
              hdr[6] = L.pst;
              hdr[7] = L.rf;
              // generic-proxy header writes before the async-proxy copies land
              asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
              mbar_arrive_tx(&full[s], b4 + bd + bx + bp + br + ST_PERM);
              // record streams: device, or the host-mapped offloaded tail
              // (the split is a chunk boundary and e_hbase <= a16 <= a4)
              const bool off = A.rec4_h && m.e0 >= A.e_split;
              const long long hb = off ? A.e_hbase : 0;
              bulk_g2s(st, (off ? A.rec4_h : A.rec4) + (m.e0 - hb), b4, &full[s], pol);
              bulk_g2s(st + L.d2, (off ? A.d2_h : A.d2) + (a4 - hb), bd, &full[s], pol);
              bulk_g2s(st + L.pix, (off ? A.pix_h : A.pix) + (a16 - hb), bx, &full[s], pol);
              bulk_g2s(st + L.pst, A.run_static + (size_t)m.k0 * 8, bp, &full[s], pol);
              bulk_g2s(st + L.rf, A.run_fn + aq, br, &full[s], pol);
              bulk_g2s(st + OFF_PERM, A.chunk_perm + (size_t)(w0 + i) * CR, ST_PERM, &full[s], pol);
            }
            __syncwarp();
          }
        }
      }
    }
    return;
  }

  // ------------------------------ consumers -------------------------------
  unsigned g = 0;
  float4* acc = s_acc + warp * 256;
  const int p = threadIdx.x;
  for (unsigned tk = 0;; ++tk) {
    const unsigned qs = tk % TQ;
    mbar_wait(&tq_full[qs], (tk / TQ) & 1u);
    const int t = tq[qs];
    const int4 ti = tqi[qs];
    const int2 tc = tqc[qs];
    __syncwarp();
    if (lane == 0) mbar_arrive(&tq_empty[qs]);
    if (t < 0) break;
    const int px = p & 15, py = p >> 4;
    const bool inside = px < (ti.w & 0xff) && py < (ti.w >> 8);
    const long long gp = (((long long)ti.y << 32) | (unsigned)ti.x) + (long long)py * ti.z + px;
    const int c0 = tc.x, c1 = tc.y;
    // per-pixel weight / input loaded up front so its latency hides behind the J pass
    float4 wt = make_float4(1.f, 1.f, 1.f, 0.f);
    if (MODE & MODE_J) {
      // only inside pixels use the weight (at the end of the J pass): the
      // load is unpredicated (outside pixels read the tile's first pixel), so
      // no select right after it waits on the load at the tile start
      const long long g0p = ((long long)ti.y << 32) | (unsigned)ti.x;
      if (A.gradr) wt = A.gradr[inside ? gp : g0p];
    } else if (MODE & MODE_DIAG) {
      wt = inside ? A.gradr[gp] : make_float4(0.f, 0.f, 0.f, 0.f);
      s_c[p] = inside && A.u ? A.u[gp] : make_float4(0.f, 0.f, 0.f, 0.f);
    } else {
      wt = inside ? A.u[gp] : make_float4(0.f, 0.f, 0.f, 0.f);
    }

    if (MODE & MODE_J) {
      for (int i = lane; i < 256; i += 32) acc[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      __syncwarp();
      // pass J: one run per warp at a time, lanes over its entries (a run
      // never repeats a pixel, so the per-warp accumulators need no atomics;
      // runs are taken in a fixed order -> deterministic).  Measured faster
      // than flat 32-entry windows with __match_any conflict resolution.
      for (int ci = c0; ci < c1; ++ci, ++g) {
        const int s = (int)(g % NSM);
        mbar_wait(&full[s], (g / NSM) & 1u);
        const uint8_t* st = stage_ptr(ring, s);
        const int* hdr = reinterpret_cast<const int*>(st + OFF_HDR);
        const int nr = hdr[0];
        const uint32_t* rf = reinterpret_cast<const uint32_t*>(st + hdr[7]) + hdr[1];
        const float4* s4 = reinterpret_cast<const float4*>(st);
        const float* sd2 = reinterpret_cast<const float*>(st + hdr[4]);
        const uint8_t* spx = st + hdr[5];
        const float4* PST = reinterpret_cast<const float4*>(st + hdr[6]);
        const float4* PDY = reinterpret_cast<const float4*>(st + hdr[6] + nr * 32);
        for (int i = (warp + ci) & (NW - 1); i < nr; i += NW) {  // rotated: no warp always gets the extra runs
          // static: q0 = (c1, c2, ka, kb), s1 = (kb, kc, io, slot)
          // pair m:  d0 = (m_opa, m0, m1, m2), d1 = (m3, m4, c0, c1), d2m = (c2, -, -, -)
          const float4 q0 = PST[i * 2], s1 = PST[i * 2 + 1];
          const float4 d0 = PDY[i * 3], d1 = PDY[i * 3 + 1];
          const float c2m = PDY[i * 3 + 2].x;
          const float a0 = s1.z * d0.x;
          const uint32_t fn = rf[i];
          const int f0 = (int)(fn & 0xffffu), n = (int)(fn >> 16);
          const float4* pr = s4 + f0;
          const float* pd = sd2 + f0;
          const uint8_t* pp = spx + f0;
          const float2 mc01 = make_float2(d1.z, d1.w);
          const RunE ke = run_e_of(q0, s1);
          for (int j = lane; j < n; j += 32) {
            const float4 r = pr[j];
            const float d2 = pd[j];
            const int pl = pp[j];
            const float2 e = run_e(ke, pl);
            // dalpha = alpha_eff (m_o/o + e1 m0 + e2 m1 + e1^2 m2 + e1 e2 m3 + e2^2 m4)
            const float t1 = fmaf(e.x, d0.w, fmaf(e.y, d1.x, d0.y)), t2 = fmaf(e.y, d1.y, d0.z);
            const float da = r.x * fmaf(e.x, t1, fmaf(e.y, t2, a0));
            float4 a = acc[pl];
            // u_ch += dc/dalpha_ch dalpha + alpha T m_col,ch
            const float2 axy = __ffma2_rn(make_float2(r.z, r.w), make_float2(da, da),
                                          __ffma2_rn(make_float2(r.y, r.y), mc01, make_float2(a.x, a.y)));
            a.x = axy.x;
            a.y = axy.y;
            a.z = fmaf(d2, da, fmaf(r.y, c2m, a.z));
            acc[pl] = a;
          }
          __syncwarp();  // the next run may update the same pixels from other lanes
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
      consumer_sync();
      float u0 = 0.f, u1 = 0.f, u2 = 0.f;
#pragma unroll
      for (int w = 0; w < NW; ++w) {  // fixed warp order -> deterministic
        const float4 a = s_acc[w * 256 + p];
        u0 += a.x;
        u1 += a.y;
        u2 += a.z;
      }
      float4 uw = make_float4(0.f, 0.f, 0.f, 0.f);
      if (inside) {
        uw = make_float4(u0 * wt.x, u1 * wt.y, u2 * wt.z, 0.f);
        if (MODE & MODE_WRITEU) A.u_out[gp] = uw;
      }
      s_u[p] = uw;
    } else {
      // J^T: u per pixel; diag: grad_r_sq per pixel (loaded above)
      s_u[p] = wt;
    }

    if (MODE & MODE_DIAG) {
      consumer_sync();
      // diag(J^T W J) (ref: jacobian.py:486-512) in moment form, plus the
      // J^T partials of the colour gradient (b = -J^T color_grad, ref
      // jacobian.py:411-413) in the same sweep over the cache.  Per entry
      // with w = alpha_eff (e1, e2, e1^2/2, e1 e2, e2^2/2), Aw = sum_ch
      // gr_ch dd_ch^2 (dd = dc/dalpha) and g_ch = gr_ch dd_ch alphaT, a run
      // accumulates
      //   S = sum Aw w w^T (15), V_ch = sum g_ch w (15), T3_ch = sum gr_ch
      //   (alphaT)^2 (3), O = sum Aw alpha_eff^2 (1),
      // so that for a parameter with chain coefficients D (da = w.D) and
      // colour coefficients c_ch, sum gr_ch (dd_ch da + alphaT c_ch)^2 =
      // D^T S D + 2 sum_ch c_ch D.V_ch + sum_ch c_ch^2 T3_ch: the backward
      // applies the pair's chain once per pair instead of once per entry.
      // Same GL-lane groups / length-sorted schedule as the J^T pass; lanes
      // past their run's end add exact zeros (selects).
      const bool rhs = A.u != nullptr;
      constexpr int GL = kDgGL, RPW = 32 / GL, RPR = NW * RPW;  // runs per warp / per round
      const int slot = lane / GL, lg = lane % GL;
      for (int ci = c0; ci < c1; ++ci, ++g) {
        const int s = (int)(g % NSM);
        mbar_wait(&full[s], (g / NSM) & 1u);
        const uint8_t* st = stage_ptr(ring, s);
        const int* hdr = reinterpret_cast<const int*>(st + OFF_HDR);
        const uint32_t* rf = reinterpret_cast<const uint32_t*>(st + hdr[7]) + hdr[1];
        const float4* s4 = reinterpret_cast<const float4*>(st);
        const float* sd2 = reinterpret_cast<const float*>(st + hdr[4]);
        const uint8_t* spx = st + hdr[5];
        for (int rd = 0; rd < CR / RPR && rd * RPR < hdr[0]; ++rd) {  // RPR runs per round, longest first
          const int ri = st[OFF_PERM + rd * RPR + ((warp + ci) & (NW - 1)) * RPW + slot];
          int n = 0, f0 = 0, sl = 0;
          float4 q0 = make_float4(0.f, 0.f, 0.f, 0.f), s1 = q0;
          float io = 0.f;
          if (ri != 0xff) {
            const float4* P4 = reinterpret_cast<const float4*>(st + hdr[6]) + ri * 2;
            q0 = P4[0];
            s1 = P4[1];
            io = s1.z;
            sl = __float_as_int(s1.w);
            const uint32_t fn = rf[ri];
            f0 = (int)(fn & 0xffffu);
            n = (int)(fn >> 16);
          }
          const int nmax = (int)__reduce_max_sync(0xffffffffu, (unsigned)n);
          if (nmax == 0) continue;
          const RunE ke = run_e_of(q0, s1);
          float m[DIAG_M];  // S (15, row-major upper triangle), V (3 x 5), T3 (3), O, pad
#pragma unroll
          for (int k = 0; k < DIAG_M; ++k) m[k] = 0.f;
          float2 a01 = make_float2(0.f, 0.f), a23 = a01, a67 = a01;  // rhs J^T partials
          float a4 = 0.f, a5 = 0.f, a8 = 0.f;
          const float4* pr = s4 + f0;
          const float* pd = sd2 + f0;
          const uint8_t* pp = spx + f0;
          for (int j = lg; j < nmax; j += GL) {
            const bool ok = j < n;
            const float4 r = pr[j];
            const int pl = pp[j];
            const float4 gr = s_u[pl];
            const float ae = ok ? r.x : 0.f, at = ok ? r.y : 0.f;
            const float dd0 = ok ? r.z : 0.f, dd1 = ok ? r.w : 0.f, dd2 = ok ? pd[j] : 0.f;
            const float2 e = run_e(ke, pl);
            const float w0 = ae * e.x, w1 = ae * e.y;
            const float w[5] = {w0, w1, 0.5f * w0 * e.x, w0 * e.y, 0.5f * w1 * e.y};
            const float g0 = gr.x * dd0, g1 = gr.y * dd1, g2 = gr.z * dd2;
            const float Aw = fmaf(g0, dd0, fmaf(g1, dd1, g2 * dd2));
            float aw[5];
#pragma unroll
            for (int i = 0; i < 5; ++i) aw[i] = Aw * w[i];
            int k = 0;
#pragma unroll
            for (int i = 0; i < 5; ++i)
#pragma unroll
              for (int jj = i; jj < 5; ++jj, ++k) m[k] = fmaf(aw[i], w[jj], m[k]);
            const float ga[3] = {g0 * at, g1 * at, g2 * at};
#pragma unroll
            for (int ch = 0; ch < 3; ++ch)
#pragma unroll
              for (int i = 0; i < 5; ++i) m[15 + ch * 5 + i] = fmaf(ga[ch], w[i], m[15 + ch * 5 + i]);
            const float at2 = at * at;
            m[30] = fmaf(gr.x, at2, m[30]);
            m[31] = fmaf(gr.y, at2, m[31]);
            m[32] = fmaf(gr.z, at2, m[32]);
            m[33] = fmaf(Aw * ae, ae, m[33]);
            if (rhs) {  // J^T partials of the colour gradient, as in the J^T pass
              const float4 uu = s_c[pl];
              const float sa = fmaf(dd0, uu.x, fmaf(dd1, uu.y, dd2 * uu.z));
              const float tt = sa * ae;
              const float2 te = __fmul2_rn(make_float2(tt, tt), e);
              a01 = __fadd2_rn(a01, te);
              a23 = __ffma2_rn(make_float2(te.x, te.x), e, a23);
              a4 = fmaf(te.y, e.y, a4);
              a5 += tt;
              a67 = __ffma2_rn(make_float2(at, at), make_float2(uu.x, uu.y), a67);
              a8 = fmaf(at, uu.z, a8);
            }
          }
          // GL-lane reduce-scatter of the 40 moment floats: lane lg ends with
          // values lg + GL b; O (value 33) carries 1/o^2 (opacity da =
          // alpha_eff dopa / o)
          float res[DIAG_M / GL];
          group_rs<GL, DIAG_M / GL>(m, res, lg);
          if (ri != 0xff) {
            float* o = A.out + (size_t)sl * DIAG_M;  // pair-run-slot order
            res[33 / GL] = lg == 33 % GL ? res[33 / GL] * io * io : res[33 / GL];
#pragma unroll
            for (int h = 0; h < DIAG_M / GL; ++h) o[GL * h + lg] = res[h];
          }
          if (rhs) {
            const float a[8] = {a01.x, a01.y, a23.x, a23.y, a4, a5, a67.x, a67.y};
            float ra[8 / GL];
            group_rs<GL, 8 / GL>(a, ra, lg);
            a8 = group_sum<GL>(a8);
            if (ri != 0xff) {
#pragma unroll
              for (int h = 0; h < 8 / GL; ++h) A.rhs8[(size_t)sl * 8 + GL * h + lg] = jt_scale(GL * h + lg, ra[h], io);
              if (lg == 0) A.rhs1[sl] = a8;
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
    }

    if (MODE & MODE_JT) {
      consumer_sync();
      // pass J^T: 32 / GL runs per warp (GL lanes each) from the chunk's
      // length-sorted schedule; the warp's slot block rotates with the chunk
      constexpr int GL = JGL, RPW = 32 / GL, RPR = NW * RPW;
      const int slot = lane / GL, lg = lane % GL;
      for (int ci = c0; ci < c1; ++ci, ++g) {
        const int s = (int)(g % NSM);
        mbar_wait(&full[s], (g / NSM) & 1u);
        const uint8_t* st = stage_ptr(ring, s);
        const int* hdr = reinterpret_cast<const int*>(st + OFF_HDR);
        const uint32_t* rf = reinterpret_cast<const uint32_t*>(st + hdr[7]) + hdr[1];
        const float4* s4 = reinterpret_cast<const float4*>(st);
        const float* sd2 = reinterpret_cast<const float*>(st + hdr[4]);
        const uint8_t* spx = st + hdr[5];
        for (int rd = 0; rd < CR / RPR && rd * RPR < hdr[0]; ++rd) {  // RPR runs per round, longest first
          const int ri = st[OFF_PERM + rd * RPR + ((warp + ci) & (NW - 1)) * RPW + slot];
          int n = 0, f0 = 0;
          float4 q0 = make_float4(0.f, 0.f, 0.f, 0.f), s1 = q0;
          float io = 0.f;
          int sl = 0;
          if (ri != 0xff) {
            const float4* P4 = reinterpret_cast<const float4*>(st + hdr[6]) + ri * 2;
            q0 = P4[0];
            s1 = P4[1];
            io = s1.z;
            sl = __float_as_int(s1.w);
            const uint32_t fn = rf[ri];
            f0 = (int)(fn & 0xffffu);
            n = (int)(fn >> 16);
          }
          const int nmax = __reduce_max_sync(0xffffffffu, (unsigned)n);
          if (nmax == 0) continue;
          // per-run partials: a01 = sum t (e1, e2), a23 = sum t e1 (e1, e2),
          // a4 = sum t e2^2, a5 = sum t, a67 / a8 = sum alpha T u (t = s_alpha
          // alpha_eff).  The group runs to the warp's longest run; lanes past
          // their run's end read in-stage data and add exact zeros (selects,
          // so garbage never reaches the sums): no branch in the loop
          float2 a01 = make_float2(0.f, 0.f), a23 = a01, a67 = a01;
          float a4 = 0.f, a5 = 0.f, a8 = 0.f;
          const float4* pr = s4 + f0;
          const float* pd = sd2 + f0;
          const uint8_t* pp = spx + f0;
          const RunE ke = run_e_of(q0, s1);
#pragma unroll(GL == 4 ? 1 : kJtUnroll)  // 4-lane groups (short runs): no unroll, -1 % at C4
          for (int j = lg; j < nmax; j += GL) {
            const bool ok = j < n;
            const float4 r = pr[j];
            const float d2 = pd[j];
            const int pl = pp[j];
            const float4 uu = s_u[pl];
            const float2 e = run_e(ke, pl);
            const float sa = fmaf(r.z, uu.x, fmaf(r.w, uu.y, d2 * uu.z));
            const float tt = ok ? sa * r.x : 0.f;
            const float ry = ok ? r.y : 0.f;
            const float2 te = __fmul2_rn(make_float2(tt, tt), e);
            a01 = __fadd2_rn(a01, te);
            a23 = __ffma2_rn(make_float2(te.x, te.x), e, a23);  // x 1/2 on a[2] in the epilogue
            a4 = fmaf(te.y, e.y, a4);                            // x 1/2 in the epilogue
            a5 += tt;
            a67 = __ffma2_rn(make_float2(ry, ry), make_float2(uu.x, uu.y), a67);
            a8 = fmaf(ry, uu.z, a8);
          }
          // GL-lane reduce-scatter of a[0..7] (lane lg ends with the group
          // sums of values lg + GL h) plus a butterfly for a8
          const float a[8] = {a01.x, a01.y, a23.x, a23.y, a4, a5, a67.x, a67.y};
          float ra[8 / GL];
          group_rs<GL, 8 / GL>(a, ra, lg);
          a8 = group_sum<GL>(a8);
          if (ri != 0xff) {
            // pair-run-slot order (read contiguously by the backward): partials
            // 0-7 as one 32-byte record, partial 8 in A.out1
#pragma unroll
            for (int h = 0; h < 8 / GL; ++h) A.out[(size_t)sl * 8 + GL * h + lg] = ra[h] * (GL * h + lg == 5 ? io : jt_scl(GL * h + lg));
            if (lg == 0) A.out1[sl] = a8;
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
    }
    consumer_sync();  // s_u / s_acc are reused by the next tile
  }
}

template <int MODE, int JGL = kJtGL>
static int launch_stream_gl(const SlmTileArgs* a, cudaStream_t st) {
  if (a->n_tiles <= 0) return SLM_OK;
  const size_t bytes = stream_smem_bytes(MODE);
  // the dynamic shared-memory opt-in and the occupancy are per device: a
  // process may drive several GPUs (one stream each)
  constexpr int kMaxDev = 64;
  static int s_per_sm[kMaxDev] = {0};   // 0: not configured on that device yet
  static int s_sms[kMaxDev] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDev) return SLM_ERR_ARG;
  if (s_per_sm[dev] == 0) {
    cudaFuncSetAttribute(k_stream<MODE, JGL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    int sms = 148, per_sm = 1;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_stream<MODE, JGL>, NT, bytes);
    s_sms[dev] = sms;
    s_per_sm[dev] = per_sm < 1 ? 1 : per_sm;
  }
  const int sms = s_sms[dev], per_sm = s_per_sm[dev];
  const int grid = (int)std::min<long long>((long long)a->n_tiles, (long long)sms * per_sm);
  if (a->tile_counter) cudaMemsetAsync(a->tile_counter, 0, sizeof(int), st);
  k_stream<MODE, JGL><<<grid, NT, bytes, st>>>(*a);
  return slm_cuda_status();
}

// J^T lanes per run: 8 by default; 4 when the runs are short (the caller sets
// jt_lanes = 4 below ~18 entries per run: C4's 13-entry runs -5 % on the
// fused kernel, C2 / C3's long runs +20 % / +3 %)
template <int MODE>
static int launch_stream(const SlmTileArgs* a, cudaStream_t st) {
  if ((MODE & MODE_JT) && a->jt_lanes == 4) return launch_stream_gl<MODE, 4>(a, st);
  return launch_stream_gl<MODE, kJtGL>(a, st);
}

extern "C" {

int slm_run_static(const SlmTileArgs* a, long long n_runs, const int* run_slot, float* out, cudaStream_t st) {
  if (n_runs <= 0) return SLM_OK;
  k_run_static<<<slm_blocks(n_runs, 256, 1LL << 30), 256, 0, st>>>(*a, n_runs, run_slot, out);
  return slm_cuda_status();
}

int slm_tile_chunks(const int* tile_run_off, int n_tiles, const long long* run_start, const int* tile_chunk_off,
                    int* out, uint8_t* chunk_perm, int fill, cudaStream_t st) {
  if (n_tiles <= 0) return SLM_OK;
  const unsigned b = slm_blocks(n_tiles, 128, 1LL << 30);
  if (!fill) {
    k_tile_chunks<false><<<b, 128, 0, st>>>(tile_run_off, n_tiles, run_start, tile_chunk_off, out);
    return slm_cuda_status();
  }
  k_tile_chunks<true><<<b, 128, 0, st>>>(tile_run_off, n_tiles, run_start, tile_chunk_off, out);
  // out[n_chunks] (= R) is written by the caller before the perm pass; read it on the device
  return slm_cuda_status();
}

int slm_chunk_perm(const int* chunk_run, long long n_chunks, const long long* run_start, uint8_t* chunk_perm,
                   uint32_t* run_fn, cudaStream_t st) {
  if (n_chunks <= 0) return SLM_OK;
  k_chunk_perm<<<slm_blocks(n_chunks * 32, 256, 1LL << 30), 256, 0, st>>>(chunk_run, n_chunks, run_start,
                                                                         chunk_perm, run_fn);
  return slm_cuda_status();
}

// u = J p (a->gradr weights it) written to a->u_out
int slm_apply_j(const SlmTileArgs* a, cudaStream_t st) { return launch_stream<MODE_J | MODE_WRITEU>(a, st); }

// diag(J^T W J) moments per run (40 floats, pair-run-slot order) from
// a->gradr; with a->u = the colour gradient also its J^T partials (the rhs)
// into a->rhs8 / a->rhs1, in the same sweep
int slm_diag_stream(const SlmTileArgs* a, cudaStream_t st) { return launch_stream<MODE_DIAG>(a, st); }

// J^T partials per run from the per-pixel a->u
int slm_apply_jt_runs(const SlmTileArgs* a, cudaStream_t st) { return launch_stream<MODE_JT>(a, st); }

// fused: J^T partials of (grad_r_sq * J p) per run; u never leaves the SM
int slm_jtwj_runs(const SlmTileArgs* a, cudaStream_t st) { return launch_stream<MODE_J | MODE_JT>(a, st); }

}  // extern "C"
