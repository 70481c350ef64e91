/*
 * splatlm_b200.h -- C ABI of the B200 (sm_100a) 3DGS-LM inner-solver library
 * libsplatlm_b200.so.
 *
 * Every entry point takes plain device pointers, sizes and a cudaStream_t,
 * never allocates, launches asynchronously and returns an int status
 * (SLM_OK = 0).  Scratch sizes for CUB-backed calls are queried with the
 * *_workspace functions.  The Python package paper_2409_12892_b200 binds this
 * header with ctypes and re-exposes the reference's
 * Python API (`splatlm.*`); the "replaces" notes cite the reference function
 * each call implements.  Reference paths are relative to
 * /root/reference/pkg/src/splatlm/.
 *
 * Cache layout ("runs"): a run is one (tile, splat) pair of a view with at
 * least one kept pixel; runs are numbered (view, tile, depth order) and each
 * run's entries are stored contiguously in tile-local pixel order, with a
 * 256-bit mask of the kept pixels.  Records are float4 {alpha_eff, alpha*T,
 * dc/dalpha_r, dc/dalpha_g} + float dc/dalpha_b + uint8 tile-local pixel index
 * (21 B/entry, three streams so one entry is three shared-memory loads).
 */
#ifndef SPLATLM_B200_H
#define SPLATLM_B200_H

#include <stdint.h>

#define SLM_CHUNK_RUNS 64 /* max runs per streaming chunk; SlmTileArgs.chunk_perm holds this many bytes per chunk */

#ifdef __CUDACC__
#include <cuda_runtime.h>
typedef uint2 slm_u2;
typedef float4 slm_f4;
#else
typedef struct CUstream_st* cudaStream_t;
typedef struct { uint32_t x, y; } slm_u2;
typedef struct { float x, y, z, w; } slm_f4;
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (mapped to the reference's exception classes in Python) */
#define SLM_OK 0
#define SLM_ERR_ARG 1     /* bad argument: ValueError */
#define SLM_ERR_CUDA 2    /* CUDA launch/runtime error: RuntimeError */
#define SLM_ERR_LAYOUT 3  /* LayoutError (scene.py:48-49) -- raised by the host layer */
#define SLM_ERR_ORDER 4   /* CacheOrderError (jacobian.py:42-43) -- host layer */
#define SLM_ERR_SIZE 5    /* size beyond the 32-bit CUB limits / ImageSizeError */

/* ---- value types --------------------------------------------------------- */

/* one pinhole view (scene.py:272-304); C = -R^T t precomputed on the host */
typedef struct {
  double R[9];
  double t[3];
  double fx, fy, cx, cy;
  double C[3];
  int W, H;
  long long pix_base; /* first subset-global pixel index of this view */
} SlmCamera;

/* RenderConfig (rasterizer.py:22-48) plus the background colour */
typedef struct {
  double alpha_min, t_stop, alpha_clamp, cov_eps, z_near;
  double cull_sigma; /* <= 0 disables the footprint cull */
  double reach_fac;  /* sqrt(max(0, 2 ln(1/alpha_min))); <= 0: unbounded bbox */
  double bg[3];
} SlmRastCfg;

/* fp64 projected splat (ProjectedSplats row, rasterizer.py:63-75), 96 B */
typedef struct {
  double mx, my, ca, cb, cc, o, c0, c1, c2;
  int x0, x1, y0, y1;
  unsigned flags; /* bit0 valid, bits1..3 colour clamp per channel */
  int pad;
} SlmSplat;

/* per (gaussian, view) pair geometry used by the entry chain, 32 B */
typedef struct {
  double mx, my;
  float ka, kb, kc, inv_o;
} SlmPairGeo;

typedef struct {
  long long pix_base;
  int W, H;
} SlmView;

/* rasteriser launch arguments (both passes) */
typedef struct {
  const slm_u2* tile_range;   /* [n_tiles] instance range of each tile */
  const uint32_t* inst_gid;   /* [n_inst] gaussian of each (tile, depth) instance */
  const SlmSplat* splats;
  int W, H, tiles_x;
  long long pix_base;
  SlmRastCfg cfg;
  /* COUNT outputs */
  uint32_t* px_count;         /* [HW] entries per pixel */
  double* rgb;                /* [HW*3] rendered colour incl. background (FILL: input) */
  double* t_final;            /* [HW] */
  uint32_t* inst_mask;        /* [n_inst*8] keep mask per instance (COUNT out, FILL in) */
  /* FILL: run-ordered cache records */
  const long long* inst_start;  /* [n_inst] first entry of the instance's run */
  slm_f4* rec4;               /* {alpha_eff, alpha*T, dc/dalpha_r, dc/dalpha_g} */
  float* rec_d2;              /* dc/dalpha_b */
  uint8_t* rec_pix;           /* tile-local pixel index (16 * ly + lx) */
  /* FILL: optional pixel-order Traversals export (rasterizer.py:209-243) */
  const long long* pix_off;
  long long view_entry_base;
  long long* trav_gid;
  double* trav_alpha;
  double* trav_T;
  /* batched mode (views != NULL): one launch over all n_tiles tiles of the
   * subset's views; tile_range / px_count / rgb / t_final are subset-global */
  const SlmView* views;
  const int* view_tile_base;
  int n_views;
  int n_tiles;
  /* FILL: cache offload ("CPU offloading of cache parts"):
   * when rec4_h != NULL, entries >= e_split are written to host-pinned,
   * device-mapped streams indexed from e_hbase (a multiple of 16, <= e_split):
   * rec4_h[e - e_hbase] etc.; the device streams hold entries [0, e_split) */
  slm_f4* rec4_h;
  float* rec_d2_h;
  uint8_t* rec_pix_h;
  long long e_split, e_hbase;
} SlmRasterArgs;

/* residual weights (residuals.py:249-296) */
typedef struct {
  const double* img;
  const void* gt;
  int gt_f32;
  int W, H;
  double lambda1, lambda2, eps_den;
  double ssim_c1, ssim_c2;
  int mode; /* 0 l1ssim, 1 l2 */
  int win;
  const double* taps;
  const double* cw_y;
  const double* cw_x;
  slm_f4* gradr;
  slm_f4* cgrad;
  double* energy_part;
  double *o_gradr, *o_cgrad, *o_rabs, *o_rssim, *o_drabs, *o_drssim;
} SlmResidArgs;

/* tile-parallel product kernels (applyJ, applyJT partials, diag sums): one
 * CTA per tile of the subset, warps over the tile's runs */
typedef struct {
  const SlmView* views;
  const int* view_tile_base; /* [n_views+1] first global tile of each view */
  int n_views;
  int n_tiles;
  const int* tile_run_off;   /* [n_tiles+1] */
  const int* tile_chunk_off; /* [n_tiles+1] chunk table (slm_tile_chunks) */
  const int* chunk_run;      /* [n_chunks+1] first run of each chunk */
  const uint8_t* chunk_perm; /* [n_chunks*SLM_CHUNK_RUNS] J^T schedule: chunk-local runs by decreasing length */
  const int* run_slot;       /* [R] position of each run in pair_runs (J^T outputs go there) */
  const long long* run_start;/* [R+1] (+2 padding slots) */
  const uint32_t* run_fn;    /* [R] chunk-local first entry | length << 16 (slm_chunk_perm) */
  const int* run_q;          /* pair of each run */
  const uint32_t* run_tile;  /* view << 24 | tile */
  const float* run_static;   /* [R*8] static run records (slm_run_static) */
  const void* pm;            /* [P*12] per-pair forward chain m (slm_pair_forward); NULL: J^T / diag only */
  const SlmPairGeo* geo;
  const slm_f4* rec4;
  const float* d2;
  const uint8_t* pix;
  const slm_f4* gradr;       /* applyJ: weighting (NULL: unweighted u_hat); diag: grad_r_sq */
  const slm_f4* u;           /* applyJT input, per pixel */
  slm_f4* u_out;             /* applyJ output, per pixel */
  float* out;                /* applyJT [R*8] run partials 0-7 (32-byte records) /
                                diag [R*40] run moments, pair-run-slot order */
  float* out1;               /* applyJT [R] run partial 8, pair-run-slot order */
  float* rhs8;               /* diag with u = colour gradient: its J^T partials 0-7 [R*8] */
  float* rhs1;               /* ... and partial 8 [R] */
  int* tile_counter;         /* streaming kernels: 1 int of device scratch for
                                dynamic tile scheduling (reset by the launch);
                                NULL: static round-robin tiles */
  /* offloaded record tail (see SlmRasterArgs): chunks starting at an entry
   * >= e_split (a chunk boundary) are streamed from the host-mapped copies */
  const slm_f4* rec4_h;
  const float* d2_h;
  const uint8_t* pix_h;
  long long e_split, e_hbase;
  int jt_lanes;              /* J^T lanes per run: 8 (0 = default) or 4 (short runs) */
  int pad_;
} SlmTileArgs;

/* per-pair forward chain (applyJ) */
typedef struct {
  const float* xs;          /* scene, attribute-major fp32 */
  long long G;
  const int* pair_gid;
  const uint32_t* pair_vm;  /* view | clamp bits << 16 */
  const SlmCamera* cams;
  int n_pairs;
  const float* p;           /* direction, p[a * sa + g * sg] (either layout) */
  long long sa, sg;
  void* pm;                 /* [P*12] out: m = dy/dx p per pair (3 float4) */
  const float* gtab;        /* per-gaussian chain rows (slm_gauss_tab) */
  int dsig;                 /* 1: p is the padded gaussian-major copy with dSigma (slm_pcg_p*) */
  const float* camf;        /* dsig = 1: [V*20] fp32 camera rows (slm_cameras_f32) */
} SlmFwdArgs;

/* per-gaussian backward chain */
typedef struct {
  const float* xs; /* scene, attribute-major fp32 */
  long long G;
  const int* gpo;           /* [G+1] gaussian -> pairs (pairs are (gid, view)-numbered) */
  const uint32_t* pair_vm;  /* view | clamp bits << 16 */
  const SlmCamera* cams;
  const float* pacc;        /* per-run partials in pair-run-slot order (the J^T /
                               diag kernels write run r to its slot in pair_runs):
                               mode 0 [R*8] partials 0-7, mode 1 [R*40] moments */
  const float* pacc1;       /* mode 0: [R] partial 8 per run slot */
  const int* pair_run_off;  /* [P+1] pair -> run slots */
  const int* warp_g0;       /* first gaussian of each 32-pair window (slm_warp_bounds) */
  const int* pair_gid;
  long long n_pairs;
  float* gm;                /* [G*P] gaussian-major scratch */
  const float* gtab;        /* per-gaussian chain rows (slm_gauss_tab) */
  float scale;
  const float* p;           /* optional: fp64 partials of p.(out + lam * max(M,1e-12) * p) */
  const float* Mdiag;
  double lam;
  int lam_out;              /* 1: out += lam * max(M,1e-12) * p as well */
  float* out;
  double* dot_part;
  const float* camf;        /* [V*20] fp32 camera rows (slm_cameras_f32), mode 0 */
} SlmBackArgs;

/* fp32 camera rows of the per-pair chains: R 9 | t 3 | C 3 | fx | fy | pad 3 per view */
int slm_cameras_f32(const SlmCamera* cams, int V, float* out, cudaStream_t s);

/* ---- sizes (ctypes layout checks) --------------------------------------- */
int slm_camera_size(void);
int slm_rastcfg_size(void);
int slm_splat_size(void);
int slm_pair_geo_size(void);
int slm_view_size(void);
int slm_raster_args_size(void);
int slm_resid_args_size(void);
int slm_tile_args_size(void);
int slm_back_args_size(void);
int slm_fwd_args_size(void);
int slm_diag_moment_floats(void);

/* ---- projection / rasterisation ------------------------------------------
 * replaces project_scene (rasterizer.py:116-165): fp64 splats of one view,
 * depth keys (fp64 bits, ~0 for culled) and gid values for the depth sort.
 * err |= 1 on non-finite parameters (rasterizer.py:124-125), 2 on a zero
 * quaternion (rasterizer.py:81-82). */
int slm_preprocess(const double* x_am, long long G, int sh_degree, const SlmCamera* cam, const SlmRastCfg* cfg,
                   SlmSplat* out, unsigned long long* depth_key, uint32_t* order_val, int* err, cudaStream_t s);
/* stable radix sort of (u64 key, u32 value) pairs -- the (depth, gid) order of
 * render (rasterizer.py:328-330) and the tile-instance sort */
long long slm_sort_pairs_u64_workspace(long long n);
int slm_sort_pairs_u64(void* ws, long long ws_bytes, const unsigned long long* keys_in, unsigned long long* keys_out,
                       const uint32_t* vals_in, uint32_t* vals_out, long long n, int begin_bit, int end_bit,
                       cudaStream_t s);
/* tile binning of the depth-sorted splats (replaces the per-splat bbox walk,
 * rasterizer.py:253-261, 283-287) */
int slm_tile_count(const uint32_t* sorted_gid, const unsigned long long* sorted_key, long long G,
                   const SlmSplat* splats, int tiles_x, int tiles_y, unsigned long long* n_inst, cudaStream_t s);
/* tile keys of every (tile, splat) instance, emitted in depth-rank order, the
 * splat as the value: after a STABLE key sort (slm_sort_pairs_u32 on the tile
 * bits) the values are each tile's instance list in depth order */
int slm_tile_emit(const uint32_t* sorted_gid, const unsigned long long* inst_off, long long G, const SlmSplat* splats,
                  int tiles_x, int tiles_y, uint32_t* keys, uint32_t* vals, cudaStream_t s);
int slm_tile_ranges(const uint32_t* keys, long long n, slm_u2* ranges, int n_tiles, cudaStream_t s);
/* render (rasterizer.py:319-358): COUNT pass = image, T_final, per-pixel
 * counts and per-instance keep masks; FILL pass = run-ordered cache records
 * (build_cache, jacobian.py:383-409) and/or the Traversals arrays */
int slm_raster_count(const SlmRasterArgs* a, cudaStream_t s);
int slm_raster_fill(const SlmRasterArgs* a, cudaStream_t s);
/* runs: per-instance counts (+ per-(view,gaussian) counts), the run table and
 * runs per tile (the pair -> runs CSR is a stable slm_sort_pairs_u32 of the
 * runs by pair + slm_invert_perm) */
int slm_inst_count(const uint32_t* mask, const uint32_t* inst_gid, long long n, long long* cnt, int* used,
                   int* pair_cnt, cudaStream_t s);
int slm_runs_emit(const uint32_t* mask, const uint32_t* inst_gid, const int* used, const int* run_of,
                  const long long* ent_of, long long ibase, long long n, const int* pidx, long long* run_start,
                  int* run_q, uint32_t* run_mask /* optional */, int* pair_nruns, long long* inst_start,
                  cudaStream_t s);
int slm_tile_runs(const slm_u2* ranges, int n_tiles, const int* used, const int* run_of, long long ibase, int view,
                  int* tile_nruns, uint32_t* run_tile, const int* view_tile_base, int n_views, cudaStream_t s);
/* subset-batched projection and binning (all V views of a cache subset per
 * launch): element v * G + g, sorted value (v << 24) | g, global tiles
 * view_tile_base[v] + ty * tiles_x + tx */
int slm_preprocess_views(const double* x, long long G, int sh_degree, const SlmCamera* cams_dev, int V,
                         const SlmRastCfg* cfg, SlmSplat* out, unsigned long long* depth_key, uint32_t* order_val,
                         int* err, cudaStream_t s);
int slm_tile_count_v(const uint32_t* sv, long long n, long long G, const SlmSplat* splats, const SlmView* views,
                     unsigned long long* n_inst, cudaStream_t s);
int slm_tile_emit_v(const uint32_t* sv, const unsigned long long* inst_off, long long n, long long G,
                    const SlmSplat* splats, const SlmView* views, const int* view_tile_base, uint32_t* keys,
                    uint32_t* vals, cudaStream_t s);
long long slm_sort_keys_u32_workspace(long long n);
int slm_sort_keys_u32(void* ws, long long ws_bytes, const uint32_t* kin, uint32_t* kout, long long n, int begin_bit,
                      int end_bit, cudaStream_t s);

/* ---- residuals: compute_residuals (residuals.py:249-296) ----------------- */
int slm_residuals(const SlmResidArgs* a, int blocks, cudaStream_t s);

/* ---- scans / pairs ----------------------------------------------------------
 * (view, gaussian) pairs in (view, gid) order: counts -> flags/scans, then
 * pair geometry / maps and the gid-major CSR (gpo, gp_list) used by the
 * per-gaussian backward chain */
long long slm_scan_i64_workspace(long long n);
int slm_scan_i64(void* ws, long long wsb, const long long* in, long long* out, long long n, cudaStream_t s);
long long slm_scan_i32_workspace(long long n);
int slm_scan_i32(void* ws, long long wsb, const int* in, int* out, long long n, cudaStream_t s);
long long slm_sort_pairs_u32_workspace(long long n);
int slm_sort_pairs_u32(void* ws, long long wsb, const uint32_t* kin, uint32_t* kout, const uint32_t* vin,
                       uint32_t* vout, long long n, int begin_bit, int end_bit, cudaStream_t s);
int slm_iota_u32(uint32_t* out, long long n, cudaStream_t s);
/* inv[perm[k]] = k for a permutation of [0, n) (run -> pair-run slot) */
int slm_invert_perm(const int* perm, long long n, int* inv, cudaStream_t s);
int slm_pairs_prepare(const int* cnt, int V, long long G, long long* cntV, int* flagV, int* flagT, cudaStream_t s);
int slm_pairs_emit(const int* cnt, int V, long long G, const int* pair_of, const long long* vscan, const int* tscan,
                   const SlmSplat* splats, long long* pair_off, int* pair_gid, uint32_t* pair_vm, SlmPairGeo* geo,
                   int* pidx, int* gpo, int n_pairs, long long n_entries, cudaStream_t s);

/* reference-order export of one view (parity / interop, not on the solve
 * path): from the run order, the pixel-sorted index arrays of build_cache
 * (jacobian.py:401-409) and the gaussian-sorted ones of
 * sort_cache_by_gaussians (jacobian.py:93-105); pos_pix[e - e_base] = the
 * pixel-order position of run-order entry e.  px_off: the view's per-pixel
 * entry offsets [HW+1]; g_off: its per-gaussian offsets [G+1] */
int slm_export_view(const int* tile_run_off, int t0, int n_tiles, int tiles_x, int W, const long long* run_start,
                    const int* run_q, const uint32_t* run_tile, const int* pair_gid, const uint32_t* pair_vm,
                    const int* pair_run_off, const int* pair_runs, int n_pairs, int view, const uint8_t* pix,
                    const long long* px_off, const long long* g_off, long long e_base, long long* pos_pix,
                    long long* pixel_ids, long long* gaussian_ids, long long* g_pixel_ids, long long* g_gaussian_ids,
                    long long* g_source_index, cudaStream_t s);

/* ---- products ----------------------------------------------------------------
 * apply_j (jacobian.py:419-455) fused with weight_residuals (458-464) when
 * a->gradr != NULL; one CTA per tile of the subset */
int slm_apply_j(const SlmTileArgs* a, cudaStream_t s);
/* apply_jt (jacobian.py:467-483), first half: 9 partials per run from a->u */
int slm_apply_jt_runs(const SlmTileArgs* a, cudaStream_t s);
/* fused apply_jt(weight_residuals(apply_j(p))) first half, tile by tile: u
 * stays in shared memory, the cache is streamed from HBM once */
int slm_jtwj_runs(const SlmTileArgs* a, cudaStream_t s);
/* static run records (once per cache): centre relative to the tile, conic,
 * 1/opacity, pair-run slot, pair; and the per-tile chunk table (fill=0:
 * counts per tile, fill=1: chunk_run) + the per-chunk J^T schedule (runs by
 * decreasing length, slm_chunk_perm) */
int slm_run_static(const SlmTileArgs* a, long long n_runs, const int* run_slot, float* out, cudaStream_t s);
int slm_tile_chunks(const int* tile_run_off, int n_tiles, const long long* run_start, const int* tile_chunk_off,
                    int* out, uint8_t* chunk_perm, int fill, cudaStream_t s);
int slm_chunk_perm(const int* chunk_run, long long n_chunks, const long long* run_start, uint8_t* chunk_perm,
                   uint32_t* run_fn, cudaStream_t s);
/* per-gaussian chain rows, slm_gauss_tab_floats(sh_degree) floats each (16-byte
 * aligned): the view-independent part of the chain (rotation, scales, the
 * quaternion-normalisation derivatives, sigma'), the position and the SH
 * coefficients; once per cache (ref: jacobian.py:159-190, 213-240) */
int slm_gauss_tab(const float* xs, long long G, int sh_degree, float* gtab, cudaStream_t s);
int slm_gauss_tab_floats(int sh_degree);
/* diag_jtj (jacobian.py:486-512), first half: slm_diag_moment_floats() moment
 * sums per run on the streaming kernel, pair-run-slot order (a->gradr =
 * grad_r_sq, a->out); with a->u = the colour gradient, the same sweep writes
 * its J^T partials (the rhs, jacobian.py:411-413) to a->rhs8 / a->rhs1 */
int slm_diag_stream(const SlmTileArgs* a, cudaStream_t s);
/* forward chain m = dy/dx p per pair (jacobian.py:434-443), 48 B per pair */
int slm_pair_forward(const SlmFwdArgs* a, int sh_degree, cudaStream_t s);
/* backward chain per gaussian, attribute-major out (jacobian.py:314-353):
 * mode 0 from the J^T run partials, mode 1 from the diag run moments */
int slm_backward_blocks(long long G);
int slm_warp_bounds(const int* gpo, long long G, int n_pairs, int* warp_g0, cudaStream_t s);
int slm_pair_backward(const SlmBackArgs* a, int mode, int sh_degree, cudaStream_t s);

/* ---- PCG (Alg. 1; SPEC pcg_solve 391-399) ------------------ */
int slm_vec_blocks(void);
/* p (attribute-major, G*P) and, when p_gm != NULL, its padded gaussian-major
 * copy p_gm[g * pg + a] (pg = slm_gm_stride(P), pad 0) for the forward chain;
 * with gtab (the cache's chain rows, slm_gauss_tab) each row also carries the
 * world-covariance perturbation of the rotation / scale block at ((P+3) & ~3) */
int slm_gm_stride(int P);
int slm_pcg_pinit(float* p, float* p_gm, const float* b, const float* M, long long G, int P, const float* gtab,
                  int gtab_stride, cudaStream_t s);
int slm_pcg_pupdate(float* p, float* p_gm, const double* r, const float* M, const double* st, long long G, int P,
                    const float* gtab, int gtab_stride, cudaStream_t s);
/* the same padded gaussian-major copy (+ dSigma) of a given attribute-major p */
int slm_gm_pack(const float* p, float* p_gm, long long G, int P, const float* gtab, int gtab_stride, cudaStream_t s);
int slm_pcg_update(int mode, double* x, double* r, const float* p, const float* g, const float* b, const float* M,
                   double lam, double* st, const double* dot_part, int n_dot, double* part, long long n,
                   cudaStream_t s);
int slm_pcg_finalize(int mode, double* st, const double* part, cudaStream_t s);

/* ---- Eq. 7 combine (SPEC solve_normal_equations_batched 400-408) --------- */
int slm_combine_acc(double* num, double* den, const double* delta, const float* M, long long n, cudaStream_t s);
int slm_combine_fin(float* out, const double* num, const double* den, long long n, cudaStream_t s);

/* ---- layouts and helpers ---------------------------------------------------
 * sort_x / sort_x_inverse (scene.py:79-92) are transposes of the P x G matrix */
int slm_transpose_f32(const float* in, float* out, long long rows, long long cols, cudaStream_t s);
int slm_transpose_f64(const double* in, double* out, long long rows, long long cols, cudaStream_t s);
int slm_f64_to_f32(const double* in, float* out, long long n, cudaStream_t s);
int slm_axpy_scene(const double* x, const float* d, double gamma, double* out, long long n, cudaStream_t s);

#ifdef __cplusplus
}
#endif
#endif /* SPLATLM_B200_H */
