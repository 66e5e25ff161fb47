/* hawkes_b200.h — C ABI of the B200 spatiotemporal-Hawkes likelihood engine.
 *
 * This is the drop-in boundary for the reference's hot path
 * (/root/reference/proj/include/hawkes/, "hphawkes"):
 *
 *   reference entry point                         replaced by
 *   ----------------------------------------------------------------------
 *   log_likelihood(Catalog, HawkesParams,          hk_create + hk_eval
 *     Partition, Precision)     engine.hpp:101-110   (grad5 == NULL: LL only)
 *   log_likelihood_t / slice_log_likelihood        hk_eval_rows
 *                               engine.hpp:65-99
 *   event_contribution          model.hpp:225-230  hk_eval_rows(b, b+1)
 *   LikelihoodWorkspace<double>::set_locations     hk_set_locations
 *                               engine.hpp:172-178
 *   LikelihoodWorkspace<double>::evaluate_*        hk_ws_eval (device-cached
 *                               engine.hpp:133-158   row sums per half)
 *   Partition::make             engine.hpp:27-40   hk_partition_make
 *   benchmark_catalog           engine.hpp:251-259 hk_benchmark_catalog
 *   (new, no reference counterpart)                hk_eval with grad5 != NULL,
 *                                                  hk_plan_shards
 *
 * Conventions (mirroring the reference's C++ error behaviour):
 *   return 0 = ok, 1 = invalid_argument, 2 = out_of_range,
 *          3 = CUDA runtime error, 4 = not implemented (e.g. single precision).
 *   hk_last_error() returns the thread-local message of the last failure; the
 *   messages for invalid inputs are the reference's own (types.hpp:45-55,
 *   :92-103; engine.hpp:28-29).
 *   Non-finite log-likelihood values are returned as values, not errors
 *   (the reference's caller rejects them, mcmc.hpp:168).
 *   A context is single-caller (like LikelihoodWorkspace); several contexts may
 *   coexist.  Results are bitwise deterministic for a fixed (catalog, params,
 *   device set).
 *
 * All arrays are host pointers unless the name says `device`.  No CUDA or
 * torch types appear in the signatures; streams are passed as void*.
 */
#ifndef HAWKES_B200_H
#define HAWKES_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HK_OK 0
#define HK_INVALID_ARGUMENT 1
#define HK_OUT_OF_RANGE 2
#define HK_RUNTIME_ERROR 3
#define HK_NOT_IMPLEMENTED 4

#define HK_VARIANT_CONSTANT 0 /* Variant::constant, types.hpp:16 */
#define HK_VARIANT_VARYING 1  /* Variant::varying */

/* HawkesParams (types.hpp:83-110).  All six must be positive and finite. */
typedef struct hk_params {
  double mu0;     /* background weight */
  double tau_t;   /* background temporal lengthscale (weeks) */
  double xi0;     /* self-excitatory weight */
  double sigma_x; /* triggering spatial lengthscale (degrees) */
  double sigma_t; /* triggering temporal lengthscale (weeks) */
  double area;    /* A, square degrees */
  int variant;    /* HK_VARIANT_* */
} hk_params;

typedef struct hk_ctx hk_ctx;

/* Builds an evaluation context for a time-sorted catalog (Catalog,
 * types.hpp:41-78; the same validation and messages).  Copies the arrays,
 * uploads them to `n_gpus` devices (0..n_gpus-1; 0 means 1) and plans
 * cost-balanced row shards, one per device.  `density` is the per-event
 * population density (Event::density); the variant is chosen per
 * evaluation by hk_params.variant.  Non-finite locations are accepted (a
 * coarse-only catalog, types.hpp:43-57 with coarse_only = true); evaluations
 * then fail with HK_INVALID_ARGUMENT until hk_set_locations supplies finite
 * ones (the cut posterior's X refresh). */
int hk_create(const double* t, const double* lon, const double* lat, const double* density,
              size_t n, int n_gpus, hk_ctx** out);

/* hk_create whose multi-device shard plan is balanced for `variant` (the
 * kernel the caller mostly runs; see hk_plan_shards_variant).  Evaluations
 * may still use either variant. */
int hk_create_variant(const double* t, const double* lon, const double* lat, const double* density,
                      size_t n, int n_gpus, int variant, hk_ctx** out);

/* hk_create_variant over an explicit device list: shard k (cost-balanced)
 * runs on devices[k].  Over distinct devices the per-evaluation 6-vectors
 * are all-gathered with NCCL (libnccl.so.2, loaded on first use) and summed
 * on the devices in device order, and hk_set_locations copies to devices[0]
 * once and NCCL-broadcasts to the rest.  A list that repeats a device (e.g.
 * {0, 0, 0, 0}: several shards on one GPU) moves the same data with CUDA
 * peer copies instead (also forced by HK_NO_NCCL=1); results are bitwise
 * identical between the two and deterministic. */
int hk_create_devices(const double* t, const double* lon, const double* lat, const double* density,
                      size_t n, const int* devices, int n_devices, int variant, hk_ctx** out);

/* One rank's shard for a one-process-per-GPU job: the full catalog is
 * uploaded to `device`, but only rows [row_begin, row_end) are evaluated.
 * hk_eval then returns this shard's partial sums; the caller reduces the
 * partials across ranks (in rank order, for determinism). */
int hk_create_shard(const double* t, const double* lon, const double* lat, const double* density,
                    size_t n, size_t row_begin, size_t row_end, int device, hk_ctx** out);

void hk_destroy(hk_ctx* ctx);

/* Replaces the event locations (LikelihoodWorkspace::set_locations,
 * engine.hpp:172-178): host arrays of length n (pinned memory makes the copy
 * asynchronous DMA), copied to the first device, checked there (a device
 * reduction: bounding box and finiteness; a non-finite location fails with
 * the reference's Catalog message and leaves the context without valid
 * locations) and broadcast to the other devices (NCCL). */
int hk_set_locations(hk_ctx* ctx, const double* lon, const double* lat);

/* Same, from device arrays resident on the context's first device (e.g. a
 * GPU location sampler's output, hk_resample_locations). */
int hk_set_locations_device(hk_ctx* ctx, const double* lon_device, const double* lat_device);

/* Full evaluation.  *ll receives the log-likelihood (sum over the context's
 * rows of ell_n, engine.hpp:65-99 / model.hpp:214-223).  If grad5 != NULL it
 * receives d ell / d (mu0, tau_t, xi0, sigma_x, sigma_t).  Synchronous. */
int hk_eval(hk_ctx* ctx, const hk_params* p, double* ll, double* grad5);

/* hk_eval that also returns the per-row terms of the SAME launches (the
 * production plan: clustered windows, split background/trigger launches):
 * ell_rows[k] = ell_n and, if grad_rows != NULL (requires grad5),
 * grad_rows[5k..5k+4] = d ell_n / d theta for the context's rows in order
 * (hk_rows: begin + k).  Either row pointer may be NULL.  For parity checks
 * of the full-evaluation path row by row. */
int hk_eval_detail(hk_ctx* ctx, const hk_params* p, double* ll, double* grad5, double* ell_rows,
                   double* grad_rows);

/* Precision::single (engine.hpp:106-109 with EvalData<float>): the
 * trigger pair sums in FP32 (centred FP32 coordinates, MUFU ex2, FP32
 * partial sums per 256-column tile accumulated in FP64); background and
 * row epilogue in FP64.  Log-likelihood only, like the reference's single
 * path.  Agrees with the double result to ~1e-6 relative (the reference's
 * own single-precision gate is 1e-4, acceptance.cpp:82). */
int hk_eval_single(hk_ctx* ctx, const hk_params* p, double* ll);

/* Workspace evaluation (LikelihoodWorkspace<double>, engine.hpp:117-229):
 * like hk_eval, but the per-row background sums [B, B2] are reused while
 * tau_t is unchanged and the trigger sums [T, Td, Tq] while sigma_x,
 * sigma_t, the variant and the locations are unchanged (two cached states
 * per half: current + proposal).  A mu0/xi0 proposal is an O(N)
 * recombination; tau_t refreshes only the background; sigma_x/sigma_t or
 * hk_set_locations only the trigger.  force != 0 recomputes both halves
 * (evaluate_full).  Results are bitwise identical to hk_eval's. */
int hk_ws_eval(hk_ctx* ctx, const hk_params* p, int force, double* ll, double* grad5);
/* LikelihoodWorkspace<float> (engine.hpp:117-229 with Real = float): the
 * hk_eval_single arithmetic with the same two-entry caches per half (keyed
 * separately from the double entries).  LL only.  Bitwise equal to
 * hk_eval_single at the same parameters. */
int hk_ws_eval_single(hk_ctx* ctx, const hk_params* p, int force, double* ll);
/* Cache hits / misses of hk_ws_eval / hk_ws_eval_single since creation. */
int hk_ws_stats(const hk_ctx* ctx, long* hits, long* misses);

/* Asynchronous form: enqueues the evaluation on the context's stream(s) and
 * leaves [ll, g_mu0, g_tau_t, g_xi0, g_sigma_x, g_sigma_t] in a device buffer
 * on the first device (hk_result_device; multi-device contexts: the
 * device-order sum after the all-gather). */
int hk_eval_async(hk_ctx* ctx, const hk_params* p, int with_grad);
/* Device pointer to the 6-double result of the last hk_eval_async. */
const double* hk_result_device(hk_ctx* ctx);
/* cudaStream_t (as void*) the context launches on, for device index `dev`. */
void* hk_stream(hk_ctx* ctx, int dev);

/* ---- GPU location sampler (the cut posterior's X refresh) ----------------
 *
 * resample_locations (mcmc.hpp:80-97) -> sample_point_in_region
 * (geo.hpp:138-161) as one GPU thread per event: area-weighted polygon part,
 * bounding-box rejection against the even-odd point-in-polygon test (outer
 * ring minus holes), 10000 attempts; point regions return their point.  The
 * random stream is Philox4x32-10 keyed by `seed` with counter (event,
 * `counter`), NOT the reference's mt19937_64: draws are reproducible for a
 * fixed (seed, counter) and match the reference in distribution.
 *
 * Region table, flattened (a RegionTable, geo.hpp:85-113):
 *   is_point[R], point_xy[2R]          Region::is_point / point
 *   region_parts[R+1]                  region r owns parts [region_parts[r], region_parts[r+1])
 *   part_rings[P+1]                    part p owns rings [part_rings[p], part_rings[p+1]);
 *                                      the first is the outer ring, the rest holes
 *   ring_verts[Rings+1], verts[2V]     ring g's vertices (lon, lat) pairs
 *   region_ids[R] (nullable)           Region::id, for error messages
 *   event_region[N]                    each catalog event's region index
 * Failures (zero-area region, exhausted attempts) return HK_RUNTIME_ERROR
 * with the reference's runtime_error message and the event index. */
typedef struct hk_regions hk_regions;
int hk_regions_create(size_t n_regions, const int* is_point, const double* point_xy,
                      const size_t* region_parts, const size_t* part_rings, const size_t* ring_verts,
                      const double* verts, const char* const* region_ids, size_t n_events,
                      const int* event_region, int device, hk_regions** out);
void hk_regions_destroy(hk_regions* regions);
/* One draw for every event into host arrays lon[N], lat[N]. */
int hk_regions_sample(hk_regions* regions, uint64_t seed, uint64_t counter, double* lon, double* lat);
/* One draw for every event straight into the context's device locations
 * (then the hk_set_locations check and broadcast); the region table must
 * live on the context's first device. */
int hk_resample_locations(hk_ctx* ctx, hk_regions* regions, uint64_t seed, uint64_t counter);

/* Per-row contributions ell_n for rows [b, e) (slice_log_likelihood on
 * single rows, engine.hpp:65-83).  ell_rows has e-b entries; grad_rows, if
 * non-NULL, has 5*(e-b) entries (row-major, 5 per row).  Rows must lie in
 * the context's row range, else HK_OUT_OF_RANGE. */
int hk_eval_rows(hk_ctx* ctx, const hk_params* p, size_t b, size_t e, double* ell_rows,
                 double* grad_rows);

/* Evaluation options (all default on).
 *   HK_OPT_BG_EXPANSION: evaluate the background sum of qualifying tile
 *     pairs by the exact block expansion instead of
 *     per pair; 0 forces the direct per-pair path everywhere. */
#define HK_OPT_BG_EXPANSION 1
/*   HK_OPT_FGT: evaluate the homogeneous trigger of the tiles earlier than
 *     each block's checkpoint by the certified Hermite expansion (fast Gauss
 *     transform) where it is cheaper; 0 forces the
 *     direct per-pair path.  Rows whose certified error bound could exceed
 *     1e-13 relative make the synchronous calls recompute directly. */
#define HK_OPT_FGT 2
/*   HK_OPT_BG_FGT: evaluate the background sums of every row by the
 *     certified 1-D Hermite expansion in time (both variants, FP64 only);
 *     0 returns them to the pair kernels (block expansion / per pair). */
#define HK_OPT_BG_FGT 3
/*   HK_OPT_TR_CUT: the density-scaled FP64 trigger drops a source for every
 *     row whose spatial factor is below e^-46 (instead of only exact zeros);
 *     the dropped weight is bounded per row and certified like the
 *     expansions (1e-13 relative to the row's rate, else recomputed). */
#define HK_OPT_TR_CUT 4
/*   HK_OPT_CELLS: the density-scaled FP64 trigger visits its sources
 *     regrouped by spatial cell (tiles of one cell, time order within it),
 *     so whole tiles beyond a block's reach are skipped; 0 visits them in
 *     time order.  Same sums, different summation order. */
#define HK_OPT_CELLS 5
/*   HK_OPT_SINGLE_FP64: Precision::single evaluations of catalogs of at least
 *     131072 events run the FP64 expansion / cut path (faster there than the
 *     FP32 direct kernels, and more accurate); 0 keeps the FP32 kernels. */
#define HK_OPT_SINGLE_FP64 6
int hk_set_option(hk_ctx* ctx, int option, int value);
/* Evaluations that used a Hermite expansion (trigger or background),
 * synchronous ones recomputed
 * directly after a failed certification, and whether the last asynchronous
 * evaluation's certification failed (1; it is not recomputed). */
int hk_fgt_stats(hk_ctx* ctx, long* evals, long* fallbacks, int* async_flagged);

/* Rows [begin, end) this context evaluates, and its device count. */
int hk_rows(const hk_ctx* ctx, size_t* begin, size_t* end, int* n_devices);

/* Device-side timing of the pair kernel (CUDA events on the launching
 * stream).  Enable before evaluating; read back accumulated milliseconds,
 * the number of pair-kernel launches, and the number of all kernel
 * launches this library made since the last reset. */
int hk_set_profiling(hk_ctx* ctx, int enable);
int hk_profile(hk_ctx* ctx, double* pair_kernel_ms, long* pair_launches, long* total_launches);
int hk_reset_profile(hk_ctx* ctx);
/* The same events split by launch kind: [0] pair launches computing both
 * halves, [1] background-only launches, [2] trigger-only launches (the
 * density-scaled plan runs one [1] and one [2] per evaluation), [3] the
 * Hermite expansion's moment launches (box assignment, increments, scan),
 * [4] its row evaluation.  ms5 and launches5 have 5 entries each. */
int hk_profile_kinds(hk_ctx* ctx, double* ms5, long* launches5);

/* Catalog invariants (types.hpp:43-57) and HawkesParams::validate
 * (types.hpp:92-103) on their own, with the reference's messages. */
int hk_validate_catalog(const double* t, const double* lon, const double* lat,
                        const double* density, size_t n);
int hk_validate_params(const hk_params* p);

/* Partition::make (engine.hpp:27-40) as g+1 boundaries. */
int hk_partition_make(size_t n, size_t g, size_t* bounds);

/* Cost-balanced contiguous row shards for g devices: boundaries (g+1) such
 * that each shard carries ~1/g of the pair work, row n costing
 * alpha*(N-1) + beta*count_before(t_n): alpha = 13, beta = 16 (FP64 per pair)
 * on the direct path, alpha = 1, beta = 46 (measured) for N >= 32768 where
 * the background block expansion applies. */
int hk_plan_shards(const double* t, size_t n, size_t g, size_t* bounds);

/* The same for the kernel variant the shards will mostly run: the
 * density-scaled (HK_VARIANT_VARYING) kernel culls its trigger spatially, so
 * its rows cost alpha*(N-1) + 4.3*count_before(t_n). */
int hk_plan_shards_variant(const double* t, size_t n, size_t g, int variant, size_t* bounds);

/* benchmark_catalog(n, seed) (engine.hpp:251-259): the reference's
 * synthetic uniform catalog, bit-identical (mt19937_64, libstdc++
 * uniform_real_distribution, stable sort by t). */
int hk_benchmark_catalog(size_t n, uint64_t seed, double* t, double* lon, double* lat,
                         double* density);

/* Measured FP64 FMA throughput of `device` in TFLOP/s (2 flop per DFMA),
 * from a short register-resident DFMA loop; the roofline denominator. */
int hk_measure_fp64_peak(int device, double* tflops, double* ms);

const char* hk_last_error(void);
const char* hk_version(void);

#ifdef __cplusplus
}
#endif

#endif /* HAWKES_B200_H */
