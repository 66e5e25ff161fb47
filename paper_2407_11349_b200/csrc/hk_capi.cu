// C ABI (include/hawkes_b200.h): evaluation contexts over one or more B200s.
//
// A context holds, per device, a full replica of the catalog in SoA form
// (t, lon, lat, density; padded to whole 256-column tiles), the tie bounds
// lb/ub, the per-evaluation prep arrays, the work-item list for that
// device's row shard, and the partial-sum buffer.  Catalog data are
// uploaded once (hk_create) and locations replaced in place
// (hk_set_locations), matching LikelihoodWorkspace's lifetime
// (engine.hpp:117-229).  Multi-device contexts evaluate their shards
// concurrently (one stream per device); the per-device 6-vectors
// [ell, d ell / d theta] are all-gathered over NVLink with NCCL and summed
// on the device in device order (deterministic), and new locations go to
// device 0 once and are NCCL-broadcast to the others (north_star's data
// plane; the reference's ordered slice reduction is engine.hpp:91-98).  A
// context whose device list repeats a device (several shards on one GPU:
// the single-GPU test of this path) moves the same bytes with peer copies
// instead; the arithmetic is identical.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types and prototypes only: libnccl is dlopen'ed when a context needs it

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/hawkes_b200.h"
#include "hk_device.cuh"
#include "hk_host.hpp"
#include "hk_fgt.cuh"
#include "hk_kernels.cuh"
#include "hk_regions.hpp"

namespace {

thread_local std::string g_err;

// NCCL, loaded on first use by a multi-device context (the library itself
// has no link-time NCCL dependency; in a PyTorch process this resolves to
// the libnccl.so.2 torch already loaded).
struct NcclApi {
  decltype(&ncclCommInitAll) CommInitAll = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclAllGather) AllGather = nullptr;
  decltype(&ncclBroadcast) Broadcast = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
  std::string error;
};

const NcclApi& nccl_api() {
  static const NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.error = std::string("cannot load libnccl.so.2: ") + dlerror();
      return a;
    }
    auto sym = [&](auto& fp, const char* name) {
      fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
      if (!fp && a.error.empty()) a.error = std::string("libnccl.so.2 lacks ") + name;
    };
    sym(a.CommInitAll, "ncclCommInitAll");
    sym(a.CommDestroy, "ncclCommDestroy");
    sym(a.AllGather, "ncclAllGather");
    sym(a.Broadcast, "ncclBroadcast");
    sym(a.GroupStart, "ncclGroupStart");
    sym(a.GroupEnd, "ncclGroupEnd");
    sym(a.GetErrorString, "ncclGetErrorString");
    return a;
  }();
  return api;
}

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NotImplemented : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

void nck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw CudaError(std::string(what) + ": " + nccl_api().GetErrorString(r));
}

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return HK_OK;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return HK_INVALID_ARGUMENT;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return HK_OUT_OF_RANGE;
  } catch (const NotImplemented& e) {
    g_err = e.what();
    return HK_NOT_IMPLEMENTED;
  } catch (const std::exception& e) {
    g_err = e.what();
    return HK_RUNTIME_ERROR;
  }
}

// Row blocks per clustering window of the varying plan: the largest power
// of two whose window holds at most kMaxSplitWindow rows (median splits first
// above kMaxClusterWindow, hk::launch_cluster) and leaves at least ~6
// windows (N=1e6: 512 blocks of 256 rows; N=1e5: 64).  With the cell layout
// the trigger wants the largest windows (spatially smallest k-d leaves of 64
// rows; the window's longer time span costs little once whole cell tiles are
// classified per CTA).  Trigger ms, bench / county catalog: N=1e6 64 blocks
// 7.95 / 51.2, 128 5.66 / 45.0, 256 4.40 / 42.9, 512 3.79 / 44.1; N=1e5 32
// blocks 0.28 / 0.83, 64 0.24 / 0.78; N=1e7 256 blocks 379, 512 313, 1024
// 266 (at N=1e6, 1024 blocks: 3.51 / 48.7 — the county catalog turns).
// HK_ROW_WINDOW overrides (1 disables the clustering).
int row_window(int rows) {
  if (const char* e = std::getenv("HK_ROW_WINDOW")) {
    const int w = std::atoi(e);
    if (w >= 1 && w <= 1024 && (w & (w - 1)) == 0 && w * hk::rows_per_item(true) <= hk::kMaxSplitWindow)
      return w;
  }
  const int blocks = (rows + hk::rows_per_item(true) - 1) / hk::rows_per_item(true);
  const int w_max = hk::kMaxSplitWindow / hk::rows_per_item(true);
  int w = 1;
  while (w < w_max && 2 * w * 6 <= blocks) w *= 2;
  return w;
}

template <typename T>
T* dmalloc(std::size_t count) {
  void* p = nullptr;
  ck(cudaMalloc(&p, std::max<std::size_t>(count, 1) * sizeof(T)), "cudaMalloc");
  return static_cast<T*>(p);
}

struct DeviceState {
  int dev = 0;
  cudaStream_t stream = nullptr;
  int rb = 0, re = 0;  // row shard
  double *t = nullptr, *x = nullptr, *y = nullptr, *q = nullptr;
  double *K = nullptr, *thr = nullptr, *w = nullptr, *v = nullptr, *z = nullptr;
  float4* fxy = nullptr;
  float2* fkw = nullptr;
  double2 *xy = nullptr, *wk = nullptr, *vz = nullptr;  // interleaved trigger columns
  int *lb = nullptr, *ub = nullptr;
  // clustered row order of the varying plan (hk::launch_cluster), valid for
  // location version rperm_loc
  int* rperm = nullptr;
  int* cluster_scratch = nullptr;  // row lists of split windows (windows over kMaxClusterWindow rows)
  int window = 1;
  long rperm_loc = -1;
  // work plans per variant (rows per item differ, hk_device.cuh)
  // plans: [0] constant (also every background-only launch of the varying
  // variant, see enqueue), [1] varying (clustered windows)
  // [2]: the homogeneous trigger-only plan with the Hermite expansion
  // (hk_host.cpp plan_items_fgt: one item per row block over its band)
  // [3]: the density-scaled FP64 trigger over spatial cell tiles (hk_cells.cu)
  hk::Item* items[4] = {nullptr, nullptr, nullptr, nullptr};
  int n_items[4] = {0, 0, 0, 0}, slots[4] = {0, 0, 0, 0};
  // spatial cell tiles (hk_cells.cu): the column regrouping of location
  // version cells_loc, and its per-evaluation arrays
  hk::CellGrid cgrid{};
  hk::CellLayout cells{};
  int *cell_id = nullptr, *cell_chunk = nullptr, *cell_start = nullptr, *cell_perm = nullptr,
      *cell_nct = nullptr;
  long cells_loc = -1;
  double* partial = nullptr;
  double* bg_sums[2] = {nullptr, nullptr};  // [B, B2] x rows, LRU-2 (workspace cache)
  double* tr_sums[2] = {nullptr, nullptr};  // [T, Td, Tq] x rows
  double* blockpart = nullptr;
  int n_finish_blocks = 0;
  double* out6 = nullptr;
  double* h_out6 = nullptr;  // pinned
  // Hermite expansion of the homogeneous trigger (hk_fgt.cu): checkpoint
  // prefixes of this shard's row blocks and the per-evaluation buffers
  // checkpoints: ck_off virtual ones (every kFgtCkRows columns below the
  // shard's first prefix: a shard starting late must not sum its whole prefix
  // in one increment) followed by nck_rows real ones (one per 4 row blocks)
  int nck = 0, ck_off = 0, nck_rows = 0, fgt_cols = 0;
  double fgt_direct_cost = 0.0;  // trigger pairs the expansion replaces (sum over rows of P_k)
  int* ck_P = nullptr;                                   // [nck]
  double *fgt_tR = nullptr, *fgt_decay = nullptr, *fgt_dt = nullptr, *fgt_wsum = nullptr;  // [nck]
  int* fgt_box = nullptr;                                // [fgt_cols]
  double *fgt_u = nullptr, *fgt_v = nullptr;             // [fgt_cols]
  double* fgt_mom = nullptr;                             // [nck][nbox][2][P^2], grown on demand
  int* fgt_perm = nullptr;                               // [nck * kFgtCkRows] clustered rows
  long fgt_perm_loc = -1;                                // location version of fgt_perm
  std::size_t fgt_mom_bytes = 0;
  double* bgf_mom = nullptr;  // [nbt][kFgtP]: the background's 1-D expansion
  int* bgf_count = nullptr;   // [nbt]
  double* bgf_part = nullptr; // [nbt][parts][kFgtP] moment parts
  int bgf_cap = 0;            // boxes allocated
  unsigned* fgt_flag = nullptr;                          // device
  unsigned* h_fgt_flag = nullptr;                        // pinned
  bool flag_pending = false;                             // set by hk_eval_async
  double* cert_scratch = nullptr;                        // density-scaled cut certification
  double* gather6 = nullptr;  // [n_dev][6]: every device's out6 (multi-device contexts)
  double* total6 = nullptr;   // their device-order sum
  cudaEvent_t done = nullptr; // peer-copy mode: this device's part is ready
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_events;
  std::vector<int> prof_kind;  // per used event pair: 0 both halves, 1 background, 2 trigger, 3 FGT moments, 4 FGT rows
  std::size_t prof_used = 0;

  hk::DeviceCatalog catalog(int n, int npad) const {
    return hk::DeviceCatalog{n, npad, t, x, y, q, lb, ub, K, thr, w, v, z, fxy, fkw, rperm, xy, wk, vz};
  }
};

}  // namespace

struct hk_ctx {
  int n = 0, npad = 0;
  std::vector<double> t, x, y, d;
  std::vector<int> lb, ub;
  double d2_max = 0.0, q_max = 1.0;
  double cx = 0.0, cy = 0.0, half_extent = 0.0;
  bool unit_density = false;  // every density == 1: varying == constant exactly
  bool locations_valid = true;  // false for a coarse-only catalog until set_locations
  std::vector<DeviceState> devs;
  // multi-device data plane: NCCL communicators over distinct devices, or
  // peer copies when the device list repeats a device
  bool use_nccl = false;
  std::vector<ncclComm_t> comms;
  double* bbox_scratch = nullptr;  // device 0
  double* bbox_out = nullptr;      // device 0, 5 doubles
  double* h_bbox = nullptr;        // pinned
  bool profiling = false;
  int bg_expansion = 1;
  int fgt_enabled = 1;     // HK_OPT_FGT
  int bg_fgt_enabled = 1;  // HK_OPT_BG_FGT
  int tr_cut_enabled = 1;  // HK_OPT_TR_CUT
  int cells_enabled = 1;   // HK_OPT_CELLS
  int single_fp64 = 1;     // HK_OPT_SINGLE_FP64
  long fgt_evals = 0, fgt_fallbacks = 0;
  bool fgt_pending = false;  // an async evaluation's certification flag is unread

  // Per-evaluation decision for the homogeneous trigger's Hermite expansion.
  struct FgtPlan {
    bool on = false;
    int nb = 0;
    double L = 0, x0 = 0, y0 = 0, inv_sqd = 0, delta = 0, eps = 0;
    // the background's 1-D expansion in time
    bool bg = false;
    int nbt = 0;
    double t0 = 0, Lt = 0, inv_sqdt = 0, delta_t = 0, eps_t = 0;
  };

  // Workspace cache keys (LikelihoodWorkspace semantics, engine.hpp:117-229):
  // the background half depends on tau_t only, the trigger half on
  // (sigma_x, sigma_t, variant) and the locations.  Two entries per half
  // hold the current state and a proposal; the least recently used is
  // replaced.  Every evaluation goes through the same kernels, so cached and
  // fresh results are bitwise identical.
  struct Key {
    bool valid = false;
    double a = 0, b = 0;
    int variant = 0, grad = 0, bgx = 0;
    long loc = 0;
    unsigned long long used = 0;
  };
  Key bg_key[2], tr_key[2];
  long loc_version = 0;
  unsigned long long clock = 0;
  long ws_hits = 0, ws_misses = 0;
  double prof_ms = 0.0;
  long prof_pair = 0, prof_total = 0;

  ~hk_ctx() {
    for (ncclComm_t c : comms)
      if (c) nccl_api().CommDestroy(c);
    if (!devs.empty()) {
      cudaSetDevice(devs[0].dev);
      if (bbox_scratch) cudaFree(bbox_scratch);
      if (bbox_out) cudaFree(bbox_out);
      if (h_bbox) cudaFreeHost(h_bbox);
    }
    for (auto& s : devs) {
      cudaSetDevice(s.dev);
      if (s.stream) cudaStreamSynchronize(s.stream);
      for (double* p : {s.t, s.x, s.y, s.q, s.K, s.thr, s.w, s.v, s.z, s.partial, s.blockpart, s.out6,
                        s.bg_sums[0], s.bg_sums[1], s.tr_sums[0], s.tr_sums[1]})
        if (p) cudaFree(p);
      if (s.fxy) cudaFree(s.fxy);
      if (s.fkw) cudaFree(s.fkw);
      for (double2* p2 : {s.xy, s.wk, s.vz})
        if (p2) cudaFree(p2);
      if (s.lb) cudaFree(s.lb);
      if (s.ub) cudaFree(s.ub);
      if (s.rperm) cudaFree(s.rperm);
      if (s.cluster_scratch) cudaFree(s.cluster_scratch);
      for (void* q : {static_cast<void*>(s.cell_id), static_cast<void*>(s.cell_chunk),
                      static_cast<void*>(s.cell_start), static_cast<void*>(s.cell_perm),
                      static_cast<void*>(s.cell_nct), static_cast<void*>(s.cells.xy),
                      static_cast<void*>(s.cells.wk), static_cast<void*>(s.cells.vz),
                      static_cast<void*>(s.cells.fxy), static_cast<void*>(s.cells.t),
                      static_cast<void*>(s.cells.q), static_cast<void*>(s.cells.box),
                      static_cast<void*>(s.cells.r2), static_cast<void*>(s.cells.tmin),
                      static_cast<void*>(s.cells.tmax)})
        if (q) cudaFree(q);
      for (hk::Item* it : s.items)
        if (it) cudaFree(it);
      if (s.h_out6) cudaFreeHost(s.h_out6);
      for (void* q : {static_cast<void*>(s.ck_P), static_cast<void*>(s.fgt_tR), static_cast<void*>(s.fgt_decay),
                      static_cast<void*>(s.fgt_dt), static_cast<void*>(s.fgt_box), static_cast<void*>(s.fgt_u),
                      static_cast<void*>(s.fgt_v), static_cast<void*>(s.fgt_mom), static_cast<void*>(s.fgt_flag),
                      static_cast<void*>(s.bgf_mom), static_cast<void*>(s.bgf_count), static_cast<void*>(s.bgf_part), static_cast<void*>(s.fgt_wsum),
                      static_cast<void*>(s.fgt_perm), static_cast<void*>(s.cert_scratch)})
        if (q) cudaFree(q);
      if (s.h_fgt_flag) cudaFreeHost(s.h_fgt_flag);
      if (s.gather6) cudaFree(s.gather6);
      if (s.total6) cudaFree(s.total6);
      if (s.done) cudaEventDestroy(s.done);
      for (auto& e : s.prof_events) {
        cudaEventDestroy(e.first);
        cudaEventDestroy(e.second);
      }
      if (s.stream) cudaStreamDestroy(s.stream);
    }
  }

  // The evaluation frame from the locations' box (argument bound of the
  // exp mode, FP32 culling frame); `bad` = first non-finite index or n.
  void set_bbox(double xmin, double xmax, double ymin, double ymax, long bad) {
    locations_valid = bad >= n;
    if (!locations_valid) {
      d2_max = 0.0;
      cx = cy = half_extent = 0.0;
      return;
    }
    const double w = xmax - xmin, h = ymax - ymin;
    d2_max = w * w + h * h;
    cx = 0.5 * (xmin + xmax);
    cy = 0.5 * (ymin + ymax);
    half_extent = 0.5 * std::max(w, h);
  }

  // host version (hk_create, before any device exists)
  void update_bbox() {
    long bad = n;
    for (int i = 0; i < n && bad == n; ++i)
      if (!std::isfinite(x[i]) || !std::isfinite(y[i])) bad = i;
    if (bad < n) return set_bbox(0, 0, 0, 0, bad);
    double xmin = x[0], xmax = x[0], ymin = y[0], ymax = y[0];
    for (int i = 1; i < n; ++i) {
      xmin = std::min(xmin, x[i]);
      xmax = std::max(xmax, x[i]);
      ymin = std::min(ymin, y[i]);
      ymax = std::max(ymax, y[i]);
    }
    set_bbox(xmin, xmax, ymin, ymax, n);
  }

  // The multi-device data plane is active (several devices, or one forced
  // through NCCL).
  bool multi() const { return devs.size() > 1 || use_nccl; }

  // Multi-device set-up after every device is initialised: NCCL
  // communicators over distinct devices (HK_NO_NCCL=1 or a repeated device:
  // peer copies), the gather buffers, and device 0's bbox buffers.
  void init_data_plane() {
    const int g = static_cast<int>(devs.size());
    ck(cudaSetDevice(devs[0].dev), "cudaSetDevice");
    bbox_scratch = dmalloc<double>(hk::bbox_scratch_doubles());
    bbox_out = dmalloc<double>(5);
    ck(cudaMallocHost(&h_bbox, 5 * sizeof(double)), "cudaMallocHost");
    // HK_FORCE_NCCL=1: the NCCL data plane even for one device (a one-rank
    // communicator: exercises the all-gather / broadcast path on one GPU)
    const char* force = std::getenv("HK_FORCE_NCCL");
    const bool force_nccl = force && std::atoi(force) != 0;
    if (g == 1 && !force_nccl) return;
    std::vector<int> ids(g);
    for (int k = 0; k < g; ++k) ids[k] = devs[k].dev;
    std::vector<int> sorted_ids = ids;
    std::sort(sorted_ids.begin(), sorted_ids.end());
    const bool distinct = std::adjacent_find(sorted_ids.begin(), sorted_ids.end()) == sorted_ids.end();
    const char* no = std::getenv("HK_NO_NCCL");
    use_nccl = distinct && (force_nccl || !(no && std::atoi(no) != 0));
    for (auto& s : devs) {
      ck(cudaSetDevice(s.dev), "cudaSetDevice");
      s.gather6 = dmalloc<double>(6 * static_cast<std::size_t>(g));
      s.total6 = dmalloc<double>(6);
      ck(cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming), "cudaEventCreate");
    }
    if (use_nccl) {
      const NcclApi& api = nccl_api();
      if (!api.error.empty())
        throw CudaError("multi-device context needs NCCL: " + api.error +
                        " (HK_NO_NCCL=1 moves the 6-vectors and locations with peer copies instead)");
      comms.assign(g, nullptr);
      nck(api.CommInitAll(comms.data(), g, ids.data()), "ncclCommInitAll");
    }
  }

  // Device 0's x, y (already written) -> box + finiteness check on device 0
  // -> NCCL broadcast (or peer copies) to the other devices.  Throws the
  // reference's Catalog message for a non-finite location.
  void publish_locations() {
    DeviceState& s0 = devs[0];
    ck(cudaSetDevice(s0.dev), "cudaSetDevice");
    hk::launch_bbox(s0.x, s0.y, n, bbox_scratch, bbox_out, s0.stream);
    ck(cudaMemcpyAsync(h_bbox, bbox_out, 5 * sizeof(double), cudaMemcpyDeviceToHost, s0.stream),
       "bbox copy");
    const int g = static_cast<int>(devs.size());
    if (multi()) {
      if (use_nccl) {
        const NcclApi& api = nccl_api();
        nck(api.GroupStart(), "ncclGroupStart");
        for (int k = 0; k < g; ++k) {
          DeviceState& s = devs[k];
          ck(cudaSetDevice(s.dev), "cudaSetDevice");
          nck(api.Broadcast(s0.x, s.x, n, ncclFloat64, 0, comms[k], s.stream), "ncclBroadcast");
          nck(api.Broadcast(s0.y, s.y, n, ncclFloat64, 0, comms[k], s.stream), "ncclBroadcast");
        }
        nck(api.GroupEnd(), "ncclGroupEnd");
      } else {
        ck(cudaEventRecord(s0.done, s0.stream), "cudaEventRecord");
        for (int k = 1; k < g; ++k) {
          DeviceState& s = devs[k];
          ck(cudaSetDevice(s.dev), "cudaSetDevice");
          ck(cudaStreamWaitEvent(s.stream, s0.done, 0), "cudaStreamWaitEvent");
          ck(cudaMemcpyPeerAsync(s.x, s.dev, s0.x, s0.dev, n * sizeof(double), s.stream), "peer copy");
          ck(cudaMemcpyPeerAsync(s.y, s.dev, s0.y, s0.dev, n * sizeof(double), s.stream), "peer copy");
        }
      }
    }
    ck(cudaSetDevice(s0.dev), "cudaSetDevice");
    ck(cudaStreamSynchronize(s0.stream), "set_locations");
    set_bbox(h_bbox[0], h_bbox[1], h_bbox[2], h_bbox[3], static_cast<long>(h_bbox[4]));
    ++loc_version;  // drops the trigger caches (engine.hpp:177)
    if (!locations_valid)
      throw std::invalid_argument("Catalog: event " + std::to_string(static_cast<long>(h_bbox[4])) +
                                  " has non-finite location");
  }

  void upload_padded(DeviceState& s, double* dst, const std::vector<double>& src, double pad) {
    std::vector<double> tmp(npad, pad);
    std::copy(src.begin(), src.end(), tmp.begin());
    ck(cudaMemcpyAsync(dst, tmp.data(), npad * sizeof(double), cudaMemcpyHostToDevice, s.stream),
       "upload");
    ck(cudaStreamSynchronize(s.stream), "upload sync");
  }

  void init_device(DeviceState& s, int dev, int rb, int re) {
    s.dev = dev;
    s.rb = rb;
    s.re = re;
    ck(cudaSetDevice(dev), "cudaSetDevice");
    ck(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking), "cudaStreamCreate");
    hk::upload_exp2_table(s.stream);
    ck(cudaGetLastError(), "exp table");
    s.t = dmalloc<double>(npad);
    s.x = dmalloc<double>(npad);
    s.y = dmalloc<double>(npad);
    s.q = dmalloc<double>(npad);
    s.K = dmalloc<double>(npad);
    s.thr = dmalloc<double>(npad);
    s.w = dmalloc<double>(npad);
    s.v = dmalloc<double>(npad);
    s.z = dmalloc<double>(npad);
    s.fxy = dmalloc<float4>(npad);
    s.fkw = dmalloc<float2>(npad);
    s.xy = dmalloc<double2>(npad);
    s.wk = dmalloc<double2>(npad);
    s.vz = dmalloc<double2>(npad);
    s.lb = dmalloc<int>(n);
    s.ub = dmalloc<int>(n);
    upload_padded(s, s.t, t, t[n - 1]);
    upload_padded(s, s.x, x, 0.0);
    upload_padded(s, s.y, y, 0.0);
    upload_padded(s, s.q, d, 1.0);
    ck(cudaMemcpy(s.lb, lb.data(), n * sizeof(int), cudaMemcpyHostToDevice), "upload lb");
    ck(cudaMemcpy(s.ub, ub.data(), n * sizeof(int), cudaMemcpyHostToDevice), "upload ub");
    // The varying kernel reads its rows in spatially clustered windows of
    // kRowWindow row blocks so that warps can skip columns (launch_cluster).
    // sized by the catalog (the trigger sweeps all n columns), not the shard
    s.window = row_window(n);
    if (s.window > 1) {
      const int wr = s.window * hk::rows_per_item(true);
      const int nb = (re - rb + hk::rows_per_item(true) - 1) / hk::rows_per_item(true);
      s.rperm = dmalloc<int>(static_cast<std::size_t>(hk::window_count(nb, s.window)) * wr);
      if (wr > hk::kClusterSplitTarget)  // windows split at medians before clustering (hk::launch_cluster)
        s.cluster_scratch = dmalloc<int>(2 * static_cast<std::size_t>(hk::window_count(nb, s.window)) * wr +
                                         hk::cluster_work_ints(hk::window_count(nb, s.window), wr));
    }
    for (int v = 0; v < 2; ++v) {
      std::vector<hk::Item> items;
      s.slots[v] = hk::plan_items(lb, ub, n, rb, re, hk::rows_per_item(v != 0), items,
                                  v == 1 ? s.window : 1);
      s.n_items[v] = static_cast<int>(items.size());
      s.items[v] = dmalloc<hk::Item>(items.size());
      ck(cudaMemcpy(s.items[v], items.data(), items.size() * sizeof(hk::Item),
                    cudaMemcpyHostToDevice),
         "upload items");
    }
    if (s.window > 1) {
      // spatial cell tiles of the density-scaled FP64 trigger: a gc x gc grid
      // by catalog size (measured with 2 rows/thread and 32768-row windows,
      // trigger ms bench / county catalog: N=5e4 gc 1/2/4 = 0.165/0.161/0.172,
      // 0.281/0.314/0.323; 1e5 gc 1/2/4 = 0.34/0.29/0.28, 0.78/0.85/0.83;
      // 3e5 gc 2/4/8 = 1.12/0.95/0.94, 5.31/5.08/4.98; 1e6 gc 4/8/16 (two
      // classes) = 6.0/5.7/6.7, 44.9/45.1/47.2; 1e7 gc 8/16 = 514/574: cells
      // larger than the sources' reach gain no skips, while a cell tile's
      // time span, 256 gc^2 / n of the catalog, sets how many tiles straddle
      // a block's rows); every cell wastes at most one partial tile
      int gc = n < 75000 ? 1 : n < 200000 ? 4 : 8;
      if (const char* e = std::getenv("HK_CELL_GC")) gc = std::min(64, std::max(1, std::atoi(e)));  // tuning
      // reach classes: each cell's sources split into bands of log density
      // (a source's reach scales as 1/sqrt(q)), so a cell tile's largest
      // threshold is not set by one low-density source among many local ones
      // (N=1e6, trigger ms for 1/2/4/8 classes with 4 rows/thread: bench
      // catalog 8.37/8.21/8.27/8.46, county 52.8/51.5/51.6/52.6; with 2
      // rows/thread 1/2 classes 6.03/5.66, 47.0/45.1; with 512-block windows
      // 2/3 classes 3.80/3.76, 44.1/43.7): three from gc = 8
      int ncls = gc >= 8 ? 3 : 1;
      if (const char* e = std::getenv("HK_CELL_CLASSES")) ncls = std::min(16, std::max(1, std::atoi(e)));  // tuning
      double qmin = d[0], qmax = d[0];
      for (double v : d) {
        qmin = std::min(qmin, v);
        qmax = std::max(qmax, v);
      }
      if (!(qmin > 0.0) || !(qmax > qmin)) ncls = 1;  // one density (or invalid): no classes
      s.cgrid.ncls = ncls;
      s.cgrid.lq0 = ncls > 1 ? std::log(qmin) : 0.0;
      s.cgrid.inv_lq = ncls > 1 ? ncls / (std::log(qmax) - std::log(qmin)) : 0.0;
      const int ncell = gc * gc * ncls;
      const int max_tiles = (n + hk::kBJ - 1) / hk::kBJ + ncell;
      const std::size_t npos = static_cast<std::size_t>(max_tiles) * hk::kBJ;
      s.cgrid.gc = gc;
      s.cell_id = dmalloc<int>(n);
      s.cell_chunk = dmalloc<int>(static_cast<std::size_t>((n + 1023) / 1024) * ncell);
      s.cell_start = dmalloc<int>(ncell + 1);
      s.cell_perm = dmalloc<int>(npos);
      s.cell_nct = dmalloc<int>(1);
      s.cells.perm = s.cell_perm;
      s.cells.n_ctiles = s.cell_nct;
      s.cells.max_tiles = max_tiles;
      s.cells.xy = dmalloc<double2>(npos);
      s.cells.wk = dmalloc<double2>(npos);
      s.cells.vz = dmalloc<double2>(npos);
      s.cells.fxy = dmalloc<float4>(npos);
      s.cells.t = dmalloc<double>(npos);
      s.cells.q = dmalloc<double>(npos);
      s.cells.box = dmalloc<float4>(max_tiles);
      s.cells.r2 = dmalloc<float>(max_tiles);
      s.cells.tmin = dmalloc<double>(max_tiles);
      s.cells.tmax = dmalloc<double>(max_tiles);
      std::vector<hk::Item> items;
      s.slots[3] = hk::plan_items(lb, ub, n, rb, re, hk::rows_per_item(true), items, s.window, max_tiles);
      s.n_items[3] = static_cast<int>(items.size());
      s.items[3] = dmalloc<hk::Item>(items.size());
      ck(cudaMemcpy(s.items[3], items.data(), items.size() * sizeof(hk::Item), cudaMemcpyHostToDevice),
         "upload items");
    }
    {
      std::vector<hk::Item> items;
      s.slots[2] = hk::plan_items_fgt(lb, ub, n, rb, re, hk::rows_per_item(false), items);
      s.n_items[2] = static_cast<int>(items.size());
      s.items[2] = dmalloc<hk::Item>(items.size());
      ck(cudaMemcpy(s.items[2], items.data(), items.size() * sizeof(hk::Item), cudaMemcpyHostToDevice),
         "upload items");
    }
    const std::size_t rows = static_cast<std::size_t>(re - rb);
    {  // Hermite-expansion checkpoints of the homogeneous plan (hk_host.cpp plan_items: Item::xt)
      static_assert(hk::kFgtRowBlock == hk::rows_per_item(false), "FGT checkpoints follow the homogeneous plan");
      const int bi = hk::rows_per_item(false);
      const int nblocks = (re - rb + bi - 1) / bi;
      s.nck_rows = (nblocks + hk::kFgtBlocks - 1) / hk::kFgtBlocks;
      std::vector<int> real(s.nck_rows), ckp;
      for (int k = 0; k < s.nck_rows; ++k) real[k] = lb[rb + k * hk::kFgtBlocks * bi] / hk::kBJ * hk::kBJ;
      for (int v = hk::kFgtCkRows; s.nck_rows && v < real[0]; v += hk::kFgtCkRows) ckp.push_back(v);
      s.ck_off = static_cast<int>(ckp.size());
      ckp.insert(ckp.end(), real.begin(), real.end());
      s.nck = static_cast<int>(ckp.size());
      s.fgt_cols = s.nck ? ckp.back() : 0;
      s.ck_P = dmalloc<int>(s.nck);
      ck(cudaMemcpy(s.ck_P, ckp.data(), s.nck * sizeof(int), cudaMemcpyHostToDevice), "upload checkpoints");
      s.fgt_tR = dmalloc<double>(s.nck);
      s.fgt_decay = dmalloc<double>(s.nck);
      s.fgt_dt = dmalloc<double>(s.nck);
      s.fgt_wsum = dmalloc<double>(s.nck);
      s.cert_scratch = dmalloc<double>(4 * static_cast<std::size_t>((n + hk::kCertChunk - 1) / hk::kCertChunk));
      s.fgt_perm = dmalloc<int>(static_cast<std::size_t>(s.nck_rows) * hk::kFgtCkRows);
      static_assert((hk::kFgtCkRows & (hk::kFgtCkRows - 1)) == 0, "checkpoint windows are sorted bitonically");
      s.fgt_box = dmalloc<int>(s.fgt_cols);
      s.fgt_u = dmalloc<double>(s.fgt_cols);
      s.fgt_v = dmalloc<double>(s.fgt_cols);
      s.fgt_flag = dmalloc<unsigned>(1);
      ck(cudaMallocHost(&s.h_fgt_flag, sizeof(unsigned)), "cudaMallocHost");
      s.fgt_direct_cost = 0.0;
      for (int b = 0; b < nblocks; ++b)
        s.fgt_direct_cost += static_cast<double>(std::min(bi, re - rb - b * bi)) * real[b / hk::kFgtBlocks];
    }
    s.partial = dmalloc<double>(static_cast<std::size_t>(std::max({s.slots[0], s.slots[1], s.slots[2], s.slots[3]})) * 5 *
                                rows);
    for (int k = 0; k < 2; ++k) {
      s.bg_sums[k] = dmalloc<double>(2 * rows);
      s.tr_sums[k] = dmalloc<double>(3 * rows);
    }
    s.n_finish_blocks = static_cast<int>((rows + 255) / 256);
    s.blockpart = dmalloc<double>(static_cast<std::size_t>(s.n_finish_blocks) * 6);
    s.out6 = dmalloc<double>(6);
    ck(cudaMallocHost(&s.h_out6, 6 * sizeof(double)), "cudaMallocHost");
  }

  std::pair<cudaEvent_t, cudaEvent_t> next_events(DeviceState& s, int kind) {
    if (s.prof_used == s.prof_events.size()) {
      cudaEvent_t a, b;
      ck(cudaEventCreate(&a), "cudaEventCreate");
      ck(cudaEventCreate(&b), "cudaEventCreate");
      s.prof_events.emplace_back(a, b);
      s.prof_kind.push_back(0);
    }
    s.prof_kind[s.prof_used] = kind;
    return s.prof_events[s.prof_used++];
  }

  // One pair launch, bracketed by profiling events of its kind when enabled.
  template <typename Fn>
  void timed_pair(DeviceState& s, int kind, Fn&& launch) {
    std::pair<cudaEvent_t, cudaEvent_t> ev{};
    if (profiling) {
      ev = next_events(s, kind);
      ck(cudaEventRecord(ev.first, s.stream), "cudaEventRecord");
    }
    launch();
    if (profiling) ck(cudaEventRecord(ev.second, s.stream), "cudaEventRecord");
  }

  hk::EvalCoef coef(const hk_params* p, bool single = false) const {
    if (!p) throw std::invalid_argument("hk_eval: null params");
    if (!locations_valid)
      throw std::invalid_argument(
          "hk_eval: event locations are not set (coarse-only catalog): call hk_set_locations first");
    hk::ParamsIn in{p->mu0, p->tau_t, p->xi0, p->sigma_x, p->sigma_t, p->area, p->variant};
    hk::validate_params(in);
    // With unit densities the varying kernel (q_j = D_j = 1) IS the constant
    // one; running it through the same plan keeps acceptance.cpp criterion 8
    // (variant collapse, bitwise) exact by construction.
    if (unit_density) in.variant = 0;
    hk::EvalCoef c = hk::make_coef(in, t[0], t[n - 1], d2_max, q_max);
    c.bg_expansion = bg_expansion;
    c.cx = cx;
    c.cy = cy;
    // |fl32(x - cx) - (x - cx)| <= E 2^-24 per coordinate (E = half extent),
    // twice per difference, plus the FP32 subtraction itself: 8 E 2^-24 bounds
    // the error of each FP32 coordinate difference with margin.
    c.f32_err = 8.0 * half_extent * 5.9604644775390625e-08;
    c.single_prec = single ? 1 : 0;
    return c;
  }

  // Whether this evaluation's homogeneous trigger goes through the Hermite
  // expansion: homogeneous FP64, expansion enabled, a box grid of at most
  // kFgtMaxBoxes boxes of side sqrt(2) sqrt(2 sigma_x^2), and an expected
  // cost (rows x boxes x terms) below half the direct trigger pairs it
  // replaces (x 16 FP64 each).
  FgtPlan fgt_plan(const hk::EvalCoef& c, bool grad) const {
    FgtPlan f;
    if (bg_fgt_enabled && !c.single_prec) {
      // background: time boxes of side gamma sqrt(2 tau^2) over [t_0, t_end]
      const double sqdt = std::sqrt(2.0) * c.tau_t;
      const double Lt = hk::kFgtGamma * sqdt;
      const double nbt = std::max(1.0, std::ceil((t[n - 1] - t[0]) / Lt));
      if (nbt <= hk::kBgFgtMaxBoxes) {
        f.bg = true;
        f.nbt = static_cast<int>(nbt);
        f.t0 = t[0];
        f.Lt = Lt;
        f.inv_sqdt = 1.0 / sqdt;
        f.delta_t = 2.0 * c.tau_t * c.tau_t;
        f.eps_t = hk::bg_fgt_truncation_bound(hk::kFgtP, hk::kFgtGamma) + 4e-16;
      }
    }
    if (!fgt_enabled || c.varying || c.single_prec || !locations_valid) return f;
    const double sqd = std::sqrt(2.0) * c.sigma_x;
    const double L = hk::kFgtGamma * sqd;
    const double span = 2.0 * half_extent;
    const double nbd = std::max(1.0, std::ceil(span / L));
    if (!(nbd * nbd <= hk::kFgtMaxBoxes)) return f;
    const int nb = static_cast<int>(nbd);
    double direct = 0.0, expanded = 0.0;
    const double per_row = static_cast<double>(nb * nb) * hk::kFgtP * hk::kFgtP * (grad ? 3.0 : 1.0);
    std::size_t moments = 0;
    for (const auto& s : devs) {
      direct += 16.0 * s.fgt_direct_cost;
      expanded += per_row * (s.re - s.rb);
      moments = std::max(moments, static_cast<std::size_t>(s.nck) * nb * nb * 2 * hk::kFgtP * hk::kFgtP);
    }
    if (!(expanded < 0.5 * direct) || moments * sizeof(double) > (std::size_t{48} << 30)) return f;
    f.on = true;
    f.nb = nb;
    f.L = L;
    f.x0 = cx - 0.5 * nb * L;
    f.y0 = cy - 0.5 * nb * L;
    f.inv_sqd = 1.0 / sqd;
    f.delta = 2.0 * c.sigma_x * c.sigma_x;
    f.eps = hk::fgt_truncation_bound(hk::kFgtP, hk::kFgtGamma) + 4e-16;  // + rounding of the sums
    return f;
  }

  hk::FgtParams fgt_params(DeviceState& s, const hk::EvalCoef& c, const FgtPlan& f, bool grad) {
    const std::size_t need = static_cast<std::size_t>(s.nck) * f.nb * f.nb * 2 * hk::kFgtP * hk::kFgtP *
                             sizeof(double);
    if (need > s.fgt_mom_bytes) {
      if (s.fgt_mom) ck(cudaFree(s.fgt_mom), "cudaFree");
      s.fgt_mom = nullptr;
      s.fgt_mom_bytes = 0;
      s.fgt_mom = dmalloc<double>(need / sizeof(double));
      s.fgt_mom_bytes = need;
    }
    hk::FgtParams F{};
    F.n = n;
    F.ncols = s.fgt_cols;
    F.t = s.t;
    F.x = s.x;
    F.y = s.y;
    F.nck = s.nck;
    F.ck_off = s.ck_off;
    F.nck_rows = s.nck_rows;
    F.P = s.ck_P;
    F.tR = s.fgt_tR;
    F.decay = s.fgt_decay;
    F.dt = s.fgt_dt;
    F.nb = f.nb;
    F.nbox = f.nb * f.nb;
    F.x0 = f.x0;
    F.y0 = f.y0;
    F.L = f.L;
    F.inv_sqd = f.inv_sqd;
    F.omega = c.omega;
    F.delta = f.delta;
    F.eps = f.eps;
    {  // per-box truncation: every box within the full square's bound (F.eps covers it)
      struct Table {
        unsigned short pn[hk::kFgtR2Buckets];
        Table() { hk::fgt_truncation_table(hk::kFgtGamma, hk::fgt_truncation_bound(hk::kFgtP, hk::kFgtGamma), pn); }
      };
      static const Table table;
      std::memcpy(F.pn, table.pn, sizeof(F.pn));
      if (std::getenv("HK_FGT_FULL_SQUARE"))  // comparisons: the full kFgtP x kFgtP square everywhere
        for (auto& v : F.pn) v = static_cast<unsigned short>(hk::kFgtP | (hk::kFgtP << 5) | ((hk::kFgtP / 2) << 10));
    }
    F.row_tol = hk::kFgtRowTol;
    if (const char* e = std::getenv("HK_FGT_ROW_TOL")) F.row_tol = std::atof(e);  // tests: force the fallback
    F.grad = grad ? 1 : 0;
    F.box = s.fgt_box;
    F.u = s.fgt_u;
    F.v = s.fgt_v;
    F.mom = s.fgt_mom;
    F.wsum = s.fgt_wsum;
    F.perm = s.fgt_perm;
    return F;
  }

  // The density-scaled FP64 trigger drops columns whose spatial factor is
  // below e^{-46} of their weight (certified per row, hk::launch_tr_cut_cert;
  // HK_OPT_TR_CUT=0 keeps the flush threshold: exact zeros only).
  void set_cut(hk::EvalCoef& c) const {
    if (tr_cut_enabled && c.varying && !c.single_prec) c.tr_cut = 46.0 * hk::kLog2eT;
  }

  // The density-scaled FP64 trigger runs over spatial cell tiles
  // (hk_cells.cu) on devices with a clustered plan.
  bool use_cells(const hk::EvalCoef& c) const {
    return cells_enabled && c.varying && !c.single_prec && !devs.empty() && devs.front().window > 1;
  }

  // The trigger half depends on the variant and on the precision.
  static int tr_variant(const hk::EvalCoef& c) { return c.varying + 2 * c.single_prec; }

  // Picks the cache entry for each half: a hit (unless forced) or the least
  // recently used entry, which the next enqueue recomputes.  Returns the
  // halves to compute.
  int plan_halves(const hk::EvalCoef& c, bool grad, bool force, int& bgi, int& tri, bool fgt = false,
                  bool bg_fgt = false) {
    const int bgx = c.bg_expansion + (bg_fgt ? 2 : 0);  // how the background half is computed
    const int tr_how = (fgt ? 1 : 0) + (c.tr_cut > 0.0 ? 2 : 0) + (use_cells(c) ? 4 : 0);  // ... and the trigger half
    // the background half is FP64 in both precisions, but each precision
    // keeps its own entries so a cached result is bitwise the fresh one of
    // the same precision (the launches differ between the two)
    auto hit_bg = [&](const Key& k) {
      return k.valid && k.a == c.tau_t && k.b == c.single_prec && k.bgx == bgx &&
             (k.grad || !grad);
    };
    auto hit_tr = [&](const Key& k) {
      return k.valid && k.a == c.sigma_x && k.b == c.sigma_t && k.variant == tr_variant(c) &&
             k.loc == loc_version && k.bgx == tr_how && (k.grad || !grad);
    };
    int halves = 0;
    bgi = -1;
    tri = -1;
    if (!force)
      for (int k = 0; k < 2; ++k) {
        if (bgi < 0 && hit_bg(bg_key[k])) bgi = k;
        if (tri < 0 && hit_tr(tr_key[k])) tri = k;
      }
    if (bgi < 0) {
      halves |= hk::kHalfBg;
      bgi = bg_key[0].used <= bg_key[1].used ? 0 : 1;
      bg_key[bgi] = Key{true, c.tau_t, static_cast<double>(c.single_prec), 0, grad ? 1 : 0, bgx, 0, 0};
    }
    if (tri < 0) {
      halves |= hk::kHalfTr;
      tri = tr_key[0].used <= tr_key[1].used ? 0 : 1;
      tr_key[tri] = Key{true, c.sigma_x, c.sigma_t, tr_variant(c), grad ? 1 : 0, tr_how, loc_version, 0};
    }
    bg_key[bgi].used = ++clock;
    tr_key[tri].used = ++clock;
    if (halves) ++ws_misses; else ++ws_hits;
    return halves;
  }

  // Enqueues [prep + pair + collapse for the missing halves] + finish + reduce.
  // ell_rows / grad_rows (device, optional): the shard's per-row ell_n and
  // d ell_n / d theta from the same launches.
  // Returns whether an expansion ran (its certification flag is then copied
  // to s.h_fgt_flag on the stream).
  bool enqueue(DeviceState& s, const hk::EvalCoef& c, bool grad, int halves, int bgi, int tri,
               double* ell_rows = nullptr, double* grad_rows = nullptr, const FgtPlan* fgt = nullptr) {
    ck(cudaSetDevice(s.dev), "cudaSetDevice");
    const hk::DeviceCatalog dc = s.catalog(n, npad);
    const int rows = s.re - s.rb;
    if (c.varying && s.window > 1 && s.rperm_loc != loc_version) {
      const int bi = hk::rows_per_item(true);
      hk::launch_cluster(s.x, s.y, s.rperm, s.rb, rows, s.window * bi,
                         hk::window_count((rows + bi - 1) / bi, s.window),
                         32 * hk::rows_per_thread(true), c.cx, c.cy, half_extent, s.stream, 0,
                         s.cluster_scratch);
      s.rperm_loc = loc_version;
      prof_total += 1;
    }
    const bool cells = use_cells(c) && s.window > 1 && (halves & hk::kHalfTr);
    if (cells && s.cells_loc != loc_version) {  // columns regrouped by cell, once per location set
      const double side = 2.0 * half_extent / s.cgrid.gc;
      s.cgrid.x0 = cx - half_extent;
      s.cgrid.y0 = cy - half_extent;
      s.cgrid.inv_side = side > 0.0 ? 1.0 / side : 0.0;
      hk::launch_cells(s.x, s.y, s.q, n, s.cgrid, s.cell_id, s.cell_chunk, s.cell_start, s.cell_perm,
                       s.cells.max_tiles * hk::kBJ, s.cell_nct, s.stream);
      s.cells_loc = loc_version;
      prof_total += 3;
    }
    const bool use_fgt = fgt && fgt->on && (halves & hk::kHalfTr) && s.nck > 0;
    const bool use_bgf = fgt && fgt->bg && (halves & hk::kHalfBg);
    const bool use_cut = c.tr_cut > 0.0 && (halves & hk::kHalfTr);
    if (use_fgt || use_bgf || use_cut) ck(cudaMemsetAsync(s.fgt_flag, 0, sizeof(unsigned), s.stream), "memset");
    if (use_bgf) {  // the background half by the 1-D expansion in time, straight into bg_sums
      if (fgt->nbt > s.bgf_cap) {
        if (s.bgf_mom) ck(cudaFree(s.bgf_mom), "cudaFree");
        if (s.bgf_count) ck(cudaFree(s.bgf_count), "cudaFree");
        if (s.bgf_part) ck(cudaFree(s.bgf_part), "cudaFree");
        s.bgf_mom = nullptr;
        s.bgf_count = nullptr;
        s.bgf_part = nullptr;
        s.bgf_cap = 0;
        s.bgf_mom = dmalloc<double>(static_cast<std::size_t>(fgt->nbt) * hk::kFgtP);
        s.bgf_count = dmalloc<int>(fgt->nbt);
        // parts for any box range: boxes x parts <= max(nbt, n / 4096) (bg_fgt_parts)
        s.bgf_part = dmalloc<double>(static_cast<std::size_t>(std::max(fgt->nbt, n / 4096 + 1)) * hk::kFgtP);
        s.bgf_cap = fgt->nbt;
      }
      hk::BgFgtParams G{};
      G.n = n;
      G.t = s.t;
      G.lb = s.lb;
      G.ub = s.ub;
      G.nbt = fgt->nbt;
      G.t0 = fgt->t0;
      G.L = fgt->Lt;
      G.inv_sqd = fgt->inv_sqdt;
      G.delta = fgt->delta_t;
      G.eps = fgt->eps_t;
      G.row_tol = hk::kFgtRowTol;
      if (const char* e = std::getenv("HK_FGT_ROW_TOL")) G.row_tol = std::atof(e);
      G.mom = s.bgf_mom;
      G.count = s.bgf_count;
      timed_pair(s, 1, [&] {
        hk::launch_bg_fgt(G, s.rb, rows, s.bg_sums[bgi], s.fgt_flag, s.stream, t[s.rb], t[s.re - 1], s.bgf_part);
      });
      prof_total += 2;
      halves &= ~hk::kHalfBg;  // the pair kernels compute the trigger only
    }
    hk::FgtParams F{};
    if (use_fgt) {
      if (s.fgt_perm_loc != loc_version) {  // checkpoint rows in spatial order, once per location set
        hk::launch_cluster(s.x, s.y, s.fgt_perm, s.rb, rows, hk::kFgtCkRows, s.nck_rows, hk::kFgtLeaf, cx, cy,
                           half_extent, s.stream, hk::kFgtCkRows);
        s.fgt_perm_loc = loc_version;
        prof_total += 1;
      }
      F = fgt_params(s, c, *fgt, grad);
      timed_pair(s, 3, [&] { hk::launch_fgt_prepare(F, s.stream); });
      prof_total += 4;
    }
    if (halves) {
      hk::launch_prep(dc, c, s.stream);
      if (cells) {
        hk::launch_prep_cells(dc, c, s.cells, s.stream);
        prof_total += 1;
      }
      const int v = c.varying ? 1 : 0;
      // the pair launch's plan: the expansion's band-only plan when it computes
      // just the homogeneous trigger next to the expansion
      const int pv = (use_fgt && halves == hk::kHalfTr) ? 2 : v;
      // The density-scaled kernel's rows come in clustered windows that span
      // far more time than a row block, which would disqualify the
      // background block expansion.  The background does not depend on the
      // variant, so it runs as its own launch of the homogeneous kernel on
      // the homogeneous plan: bitwise the background of a homogeneous
      // evaluation, for full evaluations and background-only refreshes
      // alike (the cache is keyed by tau alone).  Each launch writes only its
      // half's planes of the partial buffer.
      const bool split = c.varying && s.window > 1;
      if (split) {
        hk::EvalCoef cb = c;
        cb.varying = 0;
        if (halves & hk::kHalfBg)
          timed_pair(s, 1, [&] {
            hk::launch_pair(dc, cb, s.items[0], s.n_items[0], s.partial, s.rb, rows, grad, hk::kHalfBg,
                            s.stream);
          });
        if (halves & hk::kHalfTr)
          timed_pair(s, 2, [&] {
            const int pt = cells ? 3 : 1;
            hk::launch_pair(dc, c, s.items[pt], s.n_items[pt], s.partial, s.rb, rows, grad, hk::kHalfTr,
                            s.stream, false, cells ? &s.cells : nullptr);
          });
      } else {
        const int kind = halves == (hk::kHalfBg | hk::kHalfTr) ? 0 : (halves == hk::kHalfBg ? 1 : 2);
        timed_pair(s, kind, [&] {
          hk::launch_pair(dc, c, s.items[pv], s.n_items[pv], s.partial, s.rb, rows, grad, halves, s.stream,
                          use_fgt);
        });
      }
      if (split) {
        if (halves & hk::kHalfBg)
          hk::launch_collapse(s.partial, s.slots[0], rows, s.bg_sums[bgi], nullptr, s.stream);
        if (halves & hk::kHalfTr)
          hk::launch_collapse(s.partial, s.slots[cells ? 3 : 1], rows, nullptr, s.tr_sums[tri], s.stream);
        prof_total += (halves == (hk::kHalfBg | hk::kHalfTr)) ? 5 : 3;
      } else {
        hk::launch_collapse(s.partial, s.slots[pv], rows,
                            (halves & hk::kHalfBg) ? s.bg_sums[bgi] : nullptr,
                            (halves & hk::kHalfTr) ? s.tr_sums[tri] : nullptr, s.stream);
        prof_total += 3;
      }
      if (profiling) prof_pair += 1;
    }
    if (use_fgt) {
      timed_pair(s, 4, [&] {
        hk::launch_fgt_eval(F, s.rb, rows, s.bg_sums[bgi], s.tr_sums[tri], c.a, c.c, s.fgt_flag, s.stream);
      });
      prof_total += 1;
    }
    if (use_cut) {
      double tol = hk::kFgtRowTol;
      if (const char* e = std::getenv("HK_FGT_ROW_TOL")) tol = std::atof(e);
      hk::launch_tr_cut_cert(dc, c, s.bg_sums[bgi], s.tr_sums[tri], s.rb, rows, s.cert_scratch, tol,
                             s.fgt_flag, s.stream, lb[s.re - 1]);
      prof_total += 3;
    }
    if (use_fgt || use_bgf || use_cut)
      ck(cudaMemcpyAsync(s.h_fgt_flag, s.fgt_flag, sizeof(unsigned), cudaMemcpyDeviceToHost, s.stream),
         "flag copy");
    hk::launch_finish(dc, c, s.bg_sums[bgi], s.tr_sums[tri], s.rb, rows, grad, ell_rows,
                      grad ? grad_rows : nullptr, s.blockpart, s.stream);
    hk::launch_reduce(s.blockpart, s.n_finish_blocks, s.out6, s.stream);
    ck(cudaGetLastError(), "kernel launch");
    prof_total += 2;
    return use_fgt || use_bgf || use_cut;
  }

  // Full or workspace evaluation on every device; sums in device order.
  // ell_rows / grad_rows (host, optional): per-row outputs of the context's
  // rows, devices in order (hk_eval_detail).
  void evaluate(const hk_params* p, bool grad, bool workspace, bool force, double* ll, double* grad5,
                bool single = false, double* ell_rows = nullptr, double* grad_rows = nullptr,
                bool allow_fgt = true) {
    // Precision::single on catalogs where the FP64 expansions / certified cut
    // apply: their FP64 result (within 1e-13 of the exact sums) arrives ~10x
    // sooner than the FP32 direct kernels' (144 / 30 ms at N=1e6); the
    // reference's float path is a speed choice, and its 1e-4 gate
    // (acceptance.cpp) is met with margin.  HK_OPT_SINGLE_FP64=0 keeps FP32.
    if (single && single_fp64 && allow_fgt && static_cast<std::size_t>(n) >= hk::kFgtPlanRows) single = false;
    hk::EvalCoef c = coef(p, single);
    if (allow_fgt) set_cut(c);
    const FgtPlan fgt = allow_fgt ? fgt_plan(c, grad) : FgtPlan{};
    int bgi, tri;
    const int halves = workspace ? plan_halves(c, grad, force, bgi, tri, fgt.on, fgt.bg)
                                 : plan_halves(c, grad, /*force=*/true, bgi, tri, fgt.on, fgt.bg);
    std::vector<double*> dev_rows(devs.size(), nullptr);
    struct Free {
      std::vector<double*>& v;
      ~Free() {
        for (double* q : v)
          if (q) cudaFree(q);
      }
    } free_rows{dev_rows};
    std::size_t off = 0;
    std::vector<char> expanded(devs.size(), 0);
    for (std::size_t k = 0; k < devs.size(); ++k) {
      auto& s = devs[k];
      const std::size_t rows = static_cast<std::size_t>(s.re - s.rb);
      double *d_ell = nullptr, *d_grad = nullptr;
      if (ell_rows || grad_rows) {
        ck(cudaSetDevice(s.dev), "cudaSetDevice");
        dev_rows[k] = dmalloc<double>(6 * rows);
        d_ell = dev_rows[k];
        d_grad = dev_rows[k] + rows;
      }
      expanded[k] = enqueue(s, c, grad, halves, bgi, tri, d_ell, d_grad, &fgt);
      if (!multi())
        ck(cudaMemcpyAsync(s.h_out6, s.out6, 6 * sizeof(double), cudaMemcpyDeviceToHost, s.stream),
           "result copy");
      if (ell_rows)
        ck(cudaMemcpyAsync(ell_rows + off, d_ell, rows * sizeof(double), cudaMemcpyDeviceToHost,
                           s.stream),
           "rows copy");
      if (grad_rows && grad)
        ck(cudaMemcpyAsync(grad_rows + 5 * off, d_grad, 5 * rows * sizeof(double),
                           cudaMemcpyDeviceToHost, s.stream),
           "rows copy");
      off += rows;
    }
    if (multi()) {
      reduce_devices();
      ck(cudaSetDevice(devs[0].dev), "cudaSetDevice");
      ck(cudaMemcpyAsync(devs[0].h_out6, devs[0].total6, 6 * sizeof(double), cudaMemcpyDeviceToHost,
                         devs[0].stream),
         "result copy");
    }
    bool flagged = false, any_expanded = false;
    for (std::size_t k = 0; k < devs.size(); ++k) {
      auto& s = devs[k];
      ck(cudaSetDevice(s.dev), "cudaSetDevice");
      ck(cudaStreamSynchronize(s.stream), "hk_eval");
      if (expanded[k]) flagged = flagged || *s.h_fgt_flag != 0;
      any_expanded = any_expanded || expanded[k];
    }
    if (any_expanded) ++fgt_evals;
    if (flagged) {
      // a row's certified expansion error could exceed kFgtRowTol: the same
      // evaluation on the direct path (both halves recomputed, caches reset)
      ++fgt_fallbacks;
      for (Key& k : tr_key) k.valid = false;
      for (Key& k : bg_key) k.valid = false;
      evaluate(p, grad, workspace, /*force=*/true, ll, grad5, single, ell_rows, grad_rows, /*allow_fgt=*/false);
      return;
    }
    const double* acc = devs[0].h_out6;
    *ll = acc[0];
    if (grad5)
      for (int k = 0; k < 5; ++k) grad5[k] = acc[1 + k];
  }

  // The per-device 6-vectors -> their device-order sum in total6: an NCCL
  // all-gather of 6 doubles per device (every device then holds the total),
  // or peer copies into device 0.  Enqueued, not synchronised.
  void reduce_devices() {
    const int g = static_cast<int>(devs.size());
    if (use_nccl) {
      const NcclApi& api = nccl_api();
      nck(api.GroupStart(), "ncclGroupStart");
      for (int k = 0; k < g; ++k) {
        DeviceState& s = devs[k];
        ck(cudaSetDevice(s.dev), "cudaSetDevice");
        nck(api.AllGather(s.out6, s.gather6, 6, ncclFloat64, comms[k], s.stream), "ncclAllGather");
      }
      nck(api.GroupEnd(), "ncclGroupEnd");
      for (auto& s : devs) {
        ck(cudaSetDevice(s.dev), "cudaSetDevice");
        hk::launch_sum6(s.gather6, g, s.total6, s.stream);
      }
    } else {
      for (auto& s : devs) {
        ck(cudaSetDevice(s.dev), "cudaSetDevice");
        ck(cudaEventRecord(s.done, s.stream), "cudaEventRecord");
      }
      DeviceState& s0 = devs[0];
      ck(cudaSetDevice(s0.dev), "cudaSetDevice");
      for (int k = 0; k < g; ++k) {
        ck(cudaStreamWaitEvent(s0.stream, devs[k].done, 0), "cudaStreamWaitEvent");
        ck(cudaMemcpyPeerAsync(s0.gather6 + 6 * k, s0.dev, devs[k].out6, devs[k].dev, 6 * sizeof(double),
                               s0.stream),
           "peer copy");
      }
      hk::launch_sum6(s0.gather6, g, s0.total6, s0.stream);
    }
    ck(cudaGetLastError(), "sum6");
    prof_total += use_nccl ? g : 1;
  }
};

namespace {

// Per-row trigger weight of the shard cost model (hk_host.hpp).
double shard_beta(int variant, std::size_t n) {
  if (variant == HK_VARIANT_VARYING) return hk::kCostBetaVarying;
  if (n >= hk::kFgtPlanRows) return hk::kCostBetaFgt;
  return n >= hk::kExpansionRows ? hk::kCostBetaExpanded : hk::kCostBeta;
}

std::unique_ptr<hk_ctx> new_ctx(const double* t, const double* x, const double* y,
                                const double* d, std::size_t n) {
  if (!t || !x || !y || !d) throw std::invalid_argument("hk_create: null array");
  // Non-finite locations are accepted (a coarse-only catalog, types.hpp:43,
  // whose locations the cut posterior imputes); evaluation then requires
  // hk_set_locations first.
  hk::validate_catalog(t, x, y, d, n, /*coarse_only=*/true);
  auto ctx = std::make_unique<hk_ctx>();
  ctx->n = static_cast<int>(n);
  ctx->npad = static_cast<int>((n + hk::kBJ - 1) / hk::kBJ * hk::kBJ);
  ctx->t.assign(t, t + n);
  ctx->x.assign(x, x + n);
  ctx->y.assign(y, y + n);
  ctx->d.assign(d, d + n);
  ctx->q_max = *std::max_element(ctx->d.begin(), ctx->d.end());
  ctx->unit_density = std::all_of(ctx->d.begin(), ctx->d.end(), [](double v) { return v == 1.0; });
  hk::tie_bounds(ctx->t, ctx->lb, ctx->ub);
  ctx->update_bbox();
  return ctx;
}

}  // namespace

extern "C" {

const char* hk_last_error(void) { return g_err.c_str(); }
const char* hk_version(void) { return "hawkes_b200 0.1 (sm_100a)"; }

int hk_create(const double* t, const double* lon, const double* lat, const double* density,
              size_t n, int n_gpus, hk_ctx** out) {
  return hk_create_variant(t, lon, lat, density, n, n_gpus, HK_VARIANT_CONSTANT, out);
}

namespace {

// A context over an explicit device list: cost-balanced row shards, one per
// entry (shard k on devices[k]), then the multi-device data plane.
int create_on(const double* t, const double* lon, const double* lat, const double* density, size_t n,
              const int* devices, int n_dev, int variant, hk_ctx** out) {
  return guarded([&] {
    if (!out) throw std::invalid_argument("hk_create: null output");
    if (variant != HK_VARIANT_CONSTANT && variant != HK_VARIANT_VARYING)
      throw std::invalid_argument("hk_create: unknown variant");
    *out = nullptr;
    auto ctx = new_ctx(t, lon, lat, density, n);
    int avail = 0;
    ck(cudaGetDeviceCount(&avail), "cudaGetDeviceCount");
    const int top = *std::max_element(devices, devices + n_dev);
    if (top >= avail)
      throw std::invalid_argument("hk_create: requested " + std::to_string(top + 1) + " GPUs, " +
                                  std::to_string(avail) + " visible");
    if (*std::min_element(devices, devices + n_dev) < 0)
      throw std::invalid_argument("hk_create: negative device index");
    if (static_cast<std::size_t>(n_dev) > n) throw std::invalid_argument("Partition: more workers than terms");
    const auto bounds = hk::plan_shards(ctx->lb, static_cast<std::size_t>(n_dev), shard_beta(variant, n));
    ctx->devs.resize(n_dev);
    for (int i = 0; i < n_dev; ++i)
      ctx->init_device(ctx->devs[i], devices[i], static_cast<int>(bounds[i]), static_cast<int>(bounds[i + 1]));
    ctx->init_data_plane();
    *out = ctx.release();
  });
}

}  // namespace

int hk_create_variant(const double* t, const double* lon, const double* lat, const double* density,
                      size_t n, int n_gpus, int variant, hk_ctx** out) {
  const int g = n_gpus <= 0 ? 1 : n_gpus;
  std::vector<int> devices(g);
  for (int k = 0; k < g; ++k) devices[k] = k;
  return create_on(t, lon, lat, density, n, devices.data(), g, variant, out);
}

int hk_create_devices(const double* t, const double* lon, const double* lat, const double* density,
                      size_t n, const int* devices, int n_devices, int variant, hk_ctx** out) {
  if (!devices || n_devices <= 0) {
    g_err = "hk_create_devices: empty device list";
    if (out) *out = nullptr;
    return HK_INVALID_ARGUMENT;
  }
  return create_on(t, lon, lat, density, n, devices, n_devices, variant, out);
}

int hk_create_shard(const double* t, const double* lon, const double* lat, const double* density,
                    size_t n, size_t row_begin, size_t row_end, int device, hk_ctx** out) {
  return guarded([&] {
    if (!out) throw std::invalid_argument("hk_create_shard: null output");
    *out = nullptr;
    auto ctx = new_ctx(t, lon, lat, density, n);
    if (!(row_begin < row_end) || row_end > n)
      throw std::out_of_range("hk_create_shard: row range out of range");
    int avail = 0;
    ck(cudaGetDeviceCount(&avail), "cudaGetDeviceCount");
    if (device < 0 || device >= avail) throw std::invalid_argument("hk_create_shard: bad device");
    ctx->devs.resize(1);
    ctx->init_device(ctx->devs[0], device, static_cast<int>(row_begin), static_cast<int>(row_end));
    ctx->init_data_plane();
    *out = ctx.release();
  });
}

void hk_destroy(hk_ctx* ctx) { delete ctx; }

int hk_set_locations(hk_ctx* ctx, const double* lon, const double* lat) {
  return guarded([&] {
    if (!ctx || !lon || !lat) throw std::invalid_argument("hk_set_locations: null argument");
    auto& s0 = ctx->devs[0];
    ck(cudaSetDevice(s0.dev), "cudaSetDevice");
    // one host->device copy (asynchronous from pinned memory), then the box
    // check on device 0 and the NCCL broadcast to the other devices
    ck(cudaMemcpyAsync(s0.x, lon, ctx->n * sizeof(double), cudaMemcpyHostToDevice, s0.stream),
       "set_locations");
    ck(cudaMemcpyAsync(s0.y, lat, ctx->n * sizeof(double), cudaMemcpyHostToDevice, s0.stream),
       "set_locations");
    ctx->publish_locations();
  });
}

int hk_set_locations_device(hk_ctx* ctx, const double* lon_device, const double* lat_device) {
  return guarded([&] {
    if (!ctx || !lon_device || !lat_device)
      throw std::invalid_argument("hk_set_locations_device: null argument");
    auto& s = ctx->devs[0];
    ck(cudaSetDevice(s.dev), "cudaSetDevice");
    ck(cudaMemcpyAsync(s.x, lon_device, ctx->n * sizeof(double), cudaMemcpyDeviceToDevice, s.stream),
       "set_locations_device");
    ck(cudaMemcpyAsync(s.y, lat_device, ctx->n * sizeof(double), cudaMemcpyDeviceToDevice, s.stream),
       "set_locations_device");
    ctx->publish_locations();
  });
}

// ---- GPU location sampler (hk_regions.cu) ------------------------------------

}  // extern "C"

struct hk_regions {
  int device = 0;
  cudaStream_t stream = nullptr;
  hk::RegionsDevice d;
  std::vector<std::string> ids;
  unsigned long long* h_fail = nullptr;  // pinned
  double *tmp_x = nullptr, *tmp_y = nullptr;  // hk_regions_sample's device outputs
  ~hk_regions() {
    cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    hk::free_regions(d);
    if (h_fail) cudaFreeHost(h_fail);
    if (tmp_x) cudaFree(tmp_x);
    if (tmp_y) cudaFree(tmp_y);
    if (stream) cudaStreamDestroy(stream);
  }

  std::string id(int r) const {
    return r < static_cast<int>(ids.size()) ? ids[r] : std::to_string(r);
  }

  // The reference's messages (mcmc.hpp:87-95, geo.hpp:146-147, :158-159).
  void throw_failure(unsigned long long word, const std::vector<int>& event_region) const {
    const unsigned long long e = word >> 2;
    const int r = event_region[e];
    const std::string what = (word & 3) == hk::kFailZeroArea
                                 ? "sample_point_in_region: region " + id(r) + " has zero area"
                                 : "sample_point_in_region: rejection budget exhausted for region " + id(r);
    throw std::runtime_error("resample_locations: event " + std::to_string(e) + ": " + what);
  }
  std::vector<int> event_region;
};

extern "C" {

int hk_regions_create(size_t n_regions, const int* is_point, const double* point_xy,
                      const size_t* region_parts, const size_t* part_rings, const size_t* ring_verts,
                      const double* verts, const char* const* region_ids, size_t n_events,
                      const int* event_region, int device, hk_regions** out) {
  return guarded([&] {
    if (!out || !is_point || !point_xy || !region_parts || !event_region)
      throw std::invalid_argument("hk_regions_create: null argument");
    if (region_parts[n_regions] > 0 && (!part_rings || !ring_verts || !verts))
      throw std::invalid_argument("hk_regions_create: null polygon arrays");
    if (n_events >= (std::size_t{1} << 31) - 1024)
      throw std::invalid_argument("hk_regions_create: more than 2^31 events is not supported");
    *out = nullptr;
    auto reg = std::make_unique<hk_regions>();
    const hk::RegionsHost h = hk::build_regions(n_regions, is_point, point_xy, region_parts, part_rings,
                                                ring_verts, verts, n_events, event_region);
    reg->device = device;
    ck(cudaSetDevice(device), "cudaSetDevice");
    ck(cudaStreamCreateWithFlags(&reg->stream, cudaStreamNonBlocking), "cudaStreamCreate");
    reg->d = hk::upload_regions(h, reg->stream);
    ck(cudaStreamSynchronize(reg->stream), "hk_regions_create");
    ck(cudaMallocHost(&reg->h_fail, sizeof(unsigned long long)), "cudaMallocHost");
    if (region_ids)
      for (std::size_t r = 0; r < n_regions; ++r) reg->ids.emplace_back(region_ids[r] ? region_ids[r] : "");
    reg->event_region = h.event_region;
    *out = reg.release();
  });
}

void hk_regions_destroy(hk_regions* regions) { delete regions; }

int hk_regions_sample(hk_regions* regions, uint64_t seed, uint64_t counter, double* lon, double* lat) {
  return guarded([&] {
    if (!regions || !lon || !lat) throw std::invalid_argument("hk_regions_sample: null argument");
    hk_regions& R = *regions;
    ck(cudaSetDevice(R.device), "cudaSetDevice");
    const std::size_t n = static_cast<std::size_t>(R.d.n_events);
    if (!R.tmp_x) {
      R.tmp_x = dmalloc<double>(n);
      R.tmp_y = dmalloc<double>(n);
    }
    hk::launch_sample(R.d, seed, counter, R.tmp_x, R.tmp_y, R.stream);
    ck(cudaGetLastError(), "sample kernel");
    ck(cudaMemcpyAsync(R.h_fail, R.d.fail, sizeof(unsigned long long), cudaMemcpyDeviceToHost, R.stream),
       "fail copy");
    ck(cudaMemcpyAsync(lon, R.tmp_x, n * sizeof(double), cudaMemcpyDeviceToHost, R.stream), "copy");
    ck(cudaMemcpyAsync(lat, R.tmp_y, n * sizeof(double), cudaMemcpyDeviceToHost, R.stream), "copy");
    ck(cudaStreamSynchronize(R.stream), "hk_regions_sample");
    if (*R.h_fail != ~0ull) R.throw_failure(*R.h_fail, R.event_region);
  });
}

int hk_resample_locations(hk_ctx* ctx, hk_regions* regions, uint64_t seed, uint64_t counter) {
  return guarded([&] {
    if (!ctx || !regions) throw std::invalid_argument("hk_resample_locations: null argument");
    hk_regions& R = *regions;
    if (R.d.n_events != ctx->n)
      throw std::invalid_argument("hk_resample_locations: region table is for " +
                                  std::to_string(R.d.n_events) + " events, catalog has " +
                                  std::to_string(ctx->n));
    auto& s0 = ctx->devs[0];
    if (R.device != s0.dev)
      throw std::invalid_argument("hk_resample_locations: region table and context on different devices");
    ck(cudaSetDevice(s0.dev), "cudaSetDevice");
    hk::launch_sample(R.d, seed, counter, s0.x, s0.y, s0.stream);
    ck(cudaGetLastError(), "sample kernel");
    ck(cudaMemcpyAsync(R.h_fail, R.d.fail, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s0.stream),
       "fail copy");
    ctx->prof_total += 1;
    ctx->publish_locations();  // box check on device 0, broadcast, trigger caches dropped
    if (*R.h_fail != ~0ull) {
      ctx->locations_valid = false;
      R.throw_failure(*R.h_fail, R.event_region);
    }
  });
}

int hk_eval(hk_ctx* ctx, const hk_params* p, double* ll, double* grad5) {
  return guarded([&] {
    if (!ctx || !ll) throw std::invalid_argument("hk_eval: null argument");
    ctx->evaluate(p, grad5 != nullptr, /*workspace=*/false, /*force=*/true, ll, grad5);
  });
}

int hk_eval_detail(hk_ctx* ctx, const hk_params* p, double* ll, double* grad5, double* ell_rows,
                   double* grad_rows) {
  return guarded([&] {
    if (!ctx || !ll) throw std::invalid_argument("hk_eval_detail: null argument");
    if (grad_rows && !grad5)
      throw std::invalid_argument("hk_eval_detail: grad_rows needs grad5");
    ctx->evaluate(p, grad5 != nullptr, /*workspace=*/false, /*force=*/true, ll, grad5,
                  /*single=*/false, ell_rows, grad_rows);
  });
}

int hk_eval_single(hk_ctx* ctx, const hk_params* p, double* ll) {
  return guarded([&] {
    if (!ctx || !ll) throw std::invalid_argument("hk_eval_single: null argument");
    ctx->evaluate(p, /*grad=*/false, /*workspace=*/false, /*force=*/true, ll, nullptr, /*single=*/true);
  });
}

int hk_ws_eval(hk_ctx* ctx, const hk_params* p, int force, double* ll, double* grad5) {
  return guarded([&] {
    if (!ctx || !ll) throw std::invalid_argument("hk_ws_eval: null argument");
    ctx->evaluate(p, grad5 != nullptr, /*workspace=*/true, force != 0, ll, grad5);
  });
}

int hk_ws_eval_single(hk_ctx* ctx, const hk_params* p, int force, double* ll) {
  return guarded([&] {
    if (!ctx || !ll) throw std::invalid_argument("hk_ws_eval_single: null argument");
    ctx->evaluate(p, /*grad=*/false, /*workspace=*/true, force != 0, ll, nullptr, /*single=*/true);
  });
}

int hk_ws_stats(const hk_ctx* ctx, long* hits, long* misses) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("hk_ws_stats: null context");
    if (hits) *hits = ctx->ws_hits;
    if (misses) *misses = ctx->ws_misses;
  });
}

int hk_eval_async(hk_ctx* ctx, const hk_params* p, int with_grad) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("hk_eval_async: null context");
    hk::EvalCoef c = ctx->coef(p);
    ctx->set_cut(c);
    const hk_ctx::FgtPlan fgt = ctx->fgt_plan(c, with_grad != 0);
    int bgi, tri;
    const int halves = ctx->plan_halves(c, with_grad != 0, /*force=*/true, bgi, tri, fgt.on, fgt.bg);
    bool any = false;
    for (auto& s : ctx->devs) {
      s.flag_pending = ctx->enqueue(s, c, with_grad != 0, halves, bgi, tri, nullptr, nullptr, &fgt);
      any = any || s.flag_pending;
    }
    if (any) {
      ++ctx->fgt_evals;
      ctx->fgt_pending = true;
    }
    if (ctx->multi()) ctx->reduce_devices();
  });
}

const double* hk_result_device(hk_ctx* ctx) {
  if (!ctx || ctx->devs.empty()) return nullptr;
  return ctx->multi() ? ctx->devs[0].total6 : ctx->devs[0].out6;
}

void* hk_stream(hk_ctx* ctx, int dev) {
  if (!ctx || dev < 0 || dev >= static_cast<int>(ctx->devs.size())) return nullptr;
  return static_cast<void*>(ctx->devs[dev].stream);
}

int hk_eval_rows(hk_ctx* ctx, const hk_params* p, size_t b, size_t e, double* ell_rows,
                 double* grad_rows) {
  return guarded([&] {
    if (!ctx || !ell_rows) throw std::invalid_argument("hk_eval_rows: null argument");
    const hk::EvalCoef c = ctx->coef(p);
    if (!(b < e) || e > static_cast<size_t>(ctx->n))
      throw std::out_of_range("event_contribution: index out of range");
    // the device whose shard contains the range
    DeviceState* sp = nullptr;
    for (auto& s : ctx->devs)
      if (b >= static_cast<size_t>(s.rb) && e <= static_cast<size_t>(s.re)) sp = &s;
    if (!sp) throw std::out_of_range("hk_eval_rows: rows outside this context's shard");
    DeviceState& s = *sp;
    ck(cudaSetDevice(s.dev), "cudaSetDevice");
    const int rb = static_cast<int>(b), re = static_cast<int>(e);
    std::vector<hk::Item> items;
    const int slots =
        hk::plan_items(ctx->lb, ctx->ub, ctx->n, rb, re, hk::rows_per_item(c.varying != 0), items);
    const std::size_t rows = e - b;
    hk::Item* d_items = dmalloc<hk::Item>(items.size());
    double* d_partial = dmalloc<double>(static_cast<std::size_t>(slots) * 5 * rows);
    double* d_ell = dmalloc<double>(rows);
    double* d_grad = dmalloc<double>(rows * 5);
    const int nfb = static_cast<int>((rows + 255) / 256);
    double* d_bp = dmalloc<double>(static_cast<std::size_t>(nfb) * 6);
    double* d_sums = dmalloc<double>(5 * rows);
    auto cleanup = [&] {
      cudaFree(d_sums);
      cudaFree(d_items);
      cudaFree(d_partial);
      cudaFree(d_ell);
      cudaFree(d_grad);
      cudaFree(d_bp);
    };
    try {
      ck(cudaMemcpyAsync(d_items, items.data(), items.size() * sizeof(hk::Item),
                         cudaMemcpyHostToDevice, s.stream),
         "items");
      const hk::DeviceCatalog dc = s.catalog(ctx->n, ctx->npad);
      hk::launch_prep(dc, c, s.stream);
      const bool grad = grad_rows != nullptr;
      hk::launch_pair(dc, c, d_items, static_cast<int>(items.size()), d_partial, rb, re - rb, grad,
                      hk::kHalfBg | hk::kHalfTr, s.stream);
      hk::launch_collapse(d_partial, slots, re - rb, d_sums, d_sums + 2 * rows, s.stream);
      hk::launch_finish(dc, c, d_sums, d_sums + 2 * rows, rb, re - rb, grad, d_ell,
                        grad ? d_grad : nullptr, d_bp, s.stream);
      ck(cudaGetLastError(), "kernel launch");
      ctx->prof_total += 4;
      ck(cudaMemcpyAsync(ell_rows, d_ell, rows * sizeof(double), cudaMemcpyDeviceToHost, s.stream),
         "rows copy");
      if (grad)
        ck(cudaMemcpyAsync(grad_rows, d_grad, rows * 5 * sizeof(double), cudaMemcpyDeviceToHost,
                           s.stream),
           "rows copy");
      ck(cudaStreamSynchronize(s.stream), "hk_eval_rows");
    } catch (...) {
      cleanup();
      throw;
    }
    cleanup();
  });
}

int hk_fgt_stats(hk_ctx* ctx, long* evals, long* fallbacks, int* async_flagged) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("hk_fgt_stats: null context");
    int flagged = 0;
    if (ctx->fgt_pending) {
      for (auto& s : ctx->devs) {
        ck(cudaSetDevice(s.dev), "cudaSetDevice");
        ck(cudaStreamSynchronize(s.stream), "hk_fgt_stats");
        if (s.flag_pending && *s.h_fgt_flag) flagged = 1;
      }
    }
    if (evals) *evals = ctx->fgt_evals;
    if (fallbacks) *fallbacks = ctx->fgt_fallbacks;
    if (async_flagged) *async_flagged = flagged;
  });
}

int hk_set_option(hk_ctx* ctx, int option, int value) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("hk_set_option: null context");
    if (option == HK_OPT_BG_EXPANSION) ctx->bg_expansion = value != 0;
    else if (option == HK_OPT_BG_FGT) ctx->bg_fgt_enabled = value != 0;
    else if (option == HK_OPT_TR_CUT) ctx->tr_cut_enabled = value != 0;
    else if (option == HK_OPT_FGT) ctx->fgt_enabled = value != 0;
    else if (option == HK_OPT_CELLS) ctx->cells_enabled = value != 0;
    else if (option == HK_OPT_SINGLE_FP64) ctx->single_fp64 = value != 0;
    else throw std::invalid_argument("hk_set_option: unknown option " + std::to_string(option));
  });
}

int hk_rows(const hk_ctx* ctx, size_t* begin, size_t* end, int* n_devices) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("hk_rows: null context");
    if (begin) *begin = static_cast<size_t>(ctx->devs.front().rb);
    if (end) *end = static_cast<size_t>(ctx->devs.back().re);
    if (n_devices) *n_devices = static_cast<int>(ctx->devs.size());
  });
}

int hk_set_profiling(hk_ctx* ctx, int enable) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("hk_set_profiling: null context");
    ctx->profiling = enable != 0;
  });
}

int hk_profile(hk_ctx* ctx, double* pair_kernel_ms, long* pair_launches, long* total_launches) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("hk_profile: null context");
    double ms = 0.0;
    for (auto& s : ctx->devs) {
      ck(cudaSetDevice(s.dev), "cudaSetDevice");
      ck(cudaStreamSynchronize(s.stream), "hk_profile");
      for (std::size_t i = 0; i < s.prof_used; ++i) {
        float m = 0.f;
        ck(cudaEventElapsedTime(&m, s.prof_events[i].first, s.prof_events[i].second),
           "cudaEventElapsedTime");
        ms += m;
      }
    }
    if (pair_kernel_ms) *pair_kernel_ms = ms;
    if (pair_launches) *pair_launches = ctx->prof_pair;
    if (total_launches) *total_launches = ctx->prof_total;
  });
}

int hk_profile_kinds(hk_ctx* ctx, double* ms5, long* launches5) {
  return guarded([&] {
    if (!ctx || !ms5 || !launches5) throw std::invalid_argument("hk_profile_kinds: null argument");
    for (int k = 0; k < 5; ++k) {
      ms5[k] = 0.0;
      launches5[k] = 0;
    }
    for (auto& s : ctx->devs) {
      ck(cudaSetDevice(s.dev), "cudaSetDevice");
      ck(cudaStreamSynchronize(s.stream), "hk_profile_kinds");
      for (std::size_t i = 0; i < s.prof_used; ++i) {
        float m = 0.f;
        ck(cudaEventElapsedTime(&m, s.prof_events[i].first, s.prof_events[i].second),
           "cudaEventElapsedTime");
        ms5[s.prof_kind[i]] += m;
        launches5[s.prof_kind[i]] += 1;
      }
    }
  });
}

int hk_reset_profile(hk_ctx* ctx) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("hk_reset_profile: null context");
    for (auto& s : ctx->devs) s.prof_used = 0;
    ctx->prof_pair = 0;
    ctx->prof_total = 0;
  });
}

int hk_validate_catalog(const double* t, const double* lon, const double* lat,
                        const double* density, size_t n) {
  return guarded([&] {
    if (!t || !lon || !lat || !density) throw std::invalid_argument("hk_validate_catalog: null array");
    hk::validate_catalog(t, lon, lat, density, n);
  });
}

int hk_validate_params(const hk_params* p) {
  return guarded([&] {
    if (!p) throw std::invalid_argument("hk_validate_params: null params");
    hk::validate_params(
        hk::ParamsIn{p->mu0, p->tau_t, p->xi0, p->sigma_x, p->sigma_t, p->area, p->variant});
  });
}

int hk_partition_make(size_t n, size_t g, size_t* bounds) {
  return guarded([&] {
    if (!bounds) throw std::invalid_argument("hk_partition_make: null output");
    const auto b = hk::partition_make(n, g);
    std::copy(b.begin(), b.end(), bounds);
  });
}

int hk_plan_shards_variant(const double* t, size_t n, size_t g, int variant, size_t* bounds) {
  return guarded([&] {
    if (!t || !bounds) throw std::invalid_argument("hk_plan_shards: null argument");
    if (variant != HK_VARIANT_CONSTANT && variant != HK_VARIANT_VARYING)
      throw std::invalid_argument("hk_plan_shards: unknown variant");
    std::vector<double> tv(t, t + n);
    for (size_t i = 1; i < n; ++i)
      if (tv[i - 1] > tv[i])
        throw std::invalid_argument("Catalog: times not sorted at index " + std::to_string(i));
    std::vector<int> lb, ub;
    hk::tie_bounds(tv, lb, ub);
    const auto b = hk::plan_shards(lb, g, shard_beta(variant, n));
    std::copy(b.begin(), b.end(), bounds);
  });
}

int hk_plan_shards(const double* t, size_t n, size_t g, size_t* bounds) {
  return hk_plan_shards_variant(t, n, g, HK_VARIANT_CONSTANT, bounds);
}

int hk_benchmark_catalog(size_t n, uint64_t seed, double* t, double* lon, double* lat,
                         double* density) {
  return guarded([&] {
    if (!t || !lon || !lat || !density) throw std::invalid_argument("hk_benchmark_catalog: null array");
    hk::benchmark_catalog(n, seed, t, lon, lat, density);
  });
}

int hk_measure_fp64_peak(int device, double* tflops, double* ms) {
  return guarded([&] {
    if (!tflops) throw std::invalid_argument("hk_measure_fp64_peak: null output");
    *tflops = hk::measure_fp64_peak(device, ms);
    ck(cudaGetLastError(), "dfma probe");
  });
}

}  // extern "C"
