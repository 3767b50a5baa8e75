// Internal host-side structures of libreachplan_b200 (not part of the ABI).
#pragma once

#include "reachplan_b200.h"
#include "rp_device.cuh"

#include <algorithm>

#include <condition_variable>
#include <cstdint>
#include <cuda_runtime.h>
#include <exception>
#include <functional>
#include <initializer_list>
#include <map>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <thread>
#include <vector>

namespace rp {

using rpd::V3;

/// Thrown inside the library, converted to rp_status at the ABI.
struct Fail {
  rp_status code;
  std::string msg;
};

const char* errc_name(rp_status code);
[[noreturn]] void fail(rp_status code, const std::string& msg);
inline void require(bool ok, rp_status code, const std::string& msg) {
  if (!ok) fail(code, msg);
}
void cuda_check(cudaError_t e, const char* what);
void set_last_error(const std::string& s);

/// Every ABI entry point runs its body through this guard: nothing throws
/// across the C boundary.
template <typename F>
inline rp_status guarded(F&& f) {
  try {
    f();
    return RP_OK;
  } catch (const Fail& e) {
    set_last_error(e.msg);
    // a failed launch or API call leaves its (non-sticky) error pending on
    // this thread; clear it so the next call does not report it again
    if (e.code == RP_E_CUDA) (void)cudaGetLastError();
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("internal: host allocation failed");
    return RP_E_INTERNAL;
  } catch (const std::exception& e) {
    set_last_error(std::string("internal: ") + e.what());
    return RP_E_INTERNAL;
  }
}
#define RP_CUDA(x) ::rp::cuda_check((x), #x)

struct TimedLaunch {
  std::string name;
  cudaEvent_t start, stop;
};

}  // namespace rp

namespace rp {
/// Persistent host threads of a context (one per worker slot), started on
/// first use: run(n, f) executes f(k) on thread k for k < n and returns when
/// all are done. Spawning threads per planner call cost ~0.1 ms per window.
class HostWorkers {
 public:
  explicit HostWorkers(int device) : device_(device) {}
  ~HostWorkers();
  void run(int n, const std::function<void(int)>& f,
           const std::function<void()>& main_side = {});

 private:
  void grow(int n);
  int device_;
  std::vector<std::thread> threads_;
  std::mutex m_, call_;
  std::condition_variable cv_, done_;
  const std::function<void(int)>* job_ = nullptr;
  int n_ = 0, left_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};
}  // namespace rp

struct rp_ctx {
  int device = 0;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  bool timing = false;
  int64_t launches = 0;
  std::vector<rp::TimedLaunch> pending;
  std::vector<cudaEvent_t> event_pool;
  cudaEvent_t tl_base = nullptr;  // RP_TIMELINE: start of the first launch since reset_timing
  bool tl_armed = false;
  float tl_prev_end = 0.f;
  const rp_ctx* tl_parent = nullptr;  // worker contexts: the context they serve
  std::map<std::string, std::pair<double, int64_t>> kernel_ms;
  int sm_count = 148;
  // Small pinned staging buffer for scalar read-backs.
  void* pinned = nullptr;
  size_t pinned_bytes = 0;
  // Worker contexts (own streams, same device) for concurrent planner
  // attempts; created on first use, folded back by ctx_absorb.
  std::vector<rp_ctx*> workers;
  rp_ctx* parent = nullptr;  // worker contexts: the context they serve (same device)
  std::unique_ptr<rp::HostWorkers> pool;  // threads for the concurrent planner attempts
  // Worker contexts: a device flag that stops this worker's cooperative pass
  // (set and cleared by DMA copies), and the auxiliary stream those copies
  // use on the parent.
  int* cancel_flag = nullptr;
  cudaStream_t aux = nullptr;
  cudaEvent_t aux_ev = nullptr;  // "cancel flags cleared" on aux
  // solve_reach's temporaries (ctx_scratch): kept across solves, reused in
  // the context stream's order
  void* scratch[2] = {nullptr, nullptr};  // 0: solve_reach, 1: grid_clearance_field
  size_t scratch_bytes[2] = {0, 0};
  // Pinned upload ring (copy_to_device): kUploadSlots slots of
  // kUploadSlotBytes; a slot is reused only after the event recorded behind
  // its last copy completed, so uploads never synchronise the stream.
  char* upload_ring = nullptr;
  std::vector<cudaEvent_t> upload_ev;
  int upload_next = 0;
  int64_t upload_syncs = 0;  // uploads that still had to synchronise (too large)
  // released segment-2 cache buffers (rp_grid::Seg2Cache) for reuse by the
  // next grid: {quiver size, bits, ok}
  struct S2Buf {
    int q;
    uint32_t* bits;
    uint8_t* ok;
  };
  std::vector<S2Buf> s2_pool;
  // pinned read-back staging of copy_to_host (small reads)
  void* readback = nullptr;
};

namespace rp {
/// The k-th worker context of `parent` (created on first use).
rp_ctx* worker_ctx(rp_ctx* parent, int k);
/// True when objects of context `owner` may be used on context `user`: the
/// same context, or worker contexts of one parent (same device).
inline bool ctx_shares(const rp_ctx* user, const rp_ctx* owner) {
  const rp_ctx* a = user->parent ? user->parent : user;
  const rp_ctx* b = owner->parent ? owner->parent : owner;
  return a == b;
}
/// The context's persistent worker threads (created on first use).
rp::HostWorkers& host_workers(rp_ctx* ctx);
/// Fold a worker's launch count and kernel timings into its parent.
void ctx_absorb(rp_ctx* parent, rp_ctx* worker);
}  // namespace rp

struct rp_quiver {
  rp_ctx* ctx = nullptr;
  int n = 0;
  std::vector<double> host_xyz;  // AoS, reference order
  double* d_soa = nullptr;       // x[n], y[n], z[n]
  // ring addressing (Quiver fields, inc/reachplan/quiver.hpp:16-24); empty
  // for uploaded quivers
  std::vector<int> ring_offsets;
  std::vector<double> ring_elevations;
  double elev_step = 0.0, equator_azim_step = 0.0;
  int min_per_ring = 0;
  // device copies for direction culling (rp_rings.cuh): ring offsets
  // [n_rings + 1] and cos/sin of the ring elevations (host glibc); 0 rings
  // for uploaded quivers. d_qf = the directions as fp32 float4 (prefilters
  // only; every decision is re-taken on the fp64 SoA).
  int n_rings = 0;
  int* d_ring_off = nullptr;
  double* d_ring_c = nullptr;
  double* d_ring_s = nullptr;
  float4* d_qf = nullptr;
};

struct rp_grid {
  // every live grid is registered by a serial number, so a grid can refer to
  // another (ov_base_id) without a dangling pointer when that one is gone
  rp_grid();
  ~rp_grid();
  rp_grid(const rp_grid&) = delete;
  rp_grid& operator=(const rp_grid&) = delete;
  uint64_t id = 0;
  rp_ctx* ctx = nullptr;
  int dims[3] = {0, 0, 0};
  int wx = 0;  // 64-bit words per x row
  double origin[3] = {0, 0, 0};
  double voxel_size = 0.0;
  double dilation_radius = 0.0;
  uint64_t* bits = nullptr;
  size_t n_words = 0;
  bool empty = true;  // no occupancy since build: fused mark+dilate is exact
  // Coarse clearance field (grid_clearance_field): built lazily, cached
  // until the next modification (version) and never cached once the words
  // were exported for external writes (rp_grid_device_bits).
  uint64_t version = 0;
  bool exported = false;
  mutable uint64_t cf_version = ~0ull;
  mutable uint16_t* cf = nullptr;
  mutable cudaEvent_t cf_ready = nullptr;  // recorded after the field's build
  mutable int cf_bk = 0;
  mutable int cf_nc[3] = {0, 0, 0};
  // Segment-2 clearance cache (grid_seg2_cache): walk verdicts of
  // [root + L1 q_i, + L2 q_j] shared by the solves on this grid version.
  struct Seg2Cache {
    double key[5];  // root xyz, L1, L2
    int n;
    const rp_quiver* q;
    uint32_t* bits;  // [Q][ceil(Q/32)]: bit j of row i = clear
    uint8_t* ok;     // [Q][ceil(Q/1024)]: row chunk computed
  };
  mutable std::vector<Seg2Cache> s2;
  // Set by rp_grid_overlay: at version ov_version this grid is `ov_base` (at
  // ov_base_version) plus occupancy only inside the world box [ov_lo, ov_hi]
  // (the dynamic obstacle's dilated cells with a one-cell margin), so solves
  // on it can read the base's walk cache (grid_seg2_base_cache).
  uint64_t ov_base_id = 0;  // 0: not an overlay
  uint64_t ov_base_version = 0, ov_version = ~0ull;
  double ov_lo[3] = {0, 0, 0}, ov_hi[3] = {-1, -1, -1};
  // Segment-1 walk verdicts from the root (k_walk1_bits) for an arm (root,
  // L1, n) and quiver, shared by the planners on this grid version; `ready`
  // is recorded after the kernel on the computing stream (others wait on it).
  struct Walk1Cache {
    double key[4];
    int n = 0;
    const rp_quiver* q = nullptr;
    uint64_t version = ~0ull;
    uint32_t* bits = nullptr;
    size_t words = 0;
    cudaEvent_t ready = nullptr;
  };
  mutable Walk1Cache w1;
  mutable uint64_t s2_version = ~0ull;
  mutable std::unique_ptr<std::mutex> s2_mutex = std::make_unique<std::mutex>();

  rpd::GridView view() const {
    rpd::GridView v;
    v.bits = bits;
    v.nx = dims[0];
    v.ny = dims[1];
    v.nz = dims[2];
    v.wx = wx;
    v.ox = origin[0];
    v.oy = origin[1];
    v.oz = origin[2];
    v.vs = voxel_size;
    v.rvs = 1.0 / voxel_size;
    v.dq = (std::max(dims[0], std::max(dims[1], dims[2])) + 2.0) * 8.9e-16 + 1e-300;
    return v;
  }
};

namespace rp {

/// Device arm description used by every search kernel.
struct ArmDev {
  int nseg;
  int has_offsets;
  int any_limit;
  int lim_active[4];
  double L[4];
  double off[4];
  rpd::Limit lim[4];
  V3 root;
  double arm_radius;
  rpd::M3 base;
};

ArmDev make_arm_dev(const rp_arm& a);
void validate_arm(const rp_arm& a);            // ArmSpec::validate (src/arm_model.cpp:102-122)
void validate_reach(const rp_reach_params& r);  // ReachParams::validate (src/reach_solver.cpp:45-52)

/// Materialised pose on the host: PoseChain equivalent.
struct HostPose {
  int nseg = 0;
  bool has_elbows = false;
  V3 seg[4];
  V3 joints[5];
  V3 elbows[4];
  int qidx[4] = {-1, -1, -1, -1};
  bool no_qidx = false;  // quiver_indices empty in the reference PoseChain
  double s4dev = 0.0;
  std::vector<V3> waypoints;
};

void to_abi(const HostPose& p, rp_pose* out, double* wps, int cap);
HostPose from_abi(const rp_pose& p, const double* wps);

/// Shortcut record (ShortcutPath, inc/reachplan/reach_solver.hpp:60-74).
struct HostShortcut {
  int segment_index = 1;
  int hit = 0;
  int seg1 = -1, seg2 = -1;
  bool has_bridge = false;
  bool via_direct = false;
  V3 bridge{0, 0, 0};
  double path_length = 0.0;
  std::vector<V3> prefix;     // segment-1 samples (segment-2 hits)
  std::vector<V3> sublength;  // hit samples, or the direct origin->target samples
  HostPose basis;

  std::vector<V3> tip_waypoints(V3 target) const {
    std::vector<V3> w = prefix;
    w.insert(w.end(), sublength.begin(), sublength.end());
    if (has_bridge) w.push_back(target);
    return w;
  }
};

// Launch accounting: every kernel of the library goes through this.
void launch_begin(rp_ctx* ctx, const char* name, cudaEvent_t* ev);
void launch_end(rp_ctx* ctx, const char* name, cudaEvent_t ev);

template <typename K, typename... Args>
inline void launch(rp_ctx* ctx, const char* name, K kernel, dim3 grid, dim3 block, size_t smem,
                   Args... args) {
  cudaEvent_t ev = nullptr;
  launch_begin(ctx, name, &ev);
  kernel<<<grid, block, smem, ctx->stream>>>(args...);
  launch_end(ctx, name, ev);
}

/// launch() with programmatic dependent launch: the kernel may begin while
/// the previous kernel on the stream drains. The kernel must execute
/// griddepcontrol.wait before touching memory that kernel writes (or any
/// memory a preceding kernel produced); see k_mark_dilate_rowwise.
template <typename... KArgs, typename... Args>
inline void launch_pdl(rp_ctx* ctx, const char* name, void (*kernel)(KArgs...), dim3 grid,
                       dim3 block, size_t smem, Args... args) {
  cudaEvent_t ev = nullptr;
  launch_begin(ctx, name, &ev);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  RP_CUDA(cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...));
  launch_end(ctx, name, ev);
}

/// The context's scratch block of at least `bytes` (grown stream-ordered;
/// the contents are undefined). For temporaries of one call on the
/// context's stream: the next call's kernels run after this call's.
unsigned char* ctx_scratch(rp_ctx* ctx, size_t bytes, int slot = 0);

/// Lays typed arrays out in one block, 16-byte aligned: reserve() the
/// sizes, bind() the block, then at() the arrays.
struct ScratchCarver {
  unsigned char* base = nullptr;
  size_t off = 0;
  template <typename T>
  size_t reserve(size_t n) {
    off = (off + 15) & ~size_t{15};
    const size_t at = off;
    off += n * sizeof(T);
    return at;
  }
  void bind(unsigned char* b) { base = b; }
  template <typename T>
  T* at(size_t o) const { return reinterpret_cast<T*>(base + o); }
};

/// Stream-ordered device buffer.
template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  DevBuf() = default;
  DevBuf(size_t count, cudaStream_t stream) { alloc(count, stream); }
  void alloc(size_t count, cudaStream_t stream) {
    release();
    s = stream;
    n = count;
    if (count) RP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), stream));
  }
  void zero() {
    if (n) RP_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s));
  }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
  }
  ~DevBuf() { release(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; o.n = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    release();
    p = o.p; n = o.n; s = o.s;
    o.p = nullptr; o.n = 0;
    return *this;
  }
};

/// Host span tracing (RP_TRACE_HOST=<ms>): prints spans longer than the
/// threshold to stderr. Zero cost when the variable is unset.
struct HostSpan {
  const char* name;
  double t0;
  explicit HostSpan(const char* n);
  ~HostSpan();
};

void copy_to_host(rp_ctx* ctx, void* dst, const void* src, size_t bytes);  // syncs
/// Several device -> host reads behind one synchronisation.
struct HostRead {
  void* dst;
  const void* src;
  size_t bytes;
};
void copy_to_host_many(rp_ctx* ctx, std::initializer_list<HostRead> reads);
void copy_to_device(rp_ctx* ctx, void* dst, const void* src, size_t bytes);
/// copy_to_device of `bytes` written by `fill` straight into a pinned
/// upload slot (no host staging copy).
void copy_to_device_fill(rp_ctx* ctx, void* dst, size_t bytes,
                         const std::function<void(unsigned char*)>& fill);

// Derived reach parameters (src/reach_solver.cpp:28-43).
double nominal_spacing(const rp_arm& a, const rp_reach_params& r);
double resolved_epsilon(const rp_arm& a, const rp_reach_params& r);
double resolved_near_radius(const rp_arm& a, const rp_reach_params& r);

/// Lower bound on the distance from any point to the grid's occupied cells:
/// a squared distance d2[c] (in units of `side`^2) per coarse cell c of
/// bk^3 voxels, d2 = min over occupied blocks b of sum_i max(0, |c_i-b_i|-1)^2
/// (saturated at the transform's window). A point p in (or projected onto)
/// cell c is at least side*sqrt(d2[c]) from every occupied cell. d2 is null
/// for grids too elongated for the coarse lines (then nothing is skipped).
struct ClearanceField {
  const uint16_t* d2;
  int bk, ncx, ncy, ncz;
  double side, inv_side;
};
ClearanceField grid_clearance_field(const rp_grid* g, rp_ctx* caller = nullptr);

/// The grid's cache of segment-2 walk verdicts for an arm (root, L1, L2, n)
/// and quiver: bits[i * ceil(Q/32) + j/32] bit j%32 = walk clear, valid for
/// row i's chunk c (1024 directions) once ok[i * ceil(Q/1024) + c] != 0.
/// Walks depend on neither the target nor the rest of the arm
/// (src/reach_solver.cpp:368), so every solve on this grid version with the
/// same first two segments reuses them. False when not cacheable.
bool grid_seg2_cache(const rp_grid* g, const rp_quiver* q, const rp_arm& arm, int n,
                     uint32_t** bits, uint8_t** ok);
/// An overlay grid (rp_grid_overlay) whose base grid has the walk cache for
/// this arm and quiver: the base's verdicts, read-only, and the box holding
/// every cell the overlay added. A base verdict "blocked" holds on the
/// overlay too (cells are only added); a "clear" one holds unless the
/// segment's bounding box meets the box, in which case the solve walks it
/// again on the overlay grid (k_seg2_rows).
bool grid_seg2_base_cache(const rp_grid* g, const rp_quiver* q, const rp_arm& arm, int n,
                          const uint32_t** bits, const uint8_t** ok, V3* lo, V3* hi);

/// side * sqrt(d2) of the coarse cell holding p projected onto the grid box
/// (projection onto a convex set never increases distances to points in it),
/// shrunk by 1e-9 relative + 1e-9 m for the fp64 rounding of the cell index.
__device__ __forceinline__ double cf_distance(const ClearanceField& f, const rpd::GridView& g,
                                              V3 p) {
  if (!f.d2) return -1.0;  // no field: no sample is proven free
  int c[3];
  const double o[3] = {g.ox, g.oy, g.oz};
  const double pv[3] = {p.x, p.y, p.z};
  const int n[3] = {f.ncx, f.ncy, f.ncz};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double u = (pv[a] - o[a]) * f.inv_side;
    int k = u <= 0.0 ? 0 : (u >= n[a] ? n[a] - 1 : static_cast<int>(u));
    c[a] = k;
  }
  const unsigned d2 = __ldg(f.d2 + (static_cast<size_t>(c[2]) * f.ncy + c[1]) * f.ncx + c[0]);
  return f.side * sqrt(static_cast<double>(d2)) * (1.0 - 1e-9) - 1e-9;
}

// Grid entry points used across translation units.
rp_grid* grid_alloc_like(const rp_grid* g);
void grid_mark_dilate_boxes(rp_grid* g, const rp_obstacle* obs, int n, double radius,
                            bool or_into_existing);

}  // namespace rp
