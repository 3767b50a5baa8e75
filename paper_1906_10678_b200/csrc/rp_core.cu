// Context, errors, parameters, quiver and pose conversions of libreachplan_b200.
#include "rp_internal.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

namespace rp {

namespace {
thread_local std::string g_last_error;
constexpr double kPi = 3.14159265358979323846;
}  // namespace

const char* errc_name(rp_status code) {
  static const char* names[] = {"invalid-parameter", "capacity-exceeded", "degenerate-input",
                                "unreachable-target", "empty-cone", "no-solution", "no-path",
                                "infeasible-timing", "execution-collision", "timeout",
                                "parse-error"};
  if (code >= 1 && code <= 11) return names[code - 1];
  if (code == RP_E_CUDA) return "cuda-error";
  return "internal";
}

void fail(rp_status code, const std::string& msg) {
  throw Fail{code, std::string(errc_name(code)) + ": " + msg};
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(RP_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

void set_last_error(const std::string& s) { g_last_error = s; }

void launch_begin(rp_ctx* ctx, const char* name, cudaEvent_t* ev) {
  ++ctx->launches;
  if (!ctx->timing) return;
  cudaEvent_t e;
  if (!ctx->event_pool.empty()) {
    e = ctx->event_pool.back();
    ctx->event_pool.pop_back();
  } else {
    RP_CUDA(cudaEventCreate(&e));
  }
  RP_CUDA(cudaEventRecord(e, ctx->stream));
  *ev = e;
  if (!ctx->tl_armed) {  // the timeline's origin: this launch's start
    if (!ctx->tl_base) RP_CUDA(cudaEventCreate(&ctx->tl_base));
    RP_CUDA(cudaEventRecord(ctx->tl_base, ctx->stream));
    ctx->tl_armed = true;
  }
  (void)name;
}

void launch_end(rp_ctx* ctx, const char* name, cudaEvent_t ev) {
  RP_CUDA(cudaGetLastError());
  if (!ctx->timing || !ev) return;
  cudaEvent_t e;
  if (!ctx->event_pool.empty()) {
    e = ctx->event_pool.back();
    ctx->event_pool.pop_back();
  } else {
    RP_CUDA(cudaEventCreate(&e));
  }
  RP_CUDA(cudaEventRecord(e, ctx->stream));
  ctx->pending.push_back({name, ev, e});
}

static void drain_timing(rp_ctx* ctx) {
  if (ctx->pending.empty()) return;
  RP_CUDA(cudaStreamSynchronize(ctx->stream));
  // RP_TIMELINE=1: the device timeline of the timed launches (offsets from
  // the first launch, and the idle gap before each one)
  static const bool timeline = std::getenv("RP_TIMELINE") != nullptr;
  for (auto& t : ctx->pending) {
    float ms = 0.f;
    RP_CUDA(cudaEventElapsedTime(&ms, t.start, t.stop));
    if (timeline) {
      // offsets from the first launch since reset_timing (across drains),
      // and the idle gap since the previous launch ended on this stream
      float at = 0.f;
      const rp_ctx* o = ctx->tl_parent && ctx->tl_parent->tl_armed ? ctx->tl_parent : ctx;
      RP_CUDA(cudaEventElapsedTime(&at, o->tl_base, t.start));
      std::fprintf(stderr, "[tl] %9.3f ms +%8.3f gap %8.3f %s%s\n", at, ms, at - ctx->tl_prev_end,
                   t.name.c_str(), o != ctx ? " (worker)" : "");
      ctx->tl_prev_end = at + ms;
    }
    auto& acc = ctx->kernel_ms[t.name];
    acc.first += ms;
    acc.second += 1;
    ctx->event_pool.push_back(t.start);
    ctx->event_pool.push_back(t.stop);
  }
  ctx->pending.clear();
}

static double trace_threshold_ms() {
  static const double t = [] {
    const char* e = std::getenv("RP_TRACE_HOST");
    return e ? std::atof(e) : -1.0;
  }();
  return t;
}

static double now_ms() {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

HostSpan::HostSpan(const char* n) : name(n), t0(trace_threshold_ms() >= 0 ? now_ms() : 0.0) {}

HostSpan::~HostSpan() {
  // RP_CHECK_SPANS=1: report a CUDA error left pending inside the span
  // (debugging aid: names the host stage whose call went unchecked)
  static const bool check = std::getenv("RP_CHECK_SPANS") != nullptr;
  if (check) {
    const cudaError_t e = cudaPeekAtLastError();
    if (e != cudaSuccess) std::fprintf(stderr, "[span] %s: pending %s\n", name, cudaGetErrorString(e));
  }
  const double th = trace_threshold_ms();
  if (th < 0) return;
  const double dt = now_ms() - t0;
  if (dt >= th) std::fprintf(stderr, "[span] %-24s %9.3f ms\n", name, dt);
}

namespace {
constexpr size_t kReadbackBytes = 256 << 10;
}  // namespace

namespace {
constexpr int kGatherMax = 8;
constexpr size_t kGatherBytes = 4096;
struct GatherArgs {
  const unsigned char* src[kGatherMax];
  unsigned bytes[kGatherMax];
  unsigned off[kGatherMax];
  int n;
};
/// Small reads gathered by one kernel straight into the mapped pinned
/// read-back buffer (one launch instead of one DMA call per read).
__global__ void k_gather_to_host(GatherArgs a, unsigned char* __restrict__ dst) {
  for (int e = 0; e < a.n; ++e)
    for (unsigned k = threadIdx.x; k < a.bytes[e]; k += blockDim.x) dst[a.off[e] + k] = a.src[e][k];
}
/// Device -> mapped pinned host copy, 16 bytes per thread.
__global__ void k_copy_to_mapped(uint4* __restrict__ dst, const uint4* __restrict__ src, size_t n16) {
  const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n16) dst[i] = src[i];
}
}  // namespace

/// Device -> host copy that completes before returning. Reads up to 256 KiB
/// land in the context's pinned read-back buffer, written there by a copy
/// kernel through its mapping (a DMA call costs ~5-16 us of host time, a
/// launch ~4; RP_READBACK_DMA=1 restores the DMA).
void copy_to_host(rp_ctx* ctx, void* dst, const void* src, size_t bytes) {
  if (!bytes) return;
  if (bytes <= kReadbackBytes) {
    if (!ctx->readback) RP_CUDA(cudaMallocHost(&ctx->readback, kReadbackBytes));
    static const bool dma = std::getenv("RP_READBACK_DMA") != nullptr;
    const bool aligned = (reinterpret_cast<uintptr_t>(src) & 15) == 0 && (bytes & 15) == 0;
    if (!dma && aligned) {
      const size_t n16 = bytes / 16;
      launch(ctx, "readback", k_copy_to_mapped, dim3(static_cast<unsigned>((n16 + 255) / 256)),
             dim3(256), 0, static_cast<uint4*>(ctx->readback), static_cast<const uint4*>(src), n16);
    } else if (!dma && bytes <= kGatherBytes) {
      GatherArgs ga{};
      ga.src[0] = static_cast<const unsigned char*>(src);
      ga.bytes[0] = static_cast<unsigned>(bytes);
      ga.n = 1;
      launch(ctx, "readback", k_gather_to_host, dim3(1), dim3(256), 0, ga,
             static_cast<unsigned char*>(ctx->readback));
    } else {
      RP_CUDA(cudaMemcpyAsync(ctx->readback, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    }
    RP_CUDA(cudaStreamSynchronize(ctx->stream));
    std::memcpy(dst, ctx->readback, bytes);
    return;
  }
  RP_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  RP_CUDA(cudaStreamSynchronize(ctx->stream));
}

void copy_to_host_many(rp_ctx* ctx, std::initializer_list<HostRead> reads) {
  size_t total = 0;
  for (const HostRead& r : reads) total += (r.bytes + 15) & ~size_t{15};
  if (total > kReadbackBytes) {
    for (const HostRead& r : reads) copy_to_host(ctx, r.dst, r.src, r.bytes);
    return;
  }
  if (!ctx->readback) RP_CUDA(cudaMallocHost(&ctx->readback, kReadbackBytes));
  static const bool dma = std::getenv("RP_READBACK_DMA") != nullptr;
  if (!dma && reads.size() > 1 && reads.size() <= static_cast<size_t>(kGatherMax) &&
      total <= kGatherBytes) {
    GatherArgs ga{};
    size_t o = 0;
    for (const HostRead& r : reads) {
      ga.src[ga.n] = static_cast<const unsigned char*>(r.src);
      ga.bytes[ga.n] = static_cast<unsigned>(r.bytes);
      ga.off[ga.n] = static_cast<unsigned>(o);
      ++ga.n;
      o += (r.bytes + 15) & ~size_t{15};
    }
    launch(ctx, "readback", k_gather_to_host, dim3(1), dim3(256), 0, ga,
           static_cast<unsigned char*>(ctx->readback));
    RP_CUDA(cudaStreamSynchronize(ctx->stream));
    o = 0;
    for (const HostRead& r : reads) {
      if (r.bytes) std::memcpy(r.dst, static_cast<char*>(ctx->readback) + o, r.bytes);
      o += (r.bytes + 15) & ~size_t{15};
    }
    return;
  }
  size_t off = 0;
  for (const HostRead& r : reads) {
    if (r.bytes)
      RP_CUDA(cudaMemcpyAsync(static_cast<char*>(ctx->readback) + off, r.src, r.bytes,
                              cudaMemcpyDeviceToHost, ctx->stream));
    off += (r.bytes + 15) & ~size_t{15};
  }
  RP_CUDA(cudaStreamSynchronize(ctx->stream));
  off = 0;
  for (const HostRead& r : reads) {
    if (r.bytes) std::memcpy(r.dst, static_cast<char*>(ctx->readback) + off, r.bytes);
    off += (r.bytes + 15) & ~size_t{15};
  }
}

namespace {
constexpr int kUploadSlots = 64;
constexpr size_t kUploadSlotBytes = 64 << 10;
}  // namespace

/// Host -> device copy in stream order without synchronising the stream:
/// the source (often a temporary) is staged into the next slot of the
/// context's pinned ring and the DMA reads it from there. A pageable
/// cudaMemcpyAsync would synchronise the stream before it starts; only
/// uploads larger than a slot (a quiver or a uint8 grid, once) still do.
namespace {
/// Device copy out of a mapped pinned slot (UVA: the slot's host address is
/// valid on the device), 16 bytes per thread.
__global__ void k_copy_mapped(uint4* __restrict__ dst, const uint4* __restrict__ src, size_t n16) {
  const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n16) dst[i] = src[i];
}

/// Slot -> device in stream order. Larger uploads go through a copy kernel
/// reading the mapped slot: measured on B200 a 50 KB pinned cudaMemcpyAsync
/// costs ~16 us of host time, a kernel launch ~4.
void upload_from_slot(rp_ctx* ctx, void* dst, const void* slot, size_t bytes) {
  static const bool dma = std::getenv("RP_UPLOAD_DMA") != nullptr;
  const bool aligned = (reinterpret_cast<uintptr_t>(dst) & 15) == 0 && (bytes & 15) == 0;
  if (dma || !aligned || bytes < 4096) {
    RP_CUDA(cudaMemcpyAsync(dst, slot, bytes, cudaMemcpyHostToDevice, ctx->stream));
    return;
  }
  const size_t n16 = bytes / 16;
  launch(ctx, "upload", k_copy_mapped, dim3(static_cast<unsigned>((n16 + 255) / 256)), dim3(256), 0,
         static_cast<uint4*>(dst), static_cast<const uint4*>(slot), n16);
}
}  // namespace

void copy_to_device(rp_ctx* ctx, void* dst, const void* src, size_t bytes) {
  if (!bytes) return;
  if (bytes > kUploadSlotBytes) {
    ++ctx->upload_syncs;
    RP_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
    // The source may be a temporary host buffer: make the copy complete.
    RP_CUDA(cudaStreamSynchronize(ctx->stream));
    return;
  }
  if (!ctx->upload_ring) {
    RP_CUDA(cudaMallocHost(reinterpret_cast<void**>(&ctx->upload_ring),
                           kUploadSlots * kUploadSlotBytes));
    ctx->upload_ev.assign(kUploadSlots, nullptr);
    for (auto& e : ctx->upload_ev) RP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& e : ctx->upload_ev) RP_CUDA(cudaEventRecord(e, ctx->stream));
  }
  const int k = ctx->upload_next;
  ctx->upload_next = (k + 1) % kUploadSlots;
  // the slot's previous copy has long finished in practice (63 copies ago)
  RP_CUDA(cudaEventSynchronize(ctx->upload_ev[k]));
  char* slot = ctx->upload_ring + static_cast<size_t>(k) * kUploadSlotBytes;
  std::memcpy(slot, src, bytes);
  upload_from_slot(ctx, dst, slot, bytes);
  RP_CUDA(cudaEventRecord(ctx->upload_ev[k], ctx->stream));
}

unsigned char* ctx_scratch(rp_ctx* ctx, size_t bytes, int slot) {
  void*& p = ctx->scratch[slot];
  size_t& have = ctx->scratch_bytes[slot];
  if (bytes > have) {
    if (p) RP_CUDA(cudaFreeAsync(p, ctx->stream));
    const size_t want = std::max(bytes, have + have / 2);
    p = nullptr;
    have = 0;
    RP_CUDA(cudaMallocAsync(&p, want, ctx->stream));
    have = want;
  }
  return static_cast<unsigned char*>(p);
}

void copy_to_device_fill(rp_ctx* ctx, void* dst, size_t bytes,
                         const std::function<void(unsigned char*)>& fill) {
  if (!bytes) return;
  if (bytes > kUploadSlotBytes || !ctx->upload_ring) {
    std::vector<unsigned char> h(bytes);
    fill(h.data());
    copy_to_device(ctx, dst, h.data(), bytes);
    return;
  }
  // fill the pinned slot in place (no staging copy)
  const int k = ctx->upload_next;
  ctx->upload_next = (k + 1) % kUploadSlots;
  RP_CUDA(cudaEventSynchronize(ctx->upload_ev[k]));
  unsigned char* slot = reinterpret_cast<unsigned char*>(ctx->upload_ring) + static_cast<size_t>(k) * kUploadSlotBytes;
  fill(slot);
  upload_from_slot(ctx, dst, slot, bytes);
  RP_CUDA(cudaEventRecord(ctx->upload_ev[k], ctx->stream));
}

double nominal_spacing(const rp_arm& a, const rp_reach_params& r) {
  const int segs = (r.mode == RP_MODE_6DOF) ? 3 : a.n_segments;
  double sum = 0.0;
  for (int j = 0; j < std::min(segs, 3); ++j) sum += a.lengths[j];
  return sum / (3.0 * r.n_samples);
}

double resolved_epsilon(const rp_arm& a, const rp_reach_params& r) {
  if (r.epsilon_gap >= 0.0) return r.epsilon_gap;
  return 0.5 * a.lengths[2] / r.n_samples;
}

double resolved_near_radius(const rp_arm& a, const rp_reach_params& r) {
  if (r.near_target_radius >= 0.0) return r.near_target_radius;
  return 0.5 * nominal_spacing(a, r);
}

static double n3(const double* v) {
  const double xy = v[0] * v[0] + v[1] * v[1];
  return std::sqrt(xy + v[2] * v[2]);
}

void validate_arm(const rp_arm& a) {
  require(a.n_segments == 3 || a.n_segments == 4, RP_E_INVALID_PARAMETER,
          "arm must have 3 or 4 segments");
  for (int k = 0; k < a.n_segments; ++k)
    require(a.lengths[k] > 0.0, RP_E_INVALID_PARAMETER, "segment lengths must be > 0");
  require(a.arm_radius >= 0.0, RP_E_INVALID_PARAMETER, "arm_radius must be >= 0");
  require(a.n_limits >= 0 && a.n_limits <= 4 && a.n_offsets >= 0 && a.n_offsets <= 4,
          RP_E_INVALID_PARAMETER, "at most 4 joint limits / offsets");
  for (int k = 0; k < a.n_limits; ++k) {
    const auto& l = a.limits[k];
    require(l.elev_min >= -1e-12 && l.elev_max <= kPi + 1e-12 && l.elev_min <= l.elev_max,
            RP_E_INVALID_PARAMETER, "elevation limits must satisfy 0 <= min <= max <= pi");
    require(l.azim_min <= l.azim_max, RP_E_INVALID_PARAMETER,
            "azimuth limits must satisfy min <= max");
  }
  for (int k = 0; k < a.n_offsets; ++k)
    require(a.offsets[k] >= 0.0, RP_E_INVALID_PARAMETER, "joint offsets must be >= 0");
  require(std::abs(n3(a.base_axis) - 1.0) <= 1e-9, RP_E_INVALID_PARAMETER,
          "base_axis must be unit");
  require(std::abs(n3(a.fold_plane_normal) - 1.0) <= 1e-9, RP_E_INVALID_PARAMETER,
          "fold_plane_normal must be unit");
  const double d = (a.base_axis[0] * a.base_ref[0] + a.base_axis[1] * a.base_ref[1]) +
                   a.base_axis[2] * a.base_ref[2];
  require(std::abs(d) <= 1e-9 && std::abs(n3(a.base_ref) - 1.0) <= 1e-9, RP_E_INVALID_PARAMETER,
          "base_ref must be unit and orthogonal to base_axis");
}

void validate_reach(const rp_reach_params& r) {
  require(r.n_samples >= 1, RP_E_INVALID_PARAMETER, "n_samples must be >= 1");
  require(r.approach_half_angle >= 0.0 && r.approach_half_angle <= kPi, RP_E_INVALID_PARAMETER,
          "approach_half_angle must be in [0, pi]");
  require(std::abs(n3(r.approach_axis) - 1.0) <= 1e-9, RP_E_INVALID_PARAMETER,
          "approach_axis must be unit");
  require(r.workers >= 1, RP_E_INVALID_PARAMETER, "workers must be >= 1");
}

extern "C" rp_status rp_reach_params_validate(const rp_reach_params* rp) {
  return guarded([&] { validate_reach(*rp); });
}

ArmDev make_arm_dev(const rp_arm& a) {
  ArmDev d{};
  d.nseg = a.n_segments;
  for (int k = 0; k < 4; ++k) {
    d.L[k] = k < a.n_segments ? a.lengths[k] : 0.0;
    d.off[k] = k < a.n_offsets ? a.offsets[k] : 0.0;
    if (d.off[k] != 0.0) d.has_offsets = 1;
    if (k < a.n_limits) {
      d.lim[k] = {a.limits[k].elev_min, a.limits[k].elev_max, a.limits[k].azim_min,
                  a.limits[k].azim_max};
    } else {
      d.lim[k] = {0.0, kPi, -kPi, kPi};
    }
    d.lim_active[k] = rpd::limit_active(d.lim[k]) ? 1 : 0;
    if (d.lim_active[k]) d.any_limit = 1;
  }
  d.root = V3{a.root[0], a.root[1], a.root[2]};
  d.arm_radius = a.arm_radius;
  // base_frame (src/arm_model.cpp:94-100): columns ref, axis x ref, axis.
  const V3 axis{a.base_axis[0], a.base_axis[1], a.base_axis[2]};
  const V3 ref{a.base_ref[0], a.base_ref[1], a.base_ref[2]};
  const V3 c1 = rpd::cross(axis, ref);
  const V3 cols[3] = {ref, c1, axis};
  for (int c = 0; c < 3; ++c) {
    d.base.a[0][c] = cols[c].x;
    d.base.a[1][c] = cols[c].y;
    d.base.a[2][c] = cols[c].z;
  }
  return d;
}

void to_abi(const HostPose& p, rp_pose* out, double* wps, int cap) {
  std::memset(out, 0, sizeof(*out));
  out->n_segments = p.nseg;
  out->has_elbows = p.has_elbows ? 1 : 0;
  out->no_indices = p.no_qidx ? 1 : 0;
  for (int k = 0; k < 4; ++k) out->quiver_indices[k] = k < p.nseg ? p.qidx[k] : -1;
  out->s4_length_dev = p.s4dev;
  for (int k = 0; k < p.nseg; ++k) {
    out->segments[k][0] = p.seg[k].x;
    out->segments[k][1] = p.seg[k].y;
    out->segments[k][2] = p.seg[k].z;
    if (p.has_elbows) {
      out->elbows[k][0] = p.elbows[k].x;
      out->elbows[k][1] = p.elbows[k].y;
      out->elbows[k][2] = p.elbows[k].z;
    }
  }
  for (int k = 0; k <= p.nseg; ++k) {
    out->joints[k][0] = p.joints[k].x;
    out->joints[k][1] = p.joints[k].y;
    out->joints[k][2] = p.joints[k].z;
  }
  out->n_waypoints = static_cast<int>(p.waypoints.size());
  if (wps)
    for (int k = 0; k < out->n_waypoints && k < cap; ++k) {
      wps[3 * k] = p.waypoints[k].x;
      wps[3 * k + 1] = p.waypoints[k].y;
      wps[3 * k + 2] = p.waypoints[k].z;
    }
}

HostPose from_abi(const rp_pose& p, const double* wps) {
  HostPose h;
  h.nseg = p.n_segments;
  h.has_elbows = p.has_elbows != 0;
  h.no_qidx = p.no_indices != 0;
  for (int k = 0; k < p.n_segments; ++k) {
    h.seg[k] = V3{p.segments[k][0], p.segments[k][1], p.segments[k][2]};
    h.elbows[k] = V3{p.elbows[k][0], p.elbows[k][1], p.elbows[k][2]};
    h.qidx[k] = p.quiver_indices[k];
  }
  for (int k = 0; k <= p.n_segments; ++k)
    h.joints[k] = V3{p.joints[k][0], p.joints[k][1], p.joints[k][2]};
  h.s4dev = p.s4_length_dev;
  if (wps)
    for (int k = 0; k < p.n_waypoints; ++k)
      h.waypoints.push_back(V3{wps[3 * k], wps[3 * k + 1], wps[3 * k + 2]});
  return h;
}

}  // namespace rp

using namespace rp;

namespace rp {

HostWorkers::~HostWorkers() {
  {
    std::lock_guard<std::mutex> lk(m_);
    stop_ = true;
  }
  cv_.notify_all();
  for (auto& t : threads_) t.join();
}

void HostWorkers::grow(int n) {
  while (static_cast<int>(threads_.size()) < n) {
    const int k = static_cast<int>(threads_.size());
    const uint64_t g0 = gen_;  // before run() publishes the job: the new thread takes it
    threads_.emplace_back([this, k, g0] {
      cudaSetDevice(device_);
      std::unique_lock<std::mutex> lk(m_);
      uint64_t seen = g0;
      for (;;) {
        cv_.wait(lk, [&] { return stop_ || (gen_ != seen && k < n_); });
        if (stop_) return;
        seen = gen_;
        const auto* f = job_;
        lk.unlock();
        try {
          (*f)(k);  // callers capture their own exceptions; this only keeps the thread alive
        } catch (...) {
        }
        lk.lock();
        if (--left_ == 0) done_.notify_all();
      }
    });
  }
}

void HostWorkers::run(int n, const std::function<void(int)>& f,
                      const std::function<void()>& main_side) {
  std::lock_guard<std::mutex> one(call_);  // one window at a time per context
  std::unique_lock<std::mutex> lk(m_);
  if (n > 0) {
    grow(n);
    job_ = &f;
    n_ = n;
    left_ = n;
    ++gen_;
    cv_.notify_all();
  }
  if (main_side) {  // on the calling thread, while the workers run
    lk.unlock();
    main_side();  // must not throw (callers capture their exceptions)
    lk.lock();
  }
  done_.wait(lk, [&] { return left_ == 0; });
  job_ = nullptr;
  n_ = 0;
}

HostWorkers& host_workers(rp_ctx* ctx) {
  if (!ctx->pool) ctx->pool = std::make_unique<HostWorkers>(ctx->device);
  return *ctx->pool;
}

rp_ctx* worker_ctx(rp_ctx* parent, int k) {
  while (static_cast<int>(parent->workers.size()) <= k) {
    auto* c = new rp_ctx();
    c->device = parent->device;
    RP_CUDA(cudaSetDevice(parent->device));
    RP_CUDA(cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking));
    c->stream = c->own;
    c->sm_count = parent->sm_count;
    c->parent = parent;
    RP_CUDA(cudaMalloc(reinterpret_cast<void**>(&c->cancel_flag), sizeof(int)));
    RP_CUDA(cudaMemset(c->cancel_flag, 0, sizeof(int)));
    parent->workers.push_back(c);
  }
  rp_ctx* w = parent->workers[k];
  w->timing = parent->timing;
  w->tl_parent = parent;  // RP_TIMELINE offsets from the parent's origin
  return w;
}

void ctx_absorb(rp_ctx* parent, rp_ctx* w) {
  drain_timing(w);
  for (const auto& kv : w->kernel_ms) {
    auto& acc = parent->kernel_ms[kv.first];
    acc.first += kv.second.first;
    acc.second += kv.second.second;
  }
  w->kernel_ms.clear();
  parent->launches += w->launches;
  w->launches = 0;
}

}  // namespace rp

extern "C" {

int32_t rp_abi_version(void) { return RP_ABI_VERSION; }
const char* rp_last_error(void) { return g_last_error.c_str(); }

rp_status rp_ctx_create(int32_t device, rp_ctx** out) {
  return guarded([&] {
    require(out != nullptr, RP_E_INVALID_PARAMETER, "null output");
    int count = 0;
    RP_CUDA(cudaGetDeviceCount(&count));
    require(count > 0, RP_E_CUDA, "no CUDA device (the library has no CPU fallback)");
    require(device >= 0 && device < count, RP_E_INVALID_PARAMETER, "device index out of range");
    RP_CUDA(cudaSetDevice(device));
    auto* c = new rp_ctx();
    c->device = device;
    RP_CUDA(cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking));
    c->stream = c->own;
    cudaDeviceProp prop;
    RP_CUDA(cudaGetDeviceProperties(&prop, device));
    c->sm_count = prop.multiProcessorCount;
    // Keep freed stream-ordered allocations cached in the pool: solves and
    // plans allocate their scratch per call.
    cudaMemPool_t pool;
    RP_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t keep = UINT64_MAX;
    RP_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    *out = c;
  });
}

rp_status rp_ctx_destroy(rp_ctx* ctx) {
  return guarded([&] {
    if (!ctx) return;
    ctx->pool.reset();  // joins the worker threads
    for (rp_ctx* w : ctx->workers) rp_ctx_destroy(w);
    cudaStreamSynchronize(ctx->stream);
    for (auto& t : ctx->pending) {
      cudaEventDestroy(t.start);
      cudaEventDestroy(t.stop);
    }
    for (auto e : ctx->event_pool) cudaEventDestroy(e);
    if (ctx->tl_base) cudaEventDestroy(ctx->tl_base);
    if (ctx->pinned) cudaFreeHost(ctx->pinned);
    if (ctx->readback) cudaFreeHost(ctx->readback);
    for (cudaEvent_t e : ctx->upload_ev) cudaEventDestroy(e);
    for (auto& b : ctx->s2_pool) {
      cudaFree(b.bits);
      cudaFree(b.ok);
    }
    if (ctx->upload_ring) cudaFreeHost(ctx->upload_ring);
    if (ctx->cancel_flag) cudaFree(ctx->cancel_flag);
    if (ctx->aux) cudaStreamDestroy(ctx->aux);
    if (ctx->aux_ev) cudaEventDestroy(ctx->aux_ev);
    for (void* p : ctx->scratch)
      if (p) cudaFree(p);
    if (ctx->own) cudaStreamDestroy(ctx->own);
    delete ctx;
  });
}

rp_status rp_ctx_set_stream(rp_ctx* ctx, void* stream) {
  return guarded([&] {
    require(ctx != nullptr, RP_E_INVALID_PARAMETER, "null ctx");
    drain_timing(ctx);
    cudaStream_t next = stream ? static_cast<cudaStream_t>(stream) : ctx->own;
    // the context's scratch blocks and upload slots are reused in stream
    // order: let the old stream's work on them finish first
    if (ctx->stream && ctx->stream != next) RP_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->stream = next;
  });
}

void* rp_ctx_stream(rp_ctx* ctx) { return ctx ? ctx->stream : nullptr; }

rp_status rp_ctx_synchronize(rp_ctx* ctx) {
  return guarded([&] { RP_CUDA(cudaStreamSynchronize(ctx->stream)); });
}

rp_status rp_ctx_enable_timing(rp_ctx* ctx, int32_t enable) {
  return guarded([&] {
    drain_timing(ctx);
    ctx->timing = enable != 0;
  });
}

rp_status rp_ctx_kernel_time(rp_ctx* ctx, const char* name, double* total_ms, int64_t* launches) {
  return guarded([&] {
    drain_timing(ctx);
    auto it = ctx->kernel_ms.find(name);
    *total_ms = it == ctx->kernel_ms.end() ? 0.0 : it->second.first;
    *launches = it == ctx->kernel_ms.end() ? 0 : it->second.second;
  });
}

rp_status rp_ctx_reset_timing(rp_ctx* ctx) {
  return guarded([&] {
    drain_timing(ctx);
    ctx->kernel_ms.clear();
    ctx->tl_armed = false;
    ctx->tl_prev_end = 0.f;
  });
}

int64_t rp_ctx_launch_count(rp_ctx* ctx) { return ctx ? ctx->launches : 0; }

void rp_arm_init(rp_arm* a, int32_t n_segments, const double* lengths) {
  std::memset(a, 0, sizeof(*a));
  a->n_segments = n_segments;
  for (int k = 0; k < n_segments && k < 4; ++k) a->lengths[k] = lengths ? lengths[k] : 0.0;
  a->fold_plane_normal[1] = 1.0;
  a->fold_flex = 170.0 * (kPi / 180.0);
  a->base_axis[2] = 1.0;
  a->base_ref[0] = 1.0;
}

void rp_reach_params_init(rp_reach_params* r) {
  std::memset(r, 0, sizeof(*r));
  r->epsilon_gap = -1.0;
  r->n_samples = 8;
  r->approach_axis[0] = 1.0;
  r->near_target_radius = -1.0;
  r->mode = RP_MODE_8DOF;
  r->workers = 1;
}

void rp_path_params_init(rp_path_params* p) {
  std::memset(p, 0, sizeof(*p));
  p->epsilon_waypoint = p->d_w = p->slack = p->joint1_max_move = p->joint2_max_move = -1.0;
  p->n_relax = 3;
  p->relax_schedule[0] = 1.5;
  p->relax_schedule[1] = 2.0;
  p->relax_schedule[2] = 3.0;
  p->unfold_steps = 16;
}

double rp_nominal_spacing(const rp_arm* a, const rp_reach_params* r) {
  return nominal_spacing(*a, *r);
}
double rp_resolved_epsilon(const rp_arm* a, const rp_reach_params* r) {
  return resolved_epsilon(*a, *r);
}
double rp_resolved_near_radius(const rp_arm* a, const rp_reach_params* r) {
  return resolved_near_radius(*a, *r);
}
double rp_effective_dilation(const rp_arm* a, const rp_reach_params* r, double configured) {
  if (configured >= 0.0) return configured;
  double m = 0.0;
  for (int j = 0; j < a->n_segments; ++j) m = std::max(m, a->lengths[j] / r->n_samples);
  return a->arm_radius + 1.25 * m;
}

// ---- quiver (src/quiver.cpp:16-51): generated with the reference formula on
// the host (glibc cos/sin, so the vectors are bit-identical), then uploaded
// once as structure-of-arrays for coalesced device reads.
static rp_quiver* upload_quiver(rp_ctx* ctx, const std::vector<double>& xyz) {
  auto* q = new rp_quiver();
  q->ctx = ctx;
  q->n = static_cast<int>(xyz.size() / 3);
  q->host_xyz = xyz;
  std::vector<double> soa(3 * static_cast<size_t>(q->n));
  for (int k = 0; k < q->n; ++k) {
    soa[k] = xyz[3 * k];
    soa[q->n + k] = xyz[3 * k + 1];
    soa[2 * q->n + k] = xyz[3 * k + 2];
  }
  RP_CUDA(cudaMalloc(&q->d_soa, soa.size() * sizeof(double) + 8));
  copy_to_device(ctx, q->d_soa, soa.data(), soa.size() * sizeof(double));
  std::vector<float4> qf(q->n);
  for (int k = 0; k < q->n; ++k)
    qf[k] = make_float4(static_cast<float>(xyz[3 * k]), static_cast<float>(xyz[3 * k + 1]),
                        static_cast<float>(xyz[3 * k + 2]), 0.0f);
  RP_CUDA(cudaMalloc(&q->d_qf, std::max<size_t>(1, qf.size()) * sizeof(float4)));
  copy_to_device(ctx, q->d_qf, qf.data(), qf.size() * sizeof(float4));
  return q;
}

static void upload_rings(rp_ctx* ctx, rp_quiver* q) {
  const int nr = static_cast<int>(q->ring_offsets.size());
  std::vector<int> off(q->ring_offsets);
  off.push_back(q->n);
  std::vector<double> c(nr), s(nr);
  for (int r = 0; r < nr; ++r) {
    c[r] = std::cos(q->ring_elevations[r]);
    s[r] = std::sin(q->ring_elevations[r]);
  }
  RP_CUDA(cudaMalloc(&q->d_ring_off, off.size() * sizeof(int)));
  RP_CUDA(cudaMalloc(&q->d_ring_c, std::max(1, nr) * sizeof(double)));
  RP_CUDA(cudaMalloc(&q->d_ring_s, std::max(1, nr) * sizeof(double)));
  copy_to_device(ctx, q->d_ring_off, off.data(), off.size() * sizeof(int));
  copy_to_device(ctx, q->d_ring_c, c.data(), nr * sizeof(double));
  copy_to_device(ctx, q->d_ring_s, s.data(), nr * sizeof(double));
  q->n_rings = nr;
}

rp_status rp_quiver_generate(rp_ctx* ctx, double elev_step, double azim_step,
                             int32_t min_per_ring, rp_quiver** out) {
  return guarded([&] {
    require(elev_step > 0.0 && elev_step <= kPi / 2.0, RP_E_INVALID_PARAMETER,
            "elev_step must be in (0, pi/2]");
    require(azim_step > 0.0 && azim_step <= kPi / 2.0, RP_E_INVALID_PARAMETER,
            "equator_azim_step must be in (0, pi/2]");
    require(min_per_ring >= 1, RP_E_INVALID_PARAMETER, "min_per_ring must be >= 1");
    std::vector<double> rings;
    for (int k = 0;; ++k) {
      const double phi = -kPi / 2.0 + k * elev_step;
      if (phi >= kPi / 2.0 - 1e-12) {
        rings.push_back(kPi / 2.0);
        break;
      }
      rings.push_back(phi);
    }
    const long n_eq = std::llround(2.0 * kPi / azim_step);
    std::vector<double> xyz;
    std::vector<int> offsets;
    for (double phi : rings) {
      const long by_circ = std::llround(static_cast<double>(n_eq) * std::cos(phi));
      const int count = static_cast<int>(std::max<long>(min_per_ring, by_circ));
      offsets.push_back(static_cast<int>(xyz.size() / 3));
      const double cp = std::cos(phi), sp = std::sin(phi);
      for (int m = 0; m < count; ++m) {
        const double theta = 2.0 * kPi * m / count;
        xyz.push_back(cp * std::cos(theta));
        xyz.push_back(cp * std::sin(theta));
        xyz.push_back(sp);
      }
    }
    rp_quiver* q = upload_quiver(ctx, xyz);
    q->ring_offsets = std::move(offsets);
    q->ring_elevations = std::move(rings);
    q->elev_step = elev_step;
    q->equator_azim_step = azim_step;
    q->min_per_ring = min_per_ring;
    upload_rings(ctx, q);
    *out = q;
  });
}

rp_status rp_quiver_rings(const rp_quiver* q, int32_t* ring_offsets, double* ring_elevations,
                          int32_t cap, int32_t* n_rings, double* elev_step,
                          double* equator_azim_step, int32_t* min_per_ring) {
  return guarded([&] {
    const int n = static_cast<int>(q->ring_offsets.size());
    require(cap >= n || !ring_offsets, RP_E_CAPACITY_EXCEEDED, "ring buffer too small");
    *n_rings = n;
    for (int k = 0; ring_offsets && k < n; ++k) {
      ring_offsets[k] = q->ring_offsets[k];
      if (ring_elevations) ring_elevations[k] = q->ring_elevations[k];
    }
    if (elev_step) *elev_step = q->elev_step;
    if (equator_azim_step) *equator_azim_step = q->equator_azim_step;
    if (min_per_ring) *min_per_ring = q->min_per_ring;
  });
}

rp_status rp_quiver_upload(rp_ctx* ctx, const double* xyz, int32_t n, rp_quiver** out) {
  return guarded([&] {
    require(n > 0 && xyz != nullptr, RP_E_INVALID_PARAMETER, "empty quiver");
    *out = upload_quiver(ctx, std::vector<double>(xyz, xyz + 3 * static_cast<size_t>(n)));
  });
}

int32_t rp_quiver_size(const rp_quiver* q) { return q ? q->n : 0; }

rp_status rp_quiver_download(const rp_quiver* q, double* xyz, int32_t cap) {
  return guarded([&] {
    require(cap >= q->n, RP_E_INVALID_PARAMETER, "buffer too small");
    std::memcpy(xyz, q->host_xyz.data(), q->host_xyz.size() * sizeof(double));
  });
}

rp_status rp_quiver_destroy(rp_quiver* q) {
  return guarded([&] {
    if (!q) return;
    if (q->d_soa) cudaFree(q->d_soa);
    if (q->d_qf) cudaFree(q->d_qf);
    if (q->d_ring_off) cudaFree(q->d_ring_off);
    if (q->d_ring_c) cudaFree(q->d_ring_c);
    if (q->d_ring_s) cudaFree(q->d_ring_s);
    delete q;
  });
}

}  // extern "C"
