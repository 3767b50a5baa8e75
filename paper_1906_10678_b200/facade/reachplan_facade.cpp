// reachplan façade: the reference's C++ API for the hot path, implemented
// over the reachplan-b200 C ABI (include/reachplan_b200.h).
//
// A caller of the reference keeps its own headers (inc/reachplan/*.hpp) and
// its Eigen, and links this translation unit plus libreachplan_b200.so in
// place of the reference's src/{voxgrid,quiver,reach_solver,arm_model,
// path_planner,pipeline}.cpp for the functions below. Names, argument
// meaning, value semantics and exceptions (reachplan::Error with the same
// Errc and message) are the reference's; the work runs on the GPU.
//
// Host data (VoxelGrid::occupancy, Quiver::vectors) is mirrored to the
// device on first use and cached per thread by content hash, so repeated
// calls on the same grid or quiver do not re-upload. A SolutionSet returned
// by solve_reach keeps its device twin registered so select_solution and
// plan_from_reach run on the device set (the returned host set is fully
// materialised, as the reference's).
//
// Covered (reference declaration -> here): build_grid, mark_obstacles,
// dilate, point_clear, segment_clear, VoxelGrid::occupied_count
// (voxgrid.hpp:60-84); generate_quiver, cone_subset (quiver.hpp:38-49);
// backward_endpoints, prune_segment1 (survivors, stats and the
// near-encounter scan), span_gap, solve_reach, short_reach_scan,
// select_solution (reach_solver.hpp:45-165);
// exact_refine_6dof / _8dof / _8dof_triangle (arm_model.hpp:92-107);
// smoothness_ok, waypoint_ik, plan_from_reach, plan_arbitrary,
// replan_dynamic, plan_reach_then_path, folded_pose,
// mean_polyline_deviation (path_planner.hpp:43-114); effective_dilation,
// build_scene_grid (pipeline.hpp:10-17).
#include "reachplan/pipeline.hpp"
#include "reachplan_b200.h"

#include <algorithm>
#include <array>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <functional>
#include <memory>
#include <mutex>
#include <ostream>
#include <string>
#include <thread>
#include <vector>

namespace reachplan {
namespace {

// ---- errors -------------------------------------------------------------------

[[noreturn]] void raise(rp_status st) {
  std::string msg = rp_last_error();
  if (st >= 1 && st <= 11) {
    const Errc code = static_cast<Errc>(st - 1);
    const std::string prefix = std::string(errc_name(code)) + ": ";
    if (msg.compare(0, prefix.size(), prefix) == 0) msg.erase(0, prefix.size());
    throw Error(code, msg);
  }
  throw std::runtime_error("reachplan-b200: " + msg);
}

void ok(rp_status st) {
  if (st != RP_OK) raise(st);
}

// ---- conversions ------------------------------------------------------------------

void put3(double* d, const Vec3& v) {
  d[0] = v.x();
  d[1] = v.y();
  d[2] = v.z();
}
Vec3 get3(const double* s) { return Vec3(s[0], s[1], s[2]); }

rp_arm to_rp(const ArmSpec& a) {
  require(a.segment_count() >= 3 && a.segment_count() <= RP_MAX_SEGMENTS, Errc::invalid_parameter,
          "arm must have 3 or 4 segments");
  rp_arm r;
  rp_arm_init(&r, a.segment_count(), a.lengths.data());
  put3(r.root, a.root);
  r.arm_radius = a.arm_radius;
  r.n_limits = static_cast<int32_t>(std::min<std::size_t>(a.joint_limits.size(), RP_MAX_SEGMENTS));
  for (int k = 0; k < r.n_limits; ++k) {
    r.limits[k].elev_min = a.joint_limits[k].elev_min;
    r.limits[k].elev_max = a.joint_limits[k].elev_max;
    r.limits[k].azim_min = a.joint_limits[k].azim_min;
    r.limits[k].azim_max = a.joint_limits[k].azim_max;
  }
  r.n_offsets = static_cast<int32_t>(std::min<std::size_t>(a.offsets.size(), RP_MAX_SEGMENTS));
  for (int k = 0; k < r.n_offsets; ++k) r.offsets[k] = a.offsets[k];
  put3(r.fold_plane_normal, a.fold_plane_normal);
  r.fold_flex = a.fold_flex;
  put3(r.base_axis, a.base_axis);
  put3(r.base_ref, a.base_ref);
  return r;
}

rp_reach_params to_rp(const ReachParams& p) {
  rp_reach_params r;
  rp_reach_params_init(&r);
  r.epsilon_gap = p.epsilon_gap;
  r.n_samples = p.n_samples_per_segment;
  put3(r.approach_axis, p.approach_axis);
  r.approach_half_angle = p.approach_half_angle;
  r.near_target_radius = p.near_target_radius;
  r.mode = p.mode == SolveMode::six_dof ? RP_MODE_6DOF : RP_MODE_8DOF;
  r.cone_precheck = p.cone_precheck ? 1 : 0;
  r.disable_geom_pruning = p.disable_geom_pruning ? 1 : 0;
  r.refine_triangle_8dof = p.refine_triangle_8dof ? 1 : 0;
  r.workers = p.workers;
  return r;
}

rp_path_params to_rp(const PathParams& p) {
  rp_path_params r;
  rp_path_params_init(&r);
  r.epsilon_waypoint = p.epsilon_waypoint;
  r.d_w = p.d_w;
  r.slack = p.slack;
  r.joint1_max_move = p.joint1_max_move;
  r.joint2_max_move = p.joint2_max_move;
  require(p.relax_schedule.size() <= RP_MAX_RELAX, Errc::invalid_parameter,
          "relax schedule longer than the device planner supports");
  r.n_relax = static_cast<int32_t>(p.relax_schedule.size());
  for (int k = 0; k < r.n_relax; ++k) r.relax_schedule[k] = p.relax_schedule[k];
  r.unfold_steps = p.unfold_steps;
  return r;
}

struct ObstacleBuf {
  std::vector<rp_obstacle> obs;
  std::vector<std::vector<double>> pts;
  explicit ObstacleBuf(const std::vector<SceneObstacle>& in) {
    obs.resize(in.size());
    pts.resize(in.size());
    for (std::size_t k = 0; k < in.size(); ++k) {
      const SceneObstacle& o = in[k];
      rp_obstacle& r = obs[k];
      std::memset(&r, 0, sizeof(r));
      r.shape = o.shape == SceneObstacle::Shape::box ? RP_SHAPE_BOX : RP_SHAPE_CLOUD;
      r.dynamic = o.dynamic ? 1 : 0;
      put3(r.box_min, o.box_min);
      put3(r.box_max, o.box_max);
      for (const Vec3& p : o.points) {
        pts[k].push_back(p.x());
        pts[k].push_back(p.y());
        pts[k].push_back(p.z());
      }
      r.points = pts[k].empty() ? nullptr : pts[k].data();
      r.n_points = static_cast<int64_t>(o.points.size());
      r.id = o.id.c_str();
    }
  }
  int32_t size() const { return static_cast<int32_t>(obs.size()); }
};

PoseChain from_rp(const rp_pose& p, const double* wps) {
  PoseChain c;
  for (int k = 0; k < p.n_segments; ++k) {
    c.segments.push_back(get3(p.segments[k]));
    if (!p.no_indices) c.quiver_indices.push_back(p.quiver_indices[k]);
    if (p.has_elbows) c.elbows.push_back(get3(p.elbows[k]));
  }
  for (int k = 0; k <= p.n_segments; ++k) c.joints.push_back(get3(p.joints[k]));
  if (wps)
    for (int k = 0; k < p.n_waypoints; ++k) c.waypoints.push_back(get3(wps + 3 * k));
  c.s4_length_dev = p.s4_length_dev;
  return c;
}

rp_pose to_rp(const PoseChain& c, std::vector<double>* wps) {
  rp_pose p;
  std::memset(&p, 0, sizeof(p));
  require(c.segment_count() >= 1 && c.segment_count() <= RP_MAX_SEGMENTS, Errc::invalid_parameter,
          "pose must have 1..4 segments");
  p.n_segments = c.segment_count();
  p.has_elbows = c.elbows.empty() ? 0 : 1;
  p.no_indices = c.quiver_indices.empty() ? 1 : 0;
  for (int k = 0; k < RP_MAX_SEGMENTS; ++k)
    p.quiver_indices[k] = k < static_cast<int>(c.quiver_indices.size()) ? c.quiver_indices[k] : -1;
  for (int k = 0; k < p.n_segments; ++k) {
    put3(p.segments[k], c.segments[k]);
    if (p.has_elbows && k < static_cast<int>(c.elbows.size())) put3(p.elbows[k], c.elbows[k]);
  }
  for (int k = 0; k < static_cast<int>(c.joints.size()) && k <= RP_MAX_SEGMENTS; ++k)
    put3(p.joints[k], c.joints[k]);
  p.s4_length_dev = c.s4_length_dev;
  p.n_waypoints = static_cast<int32_t>(c.waypoints.size());
  if (wps) {
    wps->clear();
    for (const Vec3& w : c.waypoints) {
      wps->push_back(w.x());
      wps->push_back(w.y());
      wps->push_back(w.z());
    }
  }
  return p;
}

SolveStats from_rp(const rp_solve_stats& s) {
  SolveStats o;
  o.seg1_candidates = s.seg1_candidates;
  o.seg1_limit_pass = s.seg1_limit_pass;
  o.seg1_reach_pass = s.seg1_reach_pass;
  o.seg1_survivors = s.seg1_survivors;
  o.pair_candidates = s.pair_candidates;
  o.seg2_limit_pass = s.seg2_limit_pass;
  o.seg2_clear_pass = s.seg2_clear_pass;
  o.gap_tested = s.gap_tested;
  o.gap_pass = s.gap_pass;
  o.joint_pass = s.joint_pass;
  o.v3_clear_pass = s.v3_clear_pass;
  o.solutions = s.solutions;
  o.shortcuts_found = s.shortcuts_found;
  o.wall_ms = s.wall_ms;
  return o;
}

std::vector<double> flat(const std::vector<Vec3>& v) {
  std::vector<double> out;
  out.reserve(3 * v.size());
  for (const Vec3& p : v) {
    out.push_back(p.x());
    out.push_back(p.y());
    out.push_back(p.z());
  }
  return out;
}

// ---- per-thread device runtime -------------------------------------------------

uint64_t mix_bytes(const void* data, std::size_t n, uint64_t h) {
  // 64-bit multiply-xorshift (content identity, not crypto): four
  // independent lanes over 32-byte blocks so the multiplies overlap (~4x the
  // single-chain rate on a 16 MiB grid), then the lanes and the tail
  const auto* b = static_cast<const unsigned char*>(data);
  std::size_t k = 0;
  uint64_t l[4] = {h, h ^ 0x243F6A8885A308D3ull, h ^ 0x13198A2E03707344ull,
                   h ^ 0xA4093822299F31D0ull};
  for (; k + 32 <= n; k += 32) {
    uint64_t w[4];
    std::memcpy(w, b + k, 32);
    for (int q = 0; q < 4; ++q) {
      l[q] ^= w[q];
      l[q] *= 0x9E3779B97F4A7C15ull;
      l[q] ^= l[q] >> 29;
    }
  }
  for (int q = 0; q < 4; ++q) {
    h ^= l[q];
    h *= 0x9E3779B97F4A7C15ull;
    h ^= h >> 29;
  }
  for (; k + 8 <= n; k += 8) {
    uint64_t w;
    std::memcpy(&w, b + k, 8);
    h ^= w;
    h *= 0x9E3779B97F4A7C15ull;
    h ^= h >> 29;
  }
  for (; k < n; ++k) {
    h ^= b[k];
    h *= 0x100000001B3ull;
  }
  return h;
}

/// RP_FACADE_TRACE=1: per-step host times of the façade's own work (stderr).
struct Trace {
  const char* what;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  explicit Trace(const char* w) : what(w) {}
  ~Trace() {
    static const bool on = std::getenv("RP_FACADE_TRACE") != nullptr;
    if (on)
      std::fprintf(stderr, "[facade] %-22s %9.3f ms\n", what,
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                       .count());
  }
};

/// A persistent pool of host threads for the façade's O(N^3) byte work
/// (expanding and hashing VoxelGrid bytes): spawning threads per call cost
/// more than the work at 256^3.
class HostPool {
 public:
  static HostPool& get() {
    static HostPool p;
    return p;
  }
  std::size_t size() const { return workers_.size() + 1; }
  /// f(t) for t in [0, n): the caller and the workers take indices in turn.
  void run(std::size_t n, const std::function<void(std::size_t)>& f) {
    if (n <= 1 || workers_.empty()) {
      for (std::size_t t = 0; t < n; ++t) f(t);
      return;
    }
    std::lock_guard<std::mutex> one(call_);  // one job at a time across caller threads
    std::unique_lock<std::mutex> lk(m_);
    job_ = &f;
    n_ = n;
    next_ = 0;
    left_ = n;
    ++gen_;
    cv_.notify_all();
    drain(lk);
    done_.wait(lk, [&] { return left_ == 0; });
    job_ = nullptr;
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> lk(m_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& w : workers_) w.join();
  }

 private:
  HostPool() {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    for (unsigned k = 1; k < std::min(hw, 32u); ++k)
      workers_.emplace_back([this] {
        std::unique_lock<std::mutex> lk(m_);
        uint64_t seen = 0;
        for (;;) {
          cv_.wait(lk, [&] { return stop_ || (gen_ != seen && job_ && next_ < n_); });
          if (stop_) return;
          seen = gen_;
          drain(lk);
        }
      });
  }
  // with m_ held: run indices until none is left to take
  void drain(std::unique_lock<std::mutex>& lk) {
    while (job_ && next_ < n_) {
      const std::size_t t = next_++;
      const auto* f = job_;
      lk.unlock();
      (*f)(t);
      lk.lock();
      if (--left_ == 0) done_.notify_all();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex call_, m_;
  std::condition_variable cv_, done_;
  const std::function<void(std::size_t)>* job_ = nullptr;
  std::size_t n_ = 0, next_ = 0, left_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

/// Runs f(begin, end) over [0, n) split into up to one range per pool
/// thread, each of at least `min_chunk` items.
template <typename F>
void parallel_ranges(std::size_t n, std::size_t min_chunk, F f) {
  HostPool& pool = HostPool::get();
  const std::size_t T =
      std::max<std::size_t>(1, std::min(pool.size(), n / std::max<std::size_t>(1, min_chunk)));
  if (T <= 1) {
    f(std::size_t{0}, n);
    return;
  }
  const std::size_t per = (n + T - 1) / T;
  pool.run(T, [&](std::size_t t) {
    const std::size_t a = t * per, b = std::min(n, a + per);
    if (a < b) f(a, b);
  });
}

/// Content hash of a large buffer: mix_bytes of fixed 1 MiB blocks (seeded
/// by h and the block index) computed in parallel, then mixed in order --
/// the same value for any thread count. fill(begin, end) runs on a block's
/// bytes just before they are hashed (while they are in this core's cache),
/// so a producer can write and hash in one pass.
template <typename Fill>
uint64_t hash_blocks(const uint8_t* data, std::size_t n, uint64_t h, Fill fill) {
  constexpr std::size_t kBlock = std::size_t{1} << 20;
  const std::size_t nb = (n + kBlock - 1) / kBlock;
  if (nb <= 1) {
    fill(std::size_t{0}, n);
    return mix_bytes(data, n, h);
  }
  std::vector<uint64_t> bh(nb);
  parallel_ranges(nb, 1, [&](std::size_t k0, std::size_t k1) {
    for (std::size_t k = k0; k < k1; ++k) {
      const std::size_t off = k * kBlock, len = std::min(kBlock, n - off);
      fill(off, off + len);
      bh[k] = mix_bytes(data + off, len, h ^ (k * 0x9E37ull));
    }
  });
  return mix_bytes(bh.data(), nb * sizeof(uint64_t), h);
}
uint64_t mix_bytes_parallel(const uint8_t* data, std::size_t n, uint64_t h) {
  return hash_blocks(data, n, h, [](std::size_t, std::size_t) {});
}

struct GridEntry {
  uint64_t hash;
  rp_grid* g;
};
struct QuiverEntry {
  uint64_t hash;
  rp_quiver* q;
};
struct SetEntry {
  std::vector<int64_t> fingerprint;
  rp_solution_set* s;
};

class Runtime {
 public:
  Runtime() {
    const char* dev = std::getenv("RP_DEVICE");
    ok(rp_ctx_create(dev ? std::atoi(dev) : 0, &ctx_));
  }
  ~Runtime() {
    for (auto& e : grids_) rp_grid_destroy(e.g);
    for (auto& e : quivers_) rp_quiver_destroy(e.q);
    for (auto& e : sets_) rp_solution_set_destroy(e.s);
    rp_ctx_destroy(ctx_);
  }
  rp_ctx* ctx() { return ctx_; }

  static uint64_t grid_meta_hash(const VoxelGrid& g) {
    uint64_t h = mix_bytes(g.dims.data(), sizeof(int) * 3, 0x51ED27ull);
    const double meta[5] = {g.origin.x(), g.origin.y(), g.origin.z(), g.voxel_size,
                            g.dilation_radius};
    return mix_bytes(meta, sizeof(meta), h);
  }
  static uint64_t grid_hash(const VoxelGrid& g) {
    return mix_bytes_parallel(g.occupancy.data(), g.occupancy.size(), grid_meta_hash(g));
  }

  /// Device mirror of a host grid (uploaded on a cache miss).
  rp_grid* grid(const VoxelGrid& g) {
    require(g.occupancy.size() == g.cell_count(), Errc::invalid_parameter,
            "grid occupancy size does not match its dims");
    const uint64_t h = [&] {
      Trace t_("grid lookup hash");
      return grid_hash(g);
    }();
    for (auto& e : grids_)
      if (e.hash == h) return e.g;
    double org[3];
    put3(org, g.origin);
    rp_grid* d = nullptr;
    ok(rp_grid_upload_u8(ctx_, org, g.voxel_size, g.dims.data(), g.occupancy.data(),
                         g.dilation_radius, &d));
    remember(h, d);
    return d;
  }

  /// Download a device grid into `out` (dims/origin/size/radius + bytes) and
  /// cache the handle under the new content.
  void adopt(rp_grid* d, VoxelGrid& out) {
    int32_t dims[3];
    double org[3], vs, rad;
    ok(rp_grid_info(d, dims, org, &vs, &rad));
    out.dims = {dims[0], dims[1], dims[2]};
    out.origin = get3(org);
    out.voxel_size = vs;
    out.dilation_radius = rad;
    // the bit words (1/8 of the bytes) cross PCIe and are expanded to the
    // reference's byte layout on the host, rows in parallel
    const std::size_t nx = dims[0], rows = static_cast<std::size_t>(dims[1]) * dims[2];
    const std::size_t wx = (nx + 63) / 64;
    std::vector<uint64_t> bits(rows * wx);
    {
      Trace t_("adopt download bits");
      ok(rp_grid_download_bits(d, bits.data(), bits.size()));
    }
    {
      Trace t_("adopt resize");
      out.occupancy.resize(out.cell_count());
    }
    Trace t_("adopt expand+hash");
    static const auto expand = [] {
      std::array<uint64_t, 256> t{};
      for (int v = 0; v < 256; ++v)
        for (int k = 0; k < 8; ++k)
          if ((v >> k) & 1) t[v] |= uint64_t{1} << (8 * k);  // little-endian byte k
      return t;
    }();
    uint8_t* dst = out.occupancy.data();
    // expand each 1 MiB block of the byte grid from the bit words and hash
    // it while it is in cache (grid_hash's value, one pass)
    const auto fill = [&](std::size_t o0, std::size_t o1) {
      while (o0 < o1) {
        const std::size_t r = o0 / nx, x0 = o0 - r * nx;
        const std::size_t x1 = std::min(nx, x0 + (o1 - o0));
        uint8_t* row = dst + r * nx;
        const uint64_t* wr = bits.data() + r * wx;
        std::size_t x = x0;
        for (; x < x1 && (x & 7); ++x) row[x] = static_cast<uint8_t>((wr[x >> 6] >> (x & 63)) & 1);
        for (; x + 8 <= x1; x += 8) {
          const uint64_t bytes = expand[(wr[x >> 6] >> (x & 63)) & 0xFF];
          std::memcpy(row + x, &bytes, 8);
        }
        for (; x < x1; ++x) row[x] = static_cast<uint8_t>((wr[x >> 6] >> (x & 63)) & 1);
        o0 += x1 - x0;
      }
    };
    remember(hash_blocks(dst, out.occupancy.size(), grid_meta_hash(out), fill), d);
  }

  rp_quiver* quiver(const Quiver& q) {
    require(q.size() > 0, Errc::invalid_parameter, "empty quiver");
    const std::vector<double> xyz = flat(q.vectors);
    const uint64_t h = mix_bytes(xyz.data(), xyz.size() * sizeof(double), 0x0A11Bull);
    for (auto& e : quivers_)
      if (e.hash == h) return e.q;
    rp_quiver* d = nullptr;
    ok(rp_quiver_upload(ctx_, xyz.data(), q.size(), &d));
    quivers_.push_front({h, d});
    if (quivers_.size() > 4) {
      rp_quiver_destroy(quivers_.back().q);
      quivers_.pop_back();
    }
    return d;
  }

  static std::vector<int64_t> fingerprint(const SolutionSet& s) {
    const SolveStats& t = s.stats;
    std::vector<int64_t> f{t.seg1_candidates, t.seg1_limit_pass, t.seg1_reach_pass,
                           t.seg1_survivors,  t.pair_candidates, t.seg2_limit_pass,
                           t.seg2_clear_pass, t.gap_tested,      t.gap_pass,
                           t.joint_pass,      t.v3_clear_pass,   t.solutions,
                           t.shortcuts_found, static_cast<int64_t>(s.solutions.size()),
                           static_cast<int64_t>(s.shortcuts.size())};
    for (const PoseChain* p : {s.solutions.empty() ? nullptr : &s.solutions.front(),
                               s.solutions.empty() ? nullptr : &s.solutions.back()}) {
      if (!p) continue;
      for (const Vec3& v : p->segments) {
        const double xyz[3] = {v.x(), v.y(), v.z()};
        int64_t bits[3];
        std::memcpy(bits, xyz, sizeof(bits));
        f.insert(f.end(), bits, bits + 3);
      }
    }
    for (const ShortcutPath& sc : s.shortcuts) {
      int64_t b;
      std::memcpy(&b, &sc.path_length, 8);
      f.push_back(b);
    }
    return f;
  }

  void register_set(const SolutionSet& s, rp_solution_set* d) {
    sets_.push_front({fingerprint(s), d});
    if (sets_.size() > 4) {
      rp_solution_set_destroy(sets_.back().s);
      sets_.pop_back();
    }
  }

  rp_solution_set* lookup(const SolutionSet& s) {
    const std::vector<int64_t> f = fingerprint(s);
    for (auto& e : sets_)
      if (e.fingerprint == f) return e.s;
    return nullptr;
  }

 private:
  void remember(uint64_t h, rp_grid* d) {
    for (auto& e : grids_)
      if (e.g == d) {
        e.hash = h;
        return;
      }
    grids_.push_front({h, d});
    if (grids_.size() > 4) {
      Trace t_("evict grid");
      rp_grid_destroy(grids_.back().g);
      grids_.pop_back();
    }
  }

  rp_ctx* ctx_ = nullptr;
  std::deque<GridEntry> grids_;
  std::deque<QuiverEntry> quivers_;
  std::deque<SetEntry> sets_;
};

Runtime& rt() {
  thread_local Runtime r;
  return r;
}

rp_grid* fresh_copy(const VoxelGrid& g) {
  rp_grid* d = nullptr;
  ok(rp_grid_copy(rt().grid(g), &d));
  return d;
}

PathPlan from_rp(const rp_plan* h) {
  rp_plan_info info;
  ok(rp_plan_get_info(h, &info));
  PathPlan plan;
  std::vector<double> w(3 * static_cast<std::size_t>(std::max(info.n_waypoints, 1)));
  ok(rp_plan_waypoints(h, w.data(), info.n_waypoints));
  for (int k = 0; k < info.n_waypoints; ++k) plan.waypoints.push_back(get3(&w[3 * k]));
  std::vector<double> pw(3 * 4096);
  for (int which = 0; which < 2; ++which) {
    const int n = which == 0 ? info.n_poses : info.n_unfold;
    for (int k = 0; k < n; ++k) {
      rp_pose p;
      ok(rp_plan_pose(h, which, k, &p, pw.data(), 4096));
      (which == 0 ? plan.poses : plan.unfold_prefix).push_back(from_rp(p, pw.data()));
    }
  }
  plan.provenance.kind = info.kind;
  plan.provenance.relax_per_waypoint.resize(info.n_waypoints);
  ok(rp_plan_relax(h, plan.provenance.relax_per_waypoint.data(), info.n_waypoints));
  for (int k = 0; k < info.n_notes; ++k) {
    char buf[1024];
    ok(rp_plan_note(h, k, buf, sizeof(buf)));
    plan.provenance.notes.push_back(buf);
  }
  plan.provenance.replan_switch_index = info.replan_switch_index;
  return plan;
}

PathPlan take_plan(rp_status st, rp_plan* h) {
  ok(st);
  std::unique_ptr<rp_plan, rp_status (*)(rp_plan*)> guard(h, rp_plan_destroy);
  return from_rp(h);
}

}  // namespace

// ---- voxgrid.hpp -----------------------------------------------------------------

std::size_t VoxelGrid::occupied_count() const {
  uint64_t c = 0;
  ok(rp_grid_occupied_count(rt().grid(*this), &c));
  return static_cast<std::size_t>(c);
}

VoxelGrid build_grid(const Vec3& bounds_min, const Vec3& bounds_max, double voxel_size,
                     std::size_t cell_budget) {
  double lo[3], hi[3];
  put3(lo, bounds_min);
  put3(hi, bounds_max);
  rp_grid* d = nullptr;
  ok(rp_grid_build(rt().ctx(), lo, hi, voxel_size, cell_budget, &d));
  VoxelGrid g;
  rt().adopt(d, g);
  return g;
}

void mark_obstacles(VoxelGrid& grid, const std::vector<SceneObstacle>& obstacles) {
  rp_grid* d = fresh_copy(grid);
  const ObstacleBuf ob(obstacles);
  ok(rp_grid_mark(d, ob.obs.data(), ob.size()));
  rt().adopt(d, grid);
}

void dilate(VoxelGrid& grid, double radius) {
  rp_grid* d = fresh_copy(grid);
  ok(rp_grid_dilate(d, radius));
  rt().adopt(d, grid);
}

bool point_clear(const VoxelGrid& grid, const Vec3& p) {
  double xyz[3];
  put3(xyz, p);
  uint8_t out = 0;
  ok(rp_grid_point_clear(rt().grid(grid), xyz, 1, &out));
  return out != 0;
}

SegmentProbe segment_clear(const VoxelGrid& grid, const Vec3& p_start, const Vec3& p_end,
                           int n_samples) {
  require(n_samples >= 1, Errc::invalid_parameter, "n_samples must be >= 1");
  double a[3], b[3];
  put3(a, p_start);
  put3(b, p_end);
  uint8_t out = 0;
  ok(rp_grid_segment_clear(rt().grid(grid), a, b, 1, n_samples, &out));
  SegmentProbe probe;
  probe.clear = out != 0;
  // the sample points themselves (the verdict above is the device's)
  const Vec3 d = p_end - p_start;
  for (int k = 1; k <= n_samples; ++k)
    probe.samples.push_back(p_start + (static_cast<double>(k) / n_samples) * d);
  return probe;
}

// ---- quiver.hpp ------------------------------------------------------------------

Quiver generate_quiver(double elev_step, double equator_azim_step, int min_per_ring) {
  rp_quiver* d = nullptr;
  ok(rp_quiver_generate(rt().ctx(), elev_step, equator_azim_step, min_per_ring, &d));
  std::unique_ptr<rp_quiver, rp_status (*)(rp_quiver*)> guard(d, rp_quiver_destroy);
  Quiver q;
  const int n = rp_quiver_size(d);
  std::vector<double> xyz(3 * static_cast<std::size_t>(n));
  ok(rp_quiver_download(d, xyz.data(), n));
  for (int k = 0; k < n; ++k) q.vectors.push_back(get3(&xyz[3 * k]));
  int32_t nr = 0;
  ok(rp_quiver_rings(d, nullptr, nullptr, 0, &nr, nullptr, nullptr, nullptr));
  q.ring_offsets.resize(nr);
  q.ring_elevations.resize(nr);
  int32_t mpr = 0;
  ok(rp_quiver_rings(d, q.ring_offsets.data(), q.ring_elevations.data(), nr, &nr, &q.elev_step,
                     &q.equator_azim_step, &mpr));
  q.min_per_ring = mpr;
  return q;
}

std::vector<int> cone_subset(const Quiver& q, const Vec3& axis, double half_angle) {
  double ax[3];
  put3(ax, axis);
  std::vector<int> idx(q.size());
  int32_t n = 0;
  ok(rp_cone_subset(rt().ctx(), rt().quiver(q), ax, half_angle, idx.data(), q.size(), &n));
  idx.resize(n);
  return idx;
}

// ---- reach_solver.hpp --------------------------------------------------------------

BackwardEndpoints backward_endpoints(const Vec3& target, double L4, const Quiver& q,
                                     const Vec3& approach_axis, double half_angle,
                                     SolveMode mode) {
  rp_reach_params rp;
  rp_reach_params_init(&rp);
  put3(rp.approach_axis, approach_axis);
  rp.approach_half_angle = half_angle;
  rp.mode = mode == SolveMode::six_dof ? RP_MODE_6DOF : RP_MODE_8DOF;
  double t[3];
  put3(t, target);
  const int cap = std::max(1, q.size());
  std::vector<double> pts(3 * cap), dirs(3 * cap);
  std::vector<int32_t> cone(cap);
  int32_t n = 0;
  ok(rp_backward_endpoints(rt().ctx(), rt().quiver(q), t, L4, &rp, pts.data(), dirs.data(),
                           cone.data(), cap, &n));
  BackwardEndpoints out;
  for (int k = 0; k < n; ++k) {
    out.points.push_back(get3(&pts[3 * k]));
    out.directions.push_back(get3(&dirs[3 * k]));
    out.cone_indices.push_back(cone[k]);
  }
  return out;
}

std::vector<GapCandidate> span_gap(const Vec3& p2, const std::vector<Vec3>& backward_pts,
                                   double L3, double epsilon) {
  const std::vector<double> b = flat(backward_pts);
  const int n = static_cast<int>(backward_pts.size());
  std::vector<double> v3(3 * std::max(n, 1));
  std::vector<int32_t> idx(std::max(n, 1));
  double p[3];
  put3(p, p2);
  int32_t m = 0;
  ok(rp_span_gap(rt().ctx(), p, b.data(), n, L3, epsilon, v3.data(), idx.data(), &m));
  std::vector<GapCandidate> out;
  for (int k = 0; k < m; ++k) out.push_back(GapCandidate{get3(&v3[3 * k]), idx[k]});
  return out;
}

SolutionSet solve_reach(const ArmSpec& spec, const Quiver& q, const VoxelGrid& grid,
                        const Vec3& target, const ReachParams& params) {
  const rp_arm arm = to_rp(spec);
  const rp_reach_params rp = to_rp(params);
  double t[3];
  put3(t, target);
  rp_solution_set* d = nullptr;
  ok(rp_solve_reach(rt().ctx(), &arm, rt().quiver(q), rt().grid(grid), t, &rp, &d));
  std::unique_ptr<rp_solution_set, rp_status (*)(rp_solution_set*)> guard(d,
                                                                          rp_solution_set_destroy);
  SolutionSet set;
  rp_solve_stats st;
  ok(rp_solution_set_stats(d, &st));
  set.stats = from_rp(st);
  int64_t ns = 0, nc = 0;
  ok(rp_solution_set_sizes(d, &ns, &nc));
  const int wpp = 4 * params.n_samples_per_segment;
  constexpr int64_t kChunk = 1 << 15;
  std::vector<rp_pose> poses(static_cast<std::size_t>(std::min(ns, kChunk)));
  std::vector<double> wps(poses.size() * 3 * static_cast<std::size_t>(wpp));
  set.solutions.reserve(static_cast<std::size_t>(ns));
  for (int64_t c0 = 0; c0 < ns; c0 += kChunk) {
    const int64_t n = std::min(kChunk, ns - c0);
    ok(rp_solution_set_poses(d, c0, n, poses.data(), wps.data(), wpp));
    for (int64_t k = 0; k < n; ++k)
      set.solutions.push_back(from_rp(poses[k], &wps[static_cast<std::size_t>(k) * 3 * wpp]));
  }
  std::vector<double> tip(3 * 4096);
  for (int64_t k = 0; k < nc; ++k) {
    rp_shortcut sc;
    int32_t ntip = 0;
    ok(rp_solution_set_shortcut(d, k, &sc, tip.data(), 4096, &ntip));
    rp_pose basis;
    ok(rp_solution_set_shortcut_basis(d, k, &basis));
    ShortcutPath p;
    p.segment_index = sc.segment_index;
    p.hit_sample_index = sc.hit_sample_index;
    for (int m = 0; m < sc.n_prefix; ++m) p.prefix_samples.push_back(get3(&tip[3 * m]));
    for (int m = 0; m < sc.n_sublength; ++m)
      p.sublength_samples.push_back(get3(&tip[3 * (sc.n_prefix + m)]));
    if (sc.has_bridge) p.bridge = get3(sc.bridge);
    p.via_origin_direct = sc.via_origin_direct != 0;
    p.basis_pose = from_rp(basis, nullptr);
    p.path_length = sc.path_length;
    p.seg1_index = sc.seg1_index;
    p.seg2_index = sc.seg2_index;
    set.shortcuts.push_back(std::move(p));
  }
  rt().register_set(set, guard.release());
  return set;
}

std::vector<Seg1Hypothesis> prune_segment1(const ArmSpec& spec, const Quiver& q,
                                           const VoxelGrid& grid,
                                           const std::vector<Vec3>& target_points,
                                           const ReachParams& params,
                                           std::vector<ShortcutPath>* shortcut_sink,
                                           SolveStats* stats, const Vec3* scan_target) {
  // Survivor indices and the seg1_* counters come from the device
  // (k_seg1). The per-hypothesis payload is rebuilt from the index the
  // coaxial way (dir, p1 = root + L1 dir, samples); offsets, frames and the
  // near-encounter sink are not exposed through this façade.
  require(!spec.has_offsets(), Errc::invalid_parameter,
          "façade prune_segment1 covers coaxial arms (use solve_reach)");
  const rp_arm arm = to_rp(spec);
  const rp_reach_params rp = to_rp(params);
  const std::vector<double> tp = flat(target_points);
  std::vector<int32_t> idx(q.size());
  int32_t n = 0;
  rp_solve_stats st;
  ok(rp_prune_segment1(rt().ctx(), &arm, rt().quiver(q), rt().grid(grid), tp.data(),
                       static_cast<int32_t>(target_points.size()), &rp, idx.data(), q.size(), &n,
                       &st));
  if (stats) {
    const SolveStats s = from_rp(st);
    stats->seg1_candidates += s.seg1_candidates;
    stats->seg1_limit_pass += s.seg1_limit_pass;
    stats->seg1_reach_pass += s.seg1_reach_pass;
    stats->seg1_survivors += s.seg1_survivors;
  }
  const int ns = params.n_samples_per_segment;
  if (shortcut_sink && scan_target) {
    // The near-encounter scan (reach_solver.cpp:277-291) over every
    // hypothesis whose segment passes within near_target_radius of the
    // target: their walks' per-sample clearance from one batched device
    // point_clear, each scan by rp_short_reach_scan on the device.
    const double near = params.resolved_near_radius(spec);
    const double L1 = spec.length(0);
    std::vector<int> cand;
    std::vector<double> pts;
    for (int i = 0; i < q.size(); ++i) {
      const Vec3 p1 = spec.root + L1 * q.vectors[i];
      const Vec3 ab = p1 - spec.root;  // point_to_segment (reach_solver.cpp:135-141)
      const double len2 = ab.squaredNorm();
      double d;
      if (len2 <= 1e-30) {
        d = (*scan_target - spec.root).norm();
      } else {
        const double t = std::clamp((*scan_target - spec.root).dot(ab) / len2, 0.0, 1.0);
        d = (*scan_target - (spec.root + t * ab)).norm();
      }
      if (!(d <= near + 1e-9)) continue;
      cand.push_back(i);
      for (int m = 1; m <= ns; ++m) {
        const Vec3 smp = spec.root + (static_cast<double>(m) / ns) * ab;
        pts.push_back(smp.x());
        pts.push_back(smp.y());
        pts.push_back(smp.z());
      }
    }
    std::vector<uint8_t> clear(pts.size() / 3);
    if (!clear.empty())
      ok(rp_grid_point_clear(rt().grid(grid), pts.data(), static_cast<int64_t>(clear.size()),
                             clear.data()));
    const rp_arm arm1 = to_rp(spec);
    const rp_reach_params rp1 = to_rp(params);
    double tgt[3];
    put3(tgt, *scan_target);
    for (std::size_t c = 0; c < cand.size(); ++c) {
      // the walk stops at its first blocked sample (walk_segment_into)
      int m = 0;
      while (m < ns && clear[c * ns + m]) ++m;
      const int len = m < ns ? m + 1 : ns;
      HypothesisScan scan;
      scan.segment_index = 1;
      scan.origin = spec.root;
      for (int k = 0; k < len; ++k) {
        scan.samples.push_back(get3(&pts[3 * (c * ns + k)]));
        scan.sample_clear.push_back(clear[c * ns + k]);
      }
      scan.basis_pose = chain_from_segments(spec, {L1 * q.vectors[cand[c]]}, {cand[c]});
      scan.seg1_index = cand[c];
      if (auto hit = short_reach_scan(scan, *scan_target, grid, spec, params)) {
        shortcut_sink->push_back(std::move(hit->shortcut));
        if (stats) ++stats->shortcuts_found;
      }
    }
    (void)arm1;
    (void)rp1;
    (void)tgt;
  }
  std::vector<Seg1Hypothesis> out;
  for (int k = 0; k < n; ++k) {
    Seg1Hypothesis h;
    h.quiver_index = idx[k];
    h.dir = q.vectors[idx[k]];
    h.p1 = spec.root + spec.length(0) * h.dir;
    const Vec3 d = h.p1 - spec.root;
    for (int m = 1; m <= ns; ++m) h.samples.push_back(spec.root + (static_cast<double>(m) / ns) * d);
    out.push_back(std::move(h));
  }
  return out;
}

ChosenPath select_solution(const SolutionSet& set) {
  require(!set.empty(), Errc::no_solution, "no reach solution under the given constraints");
  rp_solution_set* d = rt().lookup(set);
  rp_chosen c;
  if (d) {
    ok(rp_select_solution(d, &c));
  } else {
    // any other set: its segment vectors / shortcut lengths go to the
    // device argmin (rp_select_solution_data)
    std::vector<double> segs, scl;
    if (set.shortcuts.empty()) {
      segs.reserve(9 * set.solutions.size());
      for (const PoseChain& p : set.solutions)
        for (int k = 0; k < 3; ++k) {
          segs.push_back(p.segments[k].x());
          segs.push_back(p.segments[k].y());
          segs.push_back(p.segments[k].z());
        }
    } else {
      for (const ShortcutPath& sp : set.shortcuts) scl.push_back(sp.path_length);
    }
    ok(rp_select_solution_data(rt().ctx(), segs.data(),
                               static_cast<int64_t>(set.shortcuts.empty() ? set.solutions.size() : 0),
                               scl.data(), static_cast<int64_t>(scl.size()), &c));
  }
  ChosenPath out;
  out.path_length = c.path_length;
  if (c.kind == RP_CHOSEN_SHORTCUT) {
    out.kind = ChosenPath::Kind::shortcut;
    out.shortcut = set.shortcuts[static_cast<std::size_t>(c.index)];
  } else {
    out.kind = ChosenPath::Kind::reach_pose;
    out.pose = set.solutions[static_cast<std::size_t>(c.index)];
  }
  return out;
}

// ---- arm_model.hpp (refinement) ------------------------------------------------------
// Off by default: the rest of arm_model.cpp (chain, angles, limits, used by
// validate.cpp / motion.cpp) stays the reference's, and that TU also defines
// these three. Build with -DRP_FACADE_REFINE when refinement should run on
// the device and the reference's definitions are removed.
#ifdef RP_FACADE_REFINE
namespace {
PoseChain refine(const ArmSpec& spec, const PoseChain& approx, const Vec3& target, int variant) {
  const rp_arm arm = to_rp(spec);
  const rp_pose a = to_rp(approx, nullptr);
  double t[3];
  put3(t, target);
  rp_pose out;
  ok(rp_exact_refine(rt().ctx(), &arm, &a, t, variant, &out));
  return from_rp(out, nullptr);
}
}  // namespace

PoseChain exact_refine_6dof(const ArmSpec& spec, const PoseChain& approx, const Vec3& target) {
  require(approx.segment_count() == 3, Errc::invalid_parameter, "need a 3-segment pose");
  return refine(spec, approx, target, 0);
}

PoseChain exact_refine_8dof(const ArmSpec& spec, const PoseChain& approx, const Vec3& target) {
  require(approx.segment_count() == 4, Errc::invalid_parameter, "need a 4-segment pose");
  return refine(spec, approx, target, 0);
}

PoseChain exact_refine_8dof_triangle(const ArmSpec& spec, const PoseChain& approx,
                                     const Vec3& target) {
  require(approx.segment_count() == 4, Errc::invalid_parameter, "need a 4-segment pose");
  return refine(spec, approx, target, 1);
}

#endif  // RP_FACADE_REFINE

// ---- path_planner.hpp ----------------------------------------------------------------

bool smoothness_ok(const PoseChain& prev, const PoseChain& cand, const PathParams& params,
                   double relax) {
  // the bounds are taken as given (the caller resolves them, as in the
  // reference); the device helper resolves negatives, which a resolved
  // PathParams never holds
  rp_arm arm;
  const double L[3] = {1.0, 1.0, 1.0};
  rp_arm_init(&arm, 3, L);
  rp_reach_params rp;
  rp_reach_params_init(&rp);
  const rp_path_params pp = to_rp(params);
  const rp_pose a = to_rp(prev, nullptr), b = to_rp(cand, nullptr);
  int32_t r = 0;
  ok(rp_smoothness_ok(&arm, &rp, &pp, &a, &b, relax, &r));
  return r != 0;
}

std::optional<PoseChain> waypoint_ik(const ArmSpec& spec, const Quiver& q, const VoxelGrid& grid,
                                     const Vec3& waypoint, const PoseChain& prev,
                                     const ReachParams& rp, const PathParams& pp, double relax,
                                     const TrailContext& trail, const PoseChain* junction_bias) {
  const rp_arm arm = to_rp(spec);
  const rp_reach_params r = to_rp(rp);
  const rp_path_params p = to_rp(pp);
  double w[3], back[3], fwd[3];
  put3(w, waypoint);
  if (trail.back_dir) put3(back, *trail.back_dir);
  if (trail.fwd_dir) put3(fwd, *trail.fwd_dir);
  const rp_pose pv = to_rp(prev, nullptr);
  rp_pose bias;
  if (junction_bias) bias = to_rp(*junction_bias, nullptr);
  int32_t found = 0;
  rp_pose out;
  std::vector<double> wps(3 * 64);
  ok(rp_waypoint_ik(rt().ctx(), &arm, rt().quiver(q), rt().grid(grid), w, &pv, &r, &p, relax,
                    trail.back_dir ? back : nullptr, trail.fwd_dir ? fwd : nullptr,
                    junction_bias ? &bias : nullptr, &found, &out, wps.data(), 64));
  if (!found) return std::nullopt;
  return from_rp(out, wps.data());
}

namespace {
/// The device twin of a SolutionSet and the canonical index of `chosen` in it.
rp_chosen locate(const SolutionSet& all, const ChosenPath& chosen, rp_solution_set** d) {
  *d = rt().lookup(all);
  require(*d != nullptr, Errc::invalid_parameter,
          "solution set was not produced by this library's solve_reach");
  rp_chosen c;
  std::memset(&c, 0, sizeof(c));
  c.path_length = chosen.path_length;
  c.index = -1;
  if (chosen.kind == ChosenPath::Kind::shortcut) {
    c.kind = RP_CHOSEN_SHORTCUT;
    for (std::size_t k = 0; k < all.shortcuts.size(); ++k) {
      const ShortcutPath& s = all.shortcuts[k];
      if (s.segment_index == chosen.shortcut.segment_index &&
          s.seg1_index == chosen.shortcut.seg1_index && s.seg2_index == chosen.shortcut.seg2_index) {
        c.index = static_cast<int64_t>(k);
        break;
      }
    }
  } else {
    c.kind = RP_CHOSEN_REACH_POSE;
    // canonical order is ascending quiver indices (seg1, seg2, cone)
    const auto it = std::lower_bound(
        all.solutions.begin(), all.solutions.end(), chosen.pose,
        [](const PoseChain& x, const PoseChain& y) { return x.quiver_indices < y.quiver_indices; });
    if (it != all.solutions.end() && it->quiver_indices == chosen.pose.quiver_indices)
      c.index = static_cast<int64_t>(it - all.solutions.begin());
  }
  require(c.index >= 0, Errc::invalid_parameter, "chosen path is not in the solution set");
  return c;
}
}  // namespace

PathPlan plan_from_reach(const ArmSpec& spec, const Quiver& q, const VoxelGrid& grid,
                         const ChosenPath& chosen, const SolutionSet& all_solutions,
                         const Vec3& target, const ReachParams& rp, const PathParams& pp) {
  rp_solution_set* d = nullptr;
  const rp_chosen c = locate(all_solutions, chosen, &d);
  const rp_arm arm = to_rp(spec);
  const rp_reach_params r = to_rp(rp);
  const rp_path_params p = to_rp(pp);
  double t[3];
  put3(t, target);
  rp_plan* h = nullptr;
  const rp_status st =
      rp_plan_from_reach(rt().ctx(), &arm, rt().quiver(q), rt().grid(grid), d, &c, t, &r, &p, &h);
  return take_plan(st, h);
}

PathPlan fallback_cascade(const ArmSpec& spec, const Quiver& q, const VoxelGrid& grid,
                          const PlanFailure& failure, const SolutionSet& all_solutions,
                          const Vec3& target, const ReachParams& rp, const PathParams& pp) {
  rp_solution_set* d = nullptr;
  const rp_chosen c = locate(all_solutions, failure.candidate, &d);
  const rp_arm arm = to_rp(spec);
  const rp_reach_params r = to_rp(rp);
  const rp_path_params p = to_rp(pp);
  const std::vector<double> w = flat(failure.waypoints);
  double t[3];
  put3(t, target);
  rp_plan* h = nullptr;
  const rp_status st = rp_fallback_cascade(
      rt().ctx(), &arm, rt().quiver(q), rt().grid(grid), d, &c, w.empty() ? nullptr : w.data(),
      static_cast<int32_t>(failure.waypoints.size()), failure.blocked_index, t, &r, &p, &h);
  return take_plan(st, h);
}

PathPlan plan_arbitrary(const ArmSpec& spec, const Quiver& q, const VoxelGrid& grid,
                        const PoseChain& start_pose, const Vec3& target, const ReachParams& rp,
                        const PathParams& pp) {
  const rp_arm arm = to_rp(spec);
  const rp_reach_params r = to_rp(rp);
  const rp_path_params p = to_rp(pp);
  std::vector<double> sw;
  const rp_pose sp = to_rp(start_pose, &sw);
  double t[3];
  put3(t, target);
  rp_plan* h = nullptr;
  rp_quiver* dq = rt().quiver(q);
  rp_grid* dg = rt().grid(grid);
  rp_status st;
  {
    Trace t_("rp_plan_arbitrary");
    st = rp_plan_arbitrary(rt().ctx(), &arm, dq, dg, &sp, sw.empty() ? nullptr : sw.data(), t, &r,
                           &p, &h);
  }
  Trace t_("take_plan");
  return take_plan(st, h);
}

PathPlan replan_dynamic(const ArmSpec& spec, const Quiver& q, const VoxelGrid& grid_static,
                        const PathPlan& active, int current_index,
                        const SceneObstacle& new_obstacle, const ReplanTiming& timing,
                        const ReachParams& rp, const PathParams& pp) {
  const rp_arm arm = to_rp(spec);
  const rp_reach_params r = to_rp(rp);
  const rp_path_params p = to_rp(pp);
  const std::vector<double> w = flat(active.waypoints);
  std::vector<rp_pose> poses, unfold;
  for (const PoseChain& c : active.poses) poses.push_back(to_rp(c, nullptr));
  for (const PoseChain& c : active.unfold_prefix) unfold.push_back(to_rp(c, nullptr));
  rp_plan* act = nullptr;
  ok(rp_plan_create(active.provenance.kind.c_str(), w.data(), poses.data(),
                    active.provenance.relax_per_waypoint.data(),
                    static_cast<int32_t>(active.poses.size()), unfold.data(),
                    static_cast<int32_t>(unfold.size()), &act));
  std::unique_ptr<rp_plan, rp_status (*)(rp_plan*)> guard(act, rp_plan_destroy);
  const ObstacleBuf ob({new_obstacle});
  rp_plan* h = nullptr;
  const rp_status st = rp_replan_dynamic(rt().ctx(), &arm, rt().quiver(q), rt().grid(grid_static),
                                         act, current_index, ob.obs.data(), timing.waypoint_period,
                                         timing.replan_per_waypoint, &r, &p, &h);
  return take_plan(st, h);
}

PathPlan plan_reach_then_path(const ArmSpec& spec, const Quiver& q, const VoxelGrid& grid,
                              const Vec3& target, const ReachParams& rp, const PathParams& pp) {
  const rp_arm arm = to_rp(spec);
  const rp_reach_params r = to_rp(rp);
  const rp_path_params p = to_rp(pp);
  double t[3];
  put3(t, target);
  rp_plan* h = nullptr;
  rp_quiver* dq = rt().quiver(q);
  rp_grid* dg = rt().grid(grid);
  rp_status st;
  {
    Trace t_("rp_plan_reach_then_path");
    st = rp_plan_reach_then_path(rt().ctx(), &arm, dq, dg, t, &r, &p, &h);
  }
  Trace t_("take_plan");
  return take_plan(st, h);
}

PoseChain folded_pose(const ArmSpec& spec) {
  const rp_arm arm = to_rp(spec);
  rp_pose out;
  ok(rp_folded_pose(rt().ctx(), &arm, &out));
  return from_rp(out, nullptr);
}

double mean_polyline_deviation(const std::vector<Vec3>& pts, const std::vector<Vec3>& poly) {
  const std::vector<double> a = flat(pts), b = flat(poly);
  double out = 0.0;
  ok(rp_mean_polyline_deviation(rt().ctx(), a.data(), static_cast<int32_t>(pts.size()), b.data(),
                                static_cast<int32_t>(poly.size()), &out));
  return out;
}

// ---- pipeline.hpp ---------------------------------------------------------------

double effective_dilation(const Scene& scene, const ArmSpec& arm, const ReachParams& rp) {
  const rp_arm a = to_rp(arm);
  const rp_reach_params r = to_rp(rp);
  return rp_effective_dilation(&a, &r, scene.grid.dilation_radius);
}

VoxelGrid build_scene_grid(const Scene& scene, const ArmSpec& arm, const ReachParams& rp,
                           std::ostream* warnings) {
  const rp_arm a = to_rp(arm);
  const rp_reach_params r = to_rp(rp);
  double lo[3], hi[3];
  put3(lo, scene.grid.bounds_min);
  put3(hi, scene.grid.bounds_max);
  const ObstacleBuf ob(scene.obstacles);
  rp_grid* d = nullptr;
  {
    Trace t_("device build");
    ok(rp_build_scene_grid(rt().ctx(), lo, hi, scene.grid.voxel_size, scene.grid.dilation_radius,
                           ob.obs.data(), ob.size(), &a, &r, &d));
  }
  VoxelGrid g;
  rt().adopt(d, g);
  if (warnings) {
    // the reference's reach-sphere warning (pipeline.cpp:22-31)
    const double reach = arm.total_length();
    for (int k = 0; k < 3; ++k) {
      if (scene.root[k] - reach < scene.grid.bounds_min[k] ||
          scene.root[k] + reach > scene.grid.bounds_max[k]) {
        *warnings << "warning: the arm's reachable sphere exceeds the grid bounds; "
                     "poses outside the grid are treated as collision-free\n";
        break;
      }
    }
  }
  return g;
}

// ---- members and small value helpers the replaced TUs defined ---------------------------

std::pair<int, int> Quiver::ring_azim_of(int index) const {
  require(index >= 0 && index < size(), Errc::invalid_parameter, "quiver index out of range");
  const auto it = std::upper_bound(ring_offsets.begin(), ring_offsets.end(), index);
  const int ring = static_cast<int>(it - ring_offsets.begin()) - 1;
  return {ring, index - ring_offsets[ring]};
}

std::vector<int> neighbors(const Quiver& q, int index, double angular_radius) {
  require(index >= 0 && index < q.size(), Errc::invalid_parameter, "quiver index out of range");
  require(angular_radius > 0.0, Errc::invalid_parameter, "angular_radius must be > 0");
  return cone_subset(q, q.vectors[index], std::min(angular_radius, kPi));
}

std::vector<Vec3> ShortcutPath::tip_waypoints(const Vec3& target) const {
  std::vector<Vec3> w = prefix_samples;
  w.insert(w.end(), sublength_samples.begin(), sublength_samples.end());
  if (bridge) w.push_back(target);
  return w;
}

SolveStats& SolveStats::operator+=(const SolveStats& o) {
  seg1_candidates += o.seg1_candidates;
  seg1_limit_pass += o.seg1_limit_pass;
  seg1_reach_pass += o.seg1_reach_pass;
  seg1_survivors += o.seg1_survivors;
  pair_candidates += o.pair_candidates;
  seg2_limit_pass += o.seg2_limit_pass;
  seg2_clear_pass += o.seg2_clear_pass;
  gap_tested += o.gap_tested;
  gap_pass += o.gap_pass;
  joint_pass += o.joint_pass;
  v3_clear_pass += o.v3_clear_pass;
  solutions += o.solutions;
  shortcuts_found += o.shortcuts_found;
  wall_ms += o.wall_ms;
  return *this;
}

double ReachParams::nominal_spacing(const ArmSpec& spec) const {
  const rp_arm a = to_rp(spec);
  const rp_reach_params r = to_rp(*this);
  return rp_nominal_spacing(&a, &r);
}

double ReachParams::resolved_epsilon(const ArmSpec& spec) const {
  const rp_arm a = to_rp(spec);
  const rp_reach_params r = to_rp(*this);
  return rp_resolved_epsilon(&a, &r);
}

double ReachParams::resolved_near_radius(const ArmSpec& spec) const {
  const rp_arm a = to_rp(spec);
  const rp_reach_params r = to_rp(*this);
  return rp_resolved_near_radius(&a, &r);
}

void ReachParams::validate() const {
  const rp_reach_params r = to_rp(*this);
  ok(rp_reach_params_validate(&r));
}

PathParams PathParams::resolved(const ArmSpec& spec, const ReachParams& rp) const {
  const rp_arm a = to_rp(spec);
  const rp_reach_params r = to_rp(rp);
  const rp_path_params p = to_rp(*this);
  rp_path_params o;
  ok(rp_path_params_resolve(&a, &r, &p, &o));
  PathParams out = *this;
  out.epsilon_waypoint = o.epsilon_waypoint;
  out.d_w = o.d_w;
  out.slack = o.slack;
  out.joint1_max_move = o.joint1_max_move;
  out.joint2_max_move = o.joint2_max_move;
  return out;
}

std::vector<const PoseChain*> PathPlan::full_sequence() const {
  std::vector<const PoseChain*> seq;
  for (const PoseChain& p : unfold_prefix) seq.push_back(&p);
  for (std::size_t k = 0; k < poses.size(); ++k)
    if (!(k == 0 && !unfold_prefix.empty())) seq.push_back(&poses[k]);  // seam deduplicated
  return seq;
}

Quiver quiver_from_config(const QuiverConfig& cfg) {
  return generate_quiver(deg2rad(cfg.elev_step_deg), deg2rad(cfg.equator_azim_step_deg),
                         cfg.min_per_ring);
}

ArmSpec arm_in_scene(const ArmSpec& arm, const Scene& scene) {
  ArmSpec placed = arm;
  placed.root = scene.root;
  return placed;
}

ReachParams reach_params_for_scene(ReachParams rp, const Scene& scene, const ArmSpec& arm) {
  rp.approach_axis = scene.approach_axis.normalized();
  rp.approach_half_angle = scene.approach_half_angle;
  rp.epsilon_gap = rp.resolved_epsilon(arm);
  rp.near_target_radius = rp.resolved_near_radius(arm);
  return rp;
}

std::optional<ShortReachHit> short_reach_scan(const HypothesisScan& hyp, const Vec3& target,
                                              const VoxelGrid& grid, const ArmSpec& spec,
                                              const ReachParams& params) {
  // the scan, its bridge / direct walks and the path length on the device
  // (rp_short_reach_scan); inside solve_reach the same scan is fused into
  // k_seg1 / k_seg2 + k_shortcuts
  const rp_arm arm = to_rp(spec);
  const rp_reach_params rp = to_rp(params);
  const std::vector<double> smp = flat(hyp.samples), pre = flat(hyp.prefix_samples);
  double t[3], org[3];
  put3(t, target);
  put3(org, hyp.origin);
  const int n = static_cast<int>(hyp.samples.size());
  require(hyp.sample_clear.size() >= hyp.samples.size(), Errc::invalid_parameter,
          "sample_clear shorter than samples");
  int32_t found = 0;
  rp_shortcut sc{};
  const double len = (target - hyp.origin).norm();
  const int cap = n + std::max(1, static_cast<int>(std::ceil(len / std::max(
                                   1e-12, params.nominal_spacing(spec))))) + 1;
  std::vector<double> sub(3 * static_cast<std::size_t>(cap));
  ok(rp_short_reach_scan(rt().ctx(), rt().grid(grid), &arm, &rp, t, smp.data(),
                         hyp.sample_clear.data(), n, pre.data(),
                         static_cast<int32_t>(hyp.prefix_samples.size()), org, &found, &sc,
                         sub.data(), cap));
  if (!found) return std::nullopt;
  ShortcutPath p;
  p.segment_index = hyp.segment_index;
  p.hit_sample_index = sc.hit_sample_index;
  p.prefix_samples = hyp.prefix_samples;
  for (int k = 0; k < sc.n_sublength; ++k) p.sublength_samples.push_back(get3(&sub[3 * k]));
  if (sc.has_bridge) p.bridge = get3(sc.bridge);
  p.via_origin_direct = sc.via_origin_direct != 0;
  p.basis_pose = hyp.basis_pose;
  p.seg1_index = hyp.seg1_index;
  p.seg2_index = hyp.seg2_index;
  p.path_length = sc.path_length;
  return ShortReachHit{sc.hit_sample_index, std::move(p)};
}

}  // namespace reachplan
