// Execution simulator (src/motion.cpp:8-141, inc/reachplan/motion.hpp):
// discrete-time velocity control of a delivered plan, with the per-tick
// collision re-check of every intermediate configuration on the device.
//
// The tick loop is a serial recurrence (each tick's joint angles come from
// the previous tick's), so it runs on the host with the reference's
// arithmetic (glibc sin/cos/atan2 in the forward kinematics, as the unfold
// interpolation does). The collision test of a tick depends
// only on that tick's configuration, so all of them run as one batched
// kernel afterwards; the first colliding tick is the one the reference
// would have stopped at (pose_collides, src/motion.cpp:49-59), and the
// ticks computed past it have no effect on the result.
#include "rp_path.cuh"
#include "rp_reach.cuh"

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

namespace rp {
namespace {

struct Angles {
  int n = 0;
  double az[4] = {0, 0, 0, 0};
  double el[4] = {0, 0, 0, 0};
  uint8_t deg[4] = {0, 0, 0, 0};
};

/// vectors_to_joint_angles (src/arm_model.cpp:163-176), with the flags.
Angles angles_of(const ArmDev& arm, const DevPose& p) {
  Angles q;
  q.n = p.nseg;
  rpd::M3 frame = arm.base;
  for (int k = 0; k < p.nseg; ++k) {
    const double len = rpd::norm(p.seg[k]);
    require(len > 0.0, RP_E_DEGENERATE_INPUT, "zero-length segment");
    const rpd::FrameStep st = rpd::advance_frame(frame, p.seg[k] / len);
    q.az[k] = st.theta;
    q.el[k] = st.phi;
    q.deg[k] = st.degenerate ? 1 : 0;
    frame = rpd::m_mul(rpd::m_mul(frame, rpd::rot_z(st.theta)), rpd::rot_y(st.phi));
  }
  return q;
}

V3 tracked_point(const DevPose& p) { return p.joints[p.nseg < 3 ? p.nseg : 3]; }

/// waypoint_interval (src/motion.cpp:15-18)
double waypoint_interval(V3 pw, V3 pe, double v_w) {
  require(v_w > 0.0, RP_E_INVALID_PARAMETER, "zero or negative velocity");
  return rpd::norm(pw - pe) / v_w;
}

struct Rates {
  double az[4] = {0, 0, 0, 0};
  double el[4] = {0, 0, 0, 0};
  bool clamped = false;
};

/// joint_velocities (src/motion.cpp:20-41)
Rates joint_velocities(const Angles& qw, const Angles& qc, double t_w, double max_rate) {
  require(t_w > 0.0, RP_E_INVALID_PARAMETER, "zero waypoint interval");
  require(qw.n == qc.n, RP_E_INVALID_PARAMETER, "configurations have different joint counts");
  Rates r;
  for (int j = 0; j < qw.n; ++j) {
    double wa = rpd::wrap_angle(qw.az[j] - qc.az[j]) / t_w;
    double we = (qw.el[j] - qc.el[j]) / t_w;
    if (std::abs(wa) > max_rate) {
      wa = std::copysign(max_rate, wa);
      r.clamped = true;
    }
    if (std::abs(we) > max_rate) {
      we = std::copysign(max_rate, we);
      r.clamped = true;
    }
    r.az[j] = wa;
    r.el[j] = we;
  }
  return r;
}

/// pose_collides (src/motion.cpp:49-59) for every tick: first colliding
/// tick index (atomicMin). Links = chain_links (arm_model.cpp:363-374),
/// n samples each.
__global__ void k_tick_collides(rpd::GridView g, const DevPose* __restrict__ poses, int count,
                                int n, int* first) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count) return;
  const DevPose& p = poses[t];
  bool hit = false;
  for (int j = 0; j < p.nseg && !hit; ++j) {
    if (p.has_elbows && rpd::sqnorm(p.elbows[j] - p.joints[j]) > 0.0) {
      hit = !rpd::walk_clear(g, p.joints[j], p.elbows[j], n) ||
            !rpd::walk_clear(g, p.elbows[j], p.joints[j + 1], n);
    } else {
      hit = !rpd::walk_clear(g, p.joints[j], p.joints[j + 1], n);
    }
  }
  if (hit) atomicMin(first, t);
}

unsigned nblk(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

}  // namespace
}  // namespace rp

using namespace rp;

struct rp_trace {
  std::vector<rp_tick> ticks;
  std::vector<int32_t> overshoot, clamp;
  bool reached = false;
};

namespace {

rp_tick make_tick(double time, const Angles& q, V3 tracked, int active, const Rates* r) {
  rp_tick t;
  std::memset(&t, 0, sizeof(t));
  t.time = time;
  t.n_joints = q.n;
  for (int j = 0; j < q.n; ++j) {
    t.azimuth[j] = q.az[j];
    t.elevation[j] = q.el[j];
    t.degenerate[j] = q.deg[j];
  }
  t.tracked[0] = tracked.x;
  t.tracked[1] = tracked.y;
  t.tracked[2] = tracked.z;
  t.active = active;
  if (r) {
    t.n_rates = q.n;
    t.clamped = r->clamped ? 1 : 0;
    for (int j = 0; j < q.n; ++j) {
      t.azimuth_rate[j] = r->az[j];
      t.elevation_rate[j] = r->el[j];
    }
  }
  return t;
}

}  // namespace

extern "C" rp_status rp_simulate_execution(rp_ctx* ctx, const rp_arm* arm, const rp_plan* plan,
                                           const rp_motion_params* mp, const rp_grid* grid,
                                           rp_trace** out) {
  return guarded([&] {
    // MotionParams::validate (src/motion.cpp:8-13)
    require(mp->v_w > 0.0, RP_E_INVALID_PARAMETER, "v_w must be > 0");
    require(mp->sample_rate > 0.0, RP_E_INVALID_PARAMETER, "sample_rate must be > 0");
    require(mp->max_joint_rate > 0.0, RP_E_INVALID_PARAMETER, "max_joint_rate must be > 0");
    require(mp->arrival_tolerance > 0.0, RP_E_INVALID_PARAMETER, "arrival_tolerance must be > 0");
    const auto sequence = plan->full_sequence();
    require(!sequence.empty(), RP_E_INVALID_PARAMETER, "empty plan");
    const ArmDev ad = make_arm_dev(*arm);
    std::vector<Angles> targets;
    std::vector<V3> points;
    for (const HostPose* p : sequence) {
      const DevPose d = to_dev(*p);
      targets.push_back(angles_of(ad, d));
      points.push_back(tracked_point(d));
    }
    auto tr = std::make_unique<rp_trace>();
    const double dt = 1.0 / mp->sample_rate;
    Angles q = targets.front();
    int active = sequence.size() > 1 ? 1 : 0;
    auto pose_of = [&](const Angles& a) {
      require(a.n == ad.nseg, RP_E_INVALID_PARAMETER, "joint count does not match the arm");
      return from_angles(ad, a.az, a.el);
    };
    DevPose cur = pose_of(q);
    V3 tracked = tracked_point(cur);
    tr->ticks.push_back(make_tick(0.0, q, tracked, active, nullptr));
    std::vector<DevPose> tick_poses;  // ticks 1.. (the ones the reference checks)
    std::vector<double> tick_time;
    if (sequence.size() == 1 || rpd::norm(points.back() - tracked) <= mp->arrival_tolerance) {
      tr->reached = true;
    } else {
      double nominal_total = 0.0;
      for (size_t k = 1; k < points.size(); ++k)
        nominal_total += waypoint_interval(points[k], points[k - 1], mp->v_w);
      const long max_ticks =
          static_cast<long>((nominal_total * 20.0 + 10.0) * mp->sample_rate) + 1000;
      const int npts = static_cast<int>(points.size());
      for (long tick = 1; tick <= max_ticks; ++tick) {
        const double now = tick * dt;
        bool advanced = true;
        while (advanced && active < npts) {
          advanced = false;
          const V3 pw = points[active];
          const double dist = rpd::norm(pw - tracked);
          const bool arrive = dist <= mp->arrival_tolerance;
          bool overshoot = false;
          if (!arrive) {
            const V3 leg = pw - points[active - 1];
            if (rpd::norm(leg) > 1e-12 && rpd::dot(tracked - pw, leg) > 0.0) overshoot = true;
          }
          if (arrive || overshoot) {
            if (overshoot) tr->overshoot.push_back(static_cast<int32_t>(tr->ticks.size()) - 1);
            ++active;
            advanced = true;
          }
        }
        if (active >= npts) {
          tr->reached = true;
          break;
        }
        double t_w = waypoint_interval(points[active], tracked, mp->v_w);
        t_w = std::max(t_w, dt);
        const Rates r = joint_velocities(targets[active], q, t_w, mp->max_joint_rate);
        if (r.clamped) tr->clamp.push_back(static_cast<int32_t>(tr->ticks.size()));
        for (int j = 0; j < q.n; ++j) {
          q.az[j] = rpd::wrap_angle(q.az[j] + r.az[j] * dt);
          q.el[j] += r.el[j] * dt;
        }
        cur = pose_of(q);
        tracked = tracked_point(cur);
        tick_poses.push_back(cur);
        tick_time.push_back(now);
        tr->ticks.push_back(make_tick(now, q, tracked, active, &r));
      }
    }
    if (grid && !tick_poses.empty()) {
      const int count = static_cast<int>(tick_poses.size());
      DevBuf<DevPose> d(count, ctx->stream);
      DevBuf<int> first(1, ctx->stream);
      copy_to_device(ctx, d.p, tick_poses.data(), count * sizeof(DevPose));
      const int big = INT_MAX;
      copy_to_device(ctx, first.p, &big, sizeof(int));
      launch(ctx, "motion", k_tick_collides, dim3(nblk(count, 128)), dim3(128), 0, grid->view(),
             static_cast<const DevPose*>(d.p), count, 8, first.p);
      int h = big;
      copy_to_host(ctx, &h, first.p, sizeof(int));
      if (h != big)
        fail(RP_E_EXECUTION_COLLISION,
             "arm collided during execution at t=" + std::to_string(tick_time[h]));
    }
    require(tr->reached, RP_E_TIMEOUT, "tick budget exceeded before the final waypoint");
    *out = tr.release();
  });
}

extern "C" rp_status rp_trace_info(const rp_trace* t, int64_t* n_ticks, int64_t* n_overshoot,
                                   int64_t* n_clamp, int32_t* reached_goal) {
  return guarded([&] {
    *n_ticks = static_cast<int64_t>(t->ticks.size());
    *n_overshoot = static_cast<int64_t>(t->overshoot.size());
    *n_clamp = static_cast<int64_t>(t->clamp.size());
    *reached_goal = t->reached ? 1 : 0;
  });
}

extern "C" rp_status rp_trace_ticks(const rp_trace* t, int64_t first, int64_t count, rp_tick* out) {
  return guarded([&] {
    require(first >= 0 && count >= 0 && first + count <= static_cast<int64_t>(t->ticks.size()),
            RP_E_INVALID_PARAMETER, "tick range out of bounds");
    if (count) std::memcpy(out, t->ticks.data() + first, count * sizeof(rp_tick));
  });
}

extern "C" rp_status rp_trace_events(const rp_trace* t, int32_t* overshoot, int32_t* clamp) {
  return guarded([&] {
    if (overshoot && !t->overshoot.empty())
      std::memcpy(overshoot, t->overshoot.data(), t->overshoot.size() * sizeof(int32_t));
    if (clamp && !t->clamp.empty())
      std::memcpy(clamp, t->clamp.data(), t->clamp.size() * sizeof(int32_t));
  });
}

extern "C" void rp_motion_params_init(rp_motion_params* mp) {
  std::memset(mp, 0, sizeof(*mp));
  mp->v_w = 0.05;
  mp->sample_rate = 100.0;
  mp->max_joint_rate = 30.0 * (3.14159265358979323846 / 180.0);  // deg2rad(30)
  mp->arrival_tolerance = 0.01;
}

extern "C" rp_status rp_trace_destroy(rp_trace* t) {
  return guarded([&] { delete t; });
}
