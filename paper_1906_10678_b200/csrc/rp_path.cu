// Path-planner device kernels (src/path_planner.cpp, src/arm_model.cpp):
// waypoint IK search, pose validity batches, unfold interpolation,
// refinement, polyline-deviation scoring.
#include "rp_path.cuh"
#include "rp_planner.hpp"
#include "rp_refine.cuh"
#include "rp_rings.cuh"

#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>

namespace rp {

using rpd::V3;

namespace {
constexpr unsigned FULL = 0xffffffffu;
constexpr double kPi = 3.14159265358979323846;

inline unsigned nblk(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }
}  // namespace

// ---------------------------------------------------------------------------
// Pose helpers (host + device so materialisation replays the same arithmetic).

/// link_clear_scaled (src/path_planner.cpp:41-46)
__device__ inline bool link_clear_scaled(const rpd::GridView& g, V3 from, V3 to, double spacing) {
  const double len = rpd::norm(to - from);
  if (len == 0.0) return true;
  return rpd::walk_clear(g, from, to, rpd::scaled_sample_count(len, spacing));
}

/// pose_clear (src/path_planner.cpp:50-61)
__device__ inline bool pose_clear(const rpd::GridView& g, const DevPose& p, int n, double spacing) {
  for (int j = 0; j < p.nseg; ++j) {
    V3 from = p.joints[j];
    if (p.has_elbows) {
      if (!link_clear_scaled(g, p.joints[j], p.elbows[j], spacing)) return false;
      from = p.elbows[j];
    }
    if (!rpd::walk_clear(g, from, p.joints[j + 1], n)) return false;
  }
  return true;
}

/// pose_valid (src/path_planner.cpp:63-67)
__device__ inline bool pose_valid(const rpd::GridView& g, const ArmDev& arm, const DevPose& p, int n,
                                  double spacing) {
  return pose_clear(g, p, n, spacing) && pose_limits_ok(arm, p) &&
         pose_self_free(p, 2.0 * arm.arm_radius);
}

__host__ __device__ inline rpd::M3 angle_axis(double angle, V3 axis) {
  // Eigen AngleAxis::toRotationMatrix
  rpd::M3 r;
  const V3 sa = sin(angle) * axis;
  const double c = cos(angle);
  const V3 c1 = (1.0 - c) * axis;
  double tmp = c1.x * axis.y;
  r.a[0][1] = tmp - sa.z;
  r.a[1][0] = tmp + sa.z;
  tmp = c1.x * axis.z;
  r.a[0][2] = tmp + sa.y;
  r.a[2][0] = tmp - sa.y;
  tmp = c1.y * axis.z;
  r.a[1][2] = tmp - sa.x;
  r.a[2][1] = tmp + sa.x;
  r.a[0][0] = c1.x * axis.x + c;
  r.a[1][1] = c1.y * axis.y + c;
  r.a[2][2] = c1.z * axis.z + c;
  return r;
}

__host__ __device__ inline V3 m_vec(const rpd::M3& m, V3 v) {
  const double in[3] = {v.x, v.y, v.z};
  double out[3];
  for (int r = 0; r < 3; ++r) {
    double s = m.a[r][0] * in[0];
    s = s + m.a[r][1] * in[1];
    s = s + m.a[r][2] * in[2];
    out[r] = s;
  }
  return V3{out[0], out[1], out[2]};
}

__host__ __device__ inline rpd::M3 m_transpose(const rpd::M3& m) {
  rpd::M3 t;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) t.a[r][c] = m.a[c][r];
  return t;
}

/// folded_pose (src/path_planner.cpp:711-727)
__host__ __device__ inline DevPose folded_pose(const ArmDev& arm, V3 n, double flex) {
  V3 seed{1, 0, 0};
  if (fabs(rpd::dot(n, seed)) > fabs(rpd::dot(n, V3{0, 0, 1}))) seed = V3{0, 0, 1};
  if (fabs(rpd::dot(n, seed)) > fabs(rpd::dot(n, V3{0, 1, 0}))) seed = V3{0, 1, 0};
  V3 dir = rpd::normalized(seed - rpd::dot(seed, n) * n);
  DevPose p{};
  p.nseg = arm.nseg;
  p.no_qidx = 1;  // chain_from_segments(spec, segs): no indices (path_planner.cpp:726)
  double sign = 1.0;
  for (int j = 0; j < arm.nseg; ++j) {
    p.seg[j] = arm.L[j] * dir;
    p.qidx[j] = -1;
    dir = m_vec(angle_axis(sign * flex, n), dir);
    sign = -sign;
  }
  build_chain(arm, p);
  return p;
}

__host__ __device__ inline V3 perpendicular_of(V3 dir) {
  const V3 seed = fabs(dir.z) < 0.9 ? V3{0, 0, 1} : V3{1, 0, 0};
  return rpd::normalized(rpd::cross(dir, seed));
}

/// pose_plane_normal (src/path_planner.cpp:450-454)
__host__ __device__ inline V3 pose_plane_normal(const DevPose& p) {
  const V3 n = rpd::cross(p.seg[0], p.seg[1]);
  if (rpd::norm(n) <= 1e-12) return perpendicular_of(rpd::normalized(p.seg[0]));
  return rpd::normalized(n);
}

// ---------------------------------------------------------------------------
// waypoint_ik (src/path_planner.cpp:167-291)

__device__ inline V3 wq(const WikDev& w, int i) { return V3{w.qx[i], w.qy[i], w.qz[i]}; }

/// One (i, j) candidate through every test of waypoint_ik, in order.
__device__ __noinline__ bool wik_eval(const WikDev& w, const CiData& c, int j, DevPose* out, double* metric_out,
                         int* opt_out) {
  const ArmDev& arm = w.arm;
  const V3 qj = wq(w, j);
  rpd::FrameStep st2{};
  bool have_st2 = false;
  if (w.cond2) {
    st2 = rpd::advance_frame(c.frame1, qj);
    have_st2 = true;
    if (!rpd::joint_angle_within(st2.theta, st2.phi, st2.degenerate, arm.lim[1])) return false;
  }
  V3 link2 = c.p1, elbow2{0, 0, 0};
  const bool e2 = arm.off[1] > 0.0;
  if (e2) {
    elbow2 = c.p1 + arm.off[1] * rpd::m_col(st2.after_azimuth, 0);
    link2 = elbow2;
  }
  const V3 p2 = link2 + arm.L[1] * qj;
  const double move2 = rpd::norm(p2 - w.prev_j2);
  if (move2 > w.j2max) return false;
  const V3 v3 = w.wp - p2;
  const double v3_len = rpd::norm(v3);
  if (fabs(v3_len - arm.L[2]) > w.eps || v3_len < 1e-12) return false;
  const V3 v3_hat = v3 / v3_len;
  if (w.cond3) {
    if (!have_st2) st2 = rpd::advance_frame(c.frame1, qj);
    const rpd::FrameStep st3 = rpd::advance_frame(st2.frame, v3_hat);
    if (!rpd::joint_angle_within(st3.theta, st3.phi, st3.degenerate, arm.lim[2])) return false;
  }
  double metric = c.move1 + move2;
  if (w.has_bias) metric += rpd::norm(c.p1 - w.bias_j1) + rpd::norm(p2 - w.bias_j2);
  if (!c.ok) return false;  // segment 1 blocked for every j (lazy walk1 + break)
  if (e2 && !link_clear_scaled(w.g, c.p1, elbow2, w.spacing)) return false;
  if (!rpd::walk_clear(w.g, link2, p2, w.n)) return false;
  const V3 s3 = v3_hat * arm.L[2];
  const V3 p3 = p2 + s3;
  if (!rpd::walk_clear(w.g, p2, p3, w.n)) return false;
  DevPose ch{};
  ch.nseg = 3;
  ch.seg[0] = arm.L[0] * wq(w, c.i);
  ch.seg[1] = arm.L[1] * qj;
  ch.seg[2] = s3;
  ch.qidx[0] = c.i;
  ch.qidx[1] = j;
  ch.qidx[2] = -1;
  ch.qidx[3] = -1;
  build_chain(arm, ch);
  ch.n_wp_links = 3;
  ch.wp_from[0] = c.link1; ch.wp_to[0] = c.p1;
  ch.wp_from[1] = link2;   ch.wp_to[1] = p2;
  ch.wp_from[2] = p2;      ch.wp_to[2] = p3;
  ch.n_wp[0] = ch.n_wp[1] = ch.n_wp[2] = w.n;
  int opt = -1;
  const double min_sep = 2.0 * arm.arm_radius;
  if (w.four) {
    // append_trail (src/path_planner.cpp:127-150)
    bool done = false;
    for (int o = 0; o <= w.n_opts && !done; ++o) {
      const V3 dir = o < w.n_opts ? w.opt_dir[o] : rpd::normalized(ch.seg[2]);
      DevPose cand = ch;
      cand.nseg = 4;
      cand.seg[3] = w.L4 * dir;
      cand.qidx[3] = -1;
      build_chain(arm, cand);
      if (!pose_limits_ok(arm, cand)) continue;
      if (!rpd::walk_clear(w.g, cand.joints[3], cand.joints[4], w.n)) continue;
      if (!pose_self_free(cand, min_sep)) continue;
      cand.n_wp_links = 4;
      cand.wp_from[3] = cand.joints[3];
      cand.wp_to[3] = cand.joints[4];
      cand.n_wp[3] = w.n;
      ch = cand;
      opt = o;
      done = true;
    }
    if (!done) return false;
  } else if (!pose_self_free(ch, min_sep)) {
    return false;
  }
  if (!pose_limits_ok(arm, ch)) return false;
  if (!(rpd::norm(ch.joints[1] - w.prev_j1) <= w.sm1 &&
        rpd::norm(ch.joints[2] - w.prev_j2) <= w.sm2))
    return false;
  *metric_out = metric;
  *opt_out = opt;
  if (out) *out = ch;
  return true;
}

/// wik_eval's verdict for a coaxial arm without joint limits, on joint
/// arrays only (no DevPose construction or copies): the same tests in the
/// same order with the same arithmetic (chain joints are the cumulative sums
/// chain_from_segments forms, src/arm_model.cpp:141-143).
__device__ bool wik_eval_fast(const WikDev& w, const CiData& c, int j, double* metric_out,
                              int* opt_out) {
  const ArmDev& arm = w.arm;
  const V3 qj = wq(w, j);
  const V3 p2 = c.p1 + arm.L[1] * qj;
  const double move2 = rpd::norm(p2 - w.prev_j2);
  if (move2 > w.j2max) return false;
  const V3 v3 = w.wp - p2;
  const double v3_len = rpd::norm(v3);
  if (fabs(v3_len - arm.L[2]) > w.eps || v3_len < 1e-12) return false;
  const V3 v3_hat = v3 / v3_len;
  double metric = c.move1 + move2;
  if (w.has_bias) metric += rpd::norm(c.p1 - w.bias_j1) + rpd::norm(p2 - w.bias_j2);
  if (!c.ok) return false;
  if (!rpd::walk_clear(w.g, c.p1, p2, w.n)) return false;  // link2 = p1 (coaxial)
  const V3 s3 = v3_hat * arm.L[2];
  const V3 p3 = p2 + s3;
  if (!rpd::walk_clear(w.g, p2, p3, w.n)) return false;
  V3 J[5];
  J[0] = arm.root;
  J[1] = J[0] + arm.L[0] * wq(w, c.i);
  J[2] = J[1] + arm.L[1] * qj;
  J[3] = J[2] + s3;
  const double min_sep = 2.0 * arm.arm_radius;
  int opt = -1;
  if (w.four) {
    bool done = false;
    for (int o = 0; o <= w.n_opts && !done; ++o) {
      const V3 dir = o < w.n_opts ? w.opt_dir[o] : rpd::normalized(s3);
      J[4] = J[3] + w.L4 * dir;
      if (!rpd::walk_clear(w.g, J[3], J[4], w.n)) continue;
      if (!rpd::self_collision_free(J, 4, min_sep)) continue;
      opt = o;
      done = true;
    }
      if (!done) return false;
  } else if (!rpd::self_collision_free(J, 3, min_sep)) {
    return false;
  }
  if (!(rpd::norm(J[1] - w.prev_j1) <= w.sm1 && rpd::norm(J[2] - w.prev_j2) <= w.sm2)) return false;
  *metric_out = metric;
  *opt_out = opt;
  return true;
}

/// wik_eval_fast's exact prefix (segment-2 move bound, gap band, metric):
/// false when the pair cannot qualify. Same arithmetic, same order.
__device__ __forceinline__ bool wik_pre_fast(const WikDev& w, const CiFast& c, int j, double* metric) {
  const ArmDev& arm = w.arm;
  const V3 qj = wq(w, j);
  const V3 p2 = c.p1 + arm.L[1] * qj;
  const double move2 = rpd::norm(p2 - w.prev_j2);
  if (move2 > w.j2max) return false;
  const V3 v3 = w.wp - p2;
  const double v3_len = rpd::norm(v3);
  if (fabs(v3_len - arm.L[2]) > w.eps || v3_len < 1e-12) return false;
  double m = c.move1 + move2;
  if (w.has_bias) m += rpd::norm(c.p1 - w.bias_j1) + rpd::norm(p2 - w.bias_j2);
  *metric = m;
  return c.ok != 0;
}

/// The remaining tests of wik_eval_fast for a pair that passed wik_pre_fast,
/// spread over one warp in two data-parallel steps (every lane runs the
/// same code on its own operands, so nothing serialises on divergence):
/// walks — lane 0 segment 2, lane 1 segment 3, lanes 2.. the trail segment
/// of each option; link distances — lane 3*o + p the p-th non-adjacent link
/// pair of option o's chain. Every test is a pure function of the pose, so
/// the verdict and the first qualifying trail option equal the sequential
/// evaluation's. All lanes return the same result.
__device__ bool wik_full_warp(const WikDev& w, const CiFast& c, int j, int lane, int* opt_out) {
  const ArmDev& arm = w.arm;
  const V3 qj = wq(w, j);
  const V3 p2 = c.p1 + arm.L[1] * qj;
  const V3 v3 = w.wp - p2;
  const double v3_len = rpd::norm(v3);
  const V3 v3_hat = v3 / v3_len;
  const V3 s3 = v3_hat * arm.L[2];
  const V3 p3 = p2 + s3;
  V3 J[4];
  J[0] = arm.root;
  J[1] = J[0] + arm.L[0] * wq(w, c.i);
  J[2] = J[1] + arm.L[1] * qj;
  J[3] = J[2] + s3;
  if (!(rpd::norm(J[1] - w.prev_j1) <= w.sm1 && rpd::norm(J[2] - w.prev_j2) <= w.sm2))
    return false;
  const double min_sep = 2.0 * arm.arm_radius;
  const int nopt = w.four ? w.n_opts + 1 : 0;
  // trail endpoint of option o (lane-selected below)
  auto tip = [&](int o) {
    const V3 dir = o < w.n_opts ? w.opt_dir[o] : rpd::normalized(s3);
    return J[3] + w.L4 * dir;
  };
  // step 1: walks
  bool ok = true;
  if (lane < 2 + nopt) {
    V3 from = c.p1, to = p2;
    if (lane == 1) {
      from = p2;
      to = p3;
    } else if (lane >= 2) {
      from = J[3];
      to = tip(lane - 2);
    }
    ok = rpd::walk_first_blocked_fast_seg(w.g, from, to, w.n) == 0;
  }
  const unsigned walk_fail = __ballot_sync(0xffffffffu, !ok);
  if (walk_fail & 3u) return false;
  // step 2: non-adjacent link distances
  ok = true;
  const int npairs = w.four ? 3 * nopt : 1;
  if (lane < npairs) {
    V3 a0, a1, b0, b1;
    double ha = 0.5 * arm.L[0], hb = 0.5 * arm.L[2];
    if (!w.four) {
      a0 = J[0]; a1 = J[1]; b0 = J[2]; b1 = J[3];
    } else {
      const int o = lane / 3, pr = lane % 3;
      const V3 j4 = tip(o);
      // pairs of a 4-link chain: (0,2), (0,3), (1,3)
      a0 = pr == 2 ? J[1] : J[0];
      a1 = pr == 2 ? J[2] : J[1];
      b0 = pr == 0 ? J[2] : J[3];
      b1 = pr == 0 ? J[3] : j4;
      ha = 0.5 * (pr == 2 ? arm.L[1] : arm.L[0]);
      hb = 0.5 * (pr == 0 ? arm.L[2] : w.L4);
    }
    // unit directions: |link| = L up to rounding, absorbed by the widening
    ok = rpd::links_clear_screen(a0, a1, b0, b1, ha * (1.0 + 1e-9), hb * (1.0 + 1e-9), min_sep) ||
         !(rpd::seg_seg_distance(a0, a1, b0, b1) < min_sep);
  }
  const unsigned dist_fail = __ballot_sync(0xffffffffu, !ok);
  if (!w.four) return !(dist_fail & 1u);
  for (int o = 0; o < nopt; ++o) {
    if (!((walk_fail >> (2 + o)) & 1u) && !((dist_fail >> (3 * o)) & 7u)) {
      *opt_out = o;
      return true;
    }
  }
  return false;
}

/// wik_full_warp on a half warp (16 lanes: at most 5 walks and 9 link
/// distances), so a warp evaluates two candidates at once. `sub` = lane in
/// the half, `half` = 0/1; both halves run the same code in lockstep, and an
/// idle half passes valid = false. Same verdicts as wik_full_warp.
__device__ bool wik_full_half(const WikDev& w, const CiFast& c, int j, bool valid, int sub,
                              int half, int* opt_out) {
  const ArmDev& arm = w.arm;
  const bool pr = w.prof && blockIdx.x == 0 && threadIdx.x == 0;
  long long t0 = pr ? clock64() : 0;
  bool alive = valid;
  const V3 qj = valid ? wq(w, j) : V3{0, 0, 1};
  const V3 p1 = valid ? c.p1 : arm.root;
  const V3 p2 = p1 + arm.L[1] * qj;
  V3 v3 = w.wp - p2;
  double v3_len = rpd::norm(v3);
  if (!(v3_len > 0.0)) {  // only for idle halves (screened pairs have |v3| >= 1e-12)
    v3 = V3{0, 0, 1};
    v3_len = 1.0;
  }
  const V3 v3_hat = v3 / v3_len;
  const V3 s3 = v3_hat * arm.L[2];
  const V3 p3 = p2 + s3;
  V3 J[4];
  J[0] = arm.root;
  // root + L1 * q_i: the filter's p1 (wik_filter_fast), same operations
  J[1] = valid ? c.p1 : J[0] + arm.L[0] * V3{0, 0, 1};
  J[2] = J[1] + arm.L[1] * qj;
  J[3] = J[2] + s3;
  alive = alive && rpd::norm(J[1] - w.prev_j1) <= w.sm1 && rpd::norm(J[2] - w.prev_j2) <= w.sm2;
  const double min_sep = 2.0 * arm.arm_radius;
  const int nopt = w.four ? w.n_opts + 1 : 0;
  auto tip = [&](int o) {
    const V3 dir = o < w.n_opts ? w.opt_dir[o] : rpd::normalized(s3);
    return J[3] + w.L4 * dir;
  };
  bool ok = true;
  long long t1 = pr ? clock64() : 0;
  if (alive && sub < 2 + nopt) {
    V3 from = p1, to = p2;
    if (sub == 1) {
      from = p2;
      to = p3;
    } else if (sub >= 2) {
      from = J[3];
      to = tip(sub - 2);
    }
    ok = rpd::walk_first_blocked_fast_seg(w.g, from, to, w.n) == 0;
  }
  const unsigned walk_fail = (__ballot_sync(0xffffffffu, !ok) >> (16 * half)) & 0xFFFFu;
  long long t2 = pr ? clock64() : 0;
  alive = alive && !(walk_fail & 3u);
  ok = true;
  const int npairs = w.four ? 3 * nopt : 1;
  if (alive && sub < npairs) {
    V3 a0, a1, b0, b1;
    double ha = 0.5 * arm.L[0], hb = 0.5 * arm.L[2];
    if (!w.four) {
      a0 = J[0]; a1 = J[1]; b0 = J[2]; b1 = J[3];
    } else {
      const int o = sub / 3, pr = sub % 3;
      const V3 j4 = tip(o);
      a0 = pr == 2 ? J[1] : J[0];
      a1 = pr == 2 ? J[2] : J[1];
      b0 = pr == 0 ? J[2] : J[3];
      b1 = pr == 0 ? J[3] : j4;
      ha = 0.5 * (pr == 2 ? arm.L[1] : arm.L[0]);
      hb = 0.5 * (pr == 0 ? arm.L[2] : w.L4);
    }
    ok = rpd::links_clear_screen(a0, a1, b0, b1, ha * (1.0 + 1e-9), hb * (1.0 + 1e-9), min_sep) ||
         !(rpd::seg_seg_distance(a0, a1, b0, b1) < min_sep);
  }
  const unsigned dist_fail = (__ballot_sync(0xffffffffu, !ok) >> (16 * half)) & 0xFFFFu;
  if (pr) {
    const long long t3 = clock64();
    atomicAdd(reinterpret_cast<unsigned long long*>(w.prof + 16), t1 - t0);
    atomicAdd(reinterpret_cast<unsigned long long*>(w.prof + 17), t2 - t1);
    atomicAdd(reinterpret_cast<unsigned long long*>(w.prof + 18), t3 - t2);
  }
  if (!alive) return false;
  if (!w.four) return !(dist_fail & 1u);
  for (int o = 0; o < nopt; ++o) {
    if (!((walk_fail >> (2 + o)) & 1u) && !((dist_fail >> (3 * o)) & 7u)) {
      *opt_out = o;
      return true;
    }
  }
  return false;
}

__device__ __forceinline__ bool wik_test(const WikDev& w, const CiData& c, int j, double* m,
                                         int* opt) {
  if (!w.arm.any_limit && !w.arm.has_offsets) return wik_eval_fast(w, c, j, m, opt);
  return wik_eval(w, c, j, nullptr, m, opt);
}

/// The pose wik_eval accepted for (i, j, trail option): the same arithmetic,
/// without re-running its tests.
__device__ __noinline__ DevPose wik_pose(const WikDev& w, const CiData& c, int j, int opt) {
  const ArmDev& arm = w.arm;
  const V3 qj = wq(w, j);
  V3 link2 = c.p1;
  if (arm.off[1] > 0.0) {
    const rpd::FrameStep st2 = rpd::advance_frame(c.frame1, qj);
    link2 = c.p1 + arm.off[1] * rpd::m_col(st2.after_azimuth, 0);
  }
  const V3 p2 = link2 + arm.L[1] * qj;
  const V3 v3 = w.wp - p2;
  const double v3_len = rpd::norm(v3);
  const V3 v3_hat = v3 / v3_len;
  const V3 s3 = v3_hat * arm.L[2];
  const V3 p3 = p2 + s3;
  DevPose ch{};
  ch.nseg = 3;
  ch.seg[0] = arm.L[0] * wq(w, c.i);
  ch.seg[1] = arm.L[1] * qj;
  ch.seg[2] = s3;
  ch.qidx[0] = c.i;
  ch.qidx[1] = j;
  ch.qidx[2] = -1;
  ch.qidx[3] = -1;
  build_chain(arm, ch);
  ch.n_wp_links = 3;
  ch.wp_from[0] = c.link1; ch.wp_to[0] = c.p1;
  ch.wp_from[1] = link2;   ch.wp_to[1] = p2;
  ch.wp_from[2] = p2;      ch.wp_to[2] = p3;
  ch.n_wp[0] = ch.n_wp[1] = ch.n_wp[2] = w.n;
  if (w.four && opt >= 0) {
    const V3 dir = opt < w.n_opts ? w.opt_dir[opt] : rpd::normalized(ch.seg[2]);
    ch.nseg = 4;
    ch.seg[3] = w.L4 * dir;
    build_chain(arm, ch);
    ch.n_wp_links = 4;
    ch.wp_from[3] = ch.joints[3];
    ch.wp_to[3] = ch.joints[4];
    ch.n_wp[3] = w.n;
  }
  return ch;
}

/// Candidate filters over the quiver: segment-1 directions inside the
/// reference's cone that pass the joint-1 limit and the move1 bound, and
/// segment-2 directions inside its cone (all directions for offset arms).
__device__ void wik_filter_one(const WikDev& w, double cone1, double cone2, V3 u1, V3 u2, int i,
                               CiData* ci_by_index, bool* pi_out, bool* pj_out) {
  bool pi = false, pj = false;
  {
    const V3 q = wq(w, i);
    const ArmDev& arm = w.arm;
    bool in1 = true;
    if (w.filter_j) in1 = rpd::dot(q, u1) >= cone1;
    if (in1) {
      rpd::FrameStep st{};
      if (arm.any_limit || arm.has_offsets) st = rpd::advance_frame(arm.base, q);
      bool ok = !arm.lim_active[0] || rpd::joint_angle_within(st.theta, st.phi, st.degenerate, arm.lim[0]);
      if (ok) {
        V3 link = arm.root;
        const bool elb = arm.off[0] > 0.0;
        if (elb) link = arm.root + arm.off[0] * rpd::m_col(st.after_azimuth, 0);
        const V3 p1 = link + arm.L[0] * q;
        const double move1 = rpd::norm(p1 - w.prev_j1);
        pi = !(move1 > w.j1max);
        if (pi) {
          // segment-1 data and its (lazy in the reference) walk, once per i
          CiData c;
          c.i = i;
          c.frame1 = st.frame;
          c.link1 = link;
          c.p1 = p1;
          c.move1 = move1;
          c.ok = (!elb || link_clear_scaled(w.g, arm.root, link, w.spacing)) &&
                 rpd::walk_clear(w.g, link, p1, w.n);
          ci_by_index[i] = c;
        }
      }
    }
    pj = !w.filter_j || rpd::dot(q, u2) >= cone2;
  }
  *pi_out = pi;
  *pj_out = pj;
}

/// wik_filter_one for a coaxial arm without limits: the same tests and
/// arithmetic, writing the compact CiFast record (no frame).
__device__ __forceinline__ void wik_filter_fast(const WikDev& w, double cone1, double cone2, V3 u1,
                                                V3 u2, int i, CiFast* out, bool* pi_out,
                                                bool* pj_out, V3 q, int walk1_ok,
                                                long long* prof = nullptr) {
  bool pi = false;
  if (!w.filter_j || rpd::dot(q, u1) >= cone1) {
    const V3 p1 = w.arm.root + w.arm.L[0] * q;
    const double move1 = rpd::norm(p1 - w.prev_j1);
    pi = !(move1 > w.j1max);
    if (pi) {
      const long long t1 = prof ? clock64() : 0;
      CiFast c;
      c.i = i;
      c.move1 = move1;
      c.p1 = p1;
      // segment 1 from the root is the same walk for every waypoint and
      // attempt: its verdict comes from the planner's precomputed bitmap
      c.ok = walk1_ok;
      (void)t1;
      out[i] = c;
    }
  }
  *pi_out = pi;
  *pj_out = !w.filter_j || rpd::dot(q, u2) >= cone2;
}

/// Segment-1 clearance of every quiver direction from the root (coaxial
/// arms): walk_clear(root, root + L1 q_i) as a bitmap, the verdict
/// wik_filter_fast reads instead of walking once per attempt. Cached on the
/// grid (Planner::walk1_device) for every planner of the same arm root, L1,
/// n and quiver.
__global__ void k_walk1_bits(rpd::GridView g, ArmDev arm, const double* __restrict__ qx,
                             const double* __restrict__ qy, const double* __restrict__ qz, int Q,
                             int n, uint32_t* __restrict__ bits) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  bool clear = false;
  if (i < Q) {
    const V3 p1 = arm.root + arm.L[0] * V3{qx[i], qy[i], qz[i]};
    clear = rpd::walk_first_blocked_fast(g, arm.root, p1, n) == 0;
  }
  const unsigned m = __ballot_sync(FULL, clear);
  if ((threadIdx.x & 31) == 0 && i < Q + 31) bits[i >> 5] = m;
}

__global__ void k_wik_filter(WikDev w, double cone1, double cone2, V3 u1, V3 u2,
                             uint32_t* ibits, uint32_t* jbits, CiData* ci_by_index) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  bool pi = false, pj = false;
  if (i < w.Q) wik_filter_one(w, cone1, cone2, u1, u2, i, ci_by_index, &pi, &pj);
  const unsigned mi = __ballot_sync(FULL, pi), mj = __ballot_sync(FULL, pj);
  if ((threadIdx.x & 31) == 0 && (i >> 5) < (w.Q + 31) / 32) {
    ibits[i >> 5] = mi;
    jbits[i >> 5] = mj;
  }
}

/// Ordered compaction of both candidate lists + segment-1 data (one block).
__global__ void __launch_bounds__(1024) k_wik_compact(WikDev w, WikScratch s) {
  typedef cub::BlockScan<int, 1024> Scan;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int carry;
  const int nwords = (w.Q + 31) / 32;
  for (int which = 0; which < 2; ++which) {
    const uint32_t* bits = which == 0 ? s.ibits : s.jbits;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int w0 = 0; w0 < nwords; w0 += 1024) {
      const int wd = w0 + threadIdx.x;
      const uint32_t word = wd < nwords ? bits[wd] : 0u;
      int off = 0, total = 0;
      Scan(tmp).ExclusiveSum(__popc(word), off, total);
      off += carry;
      uint32_t x = word;
      while (x) {
        const int b = __ffs(x) - 1;
        x &= x - 1;
        const int idx = wd * 32 + b;
        if (which == 0) {
          s.ci[off] = s.ci_by_index[idx];
        } else {
          s.cj[off] = idx;
        }
        ++off;
      }
      __syncthreads();
      if (threadIdx.x == 0) carry += total;
      __syncthreads();
    }
    if (threadIdx.x == 0) s.counts[which] = carry;
    __syncthreads();
  }
}

__device__ inline bool wik_better(double m, long long o, double bm, long long bo) {
  return m < bm || (m == bm && o < bo);
}

/// All (i, j) candidates; argmin of (metric, canonical order) = the first
/// strict minimum of the reference's sequential scan. The last block to
/// finish reduces the per-block winners and materialises the pose.
__global__ void __launch_bounds__(256) k_wik_pairs(WikDev w, WikScratch s) {
  const int nci = s.counts[0], ncj = s.counts[1];
  const long long total = static_cast<long long>(nci) * ncj;
  double bm = 1e308;
  long long bo = LLONG_MAX;
  int bopt = -1;
  for (long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
       t += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int a = static_cast<int>(t / ncj);
    const CiData& c = s.ci[a];
    if (!c.ok) continue;
    double m;
    int opt;
    if (wik_test(w, c, s.cj[t - static_cast<long long>(a) * ncj], &m, &opt) &&
        wik_better(m, t, bm, bo)) {
      bm = m;
      bo = t;
      bopt = opt;
    }
  }
  for (int off = 16; off > 0; off >>= 1) {
    const double om = __shfl_down_sync(FULL, bm, off);
    const long long oo = __shfl_down_sync(FULL, bo, off);
    const int op = __shfl_down_sync(FULL, bopt, off);
    if (wik_better(om, oo, bm, bo)) {
      bm = om;
      bo = oo;
      bopt = op;
    }
  }
  __shared__ WikBest wb[8];
  __shared__ bool last;
  if ((threadIdx.x & 31) == 0) wb[threadIdx.x >> 5] = WikBest{bm, bo, bopt};
  __syncthreads();
  if (threadIdx.x == 0) {
    WikBest b = wb[0];
    for (int k = 1; k < static_cast<int>(blockDim.x >> 5); ++k)
      if (wik_better(wb[k].metric, wb[k].ord, b.metric, b.ord)) b = wb[k];
    s.block_best[blockIdx.x] = b;
    __threadfence();
    const unsigned ticket = atomicAdd(s.done, 1u);
    last = ticket == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // last block: reduce the per-block winners with the whole block
  WikBest b{1e308, LLONG_MAX, -1};
  for (int k = threadIdx.x; k < static_cast<int>(gridDim.x); k += blockDim.x) {
    WikBest r;
    r.metric = __ldcg(&s.block_best[k].metric);
    r.ord = __ldcg(&s.block_best[k].ord);
    r.opt = __ldcg(&s.block_best[k].opt);
    if (wik_better(r.metric, r.ord, b.metric, b.ord)) b = r;
  }
  for (int off = 16; off > 0; off >>= 1) {
    const double om = __shfl_down_sync(FULL, b.metric, off);
    const long long oo = __shfl_down_sync(FULL, b.ord, off);
    const int op = __shfl_down_sync(FULL, b.opt, off);
    if (wik_better(om, oo, b.metric, b.ord)) b = WikBest{om, oo, op};
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) wb[threadIdx.x >> 5] = b;
  __syncthreads();
  if (threadIdx.x != 0) return;
  b = wb[0];
  for (int k = 1; k < static_cast<int>(blockDim.x >> 5); ++k)
    if (wik_better(wb[k].metric, wb[k].ord, b.metric, b.ord)) b = wb[k];
  WikResult res{};
  res.found = 0;
  if (b.ord != LLONG_MAX) {
    const int a = static_cast<int>(b.ord / ncj);
    const int j = s.cj[b.ord - static_cast<long long>(a) * ncj];
    double m;
    int opt;
    if (wik_eval(w, s.ci[a], j, &res.pose, &m, &opt)) {
      res.found = 1;
      res.i = s.ci[a].i;
      res.j = j;
      res.opt = opt;
      res.metric = m;
    }
  }
  *s.result = res;
  *s.done = 0;
}

// ---------------------------------------------------------------------------
// Persistent backward pass: one cooperative launch runs the whole sequential
// pass (src/path_planner.cpp:322-400). Per (waypoint, target, factor)
// attempt: filter over the quiver (all blocks) | barrier | every block
// compacts the candidate lists into its shared memory and evaluates its share
// of the (i, j) pairs | barrier | block 0 reduces, materialises the pose and
// publishes the decision | barrier. Blocks are co-resident (cooperative
// launch), so the barrier is a plain global-memory one; its gpu-scope fence
// also invalidates L1, so data written by other SMs is read fresh.

__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* gen = bar + 1;
    const unsigned g0 = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == nblocks - 1) {
      bar[0] = 0;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*gen == g0) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ bool pose_smooth(const DevPose& prev, const DevPose& c, double b1,
                                            double b2) {
  return rpd::norm(c.joints[1] - prev.joints[1]) <= b1 && rpd::norm(c.joints[2] - prev.joints[2]) <= b2;
}

/// Block-local ordered compaction of a quiver bit set into shared memory.
template <int NT>
__device__ int block_compact(const uint32_t* __restrict__ bits, int Q, int* out) {
  typedef cub::BlockScan<int, NT> Scan;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int nwords = (Q + 31) / 32;
  for (int w0 = 0; w0 < nwords; w0 += NT) {
    const int wd = w0 + threadIdx.x;
    const uint32_t word = wd < nwords ? __ldcg(bits + wd) : 0u;
    int off = 0, total = 0;
    Scan(tmp).ExclusiveSum(__popc(word), off, total);
    off += carry;
    uint32_t x = word;
    while (x) {
      const int b = __ffs(x) - 1;
      x &= x - 1;
      out[off++] = wd * 32 + b;
    }
    __syncthreads();
    if (threadIdx.x == 0) carry += total;
    __syncthreads();
  }
  const int result = carry;
  __syncthreads();  // every thread has read carry before a next call resets it
  return result;
}

/// Both candidate lists in one pass (Q <= 16384, so at most 512 words, two
/// per thread): one block scan of the packed (i count << 16 | j count) per
/// thread gives both ordered offsets. Returns (n_i << 16) | n_j.
template <int NT>
__device__ int block_compact_pair(const uint32_t* __restrict__ ib, const uint32_t* __restrict__ jb,
                                  int Q, int* li, int* lj) {
  typedef cub::BlockScan<int, NT> Scan;
  __shared__ typename Scan::TempStorage tmp;
  const int nwords = (Q + 31) / 32;
  const int w0 = 2 * static_cast<int>(threadIdx.x);
  uint32_t wi[2], wj[2];
  int cnt = 0;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int w = w0 + r;
    wi[r] = w < nwords ? __ldcg(ib + w) : 0u;
    wj[r] = w < nwords ? __ldcg(jb + w) : 0u;
    cnt += (__popc(wi[r]) << 16) + __popc(wj[r]);
  }
  int off = 0, total = 0;
  Scan(tmp).ExclusiveSum(cnt, off, total);
  int oi = off >> 16, oj = off & 0xFFFF;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int base = (w0 + r) * 32;
    for (uint32_t x = wi[r]; x; x &= x - 1) li[oi++] = base + __ffs(x) - 1;
    for (uint32_t x = wj[r]; x; x &= x - 1) lj[oj++] = base + __ffs(x) - 1;
  }
  __syncthreads();  // lists complete; tmp reusable
  return total;
}

/// Coherent (L2) read of a struct written by another block in this launch.
template <typename T>
__device__ __forceinline__ T ldcg_struct(const T* p) {
  static_assert(sizeof(T) % 8 == 0, "8-byte granular");
  T v;
  const long long* s = reinterpret_cast<const long long*>(p);
  long long* d = reinterpret_cast<long long*>(&v);
#pragma unroll 4
  for (int i = 0; i < static_cast<int>(sizeof(T) / 8); ++i) d[i] = __ldcg(s + i);
  return v;
}

/// wik_pose's arithmetic for a fast-pass winner (coaxial arm: link2 = p1,
/// link1 = root), from the record kept during the pass.
__device__ __noinline__ DevPose pose_from_win(const BpArgs& A, const BpWin& W) {
  const ArmDev& arm = A.arm;
  const V3 qi{A.qx[W.i], A.qy[W.i], A.qz[W.i]};
  const V3 qj{A.qx[W.j], A.qy[W.j], A.qz[W.j]};
  const V3 p2 = W.p1 + arm.L[1] * qj;
  const V3 v3 = W.wp - p2;
  const double v3_len = rpd::norm(v3);
  const V3 v3_hat = v3 / v3_len;
  const V3 s3 = v3_hat * arm.L[2];
  const V3 p3 = p2 + s3;
  DevPose ch{};
  ch.nseg = 3;
  ch.seg[0] = arm.L[0] * qi;
  ch.seg[1] = arm.L[1] * qj;
  ch.seg[2] = s3;
  ch.qidx[0] = W.i;
  ch.qidx[1] = W.j;
  ch.qidx[2] = -1;
  ch.qidx[3] = -1;
  build_chain(arm, ch);
  ch.n_wp_links = 3;
  ch.wp_from[0] = arm.root; ch.wp_to[0] = W.p1;
  ch.wp_from[1] = W.p1;     ch.wp_to[1] = p2;
  ch.wp_from[2] = p2;       ch.wp_to[2] = p3;
  ch.n_wp[0] = ch.n_wp[1] = ch.n_wp[2] = A.n;
  if (A.four && W.opt >= 0) {
    const V3 dir = W.opt < W.n_opts ? W.opt_dir[W.opt] : rpd::normalized(ch.seg[2]);
    ch.nseg = 4;
    ch.seg[3] = A.L4 * dir;
    build_chain(arm, ch);
    ch.n_wp_links = 4;
    ch.wp_from[3] = ch.joints[3];
    ch.wp_to[3] = ch.joints[4];
    ch.n_wp[3] = A.n;
  }
  return ch;
}

constexpr int kBpThreads = 256;

__global__ void __launch_bounds__(kBpThreads, 1) k_backward_pass(const __grid_constant__ BpArgs A) {
  extern __shared__ int sh_lists[];
  int* li = sh_lists;
  int* lj = sh_lists + A.Q;
  __shared__ WikBest wb[kBpThreads / 32];
  const unsigned nb = gridDim.x;
  const int lane = threadIdx.x & 31;
  // per-attempt search descriptor, built once per block in shared memory
  // (a per-thread copy would be ~700 B of local memory per thread)
  __shared__ WikDev sw;
  __shared__ V3 s_u1, s_u2, s_cu, s_cv, s_wk;
  __shared__ double s_fetch[21];
  __shared__ V3 s_prev[5];  // fast pass: joints[1], joints[2], seg[0], seg[1] of the last pose + its waypoint
  __shared__ int s_found;
  // screened candidates of one round (one pair per thread): metric, ordinal
  __shared__ double s_cm[kBpThreads];
  __shared__ long long s_ct[kBpThreads];
  __shared__ int s_nc;
  __shared__ short s_rank[kBpThreads];
  // the screened pairs' segment-1 data and j, kept for the evaluation waves
  __shared__ CiFast s_cf[kBpThreads];
  __shared__ int s_cj[kBpThreads];
  const bool fast_eval = !A.arm.any_limit && !A.arm.has_offsets;
  // fast path: block 0 rebuilds the published poses from their winners
  // before the kernel ends (every exit below goes through here)
  const auto rebuild = [&]() {
    if (!fast_eval || blockIdx.x != 0) return;
    __syncthreads();
    for (int q = threadIdx.x; q < A.m; q += blockDim.x)
      if (A.win[q].i >= 0) A.poses[q] = pose_from_win(A, A.win[q]);
  };
  V3 my_q{0, 0, 0};
  int my_w1 = 0;
  if (fast_eval) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < A.Q) {
      my_q = V3{A.qx[i], A.qy[i], A.qz[i]};
      my_w1 = static_cast<int>((__ldg(A.walk1 + (i >> 5)) >> (i & 31)) & 1u);
    }
  }
  for (int k = A.m - 2; k >= 0; --k) {
    if (k == 0 && A.has_fixed) {
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        // joints 1 and 2 of the pose at waypoint 1 (rebuilt in this block on
        // the fast path, else the pose in memory)
        V3 pj1, pj2;
        if (fast_eval && A.m > 2) {
          pj1 = s_prev[0];
          pj2 = s_prev[1];
        } else {
          const DevPose prev = ldcg_struct(A.poses + 1);
          pj1 = prev.joints[1];
          pj2 = prev.joints[2];
        }
        int found = 0;
        for (int fi = 0; fi < A.nf && !found; ++fi) {
          const double f = A.factors[fi];
          const double b1 = A.pj1 * f + 1e-12, b2 = A.pj2 * f + 1e-12;
          if (rpd::norm(A.fixed_first.joints[1] - pj1) <= b1 &&
              rpd::norm(A.fixed_first.joints[2] - pj2) <= b2) {  // pose_smooth
            A.poses[0] = A.fixed_first;
            A.relax[0] = f;
            A.kind[0] = 2;
            found = 1;
          }
        }
        A.state[0] = found;
        A.state[1] = found ? -1 : 0;
        A.state[2] = found;
      }
      rebuild();
      return;  // k == 0 is the last waypoint either way
    }
    // fetch what this waypoint needs from the previous pose and the waypoint
    // list in one round trip (21 doubles, one per thread; written by other
    // blocks in this launch, hence .cg loads), then thread 0 fills in the
    // per-waypoint fields of the search descriptor
    const bool from_block = fast_eval && k < A.m - 2;  // previous pose rebuilt in this block
    if (from_block) {
      if (threadIdx.x < 12) s_fetch[threadIdx.x] = (&s_prev[0].x)[threadIdx.x];
      else if (threadIdx.x < 18) {
        const int wi = k - 1 + (threadIdx.x - 12) / 3;  // k-1, k
        s_fetch[threadIdx.x] = wi >= 0 ? __ldcg(&A.wps[wi].x + (threadIdx.x - 12) % 3) : 0.0;
      } else if (threadIdx.x < 21) {
        s_fetch[threadIdx.x] = (&s_prev[4].x)[threadIdx.x - 18];
      }
    } else {
      const int t = threadIdx.x;
      if (t < 12) {
        const DevPose* pp = A.poses + k + 1;
        const double* src = t < 6 ? &pp->joints[1 + t / 3].x : &pp->seg[(t - 6) / 3].x;
        s_fetch[t] = __ldcg(src + t % 3);
      } else if (t < 21) {
        const int wi = k - 1 + (t - 12) / 3;  // k-1, k, k+1
        s_fetch[t] = wi >= 0 ? __ldcg(&A.wps[wi].x + (t - 12) % 3) : 0.0;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      // trail context from the (possibly cloud-substituted) waypoint list
      const V3 prev_j1{s_fetch[0], s_fetch[1], s_fetch[2]};
      const V3 prev_j2{s_fetch[3], s_fetch[4], s_fetch[5]};
      const V3 prev_s0{s_fetch[6], s_fetch[7], s_fetch[8]};
      const V3 prev_s1{s_fetch[9], s_fetch[10], s_fetch[11]};
      const V3 wk{s_fetch[15], s_fetch[16], s_fetch[17]};
      const V3 wprev = k > 0 ? V3{s_fetch[12], s_fetch[13], s_fetch[14]} : wk;
      const V3 wnext{s_fetch[18], s_fetch[19], s_fetch[20]};
      WikDev& w = sw;
      if (k == A.m - 2) {  // waypoint-independent fields, once per launch
        w = WikDev{};
        w.g = A.g;
        w.arm = A.arm;
        w.n = A.n;
        w.Q = A.Q;
        w.qx = A.qx;
        w.qy = A.qy;
        w.qz = A.qz;
        w.spacing = A.spacing;
        w.four = A.four;
        w.L4 = A.L4;
        w.cond2 = A.cond2;
        w.cond3 = A.cond3;
        w.filter_j = A.filter_j;
        w.prof = blockIdx.x == 0 ? A.prof : nullptr;
      }
      w.prev_j1 = prev_j1;
      w.prev_j2 = prev_j2;
      w.n_opts = 0;
      if (k > 0) {
        const V3 d = wprev - wk;
        if (rpd::norm(d) > 1e-12) w.opt_dir[w.n_opts++] = rpd::normalized(d);
      }
      if (k + 1 < A.m) {
        const V3 d = wnext - wk;
        if (rpd::norm(d) > 1e-12) w.opt_dir[w.n_opts++] = rpd::normalized(d);
      }
      const bool fixed_bias = A.has_fixed && k == 1;
      w.has_bias = (fixed_bias || A.has_bias) ? 1 : 0;
      if (w.has_bias) {
        const DevPose& b = fixed_bias ? A.fixed_first : A.bias;
        w.bias_j1 = b.joints[1];
        w.bias_j2 = b.joints[2];
      }
      s_u1 = rpd::normalized(prev_s0);
      s_u2 = rpd::normalized(prev_s1);
      s_wk = wk;
      // cloud ring frame (src/path_planner.cpp:368-377)
      s_cu = V3{0, 0, 0};
      s_cv = V3{0, 0, 0};
      if (A.cloud) {
        V3 dir = wnext - wk;
        if (rpd::norm(dir) < 1e-12 && k > 0) dir = wk - wprev;
        if (rpd::norm(dir) < 1e-12) dir = V3{0, 0, 1};
        dir = rpd::normalized(dir);
        s_cu = perpendicular_of(dir);
        s_cv = rpd::cross(dir, s_cu);
      }
    }
    __syncthreads();
    const WikDev& w = sw;
    const V3 u1 = s_u1, u2 = s_u2;
    bool found = false;
    const int n_targets = A.cloud ? 9 : 1;
    for (int t = 0; t < n_targets && !found; ++t) {
      for (int fi = 0; fi < A.nf && !found; ++fi) {
        const double f = A.factors[fi];
        if (threadIdx.x == 0) {
          sw.wp = t == 0 ? s_wk
                         : s_wk + A.cloud_radius * (A.ring_c[t - 1] * s_cu + A.ring_s[t - 1] * s_cv);
          // waypoint_ik's relaxed bounds (src/path_planner.cpp:172-174)
          sw.eps = A.eps_wp * f + 1e-12;
          sw.j1max = A.pj1 * f + 1e-12;
          sw.j2max = A.pj2 * f + 1e-12;
          sw.sm1 = sw.j1max;
          sw.sm2 = sw.j2max;
        }
        __syncthreads();
        const bool prof = A.prof && blockIdx.x == 0 && threadIdx.x == 0;
        long long c0 = prof ? clock64() : 0;
        // phase A: candidate filters
        for (int i0 = blockIdx.x * blockDim.x; i0 < A.Q; i0 += nb * blockDim.x) {
          const int i = i0 + threadIdx.x;
          bool pi = false, pj = false;
          const long long f0 = A.prof ? clock64() : 0;
          if (i < A.Q) {
            if (fast_eval)
            {
              // this thread's direction and its segment-1 verdict are the same
              // for the whole pass: kept in registers when the grid covers Q
              const bool cached = i0 == static_cast<int>(blockIdx.x * blockDim.x);
              const V3 q = cached ? my_q : wq(w, i);
              const int ok1 =
                  cached ? my_w1 : static_cast<int>((__ldg(A.walk1 + (i >> 5)) >> (i & 31)) & 1u);
              wik_filter_fast(w, A.cone1[fi], A.cone2[fi], u1, u2, i, A.ci_fast, &pi, &pj, q, ok1,
                              A.prof);
            }
            else
              wik_filter_one(w, A.cone1[fi], A.cone2[fi], u1, u2, i, A.ci_by_index, &pi, &pj);
          }
          (void)f0;
          const unsigned mi = __ballot_sync(FULL, pi), mj = __ballot_sync(FULL, pj);
          if (lane == 0 && (i >> 5) < (A.Q + 31) / 32) {
            A.ibits[i >> 5] = mi;
            A.jbits[i >> 5] = mj;
          }
        }
        const long long cb = prof ? clock64() : 0;
        grid_barrier(A.bar, nb);
        long long c1 = prof ? clock64() : 0;
        if (prof) A.prof[13] += c1 - cb;
        // phase B: block-local compaction + this block's share of the pairs
        int nci, ncj;
        if (A.Q <= 2 * 32 * kBpThreads && A.Q < 65536) {
          const int both = block_compact_pair<kBpThreads>(A.ibits, A.jbits, A.Q, li, lj);
          nci = both >> 16;
          ncj = both & 0xFFFF;
        } else {
          nci = block_compact<kBpThreads>(A.ibits, A.Q, li);
          ncj = block_compact<kBpThreads>(A.jbits, A.Q, lj);
        }
        long long c2 = prof ? clock64() : 0;
        double bm = 1e308;
        long long bo = LLONG_MAX;
        int bopt = -1;
        const long long total = static_cast<long long>(nci) * ncj;
        // pairs dealt round-robin over the blocks (pair tt -> block tt % nb),
        // so a few thousand pairs spread over every SM of the grid
        if (fast_eval) {
          // Each round every thread screens one pair with the exact prefix
          // of the test (move bound, gap band, metric); the survivors are
          // evaluated one warp per pair (wik_full_warp), which cuts the
          // serial chain of a full evaluation from ~30k to a few k cycles.
          long long tt = static_cast<long long>(threadIdx.x) * nb + blockIdx.x;
          const long long stride = static_cast<long long>(nb) * blockDim.x;
          const int warp = threadIdx.x >> 5;
          for (;;) {
            if (threadIdx.x == 0) s_nc = 0;
            __syncthreads();
            if (tt < total) {
              const int a = static_cast<int>(tt / ncj);
              if (__ldcg(&A.ci_fast[li[a]].ok)) {
                const CiFast c = ldcg_struct(A.ci_fast + li[a]);
                const int jj = lj[tt - static_cast<long long>(a) * ncj];
                double mm;
                if (wik_pre_fast(w, c, jj, &mm)) {
                  const int k = atomicAdd(&s_nc, 1);
                  s_cm[k] = mm;
                  s_ct[k] = tt;
                  s_cf[k] = c;
                  s_cj[k] = jj;
                }
              }
              tt += stride;
            }
            const bool more = __syncthreads_or(tt < total);
            const int nc = s_nc;
            const long long ps1 = prof ? clock64() : 0;

            // rank the screened candidates by (metric, ordinal) ...
            if (threadIdx.x < nc) {
              const double mm = s_cm[threadIdx.x];
              const long long t2 = s_ct[threadIdx.x];
              int r = 0;
              for (int k = 0; k < nc; ++k) r += wik_better(s_cm[k], s_ct[k], mm, t2) ? 1 : 0;
              s_rank[r] = static_cast<short>(threadIdx.x);
            }
            __syncthreads();
            if (prof) A.prof[15] += clock64() - ps1;
            // ... and evaluate them in waves of one candidate per warp, best
            // first: the first wave with a qualifying pair holds the round's
            // answer (every later candidate ranks below it)
            // (two candidates per warp, one per half warp: 16 per wave)
            const int half = lane >> 4, sub = lane & 15;
            for (int w0 = 0; w0 < nc; w0 += 2 * (kBpThreads / 32)) {
              const int k = w0 + 2 * warp + half;
              bool hit = false;
              int opt = -1;
              bool valid = false;
              double mm = 0.0;
              long long t2 = 0;
              CiFast c{};
              int jj = 0;
              if (k < nc) {
                const int e = s_rank[k];
                mm = s_cm[e];
                t2 = s_ct[e];
                if (wik_better(mm, t2, bm, bo)) {  // else it cannot improve this half's best
                  c = s_cf[e];
                  jj = s_cj[e];
                  valid = true;
                }
              }
              hit = wik_full_half(w, c, jj, valid, sub, half, &opt);
              if (prof) A.prof[14] += 1;
              if (hit) {
                bm = mm;
                bo = t2;
                bopt = opt;
              }
              if (__syncthreads_or(hit)) break;
            }
            __syncthreads();
            if (prof) {
              const long long ps3 = clock64();
              A.prof[10] += ps1 - c2;  // screening (first round)
              A.prof[11] += ps3 - ps1;  // rank + evaluation waves
              A.prof[12] += nc;
            }
            if (!more) break;
          }
        } else
        for (long long tt = static_cast<long long>(threadIdx.x) * nb + blockIdx.x; tt < total;
             tt += static_cast<long long>(nb) * blockDim.x) {
          const int a = static_cast<int>(tt / ncj);
          const long long q0 = A.prof ? clock64() : 0;
          if (!__ldcg(&A.ci_by_index[li[a]].ok)) continue;
          const CiData c = ldcg_struct(A.ci_by_index + li[a]);
          const long long q1 = A.prof ? clock64() : 0;
          double mm;
          int opt;
          const bool hit = wik_test(w, c, lj[tt - static_cast<long long>(a) * ncj], &mm, &opt);
          if (A.prof && blockIdx.x == 0) {
            const long long q2 = clock64();
            atomicMax(reinterpret_cast<unsigned long long*>(A.prof + 8), q1 - q0);
            atomicMax(reinterpret_cast<unsigned long long*>(A.prof + 9), q2 - q1);
          }
          if (hit && wik_better(mm, tt, bm, bo)) {
            bm = mm;
            bo = tt;
            bopt = opt;
          }
        }
        for (int off = 16; off > 0; off >>= 1) {
          const double om = __shfl_down_sync(FULL, bm, off);
          const long long oo = __shfl_down_sync(FULL, bo, off);
          const int op = __shfl_down_sync(FULL, bopt, off);
          if (wik_better(om, oo, bm, bo)) {
            bm = om;
            bo = oo;
            bopt = op;
          }
        }
        if (lane == 0) wb[threadIdx.x >> 5] = WikBest{bm, bo, bopt, -1, -1, V3{0, 0, 0}};
        __syncthreads();
        if (threadIdx.x == 0) {
          WikBest b = wb[0];
          for (int q = 1; q < kBpThreads / 32; ++q)
            if (wik_better(wb[q].metric, wb[q].ord, b.metric, b.ord)) b = wb[q];
          if (fast_eval && b.ord != LLONG_MAX) {
            const int a = static_cast<int>(b.ord / ncj);
            const CiFast cf = ldcg_struct(A.ci_fast + li[a]);
            b.i = cf.i;
            b.p1 = cf.p1;
            b.j = lj[b.ord - static_cast<long long>(a) * ncj];
          }
          A.block_best[blockIdx.x] = b;
          // cancellation is sampled by block 0 before the barrier and read
          // by every block after it, so all blocks leave together
          if (fast_eval && A.cancel && blockIdx.x == 0)
            A.state[3] = *reinterpret_cast<const volatile int*>(A.cancel);
        }
        long long c3 = prof ? clock64() : 0;
        grid_barrier(A.bar, nb);
        long long c4 = prof ? clock64() : 0;
        if (fast_eval && A.cancel && __ldcg(A.state + 3)) {
          rebuild();
          return;  // state[3] != 0 tells the host the pass was cancelled
        }
        if (fast_eval) {
          // Every block reduces the per-block winners itself and rebuilds the
          // winning pose (the candidate travels in block_best), so the next
          // waypoint starts without another grid barrier; block 0 also
          // records the pose for the host. block_best is rewritten only after
          // the next attempt's filter barrier, which every block reaches only
          // after this reduction.
          WikBest b{1e308, LLONG_MAX, -1, -1, -1, V3{0, 0, 0}};
          for (unsigned q = threadIdx.x; q < nb; q += blockDim.x) {
            const WikBest r = ldcg_struct(A.block_best + q);
            if (wik_better(r.metric, r.ord, b.metric, b.ord)) b = r;
          }
          for (int off = 16; off > 0; off >>= 1) {
            WikBest o;
            o.metric = __shfl_down_sync(FULL, b.metric, off);
            o.ord = __shfl_down_sync(FULL, b.ord, off);
            o.opt = __shfl_down_sync(FULL, b.opt, off);
            o.i = __shfl_down_sync(FULL, b.i, off);
            o.j = __shfl_down_sync(FULL, b.j, off);
            o.p1.x = __shfl_down_sync(FULL, b.p1.x, off);
            o.p1.y = __shfl_down_sync(FULL, b.p1.y, off);
            o.p1.z = __shfl_down_sync(FULL, b.p1.z, off);
            if (wik_better(o.metric, o.ord, b.metric, b.ord)) b = o;
          }
          __syncthreads();
          if (lane == 0) wb[threadIdx.x >> 5] = b;
          __syncthreads();
          if (threadIdx.x == 0) {
            b = wb[0];
            for (int q = 1; q < kBpThreads / 32; ++q)
              if (wik_better(wb[q].metric, wb[q].ord, b.metric, b.ord)) b = wb[q];
            int ok = 0;
            if (b.ord != LLONG_MAX) {
              // the fields the next waypoint needs, with wik_pose's
              // arithmetic (chain = cumulative sums on a coaxial arm)
              const V3 s0 = A.arm.L[0] * V3{A.qx[b.i], A.qy[b.i], A.qz[b.i]};
              const V3 s1 = A.arm.L[1] * V3{A.qx[b.j], A.qy[b.j], A.qz[b.j]};
              const V3 j1 = A.arm.root + s0;
              s_prev[0] = j1;
              s_prev[1] = j1 + s1;
              s_prev[2] = s0;
              s_prev[3] = s1;
              s_prev[4] = t > 0 ? w.wp : s_wk;  // waypoint k as the pass leaves it
              if (blockIdx.x == 0) {
                BpWin W;
                W.i = b.i;
                W.j = b.j;
                W.opt = b.opt;
                W.n_opts = w.n_opts;
                W.p1 = b.p1;
                W.wp = w.wp;
                W.opt_dir[0] = w.opt_dir[0];
                W.opt_dir[1] = w.opt_dir[1];
                A.win[k] = W;
                A.relax[k] = f;
                A.kind[k] = t > 0 ? 1 : 0;
                if (t > 0) A.wps[k] = w.wp;
              }
              ok = 1;
            }
            s_found = ok;
            if (blockIdx.x == 0) A.state[0] = ok;
          }
          __syncthreads();
        }
        long long c5f = prof ? clock64() : 0;
        if (fast_eval && prof) {
          A.prof[0] += c1 - c0;
          A.prof[1] += c2 - c1;
          A.prof[2] += c3 - c2;
          A.prof[3] += c4 - c3;
          A.prof[4] += c5f - c4;
          A.prof[6] += 1;
          A.prof[7] += static_cast<long long>(nci) * ncj;
        }
        if (fast_eval) {
          found = s_found != 0;
          continue;
        }
        // phase C: block 0 picks the first strict minimum and publishes it
        if (blockIdx.x == 0) {
          WikBest b{1e308, LLONG_MAX, -1};
          for (unsigned q = threadIdx.x; q < nb; q += blockDim.x) {
            const WikBest r = ldcg_struct(A.block_best + q);
            if (wik_better(r.metric, r.ord, b.metric, b.ord)) b = r;
          }
          for (int off = 16; off > 0; off >>= 1) {
            const double om = __shfl_down_sync(FULL, b.metric, off);
            const long long oo = __shfl_down_sync(FULL, b.ord, off);
            const int op = __shfl_down_sync(FULL, b.opt, off);
            if (wik_better(om, oo, b.metric, b.ord)) b = WikBest{om, oo, op};
          }
          __syncthreads();
          if (lane == 0) wb[threadIdx.x >> 5] = b;
          __syncthreads();
          if (threadIdx.x == 0) {
            b = wb[0];
            for (int q = 1; q < kBpThreads / 32; ++q)
              if (wik_better(wb[q].metric, wb[q].ord, b.metric, b.ord)) b = wb[q];
            int ok = 0;
            if (b.ord != LLONG_MAX) {
              const int a = static_cast<int>(b.ord / ncj);
              CiData cd;
              if (fast_eval) {
                const CiFast f = ldcg_struct(A.ci_fast + li[a]);
                cd.i = f.i;
                cd.ok = f.ok;
                cd.move1 = f.move1;
                cd.p1 = f.p1;
                cd.link1 = A.arm.root;
                cd.frame1 = rpd::m_identity();  // unused without offsets
              } else {
                cd = ldcg_struct(A.ci_by_index + li[a]);
              }
              A.poses[k] = wik_pose(w, cd, lj[b.ord - static_cast<long long>(a) * ncj], b.opt);
              A.relax[k] = f;
              A.kind[k] = t > 0 ? 1 : 0;
              if (t > 0) A.wps[k] = w.wp;
              ok = 1;
            }
            A.state[0] = ok;
          }
        }
        long long c5 = prof ? clock64() : 0;
        grid_barrier(A.bar, nb);
        if (prof) {
          const long long c6 = clock64();
          A.prof[0] += c1 - c0;  // filter + barrier
          A.prof[1] += c2 - c1;  // compaction
          A.prof[2] += c3 - c2;  // pairs (block 0's share)
          A.prof[3] += c4 - c3;  // barrier wait (slowest block)
          A.prof[4] += c5 - c4;  // publish
          A.prof[5] += c6 - c5;  // barrier
          A.prof[6] += 1;
          A.prof[7] += static_cast<long long>(nci) * ncj;
        }
        found = __ldcg(A.state) != 0;
      }
    }
    if (!found) {
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        A.state[1] = k;
        A.state[2] = 0;
      }
      rebuild();
      return;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    A.state[1] = -1;
    A.state[2] = 1;
  }
  rebuild();
}

// ---------------------------------------------------------------------------
// Cluster backward pass (coaxial arms without joint limits, generated
// quivers): the whole sequential pass (src/path_planner.cpp:322-400) in ONE
// thread-block cluster of CL CTAs. Per (waypoint, target, factor) attempt:
//  F  every CTA builds both candidate lists itself (no exchange): the
//     cones around the previous segment directions are enumerated ring by
//     ring (rp_rings.cuh: <= 2 azimuth arcs per latitude ring, a superset)
//     and each visited direction gets waypoint_ik's exact fp64 cone and
//     move1 tests; ordered compaction by block scans of packed counts.
//  S  the (i, j) pairs are dealt over the cluster's warps (32 j per warp
//     item); an fp32 prefilter with 1e-5 m margins drops the pairs that
//     cannot pass the move2 bound or the gap band, the rest queue in shared
//     memory (warp-aggregated appends).
//  E  the queue is evaluated data-parallel in flat item lists instead of
//     candidate by candidate: the exact prefix (wik_pre_fast) and the
//     smoothness bound per candidate, then every walk of every live
//     candidate (segments 2, 3 and each trail option) one per thread, then
//     every non-adjacent link distance, then the verdicts (the first trail
//     option whose walk and links are clear, as append_trail takes it) and
//     the CTA's (metric, ordinal) minimum.
//  R  one cluster barrier; lane r of warp 0 reads CTA r's winner over DSMEM
//     and every CTA reduces identically, so all continue with the same pose
//     and no second barrier is needed (slots are double-buffered by attempt
//     parity).
// Exactness: the lists are supersets filtered by the reference's own fp64
// tests (ascending index order, so ordinals compare like the reference's
// (cand_i, cand_j) scan), the prefilter only drops pairs the exact prefix
// would reject, every test is the reference's predicate on the same fp64
// pose, and the winner is the (metric, ordinal) minimum over every
// qualifying pair -- the first strict minimum of the reference's loop.

namespace cg = cooperative_groups;

constexpr int kBpcThreads = 512;
constexpr int kBpcWarps = kBpcThreads / 32;
constexpr int kBpcQueue = 768;   // prefiltered pairs per round per CTA (> 32 x warps)
constexpr int kBpcRings = 256;   // latitude rings (2 deg: 91, 1 deg: 181)
constexpr int kBpcCiCap = 1024;  // segment-1 points cached as fp32 in shared memory
constexpr int kBpcBatch = 64;    // candidates evaluated together (best first)
static_assert(kBpcQueue > 32 * kBpcWarps, "a round must fit every warp's last item");

struct BpcSlot {  // one CTA's winner of an attempt
  double metric;
  long long ord;
  int opt, i, j;
  V3 p1;
};

struct BpcShared {
  WikDev sw;
  V3 u1, u2, cu, cv, wk;
  double fetch[21];
  V3 prev[5];
  int found;
  int nci, ncj;
  int tot[2];
  int nq, nl;  // queued pairs, live candidates
  int win_rank;
  // cluster-visible, [attempt parity]: best-hit bound (metric bits),
  // winner slot, cancel flag
  unsigned long long bound[2];
  BpcSlot slot[2];
  int cancel[2];
  // ring intervals of both cones
  int rcnt[2 * kBpcRings];
  int rbase[2 * kBpcRings + 1];
  int2 riv[2 * kBpcRings][4];
  signed char rniv[2 * kBpcRings];
  // prefiltered pairs of a round: ordinal a * ncj + b, exact metric,
  // candidate geometry (p2, s3) and walk / distance failure bits
  double qm[kBpcQueue];
  unsigned qo[kBpcQueue];
  V3 cj2[kBpcQueue];
  V3 cs3[kBpcQueue];
  V3 cdl[kBpcQueue];  // normalized(s3): the straight trail option
  int cflag[kBpcQueue];
  short qs[kBpcQueue];  // the current batch
  short ql[kBpcQueue];  // live candidates (any order)
  unsigned char cbin[kBpcQueue];
  int hist[256], cum[256];
  unsigned long long mlo, mhi, bmin;
  int nb;
  float4 p1f[kBpcCiCap];
  WikBest wb[kBpcWarps];
};


__device__ __forceinline__ unsigned long long metric_bits(double m) {
  return static_cast<unsigned long long>(__double_as_longlong(m));  // m >= 0: monotone
}

__global__ void __launch_bounds__(kBpcThreads, 1) k_bp_cluster(const __grid_constant__ BpArgs A) {
  // dynamic shared memory: [BpcShared][li: list_cap x u16][lj: list_cap x u16]
  extern __shared__ __align__(16) unsigned char bpc_smem[];
  BpcShared& S = *reinterpret_cast<BpcShared*>(bpc_smem);
  unsigned short* li = reinterpret_cast<unsigned short*>(bpc_smem + sizeof(BpcShared));
  unsigned short* lj = li + A.list_cap;
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = static_cast<int>(cluster.block_rank());
  const int CL = static_cast<int>(cluster.num_blocks());
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool prof = A.prof && rank == 0 && tid == 0;
  const ArmDev& arm = A.arm;
  const auto rebuild = [&]() {
    if (rank != 0) return;
    __syncthreads();
    for (int q = tid; q < A.m; q += blockDim.x)
      if (A.win[q].i >= 0) A.poses[q] = pose_from_win(A, A.win[q]);
  };
  if (tid == 0) {
    S.bound[0] = S.bound[1] = metric_bits(1e308);
    S.cancel[0] = S.cancel[1] = 0;
  }
  cluster.sync();  // bound and flags initialised before any CTA reads CTA 0's
  unsigned long long* bound0 = cluster.map_shared_rank(&S.bound[0], 0);
  const int* cancel0 = cluster.map_shared_rank(&S.cancel[0], 0);
  int par = 0;  // attempt parity (identical in every CTA)
  const int nr = A.nrings;
  for (int k = A.m - 2; k >= 0; --k) {
    if (k == 0 && A.has_fixed) {
      if (rank == 0 && tid == 0) {
        V3 pj1, pj2;
        if (A.m > 2) {
          pj1 = S.prev[0];
          pj2 = S.prev[1];
        } else {
          const DevPose pv = ldcg_struct(A.poses + 1);
          pj1 = pv.joints[1];
          pj2 = pv.joints[2];
        }
        int found = 0;
        for (int fi = 0; fi < A.nf && !found; ++fi) {
          const double f = A.factors[fi];
          const double b1 = A.pj1 * f + 1e-12, b2 = A.pj2 * f + 1e-12;
          if (rpd::norm(A.fixed_first.joints[1] - pj1) <= b1 &&
              rpd::norm(A.fixed_first.joints[2] - pj2) <= b2) {  // pose_smooth
            A.poses[0] = A.fixed_first;
            A.relax[0] = f;
            A.kind[0] = 2;
            found = 1;
          }
        }
        A.state[0] = found;
        A.state[1] = found ? -1 : 0;
        A.state[2] = found;
      }
      rebuild();
      cluster.sync();  // no CTA leaves while another may still read its slots
      return;
    }
    // previous pose (anchor from memory, later ones from the last winner)
    // and the waypoint list around k
    if (k == A.m - 2) {
      if (tid < 12) {
        const DevPose* pp = A.poses + k + 1;
        const double* src = tid < 6 ? &pp->joints[1 + tid / 3].x : &pp->seg[(tid - 6) / 3].x;
        S.fetch[tid] = __ldcg(src + tid % 3);
      }
    } else if (tid < 12) {
      S.fetch[tid] = (&S.prev[0].x)[tid];
    }
    if (tid >= 12 && tid < 21) {
      const int wi = k - 1 + (tid - 12) / 3;  // k-1, k, k+1
      S.fetch[tid] = wi >= 0 ? __ldcg(&A.wps[wi].x + (tid - 12) % 3) : 0.0;
    }
    __syncthreads();
    if (tid == 0) {
      const V3 prev_j1{S.fetch[0], S.fetch[1], S.fetch[2]};
      const V3 prev_j2{S.fetch[3], S.fetch[4], S.fetch[5]};
      const V3 prev_s0{S.fetch[6], S.fetch[7], S.fetch[8]};
      const V3 prev_s1{S.fetch[9], S.fetch[10], S.fetch[11]};
      const V3 wk{S.fetch[15], S.fetch[16], S.fetch[17]};
      const V3 wprev = k > 0 ? V3{S.fetch[12], S.fetch[13], S.fetch[14]} : wk;
      const V3 wnext{S.fetch[18], S.fetch[19], S.fetch[20]};
      WikDev& w = S.sw;
      if (k == A.m - 2) {
        w = WikDev{};
        w.g = A.g;
        w.arm = A.arm;
        w.n = A.n;
        w.Q = A.Q;
        w.qx = A.qx;
        w.qy = A.qy;
        w.qz = A.qz;
        w.spacing = A.spacing;
        w.four = A.four;
        w.L4 = A.L4;
        w.cond2 = A.cond2;
        w.cond3 = A.cond3;
        w.filter_j = A.filter_j;
        w.prof = nullptr;
      }
      w.prev_j1 = prev_j1;
      w.prev_j2 = prev_j2;
      w.n_opts = 0;
      if (k > 0) {
        const V3 d = wprev - wk;
        if (rpd::norm(d) > 1e-12) w.opt_dir[w.n_opts++] = rpd::normalized(d);
      }
      if (k + 1 < A.m) {
        const V3 d = wnext - wk;
        if (rpd::norm(d) > 1e-12) w.opt_dir[w.n_opts++] = rpd::normalized(d);
      }
      const bool fixed_bias = A.has_fixed && k == 1;
      w.has_bias = (fixed_bias || A.has_bias) ? 1 : 0;
      if (w.has_bias) {
        const DevPose& b = fixed_bias ? A.fixed_first : A.bias;
        w.bias_j1 = b.joints[1];
        w.bias_j2 = b.joints[2];
      }
      S.u1 = rpd::normalized(prev_s0);
      S.u2 = rpd::normalized(prev_s1);
      S.wk = wk;
      S.cu = V3{0, 0, 0};
      S.cv = V3{0, 0, 0};
      if (A.cloud) {
        V3 dir = wnext - wk;
        if (rpd::norm(dir) < 1e-12 && k > 0) dir = wk - wprev;
        if (rpd::norm(dir) < 1e-12) dir = V3{0, 0, 1};
        dir = rpd::normalized(dir);
        S.cu = perpendicular_of(dir);
        S.cv = rpd::cross(dir, S.cu);
      }
    }
    __syncthreads();
    const WikDev& w = S.sw;
    bool found = false;
    const int n_targets = A.cloud ? 9 : 1;
    for (int t = 0; t < n_targets && !found; ++t) {
      for (int fi = 0; fi < A.nf && !found; ++fi, par ^= 1) {
        const double f = A.factors[fi];
        long long c0 = prof ? clock64() : 0;
        if (tid == 0) {
          S.sw.wp = t == 0 ? S.wk : S.wk + A.cloud_radius * (A.ring_c[t - 1] * S.cu +
                                                           A.ring_s[t - 1] * S.cv);
          S.sw.eps = A.eps_wp * f + 1e-12;
          S.sw.j1max = A.pj1 * f + 1e-12;
          S.sw.j2max = A.pj2 * f + 1e-12;
          S.sw.sm1 = S.sw.j1max;
          S.sw.sm2 = S.sw.j2max;
          S.nq = 0;
          S.nl = 0;
          S.mlo = metric_bits(1e308);
          S.mhi = 0ull;
          // the other parity's bound is free: every CTA passed the barrier of
          // the attempt that used it
          if (rank == 0) S.bound[par ^ 1] = metric_bits(1e308);
        }
        if (tid < 256) S.hist[tid] = 0;
        __syncthreads();
        const V3 u1 = S.u1, u2 = S.u2;
        const double cone1 = A.cone1[fi], cone2 = A.cone2[fi];
        // ---- F: ring intervals of both cones
        for (int r2 = tid; r2 < 2 * nr; r2 += blockDim.x) {
          const int cone = r2 >= nr, r = cone ? r2 - nr : r2;
          const int off = __ldg(A.ring_off + r), cnt = __ldg(A.ring_off + r + 1) - off;
          int a0[2], ln[2], is[4], ie[4];
          const int na = ring_arcs(__ldg(A.qring_c + r), __ldg(A.qring_s + r), cnt, cone ? u2 : u1,
                                   cone ? cone2 : cone1, 2.0, a0, ln);
          int m = ring_intervals(cnt, a0, ln, na, is, ie);
          if (m < 0) {
            m = 1;
            is[0] = 0;
            ie[0] = cnt;
          }
          int c = 0;
          for (int q = 0; q < m; ++q) {
            S.riv[r2][q] = make_int2(off + is[q], ie[q] - is[q]);
            c += ie[q] - is[q];
          }
          S.rniv[r2] = static_cast<signed char>(m);
          S.rcnt[r2] = c;
        }
        __syncthreads();
        if (prof) A.prof[16] += clock64() - c0;
        {
          typedef cub::BlockScan<int, kBpcThreads> Scan;
          __shared__ typename Scan::TempStorage scan_tmp;
          int v = 0;
          const int per = (2 * nr + kBpcThreads - 1) / kBpcThreads;  // <= 1 for nr <= 256
          (void)per;
          v = tid < 2 * nr ? S.rcnt[tid] : 0;
          int ex = 0, tot = 0;
          Scan(scan_tmp).ExclusiveSum(v, ex, tot);
          if (tid < 2 * nr) S.rbase[tid] = ex;
          if (tid == 0) S.rbase[2 * nr] = tot;
          __syncthreads();
          if (tid == 0) {
            S.tot[0] = S.rbase[nr];
            S.tot[1] = tot;  // positions [tot0, tot) are the j cone's
            S.nci = 0;
            S.ncj = 0;
          }
          __syncthreads();
          if (prof) {
            A.prof[17] += clock64() - c0;
            A.prof[18] += S.tot[1];
          }
          // expand positions in order, exact tests, ordered compaction with
          // packed (i count << 16 | j count) block scans
          const int total = S.tot[1], tot0 = S.tot[0];
          int carry = 0;  // packed running counts (every thread holds it)
          for (int p0 = 0; p0 < total; p0 += kBpcThreads) {
            const int p = p0 + tid;
            int flag = 0, idx = 0;
            V3 p1{0, 0, 0};
            if (p < total) {
              // ring-interval of position p: binary search over the bases
              int lo = p < tot0 ? 0 : nr, hi = p < tot0 ? nr - 1 : 2 * nr - 1;
              while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (S.rbase[mid] <= p) lo = mid;
                else hi = mid - 1;
              }
              int rem = p - S.rbase[lo];
              int q = 0;
              while (rem >= S.riv[lo][q].y) {
                rem -= S.riv[lo][q].y;
                ++q;
              }
              idx = S.riv[lo][q].x + rem;
              const V3 qv{A.qx[idx], A.qy[idx], A.qz[idx]};
              if (p < tot0) {
                // wik_filter_fast: cone, then the move1 bound
                if (rpd::dot(qv, u1) >= cone1) {
                  p1 = arm.root + arm.L[0] * qv;
                  const double move1 = rpd::norm(p1 - w.prev_j1);
                  flag = !(move1 > w.j1max) ? (1 << 16) : 0;
                }
              } else {
                flag = rpd::dot(qv, u2) >= cone2 ? 1 : 0;
              }
            }
            int ex2 = 0, tot2 = 0;
            Scan(scan_tmp).ExclusiveSum(flag, ex2, tot2);
            const int pos = carry + ex2;
            if (flag >> 16) {
              const int a = pos >> 16;
              if (a < A.list_cap) li[a] = static_cast<unsigned short>(idx);
              if (a < kBpcCiCap) {
                const float ok = static_cast<float>((__ldg(A.walk1 + (idx >> 5)) >> (idx & 31)) & 1u);
                S.p1f[a] = make_float4(static_cast<float>(p1.x), static_cast<float>(p1.y),
                                       static_cast<float>(p1.z), ok);
              }
            } else if (flag) {
              if ((pos & 0xFFFF) < A.list_cap) lj[pos & 0xFFFF] = static_cast<unsigned short>(idx);
            }
            carry += tot2;
            __syncthreads();  // scan_tmp reuse
          }
          if (tid == 0) {
            S.nci = carry >> 16;
            S.ncj = carry & 0xFFFF;
          }
          __syncthreads();
        }
        long long c1 = prof ? clock64() : 0;
        const int nci = S.nci, ncj = S.ncj;
        if (nci > A.list_cap || ncj > A.list_cap) {
          // a cone larger than the shared-memory lists (1-degree quivers
          // with large relax factors): every CTA built the same lists, so
          // all leave here together; the host reruns the pass sequenced
          rebuild();
          if (rank == 0 && tid == 0) A.state[3] = 2;
          cluster.sync();
          return;
        }
        // ---- S + E in rounds of at most kBpcQueue prefiltered pairs per CTA
        double bm = 1e308;
        long long bo = LLONG_MAX;
        int bopt = -1;
        const int nbj = (ncj + 31) >> 5;
        const long long items = static_cast<long long>(nci) * nbj;
        long long it = static_cast<long long>(rank) * kBpcWarps + warp;
        const long long istride = static_cast<long long>(CL) * kBpcWarps;
        const float L1f = static_cast<float>(arm.L[0]), L2f = static_cast<float>(arm.L[1]);
        const float rx = static_cast<float>(arm.root.x), ry = static_cast<float>(arm.root.y),
                    rz = static_cast<float>(arm.root.z);
        const float pjx = static_cast<float>(w.prev_j2.x), pjy = static_cast<float>(w.prev_j2.y),
                    pjz = static_cast<float>(w.prev_j2.z);
        const float wpx = static_cast<float>(w.wp.x), wpy = static_cast<float>(w.wp.y),
                    wpz = static_cast<float>(w.wp.z);
        const float m2max = static_cast<float>((w.j2max + 1e-5) * (w.j2max + 1e-5));
        const double bhi = arm.L[2] + w.eps + 1e-5, blo = fmax(0.0, arm.L[2] - w.eps - 1e-5);
        const float b2hi = static_cast<float>(bhi * bhi), b2lo = static_cast<float>(blo * blo);
        const int thresh = kBpcQueue - 32 * kBpcWarps;
        // walk / distance items per candidate: walks = segment 2, segment 3
        // and (8DOF) the trail segment of each option; distances = link pair
        // (0,2) and per option (0,3), (1,3) -- or (0,2) alone for 6DOF
        const int nopt = A.four ? w.n_opts + 1 : 0;
        const int nwalk = 2 + nopt, ndist = 1 + 2 * nopt;
        const double min_sep = 2.0 * arm.arm_radius;
        long long cs = 0, ce = 0;
        for (;;) {
          const long long s0 = prof ? clock64() : 0;
          // S: fp32 prefilter, survivors' ordinals queued
          while (it < items && *reinterpret_cast<volatile int*>(&S.nq) < thresh) {
            const int a = static_cast<int>(it / nbj);
            const int b = static_cast<int>(it - static_cast<long long>(a) * nbj) * 32 + lane;
            it += istride;
            float4 pf;
            if (a < kBpcCiCap) {
              pf = S.p1f[a];
            } else {
              const int i = li[a];
              const float4 qi = __ldg(A.qf + i);
              pf = make_float4(rx + L1f * qi.x, ry + L1f * qi.y, rz + L1f * qi.z,
                               static_cast<float>((__ldg(A.walk1 + (i >> 5)) >> (i & 31)) & 1u));
            }
            if (pf.w == 0.0f) continue;  // segment 1 blocked: no pair of this i qualifies
            bool keep = false;
            if (b < ncj) {
              const float4 qj = __ldg(A.qf + lj[b]);
              const float x2 = pf.x + L2f * qj.x, y2 = pf.y + L2f * qj.y, z2 = pf.z + L2f * qj.z;
              const float dx = x2 - pjx, dy = y2 - pjy, dz = z2 - pjz;
              const float vx = wpx - x2, vy = wpy - y2, vz = wpz - z2;
              const float m2 = dx * dx + dy * dy + dz * dz;
              const float v2 = vx * vx + vy * vy + vz * vz;
              keep = m2 <= m2max && v2 <= b2hi && v2 >= b2lo;
            }
            const unsigned km = __ballot_sync(FULL, keep);
            if (km) {
              int base = 0;
              if (lane == 0) base = atomicAdd(&S.nq, __popc(km));
              base = __shfl_sync(FULL, base, 0);
              if (keep)
                S.qo[base + __popc(km & ((1u << lane) - 1u))] =
                    static_cast<unsigned>(a) * static_cast<unsigned>(ncj) + static_cast<unsigned>(b);
            }
          }
          const bool more = __syncthreads_or(it < items);
          const int nq = S.nq;
          const long long s1 = prof ? clock64() : 0;
          if (nq > 0) {
            // E0: exact prefix (wik_pre_fast) + smoothness bound per candidate;
            // geometry kept for the walk and distance items; dead = +inf
            long long t_e = prof ? clock64() : 0;
            for (int e = tid; e < nq; e += kBpcThreads) {
              const unsigned od = S.qo[e];
              const int a = static_cast<int>(od / static_cast<unsigned>(ncj));
              const int j = lj[od - static_cast<unsigned>(a) * static_cast<unsigned>(ncj)];
              const int i = li[a];
              CiFast c;
              c.i = i;
              c.ok = 1;
              c.p1 = arm.root + arm.L[0] * V3{A.qx[i], A.qy[i], A.qz[i]};
              c.move1 = rpd::norm(c.p1 - w.prev_j1);
              double mm = 1e308;
              int flag = 1 << 30;  // dead
              if (wik_pre_fast(w, c, j, &mm)) {
                const V3 qj{A.qx[j], A.qy[j], A.qz[j]};
                const V3 p2 = c.p1 + arm.L[1] * qj;
                const V3 v3 = w.wp - p2;
                const V3 s3 = (v3 / rpd::norm(v3)) * arm.L[2];
                S.cj2[e] = p2;
                S.cs3[e] = s3;
                S.cdl[e] = A.four ? rpd::normalized(s3) : V3{0, 0, 0};  // straight trail
                // chain joints 1, 2 are p1, p2 (cumulative sums)
                if (rpd::norm(c.p1 - w.prev_j1) <= w.sm1 && rpd::norm(p2 - w.prev_j2) <= w.sm2)
                  flag = 0;
              }
              if (flag) mm = 1e308;
              S.qm[e] = mm;
              S.cflag[e] = flag;
              if (!flag) {
                S.ql[atomicAdd(&S.nl, 1)] = static_cast<short>(e);
                atomicMin(&S.mlo, metric_bits(mm));
                atomicMax(&S.mhi, metric_bits(mm));
              }
            }
            __syncthreads();
            // best first: (metric, ordinal) order, evaluated kBpcBatch at a
            // time; the first batch with a hit holds this CTA's answer, and a
            // batch starting above the cluster's best hit cannot win
            if (prof) { A.prof[19] += clock64() - t_e; t_e = clock64(); }
            // best first without sorting: the live metrics go into 256 equal
            // bins over [min, max]; batch t = the candidates of the bins after
            // batch t-1's up to the first bin that brings >= kBpcBatch more.
            // A bin index is monotone in the metric, so every candidate of a
            // later batch has a strictly larger metric than every candidate
            // of an earlier one: the first batch with a hit holds this CTA's
            // (metric, ordinal) minimum.
            const int nl = S.nl;
            const double mlo = __longlong_as_double(static_cast<long long>(S.mlo));
            const double bw = (__longlong_as_double(static_cast<long long>(S.mhi)) - mlo) / 256.0;
            for (int x = tid; x < nl; x += kBpcThreads) {
              const int e = S.ql[x];
              const int bin = bw > 0.0 ? min(255, static_cast<int>((S.qm[e] - mlo) / bw)) : 0;
              S.cbin[e] = static_cast<unsigned char>(bin);
              atomicAdd(&S.hist[bin], 1);
            }
            __syncthreads();
            if (warp == 0) {  // inclusive prefix sums of the 256 bins
              int run = 0;
              for (int c = 0; c < 256; c += 32) {
                int v = S.hist[c + lane];
                for (int off = 1; off < 32; off <<= 1) {
                  const int u = __shfl_up_sync(FULL, v, off);
                  if (lane >= off) v += u;
                }
                S.cum[c + lane] = run + v;
                run += __shfl_sync(FULL, v, 31);
              }
            }
            __syncthreads();
            if (prof) { A.prof[20] += clock64() - t_e; t_e = clock64(); }
            int prev = -1, done = 0;
            while (done < nl) {
              // last bin of this batch: the first whose cumulative count
              // reaches done + kBpcBatch (binary search, block-uniform)
              int lo = prev + 1, hi = 255;
              while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (S.cum[mid] >= done + kBpcBatch) hi = mid;
                else lo = mid + 1;
              }
              const int kb = lo;
              if (tid == 0) {
                S.nb = 0;
                S.bmin = metric_bits(1e308);
              }
              __syncthreads();
              for (int x = tid; x < nl; x += kBpcThreads) {
                const int e = S.ql[x];
                const int bin = S.cbin[e];
                if (bin > prev && bin <= kb) {
                  S.qs[atomicAdd(&S.nb, 1)] = static_cast<short>(e);
                  atomicMin(&S.bmin, metric_bits(S.qm[e]));
                }
              }
              __syncthreads();
              const int nb = S.nb;
              prev = kb;
              done = S.cum[kb];
              // the bound moves under other CTAs' hits: decide it block-uniformly
              const double first = __longlong_as_double(static_cast<long long>(S.bmin));
              const double gb = __longlong_as_double(static_cast<long long>(
                  *reinterpret_cast<volatile unsigned long long*>(bound0 + par)));
              if (__syncthreads_or(first > gb)) break;
              // E1: every walk of the batch's live candidates, one per thread
              for (int t = tid; t < nb * nwalk; t += kBpcThreads) {
                const int e = S.qs[t / nwalk], k = t % nwalk;
                if (S.cflag[e]) continue;
                const V3 p2 = S.cj2[e], s3 = S.cs3[e];
                const V3 j3 = p2 + s3;
                V3 from, to;
                if (k == 0) {
                  const int i = li[S.qo[e] / static_cast<unsigned>(ncj)];
                  from = arm.root + arm.L[0] * V3{A.qx[i], A.qy[i], A.qz[i]};
                  to = p2;
                } else if (k == 1) {
                  from = p2;
                  to = j3;
                } else {
                  const int o = k - 2;
                  const V3 dir = o < w.n_opts ? w.opt_dir[o] : S.cdl[e];
                  from = j3;
                  to = j3 + w.L4 * dir;
                }
                if (rpd::walk_first_blocked_fast_seg(w.g, from, to, w.n) != 0)
                  atomicOr(&S.cflag[e], 1 << k);
              }
              __syncthreads();
              if (prof) { A.prof[21] += clock64() - t_e; t_e = clock64(); }
              // E2: the non-adjacent link distances of candidates whose
              // segment-2/3 walks are clear (per option only if its trail is)
              for (int t = tid; t < nb * ndist; t += kBpcThreads) {
                const int e = S.qs[t / ndist], d = t % ndist;
                const int fl = S.cflag[e];
                if (fl & ((1 << 30) | 3)) continue;
                const int o = d == 0 ? -1 : (d - 1) >> 1;
                if (o >= 0 && ((fl >> (2 + o)) & 1)) continue;
                const V3 p2 = S.cj2[e], s3 = S.cs3[e];
                const V3 j3 = p2 + s3;
                const int i = li[S.qo[e] / static_cast<unsigned>(ncj)];
                const V3 j1 = arm.root + arm.L[0] * V3{A.qx[i], A.qy[i], A.qz[i]};
                V3 a0, a1, b0v, b1;
                double ha, hb;
                if (d == 0) {  // links 0 and 2
                  a0 = arm.root; a1 = j1; b0v = p2; b1 = j3;
                  ha = 0.5 * arm.L[0];
                  hb = 0.5 * arm.L[2];
                } else {
                  const V3 dir = o < w.n_opts ? w.opt_dir[o] : S.cdl[e];
                  const V3 j4 = j3 + w.L4 * dir;
                  const bool p03 = ((d - 1) & 1) == 0;  // links 0 and 3, else 1 and 3
                  a0 = p03 ? arm.root : j1;
                  a1 = p03 ? j1 : p2;
                  b0v = j3;
                  b1 = j4;
                  ha = 0.5 * (p03 ? arm.L[0] : arm.L[1]);
                  hb = 0.5 * w.L4;
                }
                const bool ok =
                    rpd::links_clear_screen(a0, a1, b0v, b1, ha * (1.0 + 1e-9), hb * (1.0 + 1e-9),
                                            min_sep) ||
                    !(rpd::seg_seg_distance(a0, a1, b0v, b1) < min_sep);
                if (!ok) atomicOr(&S.cflag[e], 1 << (8 + d));
              }
              __syncthreads();
              if (prof) { A.prof[22] += clock64() - t_e; t_e = clock64(); }
              // E3: verdicts (the first trail option whose walk and links are
              // clear, like append_trail) and this thread's (metric, ordinal) min
              bool hit = false;
              for (int x = tid; x < nb; x += kBpcThreads) {
                const int e = S.qs[x];
                const int fl = S.cflag[e];
                if (fl & ((1 << 30) | 3)) continue;
                int opt = -1;
                bool h = false;
                if (!A.four) {
                  h = !((fl >> 8) & 1);
                } else if (!((fl >> 8) & 1)) {
                  for (int o = 0; o < nopt && !h; ++o)
                    if (!((fl >> (2 + o)) & 1) && !((fl >> (9 + 2 * o)) & 3)) {
                      h = true;
                      opt = o;
                    }
                }
                const double mm = S.qm[e];
                const long long od = S.qo[e];
                if (h && wik_better(mm, od, bm, bo)) {
                  bm = mm;
                  bo = od;
                  bopt = opt;
                  atomicMin(bound0 + par, metric_bits(mm));
                }
                hit |= h;
              }
              if (prof) A.prof[14] += 1;
              if (__syncthreads_or(hit)) break;
            }
            if (prof) A.prof[12] += nq;
          }
          __syncthreads();
          if (tid == 0) {
            S.nq = 0;
            S.nl = 0;
            S.mlo = metric_bits(1e308);
            S.mhi = 0ull;
          }
          if (tid < 256) S.hist[tid] = 0;
          __syncthreads();
          if (prof) {
            cs += s1 - s0;
            ce += clock64() - s1;
          }
          if (!more) break;
        }
        long long c2 = prof ? clock64() : 0;
        // ---- R: this CTA's winner -> its slot; cluster barrier; reduce
        for (int off = 16; off > 0; off >>= 1) {
          const double om = __shfl_down_sync(FULL, bm, off);
          const long long oo = __shfl_down_sync(FULL, bo, off);
          const int op = __shfl_down_sync(FULL, bopt, off);
          if (wik_better(om, oo, bm, bo)) {
            bm = om;
            bo = oo;
            bopt = op;
          }
        }
        if (lane == 0) S.wb[warp] = WikBest{bm, bo, bopt, -1, -1, V3{0, 0, 0}};
        __syncthreads();
        if (tid == 0) {
          WikBest b = S.wb[0];
          for (int q = 1; q < kBpcWarps; ++q)
            if (wik_better(S.wb[q].metric, S.wb[q].ord, b.metric, b.ord)) b = S.wb[q];
          BpcSlot sl{b.metric, b.ord, b.opt, -1, -1, V3{0, 0, 0}};
          if (b.ord != LLONG_MAX) {
            const int a = static_cast<int>(b.ord / ncj);
            sl.i = li[a];
            sl.j = lj[b.ord - static_cast<long long>(a) * ncj];
            sl.p1 = arm.root + arm.L[0] * V3{A.qx[sl.i], A.qy[sl.i], A.qz[sl.i]};
          }
          S.slot[par] = sl;
          if (rank == 0 && A.cancel) S.cancel[par] = *reinterpret_cast<const volatile int*>(A.cancel);
        }
        long long c3 = prof ? clock64() : 0;
        cluster.sync();
        long long c4 = prof ? clock64() : 0;
        if (A.cancel && cancel0[par]) {
          rebuild();
          if (rank == 0 && tid == 0) A.state[3] = 1;
          cluster.sync();
          return;
        }
        if (warp == 0) {
          // lane r reads CTA r's winner; the lanes reduce (metric, ordinal)
          double rm = 1e308;
          long long ro = LLONG_MAX;
          int rr = -1;
          if (lane < CL) {
            const BpcSlot* o = cluster.map_shared_rank(&S.slot[par], lane);
            rm = o->metric;
            ro = o->ord;
            rr = lane;
          }
          for (int off = 16; off > 0; off >>= 1) {
            const double om = __shfl_down_sync(FULL, rm, off);
            const long long oo = __shfl_down_sync(FULL, ro, off);
            const int orr = __shfl_down_sync(FULL, rr, off);
            if (wik_better(om, oo, rm, ro)) {
              rm = om;
              ro = oo;
              rr = orr;
            }
          }
          if (lane == 0) S.win_rank = ro != LLONG_MAX ? rr : -1;
        }
        __syncthreads();
        if (tid == 0) {
          BpcSlot b{1e308, LLONG_MAX, -1, -1, -1, V3{0, 0, 0}};
          if (S.win_rank >= 0) b = *cluster.map_shared_rank(&S.slot[par], S.win_rank);
          int ok = 0;
          if (b.ord != LLONG_MAX) {
            const V3 s0 = arm.L[0] * V3{A.qx[b.i], A.qy[b.i], A.qz[b.i]};
            const V3 s1 = arm.L[1] * V3{A.qx[b.j], A.qy[b.j], A.qz[b.j]};
            const V3 j1 = arm.root + s0;
            S.prev[0] = j1;
            S.prev[1] = j1 + s1;
            S.prev[2] = s0;
            S.prev[3] = s1;
            S.prev[4] = t > 0 ? w.wp : S.wk;
            if (rank == 0) {
              BpWin W;
              W.i = b.i;
              W.j = b.j;
              W.opt = b.opt;
              W.n_opts = w.n_opts;
              W.p1 = b.p1;
              W.wp = w.wp;
              W.opt_dir[0] = w.opt_dir[0];
              W.opt_dir[1] = w.opt_dir[1];
              A.win[k] = W;
              A.relax[k] = f;
              A.kind[k] = t > 0 ? 1 : 0;
              if (t > 0) A.wps[k] = w.wp;
              A.state[0] = 1;
            }
            ok = 1;
          }
          S.found = ok;
        }
        __syncthreads();
        found = S.found != 0;
        if (prof) {
          const long long c5 = clock64();
          A.prof[0] += c1 - c0;  // F: lists
          A.prof[10] += cs;      // S: screening
          A.prof[11] += ce;      // E: sort + evaluation waves
          A.prof[2] += c2 - c1;  // S + E
          A.prof[3] += c4 - c3;  // cluster barrier
          A.prof[4] += c5 - c4;  // reduce + publish
          A.prof[6] += 1;
          A.prof[7] += static_cast<long long>(nci) * ncj;
        }
      }
    }
    if (!found) {
      if (rank == 0 && tid == 0) {
        A.state[1] = k;
        A.state[2] = 0;
      }
      rebuild();
      cluster.sync();
      return;
    }
  }
  if (rank == 0 && tid == 0) {
    A.state[1] = -1;
    A.state[2] = 1;
  }
  rebuild();
  cluster.sync();
}

// ---------------------------------------------------------------------------
// Single-pose operations (one thread): refinement and trail folding.

/// mode 0: exact_refine_8dof, 1: _8dof_triangle, 2: exact_refine_6dof
/// (src/arm_model.cpp:258-324); the math lives in rp_refine.cuh.
__global__ void k_refine(ArmDev arm, DevPose ap, V3 target, int mode, PoseOpOut* out) {
  PoseOpOut r{};
  r.pose = ap;
  r.status = refine_pose(arm, r.pose, target, mode, &r.msg);
  *out = r;
}
/// k_refine of a pose already on the device (a materialised solution).
__global__ void k_refine_from(ArmDev arm, const DevPose* ap, V3 target, int mode, PoseOpOut* out) {
  PoseOpOut r{};
  r.pose = *ap;
  r.status = refine_pose(arm, r.pose, target, mode, &r.msg);
  *out = r;
}

/// append_trail on a 3-segment chain (src/path_planner.cpp:127-150).
__global__ void k_append_trail(rpd::GridView g, ArmDev arm, DevPose ch, int n_opts, V3 o0, V3 o1,
                               int n, PoseOpOut* out) {
  PoseOpOut r{};
  r.status = RP_E_NO_PATH;
  const V3 opts[2] = {o0, o1};
  for (int o = 0; o <= n_opts; ++o) {
    const V3 dir = o < n_opts ? opts[o] : rpd::normalized(ch.seg[2]);
    DevPose cand = ch;
    cand.nseg = 4;
    cand.seg[3] = arm.L[3] * dir;
    cand.qidx[3] = -1;
    build_chain(arm, cand);
    if (!pose_limits_ok(arm, cand)) continue;
    if (!rpd::walk_clear(g, cand.joints[3], cand.joints[4], n)) continue;
    if (!pose_self_free(cand, 2.0 * arm.arm_radius)) continue;
    r.status = 0;
    r.pose = cand;
    break;
  }
  *out = r;
}

// ---------------------------------------------------------------------------
// Unfold (src/path_planner.cpp:405-484)

/// smoothness_ok over consecutive poses of the sequence, relax 1.
__global__ void k_seq_smooth(const DevPose* __restrict__ seq, int count, double sm1, double sm2,
                             int* __restrict__ rough) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s + 1 >= count) return;
  const DevPose& a = seq[s];
  const DevPose& b = seq[s + 1];
  if (!(rpd::norm(b.joints[1] - a.joints[1]) <= sm1 && rpd::norm(b.joints[2] - a.joints[2]) <= sm2))
    atomicExch(rough, 1);
}

// ---------------------------------------------------------------------------
// validate_plan / check_pose (src/validate.cpp:20-108): every check of the
// independent plan validator as one launch, one thread per item: the poses
// of the executable sequence, the tracked point at each waypoint, each
// consecutive pose pair's smoothness and the unfold seam. The host turns
// the flags (and the measured values the messages print) into the report.

struct VPose {
  double len_diff[4];  // |s_j| - L_j
  unsigned char len_bad[4], off_hit[4], seg_hit[4];
  unsigned char limits_bad, self_bad, _pad[6];
};

struct VArgs {
  rpd::GridView g;
  ArmDev arm;
  const DevPose* seq;  // full_sequence()
  int nseq;
  const DevPose* poses;  // plan.poses (tracked points)
  const V3* wps;
  const double* relax;       // per waypoint
  const double* pair_relax;  // per sequence pair
  int m;
  int n;
  double s4tol, eps_wp, j1, j2;
  int has_unfold;
  VPose* out_pose;
  double* out_dist;     // per waypoint: tracked-point distance
  uint8_t* out_wp_bad;  // per waypoint
  uint8_t* out_pair_bad;
  uint8_t* out_seam_bad;
};

__global__ void k_validate_plan(VArgs a) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < a.nseq) {
    const DevPose& p = a.seq[t];
    VPose r{};
    for (int j = 0; j < p.nseg; ++j) {
      const double len = rpd::norm(p.seg[j]);
      const double expected = a.arm.L[j];
      const double tol = (j == 3) ? a.s4tol : 1e-9 * fmax(1.0, expected);
      r.len_diff[j] = len - expected;
      r.len_bad[j] = fabs(len - expected) > tol ? 1 : 0;
      V3 from = p.joints[j];
      if (p.has_elbows) {
        const int n_off = max(1, static_cast<int>(ceil(rpd::norm(p.elbows[j] - p.joints[j]) /
                                                      fmax(1e-12, expected / a.n))));
        r.off_hit[j] = rpd::walk_clear(a.g, p.joints[j], p.elbows[j], n_off) ? 0 : 1;
        from = p.elbows[j];
      }
      r.seg_hit[j] = rpd::walk_clear(a.g, from, p.joints[j + 1], a.n) ? 0 : 1;
    }
    r.limits_bad = pose_limits_ok(a.arm, p) ? 0 : 1;
    r.self_bad = pose_self_free(p, 2.0 * a.arm.arm_radius) ? 0 : 1;
    a.out_pose[t] = r;
    return;
  }
  t -= a.nseq;
  if (t < a.m) {
    const DevPose& p = a.poses[t];
    const int tj = p.nseg < 3 ? p.nseg : 3;  // PoseChain::tracked_point
    const double dist = rpd::norm(p.joints[tj] - a.wps[t]);
    a.out_dist[t] = dist;
    a.out_wp_bad[t] = dist > a.eps_wp * a.relax[t] + 1e-9 ? 1 : 0;
    return;
  }
  t -= a.m;
  if (t < a.nseq - 1) {
    const DevPose& p = a.seq[t];
    const DevPose& q = a.seq[t + 1];
    const double f = a.pair_relax[t];
    const bool ok = rpd::norm(q.joints[1] - p.joints[1]) <= a.j1 * f + 1e-12 &&
                    rpd::norm(q.joints[2] - p.joints[2]) <= a.j2 * f + 1e-12;
    a.out_pair_bad[t] = ok ? 0 : 1;
    return;
  }
  t -= (a.nseq > 0 ? a.nseq - 1 : 0);
  if (t == 0 && a.has_unfold) {
    const DevPose& u = a.seq[a.nseq - a.m];  // unfold.back() sits just before poses[1]
    const DevPose& p0 = a.poses[0];
    *a.out_seam_bad = rpd::norm(u.joints[u.nseg] - p0.joints[p0.nseg]) > 1e-9 ? 1 : 0;
  }
}

/// pose_clear / pose_valid for a batch (replan collide scan).
__global__ void k_pose_check(rpd::GridView g, ArmDev arm, const DevPose* __restrict__ poses, int count,
                             int n, double spacing, int full, int* __restrict__ first_bad) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= count) return;
  const bool ok = full ? pose_valid(g, arm, poses[k], n, spacing)
                       : pose_clear(g, poses[k], n, spacing);
  if (!ok) atomicMin(first_bad, k);
}

// ---------------------------------------------------------------------------
// mean_polyline_deviation (src/path_planner.cpp:76-87) over solution tip paths.

__device__ inline double polyline_dist(V3 p, const V3* poly, int np) {
  double best = rpd::norm(p - poly[0]);
  for (int i = 0; i + 1 < np; ++i) {
    const double d = rpd::point_to_segment(p, poly[i], poly[i + 1]);
    best = d < best ? d : best;  // std::min(best, d)
  }
  return best;
}

/// Scores every solution of a set: tip path = [lead?] + the first 3 sample
/// blocks of the pose (candidate_tip_path / the replan tip list).
__global__ void k_score_solutions(SolveDev a, const SurvDev* __restrict__ sv,
                                  const long long* __restrict__ keys, int64_t count,
                                  const V3* __restrict__ poly, int npoly, int has_lead, V3 lead,
                                  unsigned long long* __restrict__ dev_bits,
                                  long long* __restrict__ ordinal, long long ord_base) {
  extern __shared__ V3 spoly[];
  for (int k = threadIdx.x; k < npoly; k += blockDim.x) spoly[k] = poly[k];
  __syncthreads();
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= count) return;
  const long long key = keys[t];
  const long long p = key / a.B;
  const int bi = static_cast<int>(key - p * a.B);
  const int s = static_cast<int>(p / a.Q);
  const int j = static_cast<int>(p - static_cast<long long>(s) * a.Q);
  const SurvDev h = sv[s];
  const ArmDev& arm = a.arm;
  const V3 dir2 = qvec(a, j);
  V3 link2 = h.p1;
  if (arm.off[1] > 0.0) {
    const rpd::FrameStep st2 = rpd::advance_frame(h.frame, dir2);
    link2 = h.p1 + arm.off[1] * rpd::m_col(st2.after_azimuth, 0);
  }
  const V3 p2 = link2 + arm.L[1] * dir2;
  const V3 from[3] = {h.link_start, link2, p2};
  const V3 to[3] = {h.p1, p2, a.bpts[bi]};
  double acc = 0.0;
  int cnt = 0;
  if (has_lead) {
    acc += polyline_dist(lead, spoly, npoly);
    ++cnt;
  }
  for (int l = 0; l < 3; ++l) {
    const V3 diff = to[l] - from[l];
    for (int k = 1; k <= a.n; ++k) {
      acc += polyline_dist(rpd::walk_sample(from[l], diff, k, a.n), spoly, npoly);
      ++cnt;
    }
  }
  const double dev = acc / static_cast<double>(cnt);
  dev_bits[t] = __double_as_longlong(dev);
  ordinal[t] = ord_base + t;
}

/// The failed path as a per-launch table in the kernel-parameter constant
/// bank: segment start a, direction ab = b - a, end a + 1*ab and |ab|^2,
/// all computed on the host with the same fp64 operations the reference
/// performs inside point_to_segment; plus an fp32 copy (a, ab, 1/|ab|^2) for
/// the screening pass and the screen's error-bound constant.
constexpr int kPolyMax = 32;  // segments (waypoints <= 33)
struct PolyTable {
  int nseg;
  float screen_c;  // max_i (|a_i|_1 + |ab_i|_1), rounded up
  double p0x, p0y, p0z;
  double ax[kPolyMax], ay[kPolyMax], az[kPolyMax];
  double bx[kPolyMax], by[kPolyMax], bz[kPolyMax];
  double ex[kPolyMax], ey[kPolyMax], ez[kPolyMax];
  double len2[kPolyMax];
  float fax[kPolyMax], fay[kPolyMax], faz[kPolyMax];
  float fbx[kPolyMax], fby[kPolyMax], fbz[kPolyMax];
  float finv[kPolyMax];
};

/// point_to_segment^2 for table segment i exactly as the reference computes
/// it (src/path_planner.cpp point_to_segment): the clamp of t = dot/len2 is
/// decided from the signs of dot and len2 - dot (dot <= 0 gives t in
/// {-0, 0}, dot >= len2 gives t = 1), so the IEEE division runs only for
/// interior projections, where it is computed exactly as written.
__device__ __forceinline__ double seg_sq_exact(V3 p, const PolyTable& T, int i) {
  const double wx = p.x - T.ax[i], wy = p.y - T.ay[i], wz = p.z - T.az[i];
  const double len2 = T.len2[i];
  if (len2 <= 1e-30) return (wx * wx + wy * wy) + wz * wz;
  const double dot = (wx * T.bx[i] + wy * T.by[i]) + wz * T.bz[i];
  if (dot <= 0.0) return (wx * wx + wy * wy) + wz * wz;
  if (dot >= len2) {
    const double dx = p.x - T.ex[i], dy = p.y - T.ey[i], dz = p.z - T.ez[i];
    return (dx * dx + dy * dy) + dz * dz;
  }
  const double t = rpd::clampd(dot / len2, 0.0, 1.0);
  const double dx = p.x - (T.ax[i] + t * T.bx[i]);
  const double dy = p.y - (T.ay[i] + t * T.by[i]);
  const double dz = p.z - (T.az[i] + t * T.bz[i]);
  return (dx * dx + dy * dy) + dz * dz;
}

/// polyline_dist with identical results. sqrt is monotone and correctly
/// rounded, so min_i sqrt(d_i^2) == sqrt(min_i d_i^2), and only the minimum
/// VALUE matters, so any segment that provably cannot hold it may be
/// skipped. A branch-free fp32 pass computes every segment's squared
/// distance s_i to within e of the exact one (error analysis in DESIGN.md:
/// e <= 10 u M^2, u = 2^-24, M = |p|_1 + |a_i|_1 + |ab_i|_1; the clamped
/// projection parameter only enters to second order); the segment holding
/// the true minimum then has s_i <= min_j s_j + 2e, so the exact fp64
/// formula runs only on segments inside that band (tol = 64 u M^2, >3x
/// margin) -- usually one or two per point.
template <int NS>
__device__ __forceinline__ double polyline_dist_tab(V3 p, const PolyTable& T) {
  double best;
  {
    const double dx = p.x - T.p0x, dy = p.y - T.p0y, dz = p.z - T.p0z;
    best = (dx * dx + dy * dy) + dz * dz;
  }
  const float px = static_cast<float>(p.x), py = static_cast<float>(p.y),
              pz = static_cast<float>(p.z);
  // branch-free over NS >= nseg entries (the host pads the table with a
  // far-away segment whose screen value is +inf), so the segments interleave
  float sq[NS];
  float lo = INFINITY;
#pragma unroll
  for (int i = 0; i < NS; ++i) {
    const float wx = px - T.fax[i], wy = py - T.fay[i], wz = pz - T.faz[i];
    const float dot = fmaf(wz, T.fbz[i], fmaf(wy, T.fby[i], wx * T.fbx[i]));
    const float t = fminf(fmaxf(dot * T.finv[i], 0.0f), 1.0f);
    const float dx = fmaf(-t, T.fbx[i], wx), dy = fmaf(-t, T.fby[i], wy),
                dz = fmaf(-t, T.fbz[i], wz);
    sq[i] = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
    lo = fminf(lo, sq[i]);
  }
  const float m = (fabsf(px) + fabsf(py)) + fabsf(pz) + T.screen_c;
  const float thr = lo + (64.0f * 5.9604645e-8f) * 1.0001f * (m * m);
  unsigned cand = 0;
#pragma unroll
  for (int i = 0; i < NS; ++i) cand |= (sq[i] <= thr ? 1u : 0u) << i;
  while (cand) {
    const int i = __ffs(cand) - 1;
    cand &= cand - 1;
    const double e = seg_sq_exact(p, T, i);
    best = e < best ? e : best;
  }
  return sqrt(best);
}

/// Running deviation sums that depend on the survivor row only: the lead
/// point (replan tip lists) and the n samples of segment 1, accumulated in
/// the reference's order, so k_score_solutions_tab continues each sum
/// exactly where the per-solution loop would be.
template <int NS>
__global__ void __launch_bounds__(256) k_score_rows(SolveDev a, const SurvDev* __restrict__ sv, int S1,
                                                    const __grid_constant__ PolyTable T, int has_lead,
                                                    V3 lead, double* __restrict__ row_acc) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S1) return;
  const SurvDev& h = sv[s];
  double acc = 0.0;
  if (has_lead) acc += polyline_dist_tab<NS>(lead, T);
  const V3 diff = h.p1 - h.link_start;
  for (int k = 1; k <= a.n; ++k) acc += polyline_dist_tab<NS>(rpd::walk_sample(h.link_start, diff, k, a.n), T);
  row_acc[s] = acc;
}

/// k_score_solutions with the polyline in the parameter bank (npoly - 1 <=
/// kPolyMax) and the row-only prefix of each sum from k_score_rows;
/// bit-identical deviations. (A per-segment bounding-box skip measured
/// 2.2x slower: it breaks the unrolled constant-operand stream.)
template <int NS>
__global__ void __launch_bounds__(256) k_score_solutions_tab(
    SolveDev a, const SurvDev* __restrict__ sv, const long long* __restrict__ keys, int64_t count,
    const __grid_constant__ PolyTable T, int has_lead, const double* __restrict__ row_acc,
    unsigned long long* __restrict__ dev_bits, long long* __restrict__ ordinal, long long ord_base) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= count) return;
  const long long key = keys[t];
  const long long p = key / a.B;
  const int bi = static_cast<int>(key - p * a.B);
  const int s = static_cast<int>(p / a.Q);
  const int j = static_cast<int>(p - static_cast<long long>(s) * a.Q);
  const SurvDev& h = sv[s];
  const ArmDev& arm = a.arm;
  const V3 dir2 = qvec(a, j);
  V3 link2 = h.p1;
  if (arm.off[1] > 0.0) {
    const rpd::FrameStep st2 = rpd::advance_frame(h.frame, dir2);
    link2 = h.p1 + arm.off[1] * rpd::m_col(st2.after_azimuth, 0);
  }
  const V3 p2 = link2 + arm.L[1] * dir2;
  double acc = row_acc[s];
  const int cnt = (has_lead ? 1 : 0) + 3 * a.n;
  {
    const V3 diff = p2 - link2;
    for (int k = 1; k <= a.n; ++k) acc += polyline_dist_tab<NS>(rpd::walk_sample(link2, diff, k, a.n), T);
  }
  {
    const V3 b = a.bpts[bi];
    const V3 diff = b - p2;
    for (int k = 1; k <= a.n; ++k) acc += polyline_dist_tab<NS>(rpd::walk_sample(p2, diff, k, a.n), T);
  }
  const double dev = acc / static_cast<double>(cnt);
  dev_bits[t] = __double_as_longlong(dev);
  ordinal[t] = ord_base + t;
}

/// Scores explicit point lists (shortcut tip paths).
__global__ void k_score_lists(const V3* __restrict__ pts, const int* __restrict__ offs, int count,
                              const V3* __restrict__ poly, int npoly,
                              unsigned long long* __restrict__ dev_bits, long long* __restrict__ ordinal) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count) return;
  double acc = 0.0;
  const int b = offs[t], e = offs[t + 1];
  for (int k = b; k < e; ++k) acc += polyline_dist(pts[k], poly, npoly);
  dev_bits[t] = __double_as_longlong(acc / static_cast<double>(e - b));
  ordinal[t] = t;
}

/// mean_polyline_deviation of one point list: block-parallel over points,
/// summed in the reference's sequential order by thread 0.
__global__ void k_mean_dev(const V3* __restrict__ pts, int npts, const V3* __restrict__ poly,
                           int npoly, double* __restrict__ scratch, double* out) {
  for (int k = threadIdx.x; k < npts; k += blockDim.x) scratch[k] = polyline_dist(pts[k], poly, npoly);
  __syncthreads();
  if (threadIdx.x == 0) {
    double acc = 0.0;
    for (int k = 0; k < npts; ++k) acc += scratch[k];
    *out = acc / static_cast<double>(npts);
  }
}

// ---------------------------------------------------------------------------
// Host wrappers

/// waypoint_ik's candidate cones (src/path_planner.cpp:190-193) as a
/// conservative dot-product bound: cos of the half angle widened by 1e-9 rad
/// (and 1e-12 on the cosine). Every candidate that passes the move tests is
/// at least 1e-9 rad inside the reference's cone, so the filter only drops
/// directions the reference's own tests would reject.
static double cone_cos(double half_angle) {
  return std::cos(std::min(half_angle + 1e-9, kPi)) - 1e-12;
}

/// folded_pose with glibc sin/cos (bit-identical to the reference's).
HostPose folded_pose_host(rp_ctx* ctx, const rp_arm& arm) {
  (void)ctx;
  const DevPose h = folded_pose(
      make_arm_dev(arm),
      V3{arm.fold_plane_normal[0], arm.fold_plane_normal[1], arm.fold_plane_normal[2]},
      arm.fold_flex);
  return host_pose_from_dev(h);
}

double mean_polyline_deviation(rp_ctx* ctx, const std::vector<V3>& pts, const std::vector<V3>& poly) {
  require(!pts.empty() && !poly.empty(), RP_E_INVALID_PARAMETER, "empty polyline");
  DevBuf<V3> dp(pts.size(), ctx->stream), dq(poly.size(), ctx->stream);
  DevBuf<double> sc(pts.size(), ctx->stream), o(1, ctx->stream);
  copy_to_device(ctx, dp.p, pts.data(), pts.size() * sizeof(V3));
  copy_to_device(ctx, dq.p, poly.data(), poly.size() * sizeof(V3));
  launch(ctx, "score", k_mean_dev, dim3(1), dim3(256), 0, static_cast<const V3*>(dp.p),
         static_cast<int>(pts.size()), static_cast<const V3*>(dq.p), static_cast<int>(poly.size()),
         sc.p, o.p);
  double h = 0.0;
  copy_to_host(ctx, &h, o.p, sizeof(h));
  return h;
}

DevPose to_dev(const HostPose& h) {
  DevPose d{};
  d.nseg = h.nseg;
  d.has_elbows = h.has_elbows ? 1 : 0;
  d.no_qidx = h.no_qidx ? 1 : 0;
  for (int k = 0; k < 4; ++k) d.qidx[k] = k < h.nseg ? h.qidx[k] : -1;
  for (int k = 0; k < h.nseg; ++k) {
    d.seg[k] = h.seg[k];
    d.elbows[k] = h.elbows[k];
  }
  for (int k = 0; k <= h.nseg; ++k) d.joints[k] = h.joints[k];
  d.s4dev = h.s4dev;
  d.n_wp_links = 0;
  return d;
}

Planner::Planner(rp_ctx* c, const rp_arm& a, const rp_quiver* qv, const rp_grid* gr,
                 const rp_reach_params& r, const rp_path_params& p)
    : ctx(c), arm(a), q(qv), g(gr), rp(r), pp_in(p) {
  HostSpan span_("Planner::Planner");
  ad = make_arm_dev(a);
  pp = resolve_path_params(p, a, r);
  n = r.n_samples;
  spacing = nominal_spacing(a, r);
  cudaStream_t st = ctx->stream;
  wik_blocks = ctx->sm_count;
  opout.alloc(1, st);
  // pinned read-back slot: one per context, reused by every planner
  if (!ctx->pinned || ctx->pinned_bytes < sizeof(WikResult)) {
    if (ctx->pinned) RP_CUDA(cudaFreeHost(ctx->pinned));
    ctx->pinned_bytes = std::max<size_t>(sizeof(WikResult), 4096);
    RP_CUDA(cudaMallocHost(&ctx->pinned, ctx->pinned_bytes));
  }
  h_result = static_cast<WikResult*>(ctx->pinned);
}

Planner::~Planner() {}

void Planner::ensure_scratch() {
  // the sequenced waypoint_ik's and the cooperative pass's scratch (the
  // cluster pass keeps its lists in shared memory): allocated on first use
  if (scratch_ready) return;
  cudaStream_t st = ctx->stream;
  const int qw = (q->n + 31) / 32 + 1;
  ibits.alloc(qw, st);
  jbits.alloc(qw, st);
  cj.alloc(q->n + 1, st);
  ci.alloc(q->n + 1, st);
  ci_by_index.alloc(q->n + 1, st);
  ci_fast.alloc(q->n + 1, st);
  counts.alloc(2, st);
  block_best.alloc(wik_blocks, st);
  done.alloc(1, st);
  done.zero();
  result.alloc(1, st);
  scratch_ready = true;
}

bool Planner::waypoint_ik(V3 wp, const HostPose& prev, double relax, const Trail& tr,
                          const HostPose* bias, HostPose* out) {
  WikDev w{};
  w.g = g->view();
  w.arm = ad;
  w.n = n;
  w.Q = q->n;
  w.qx = q->d_soa;
  w.qy = q->d_soa + q->n;
  w.qz = q->d_soa + 2 * static_cast<size_t>(q->n);
  w.spacing = spacing;
  w.wp = wp;
  w.prev_j1 = prev.joints[1];
  w.prev_j2 = prev.joints[2];
  w.eps = pp.eps_wp * relax + 1e-12;
  w.j1max = pp.j1 * relax + 1e-12;
  w.j2max = pp.j2 * relax + 1e-12;
  w.sm1 = pp.j1 * relax + 1e-12;
  w.sm2 = pp.j2 * relax + 1e-12;
  w.has_bias = bias ? 1 : 0;
  if (bias) {
    w.bias_j1 = bias->joints[1];
    w.bias_j2 = bias->joints[2];
  }
  w.four = arm.n_segments == 4;
  w.n_opts = 0;
  if (tr.has_back) w.opt_dir[w.n_opts++] = tr.back;
  if (tr.has_fwd) w.opt_dir[w.n_opts++] = tr.fwd;
  w.L4 = arm.n_segments == 4 ? arm.lengths[3] : 0.0;
  const rpd::Limit& l2 = ad.lim[1];
  const rpd::Limit& l3 = ad.lim[2];
  w.cond2 = (ad.off[1] > 0.0 || !rpd::full_azimuth(l2) || l2.elev_min > 0.0 || l2.elev_max < kPi);
  w.cond3 = (!rpd::full_azimuth(l3) || l3.elev_min > 0.0 || l3.elev_max < kPi);
  // candidate cones (src/path_planner.cpp:184-194); none for offset arms
  w.filter_j = ad.has_offsets ? 0 : 1;
  double cone1 = 0, cone2 = 0;
  V3 u1{0, 0, 1}, u2{0, 0, 1};
  if (w.filter_j) {
    auto chord_to_angle = [](double chord) {
      return 2.0 * std::asin(std::clamp(chord / 2.0, 0.0, 1.0));
    };
    const double ang1 = chord_to_angle(w.j1max / arm.lengths[0]) + 1e-9;
    const double ang2 = chord_to_angle((w.j1max + w.j2max) / arm.lengths[1]) + 1e-9;
    u1 = rpd::normalized(prev.seg[0]);
    u2 = rpd::normalized(prev.seg[1]);
    require(std::abs(rpd::norm(u1) - 1.0) <= 1e-9 && std::abs(rpd::norm(u2) - 1.0) <= 1e-9,
            RP_E_INVALID_PARAMETER, "cone axis must be unit");
    cone1 = cone_cos(std::min(kPi, ang1) + 1e-12);
    cone2 = cone_cos(std::min(kPi, ang2) + 1e-12);
  }
  ensure_scratch();
  WikScratch s{ibits.p, jbits.p, cj.p, ci.p, ci_by_index.p, counts.p, block_best.p, done.p,
               result.p, wik_blocks};
  launch(ctx, "wik_filter", k_wik_filter, dim3(nblk(q->n, 256)), dim3(256), 0, w, cone1, cone2, u1,
         u2, ibits.p, jbits.p, ci_by_index.p);
  launch(ctx, "wik_compact", k_wik_compact, dim3(1), dim3(1024), 0, w, s);
  launch(ctx, "wik_pairs", k_wik_pairs, dim3(wik_blocks), dim3(256), 0, w, s);
  RP_CUDA(cudaMemcpyAsync(h_result, result.p, sizeof(WikResult), cudaMemcpyDeviceToHost,
                          ctx->stream));
  RP_CUDA(cudaStreamSynchronize(ctx->stream));
  ++wik_calls;
  if (!h_result->found) return false;
  *out = host_pose_from_dev(h_result->pose);
  return true;
}

bool Planner::backward_pass_device(const std::vector<V3>& wps, const HostPose& anchor,
                                   const std::vector<double>& factors, bool cloud,
                                   double cloud_radius, const HostPose* fixed_first,
                                   const HostPose* bias, BpOut* out) {
  HostSpan span_("Planner::backward_pass_device");
  if (!bp_launch(wps, anchor, factors, cloud, cloud_radius, fixed_first, bias)) return false;
  return bp_finish(out);
}

bool Planner::bp_launch(const std::vector<V3>& wps, const HostPose& anchor,
                        const std::vector<double>& factors, bool cloud, double cloud_radius,
                        const HostPose* fixed_first, const HostPose* bias) {
  HostSpan span_("bp launch");
  if (!use_device_pass || factors.size() > static_cast<size_t>(kBpMaxFactors) || wps.size() < 2)
    return false;
  cudaStream_t st = ctx->stream;
  const size_t smem = 2 * static_cast<size_t>(q->n) * sizeof(int);
  // the cluster pass (k_bp_cluster) takes coaxial limit-free arms on
  // generated quivers (up to 65535 directions: 16-bit list entries; the
  // lists hold what shared memory allows, ~20k entries each, and a cone
  // larger than that falls back below); RP_BP_COOP=1 forces the
  // cooperative grid pass (Q <= 16384: two int arrays of Q in shared memory)
  static const bool force_coop = std::getenv("RP_BP_COOP") != nullptr;
  // shared memory left for the lists: the opt-in maximum per block minus
  // the kernel's static and BpcShared parts (once per device)
  static std::mutex cap_mutex;
  static std::map<int, size_t> list_room;
  size_t room = 0;
  {
    std::lock_guard<std::mutex> lock(cap_mutex);
    auto it = list_room.find(ctx->device);
    if (it == list_room.end()) {
      int optin = 0;
      RP_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
      cudaFuncAttributes fa{};
      RP_CUDA(cudaFuncGetAttributes(&fa, k_bp_cluster));
      const size_t fixed = sizeof(BpcShared) + fa.sharedSizeBytes + 256;
      it = list_room.emplace(ctx->device, static_cast<size_t>(optin) > fixed ? optin - fixed : 0).first;
    }
    room = it->second;
  }
  int list_cap = std::min<int>(q->n, static_cast<int>(room / (2 * sizeof(unsigned short))) & ~7);
  const bool cluster = !force_coop && !ad.any_limit && !ad.has_offsets && q->n_rings > 0 &&
                       q->n_rings <= kBpcRings && q->n <= 65535 && list_cap >= 1024;
  if (!cluster && q->n > 16384) return false;
  if (const char* e = std::getenv("RP_BPC_LIST_CAP"))  // tests: force the overflow fallback
    list_cap = std::min(list_cap, std::max(64, std::atoi(e)));
  if (!cluster && bp_blocks == 0) {
    // kernel attribute + occupancy: once per device and shared-memory size
    // (the attribute is per device; planners may run on several threads)
    static std::mutex attr_mutex;
    static std::map<int, std::pair<size_t, int>> configured;  // device -> (smem, per_sm)
    std::lock_guard<std::mutex> lock(attr_mutex);
    auto& cfg = configured[ctx->device];
    if (cfg.first < smem) {
      RP_CUDA(cudaFuncSetAttribute(k_backward_pass, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
      RP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&cfg.second, k_backward_pass,
                                                            kBpThreads, smem));
      cfg.first = smem;
    }
    const int per_sm = cfg.second;
    if (per_sm < 1) {
      use_device_pass = false;
      return false;
    }
    // The pass is latency-bound (a short serial chain per attempt): a few
    // dozen resident blocks keep every phase parallel while making the grid
    // barriers cheaper and the grid's L1 reuse higher.
    const char* env = std::getenv("RP_BP_BLOCKS");
    bp_blocks = std::min(ctx->sm_count * per_sm, env ? std::max(1, std::atoi(env)) : 64);
    if (bp_blocks_cap > 0) bp_blocks = std::min(bp_blocks, bp_blocks_cap);
    bp_bar.alloc(2, st);
    bp_best.alloc(bp_blocks, st);
  }
  const int m = static_cast<int>(wps.size());
  BpArgs A{};
  A.g = g->view();
  A.arm = ad;
  A.n = n;
  A.Q = q->n;
  A.four = arm.n_segments == 4;
  const rpd::Limit& l2 = ad.lim[1];
  const rpd::Limit& l3 = ad.lim[2];
  A.cond2 = (ad.off[1] > 0.0 || !rpd::full_azimuth(l2) || l2.elev_min > 0.0 || l2.elev_max < kPi);
  A.cond3 = (!rpd::full_azimuth(l3) || l3.elev_min > 0.0 || l3.elev_max < kPi);
  A.filter_j = ad.has_offsets ? 0 : 1;
  A.qx = q->d_soa;
  A.qy = q->d_soa + q->n;
  A.qz = q->d_soa + 2 * static_cast<size_t>(q->n);
  A.spacing = spacing;
  A.L4 = arm.n_segments == 4 ? arm.lengths[3] : 0.0;
  A.pj1 = pp.j1;
  A.pj2 = pp.j2;
  A.eps_wp = pp.eps_wp;
  A.m = m;
  A.nf = static_cast<int>(factors.size());
  auto chord_to_angle = [](double chord) {
    return 2.0 * std::asin(std::clamp(chord / 2.0, 0.0, 1.0));
  };
  for (int fi = 0; fi < A.nf; ++fi) {
    const double f = factors[fi];
    A.factors[fi] = f;
    const double j1max = pp.j1 * f + 1e-12, j2max = pp.j2 * f + 1e-12;
    A.cone1[fi] = cone_cos(std::min(kPi, chord_to_angle(j1max / arm.lengths[0]) + 1e-9) + 1e-12);
    A.cone2[fi] =
        cone_cos(std::min(kPi, chord_to_angle((j1max + j2max) / arm.lengths[1]) + 1e-9) + 1e-12);
  }
  A.cloud = cloud ? 1 : 0;
  A.cloud_radius = cloud_radius;
  for (int t = 0; t < 8; ++t) {
    const double a = 2.0 * kPi * t / 8.0;
    A.ring_c[t] = std::cos(a);
    A.ring_s[t] = std::sin(a);
  }
  A.has_fixed = fixed_first ? 1 : 0;
  if (fixed_first) A.fixed_first = to_dev(*fixed_first);
  A.has_bias = bias ? 1 : 0;
  if (bias) A.bias = to_dev(*bias);
  // The pass's inputs and outputs in one device block, filled by one upload
  // and read back by one copy: [state][wps][poses][relax][kind][win]
  auto al = [](size_t x) { return (x + 15) & ~size_t{15}; };
  const size_t o_wps = al(4 * sizeof(int));
  const size_t o_poses = o_wps + al(m * sizeof(V3));
  const size_t o_relax = o_poses + al(m * sizeof(DevPose));
  const size_t o_kind = o_relax + al(m * sizeof(double));
  const size_t o_win = o_kind + al(m * sizeof(int));
  const size_t io_bytes = o_win + al(m * sizeof(BpWin));
  if (bp_io.n < io_bytes) bp_io.alloc(io_bytes, st);
  copy_to_device_fill(ctx, bp_io.p, io_bytes, [&](unsigned char* h) {
    std::memset(h, 0, io_bytes);
    std::memcpy(h + o_wps, wps.data(), m * sizeof(V3));
    const DevPose da = to_dev(anchor);
    std::memcpy(h + o_poses + (m - 1) * sizeof(DevPose), &da, sizeof(DevPose));
    for (int k = 0; k < m; ++k) {
      const double one = 1.0;
      std::memcpy(h + o_relax + k * sizeof(double), &one, sizeof(double));
    }
    std::memset(h + o_win, 0xFF, m * sizeof(BpWin));  // i = -1: not published
  });
  unsigned char* io = bp_io.p;
  if (!cluster) bp_bar.zero();
  A.wps = reinterpret_cast<V3*>(io + o_wps);
  A.poses = reinterpret_cast<DevPose*>(io + o_poses);
  A.relax = reinterpret_cast<double*>(io + o_relax);
  A.kind = reinterpret_cast<int*>(io + o_kind);
  if (!cluster) ensure_scratch();
  A.ibits = ibits.p;
  A.jbits = jbits.p;
  A.ci_by_index = ci_by_index.p;
  A.ci_fast = ci_fast.p;
  A.win = reinterpret_cast<BpWin*>(io + o_win);
  A.walk1 = (!ad.any_limit && !ad.has_offsets) ? walk1_device() : walk1_bits.p;
  A.block_best = bp_best.p;
  A.bar = bp_bar.p;
  A.state = reinterpret_cast<int*>(io);
  A.cancel = cancel_flag;
  static const bool profile = std::getenv("RP_PROFILE_PASS") != nullptr;
  DevBuf<long long>& prof = bp_prof;
  if (profile) {
    prof.alloc(24, st);
    prof.zero();
    A.prof = prof.p;
  }
  cudaEvent_t ev = nullptr;
  if (cluster) {
    A.nrings = q->n_rings;
    A.ring_off = q->d_ring_off;
    A.qring_c = q->d_ring_c;
    A.qring_s = q->d_ring_s;
    A.qf = q->d_qf;
    A.list_cap = list_cap;
    const size_t csmem = sizeof(BpcShared) + 2 * static_cast<size_t>(list_cap) * sizeof(unsigned short);
    static const int ctas = [] {
      const char* e = std::getenv("RP_BPC_CTAS");
      const int c = e ? std::atoi(e) : 16;
      return c >= 16 ? 16 : (c >= 8 ? 8 : (c >= 4 ? 4 : (c >= 2 ? 2 : 1)));
    }();
    {
      // per device and shared-memory size (planners may run on several threads)
      static std::mutex attr_mutex;
      static std::map<int, size_t> configured;
      std::lock_guard<std::mutex> lock(attr_mutex);
      size_t& have = configured[ctx->device];
      if (have < csmem) {
        RP_CUDA(cudaFuncSetAttribute(k_bp_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(csmem)));
        RP_CUDA(cudaFuncSetAttribute(k_bp_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed,
                                     1));
        have = csmem;
      }
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(ctas);
    cfg.blockDim = dim3(kBpcThreads);
    cfg.dynamicSmemBytes = csmem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = ctas;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    launch_begin(ctx, "backward_pass", &ev);
    RP_CUDA(cudaLaunchKernelEx(&cfg, k_bp_cluster, A));
    launch_end(ctx, "backward_pass", ev);
  } else {
    void* args[] = {&A};
    launch_begin(ctx, "backward_pass", &ev);
    RP_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_backward_pass), dim3(bp_blocks),
                                        dim3(kBpThreads), args, smem, st));
    launch_end(ctx, "backward_pass", ev);
  }
  bp_pend = BpPending{true, m, o_wps, o_poses, o_relax, o_kind, o_win, cluster};
  return true;
}

bool Planner::bp_finish(BpOut* out) {
  HostSpan span_("bp finish");
  require(bp_pend.active, RP_E_INTERNAL, "no backward pass in flight");
  const BpPending pd = bp_pend;
  bp_pend.active = false;
  const int m = pd.m;
  const size_t o_wps = pd.o_wps, o_poses = pd.o_poses, o_relax = pd.o_relax, o_kind = pd.o_kind,
               o_win = pd.o_win;
  const bool cluster = pd.cluster;
  unsigned char* io = bp_io.p;
  static const bool profile = std::getenv("RP_PROFILE_PASS") != nullptr;
  DevBuf<long long>& prof = bp_prof;
  // the state and the pass's outputs in one read-back
  int hs[4];
  {
    std::vector<unsigned char> h(o_win);
    copy_to_host(ctx, h.data(), io, o_win);
    std::memcpy(hs, h.data(), sizeof(hs));
    out->poses.resize(m);
    out->relax.resize(m);
    out->kind.resize(m);
    out->wps.resize(m);
    std::memcpy(out->wps.data(), h.data() + o_wps, m * sizeof(V3));
    std::memcpy(out->poses.data(), h.data() + o_poses, m * sizeof(DevPose));
    std::memcpy(out->relax.data(), h.data() + o_relax, m * sizeof(double));
    std::memcpy(out->kind.data(), h.data() + o_kind, m * sizeof(int));
  }
  if (profile) {
    long long hp[24];
    copy_to_host(ctx, hp, prof.p, sizeof(hp));
    if (cluster)
      std::fprintf(stderr,
                   "[bpc] lists: arcs %lld arcs+scan %lld cycles, %lld positions | E0 %lld sort "
                   "%lld walks %lld dists %lld\n",
                   hp[16], hp[17], hp[18], hp[19], hp[20], hp[21], hp[22]);
    else
      std::fprintf(stderr, "[half] setup %lld walks %lld dists %lld cycles\n", hp[16], hp[17], hp[18]);
    std::fprintf(stderr, "[pairs] screening %lld, rank+eval %lld cycles (rank %lld, waves %lld); screened %lld\n", hp[10],
                 hp[11], hp[15], hp[14], hp[12]);
    std::fprintf(stderr,
                 "[pass] m=%d attempts=%lld pairs=%lld cyc: filter %lld compact %lld pairs %lld "
                 "wait %lld publish %lld barrier %lld | max ci-load %lld max eval %lld\n",
                 m, hp[6], hp[7], hp[0], hp[1], hp[2], hp[3], hp[4], hp[5], hp[8], hp[9]);
  }
  if (hs[3] == 2) return false;  // list overflow: the sequenced pass decides
  out->ok = hs[2] != 0;
  out->failed_index = hs[1];
  out->cancelled = hs[3] != 0;
  if (out->cancelled) {
    out->ok = false;
    return true;
  }
  return true;
}

PoseOpOut run_pose_op(Planner& P) {
  PoseOpOut h;
  copy_to_host(P.ctx, &h, P.opout.p, sizeof(PoseOpOut));
  return h;
}

HostPose Planner::refine(const HostPose& approx, V3 target, int mode) {
  HostSpan span_("Planner::refine");
  launch(ctx, "refine", k_refine, dim3(1), dim3(1), 0, ad, to_dev(approx), target, mode,
         opout.p);
  PoseOpOut r = run_pose_op(*this);
  if (r.status) fail(r.status, refine_msg(r.msg));
  HostPose h = host_pose_from_dev(r.pose);
  h.waypoints = approx.waypoints;  // PoseChain out = approx
  return h;
}

const uint32_t* Planner::walk1_device() {
  cudaStream_t st = ctx->stream;
  if (walk1_ready) return walk1_ptr;
  const double key[4] = {arm.root[0], arm.root[1], arm.root[2], arm.lengths[0]};
  auto& c = g->w1;
  std::lock_guard<std::mutex> lock(*g->s2_mutex);
  const bool current = c.bits && c.version == g->version && !g->exported;
  const bool hit = current && c.q == q && c.n == n && std::memcmp(c.key, key, sizeof(key)) == 0;
  if (current && !hit) {
    // another arm's verdicts are cached for this grid version (planners may
    // be reading them): compute this planner's own copy
    walk1_bits.alloc((q->n + 31) / 32 + 1, st);
    launch(ctx, "walk1", k_walk1_bits, dim3(nblk(q->n, 128)), dim3(128), 0, g->view(), ad,
           static_cast<const double*>(q->d_soa), static_cast<const double*>(q->d_soa + q->n),
           static_cast<const double*>(q->d_soa + 2 * static_cast<size_t>(q->n)), q->n, n,
           walk1_bits.p);
    walk1_ptr = walk1_bits.p;
    walk1_ready = true;
    return walk1_ptr;
  }
  if (!hit) {
    const size_t words = (q->n + 31) / 32 + 1;
    if (c.words < words) {
      if (c.bits) RP_CUDA(cudaFreeAsync(c.bits, st));
      RP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&c.bits), words * sizeof(uint32_t), st));
      c.words = words;
    } else if (c.ready) {
      RP_CUDA(cudaStreamWaitEvent(st, c.ready, 0));  // readers of the old verdicts
    }
    launch(ctx, "walk1", k_walk1_bits, dim3(nblk(q->n, 128)), dim3(128), 0, g->view(), ad,
           static_cast<const double*>(q->d_soa), static_cast<const double*>(q->d_soa + q->n),
           static_cast<const double*>(q->d_soa + 2 * static_cast<size_t>(q->n)), q->n, n, c.bits);
    if (!c.ready) RP_CUDA(cudaEventCreateWithFlags(&c.ready, cudaEventDisableTiming));
    RP_CUDA(cudaEventRecord(c.ready, st));
    std::memcpy(c.key, key, sizeof(key));
    c.n = n;
    c.q = q;
    c.version = g->version;
  } else {
    RP_CUDA(cudaStreamWaitEvent(st, c.ready, 0));  // computed on another stream
  }
  walk1_ptr = c.bits;
  walk1_ready = true;
  return walk1_ptr;
}

void Planner::refine_launch(const DevPose* d_approx, V3 target, int mode) {
  launch(ctx, "refine", k_refine_from, dim3(1), dim3(1), 0, ad, d_approx, target, mode, opout.p);
}

HostPose Planner::refine_result(const PoseOpOut& r, const HostPose& approx) {
  if (r.status) fail(r.status, refine_msg(r.msg));
  HostPose h = host_pose_from_dev(r.pose);
  h.waypoints = approx.waypoints;  // PoseChain out = approx
  return h;
}

bool Planner::append_trail(const HostPose& chain3, const Trail& tr, HostPose* out) {
  V3 o[2] = {V3{0, 0, 0}, V3{0, 0, 0}};
  int no = 0;
  if (tr.has_back) o[no++] = tr.back;
  if (tr.has_fwd) o[no++] = tr.fwd;
  launch(ctx, "trail", k_append_trail, dim3(1), dim3(1), 0, g->view(), ad, to_dev(chain3), no, o[0],
         o[1], n, opout.p);
  PoseOpOut r = run_pose_op(*this);
  if (r.status) return false;
  HostPose h = host_pose_from_dev(r.pose);
  h.waypoints = chain3.waypoints;
  const V3 diff = h.joints[4] - h.joints[3];
  for (int k = 1; k <= n; ++k) h.waypoints.push_back(rpd::walk_sample(h.joints[3], diff, k, n));
  *out = h;
  return true;
}

std::optional<std::vector<HostPose>> Planner::interpolate(const HostPose* from_or_null,
                                                          const HostPose& to, int base_steps,
                                                          bool* rotated_valid) {
  HostSpan span_("Planner::interpolate");
  // The joint-space interpolation is evaluated with the host's glibc
  // transcendentals, exactly as the reference does: the folded zig-zag puts
  // azimuths at +-pi, so the direction of wrap_angle(qb - qa) -- and with it
  // every interpolated pose -- is decided by the sign of last-ulp noise in
  // sin/atan2 (CUDA's libm differs in the last ulp). The device does the
  // bulk of the work: collision / limit / self-collision validity of every
  // pose and the smoothness of every consecutive pair.
  cudaStream_t st = ctx->stream;
  HostPose from;
  DevPose dfrom;
  if (from_or_null) {
    from = *from_or_null;
    dfrom = to_dev(from);
  } else {
    // build_unfold (src/path_planner.cpp:458-484): rotate the folded pose so
    // its first segment and fold plane co-align with the triangle pose.
    const V3 fn{arm.fold_plane_normal[0], arm.fold_plane_normal[1], arm.fold_plane_normal[2]};
    const DevPose fold = folded_pose(ad, fn, arm.fold_flex);
    const DevPose tri = to_dev(to);
    const V3 u1f = rpd::normalized(fold.seg[0]);
    const V3 u1t = rpd::normalized(tri.seg[0]);
    const V3 nf = pose_plane_normal(fold);
    const V3 nt = pose_plane_normal(tri);
    rpd::M3 a, b;
    const V3 ca[3] = {u1f, rpd::cross(nf, u1f), nf};
    const V3 cb[3] = {u1t, rpd::cross(nt, u1t), nt};
    for (int c = 0; c < 3; ++c) {
      a.a[0][c] = ca[c].x; a.a[1][c] = ca[c].y; a.a[2][c] = ca[c].z;
      b.a[0][c] = cb[c].x; b.a[1][c] = cb[c].y; b.a[2][c] = cb[c].z;
    }
    const rpd::M3 rot = rpd::m_mul(b, m_transpose(a));
    dfrom = DevPose{};
    dfrom.nseg = fold.nseg;
    dfrom.no_qidx = 1;  // path_planner.cpp:479
    for (int k = 0; k < fold.nseg; ++k) {
      dfrom.seg[k] = m_vec(rot, fold.seg[k]);
      dfrom.qidx[k] = -1;
    }
    build_chain(ad, dfrom);
    from = host_pose_from_dev(dfrom);
    from.waypoints.clear();
    // the rotated pose's validity is checked with the first interpolation
    // (same launch, same read-back): index 0 of the checked range
  }
  bool check_from = from_or_null == nullptr;
  double qa_az[4], qa_el[4], qb_az[4], qb_el[4];
  if (!to_angles(ad, dfrom, qa_az, qa_el) || !to_angles(ad, to_dev(to), qb_az, qb_el)) {
    if (check_from) {  // the reference checks the rotated pose first
      const bool ok = valid_poses(&dfrom, 1) < 0;
      if (rotated_valid) *rotated_valid = ok;
      if (!ok) return std::nullopt;
    }
    fail(RP_E_DEGENERATE_INPUT, "zero-length segment");
  }
  for (int steps = std::max(1, base_steps); steps <= 4096; steps *= 2) {
    std::vector<DevPose> seq(steps + 1);
    seq[0] = dfrom;
    seq[steps] = to_dev(to);
    for (int s = 1; s < steps; ++s) {
      const double t = static_cast<double>(s) / steps;
      double az[4], el[4];
      for (int j = 0; j < ad.nseg; ++j) {
        az[j] = qa_az[j] + t * rpd::wrap_angle(qb_az[j] - qa_az[j]);
        el[j] = qa_el[j] + t * (qb_el[j] - qa_el[j]);
      }
      seq[s] = from_angles(ad, az, el);
    }
    // flags (first invalid pose, smoothness failure) and the sequence in
    // one block and one upload
    const size_t o_seq = 16, bytes = o_seq + (steps + 1) * sizeof(DevPose);
    DevBuf<unsigned char> blk(bytes, st);
    {
      std::vector<unsigned char> h(bytes, 0);
      const int init[2] = {INT_MAX, 0};
      std::memcpy(h.data(), init, sizeof(init));
      std::memcpy(h.data() + o_seq, seq.data(), (steps + 1) * sizeof(DevPose));
      copy_to_device(ctx, blk.p, h.data(), bytes);
    }
    int* flags = reinterpret_cast<int*>(blk.p);
    const DevPose* dseq = reinterpret_cast<const DevPose*>(blk.p + o_seq);
    // poses 1..steps-1 (and 0, the rotated folded pose, on the first round)
    const int c0 = check_from ? 0 : 1;
    if (steps - c0 > 0)
      launch(ctx, "unfold", k_pose_check, dim3(nblk(steps - c0, 64)), dim3(64), 0, g->view(), ad,
             dseq + c0, steps - c0, n, spacing, 1, flags);
    launch(ctx, "unfold", k_seq_smooth, dim3(nblk(steps, 128)), dim3(128), 0, dseq, steps + 1,
           pp.j1 * 1.0 + 1e-12, pp.j2 * 1.0 + 1e-12, flags + 1);
    int hf[2];
    copy_to_host(ctx, hf, flags, sizeof(hf));
    if (check_from) {
      const bool ok = hf[0] != 0;  // index 0 = the rotated pose
      if (rotated_valid) *rotated_valid = ok;
      if (!ok) return std::nullopt;
      check_from = false;
    }
    if (hf[0] != INT_MAX) return std::nullopt;
    if (!hf[1]) {
      std::vector<HostPose> out;
      out.push_back(from);
      for (int s = 1; s < steps; ++s) {
        HostPose h = host_pose_from_dev(seq[s]);
        h.waypoints.clear();
        out.push_back(h);
      }
      out.push_back(to);
      return out;
    }
  }
  return std::nullopt;
}

int Planner::first_colliding(const std::vector<HostPose>& poses, const rp_grid* grid) {
  if (poses.empty()) return -1;
  cudaStream_t st = ctx->stream;
  std::vector<DevPose> d(poses.size());
  for (size_t k = 0; k < poses.size(); ++k) d[k] = to_dev(poses[k]);
  DevBuf<DevPose> dp(d.size(), st);
  copy_to_device(ctx, dp.p, d.data(), d.size() * sizeof(DevPose));
  DevBuf<int> first(1, st);
  const int init = INT_MAX;
  copy_to_device(ctx, first.p, &init, sizeof(int));
  launch(ctx, "pose_check", k_pose_check, dim3(nblk(static_cast<int64_t>(d.size()), 64)), dim3(64),
         0, grid->view(), ad, static_cast<const DevPose*>(dp.p), static_cast<int>(d.size()), n,
         spacing, 0, first.p);
  int h = INT_MAX;
  copy_to_host(ctx, &h, first.p, sizeof(int));
  return h == INT_MAX ? -1 : h;
}

int Planner::valid_poses(const DevPose* poses, int count) {
  cudaStream_t st = ctx->stream;
  DevBuf<DevPose> dp(count, st);
  copy_to_device(ctx, dp.p, poses, count * sizeof(DevPose));
  DevBuf<int> first(1, st);
  const int init = INT_MAX;
  copy_to_device(ctx, first.p, &init, sizeof(int));
  launch(ctx, "pose_check", k_pose_check, dim3(nblk(count, 64)), dim3(64), 0, g->view(), ad,
         static_cast<const DevPose*>(dp.p), count, n, spacing, 1, first.p);
  int h = INT_MAX;
  copy_to_host(ctx, &h, first.p, sizeof(int));
  return h == INT_MAX ? -1 : h;
}

// ---- head / tail selection of the ranked order (rank_by_deviation) ---------
constexpr int kRankBinBits = 12;
constexpr int kRankBins = 1 << kRankBinBits;

__global__ void k_key_range(const unsigned long long* __restrict__ k, int64_t n,
                            unsigned long long* range) {
  unsigned long long lo = ~0ull, hi = 0ull;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const unsigned long long v = k[i];
    lo = v < lo ? v : lo;
    hi = v > hi ? v : hi;
  }
  for (int off = 16; off > 0; off >>= 1) {
    const unsigned long long a = __shfl_down_sync(0xffffffffu, lo, off);
    const unsigned long long b = __shfl_down_sync(0xffffffffu, hi, off);
    lo = a < lo ? a : lo;
    hi = b > hi ? b : hi;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(range, lo);
    atomicMax(range + 1, hi);
  }
}

__global__ void k_key_hist(const unsigned long long* __restrict__ k, int64_t n,
                           unsigned long long base, int shift, unsigned* hist) {
  __shared__ unsigned h[kRankBins];
  for (int b = threadIdx.x; b < kRankBins; b += blockDim.x) h[b] = 0;
  __syncthreads();
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    atomicAdd(&h[static_cast<int>((k[i] - base) >> shift)], 1u);
  __syncthreads();
  for (int b = threadIdx.x; b < kRankBins; b += blockDim.x)
    if (h[b]) atomicAdd(hist + b, h[b]);
}

__global__ void k_key_flags(const unsigned long long* __restrict__ k, int64_t n,
                            unsigned long long tlo, unsigned long long thi, uint8_t* flags) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) flags[i] = (k[i] <= tlo || k[i] >= thi) ? 1 : 0;
}

/// Mean polyline deviation of every solution's traversal (segments 1-3,
/// the reach pose's candidate_tip_path) from `poly`, as ordered bits of the
/// fp64 value, with ordinals ord_base + t (alternate_candidates' scores,
/// src/path_planner.cpp:612-663, and mean_polyline_deviation, :76-87).
void score_set_solutions(rp_ctx* ctx, rp_solution_set* set, const std::vector<V3>& poly,
                         const V3* dpoly, bool lead, V3 lead_pt, unsigned long long* dev_bits,
                         long long* ord, long long ord_base) {
  cudaStream_t st = ctx->stream;
  const int64_t nsol = set->n_solutions;
  const long long ns = ord_base;
  ensure_keys(set);
  static const bool no_tab = std::getenv("RP_SCORE_PLAIN") != nullptr;
  if (poly.size() >= 2 && poly.size() - 1 <= static_cast<size_t>(kPolyMax) && !no_tab) {
    PolyTable T{};
    T.nseg = static_cast<int>(poly.size()) - 1;
    T.p0x = poly[0].x;
    T.p0y = poly[0].y;
    T.p0z = poly[0].z;
    for (int i = 0; i < T.nseg; ++i) {
      const V3 a = poly[i], ab = poly[i + 1] - poly[i];
      const V3 e = a + 1.0 * ab;
      T.ax[i] = a.x; T.ay[i] = a.y; T.az[i] = a.z;
      T.bx[i] = ab.x; T.by[i] = ab.y; T.bz[i] = ab.z;
      T.ex[i] = e.x; T.ey[i] = e.y; T.ez[i] = e.z;
      T.len2[i] = rpd::sqnorm(ab);
      T.fax[i] = static_cast<float>(a.x); T.fay[i] = static_cast<float>(a.y);
      T.faz[i] = static_cast<float>(a.z);
      T.fbx[i] = static_cast<float>(ab.x); T.fby[i] = static_cast<float>(ab.y);
      T.fbz[i] = static_cast<float>(ab.z);
      T.finv[i] = T.len2[i] > 1e-30 ? static_cast<float>(1.0 / T.len2[i]) : 0.0f;
      const double c = std::fabs(a.x) + std::fabs(a.y) + std::fabs(a.z) + std::fabs(ab.x) +
                       std::fabs(ab.y) + std::fabs(ab.z);
      T.screen_c = std::max(T.screen_c, static_cast<float>(c * (1.0 + 1e-6)));
    }
    for (int i = T.nseg; i < kPolyMax; ++i) {  // screen value +inf, never a candidate
      T.fax[i] = T.fay[i] = T.faz[i] = 1e30f;
      T.fbx[i] = T.fby[i] = T.fbz[i] = T.finv[i] = 0.0f;
    }
    DevBuf<double> row_acc(std::max(1, set->S1), st);
    auto run = [&](auto rows, auto sols) {
      launch(ctx, "score", rows, dim3(nblk(std::max(1, set->S1), 256)), dim3(256), 0, set->sd,
             static_cast<const SurvDev*>(set->surv.p), set->S1, T, lead ? 1 : 0, lead_pt,
             row_acc.p);
      launch(ctx, "score", sols, dim3(nblk(nsol, 256)), dim3(256), 0, set->sd,
             static_cast<const SurvDev*>(set->surv.p), static_cast<const long long*>(set->keys.p),
             nsol, T, lead ? 1 : 0, static_cast<const double*>(row_acc.p), dev_bits, ord,
             static_cast<long long>(ns));
    };
    if (T.nseg <= 8) run(k_score_rows<8>, k_score_solutions_tab<8>);
    else if (T.nseg <= 16) run(k_score_rows<16>, k_score_solutions_tab<16>);
    else if (T.nseg <= 24) run(k_score_rows<24>, k_score_solutions_tab<24>);
    else run(k_score_rows<32>, k_score_solutions_tab<32>);
  } else {
    launch(ctx, "score", k_score_solutions, dim3(nblk(nsol, 256)), dim3(256),
           poly.size() * sizeof(V3), set->sd, static_cast<const SurvDev*>(set->surv.p),
           static_cast<const long long*>(set->keys.p), nsol, dpoly,
           static_cast<int>(poly.size()), lead ? 1 : 0, lead_pt, dev_bits, ord,
           static_cast<long long>(ns));
  }
}

/// Scores of (shortcut tip lists, solutions) against a polyline, sorted by
/// (deviation, ordinal); returns the ordinals in sorted order.
std::vector<long long> Planner::rank_by_deviation(rp_solution_set* set,
                                                  const std::vector<std::vector<V3>>& lists,
                                                  const std::vector<V3>& poly, bool lead,
                                                  V3 lead_pt, int64_t* total_out,
                                                  std::vector<long long>* tail, int head_n,
                                                  int tail_n) {
  HostSpan span_("Planner::rank_by_deviation");
  cudaStream_t st = ctx->stream;
  const int64_t ns = static_cast<int64_t>(lists.size());
  const int64_t nsol = set ? set->n_solutions : 0;
  const int64_t total = ns + nsol;
  *total_out = total;
  std::vector<long long> head;
  if (total == 0) return head;
  DevBuf<unsigned long long> dev(total, st), dev_sorted(total, st);
  DevBuf<long long> ord(total, st), ord_sorted(total, st);
  DevBuf<V3> dpoly(poly.size(), st);
  copy_to_device(ctx, dpoly.p, poly.data(), poly.size() * sizeof(V3));
  if (ns > 0) {
    std::vector<V3> pts;
    std::vector<int> offs{0};
    for (const auto& l : lists) {
      pts.insert(pts.end(), l.begin(), l.end());
      offs.push_back(static_cast<int>(pts.size()));
    }
    DevBuf<V3> dpts(pts.size() + 1, st);
    DevBuf<int> doffs(offs.size(), st);
    copy_to_device(ctx, dpts.p, pts.data(), pts.size() * sizeof(V3));
    copy_to_device(ctx, doffs.p, offs.data(), offs.size() * sizeof(int));
    launch(ctx, "score", k_score_lists, dim3(nblk(ns, 128)), dim3(128), 0,
           static_cast<const V3*>(dpts.p), static_cast<const int*>(doffs.p), static_cast<int>(ns),
           static_cast<const V3*>(dpoly.p), static_cast<int>(poly.size()), dev.p, ord.p);
  }
  if (nsol > 0)
    score_set_solutions(ctx, set, poly, static_cast<const V3*>(dpoly.p), lead, lead_pt, dev.p + ns,
                        ord.p + ns, static_cast<long long>(ns));
  const int64_t nh = std::min<int64_t>(head_n, total);
  const int64_t nt = tail ? std::min<int64_t>(tail_n, total) : 0;
  // Only the first nh and last nt of the stable (deviation, ordinal) order
  // are used: bucket the keys (4096 equal-width bins over [min, max]), keep
  // the bins that hold them and stable-sort just those candidates -- the
  // same head and tail as the full sort (ordinals ascend with the index).
  static const bool full_sort = std::getenv("RP_RANK_FULL_SORT") != nullptr;
  const unsigned long long* keys_in = dev.p;
  const long long* vals_in = ord.p;
  int64_t m = total;
  DevBuf<unsigned long long> ck;
  DevBuf<long long> cv;
  if (!full_sort && total > 65536) {
    DevBuf<unsigned long long> range(2, st);
    const unsigned long long init[2] = {~0ull, 0ull};
    copy_to_device(ctx, range.p, init, sizeof(init));
    const int gb = ctx->sm_count * 4;
    launch(ctx, "rank", k_key_range, dim3(gb), dim3(256), 0,
           static_cast<const unsigned long long*>(dev.p), total, range.p);
    unsigned long long hr[2];
    copy_to_host(ctx, hr, range.p, sizeof(hr));
    const unsigned long long span = hr[1] - hr[0];
    const int bits = span ? 64 - __builtin_clzll(span) : 0;
    const int shift = std::max(0, bits - kRankBinBits);
    DevBuf<unsigned> hist(kRankBins, st);
    hist.zero();
    launch(ctx, "rank", k_key_hist, dim3(gb), dim3(256), 0,
           static_cast<const unsigned long long*>(dev.p), total, hr[0], shift, hist.p);
    std::vector<unsigned> hh(kRankBins);
    copy_to_host(ctx, hh.data(), hist.p, kRankBins * sizeof(unsigned));
    int blo = 0, bhi = kRankBins - 1;
    int64_t clo = 0, chi = 0;
    for (; blo < kRankBins; ++blo)
      if ((clo += hh[blo]) >= nh) break;
    if (nt > 0) {
      for (; bhi >= 0; --bhi)
        if ((chi += hh[bhi]) >= nt) break;
    } else {
      bhi = kRankBins;  // no tail wanted
    }
    if (blo < bhi && clo + chi <= (1 << 20)) {
      const unsigned long long tlo = hr[0] + ((static_cast<unsigned long long>(blo) + 1) << shift) - 1;
      const unsigned long long thi =
          bhi < kRankBins ? hr[0] + (static_cast<unsigned long long>(bhi) << shift) : ~0ull;
      DevBuf<uint8_t> flags(total, st);
      launch(ctx, "rank", k_key_flags, dim3(nblk(total, 256)), dim3(256), 0,
             static_cast<const unsigned long long*>(dev.p), total, tlo, thi, flags.p);
      m = clo + chi;
      ck.alloc(m, st);
      cv.alloc(m, st);
      DevBuf<int> nsel(1, st);
      size_t tbs = 0;
      cub::DeviceSelect::Flagged(nullptr, tbs, dev.p, flags.p, ck.p, nsel.p, total, st);
      DevBuf<unsigned char> tsel(tbs, st);
      RP_CUDA(cub::DeviceSelect::Flagged(tsel.p, tbs, dev.p, flags.p, ck.p, nsel.p, total, st));
      RP_CUDA(cub::DeviceSelect::Flagged(tsel.p, tbs, ord.p, flags.p, cv.p, nsel.p, total, st));
      keys_in = ck.p;
      vals_in = cv.p;
    }
  }
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, keys_in, dev_sorted.p, vals_in, ord_sorted.p,
                                  static_cast<int>(m), 0, 64, st);
  DevBuf<unsigned char> tmp(tb, st);
  RP_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, keys_in, dev_sorted.p, vals_in, ord_sorted.p,
                                          static_cast<int>(m), 0, 64, st));
  head.resize(nh);
  copy_to_host(ctx, head.data(), ord_sorted.p, nh * sizeof(long long));
  if (tail) {
    tail->resize(nt);
    copy_to_host(ctx, tail->data(), ord_sorted.p + (m - nt), nt * sizeof(long long));
  }
  return head;
}

}  // namespace rp

using namespace rp;

/// Deviation scores of solutions [first, first + count) against a polyline
/// (the quantity alternate_candidates ranks by, src/path_planner.cpp:612-663).
extern "C" rp_status rp_solution_set_deviations(rp_solution_set* set, const double* poly,
                                                int32_t n_poly, int64_t first, int64_t count,
                                                double* out) {
  return guarded([&] {
    if (n_poly < 1 || first < 0 || count < 0 || first + count > set->n_solutions)
      fail(RP_E_INVALID_PARAMETER, "deviation range or polyline");
    if (count == 0) return;
    rp_ctx* ctx = set->ctx;
    cudaStream_t st = ctx->stream;
    std::vector<V3> pl(n_poly);
    std::memcpy(pl.data(), poly, n_poly * sizeof(V3));
    DevBuf<V3> dpoly(n_poly, st);
    copy_to_device(ctx, dpoly.p, pl.data(), n_poly * sizeof(V3));
    DevBuf<unsigned long long> dev(set->n_solutions, st);
    DevBuf<long long> ord(set->n_solutions, st);
    score_set_solutions(ctx, set, pl, dpoly.p, false, V3{0, 0, 0}, dev.p, ord.p, 0);
    copy_to_host(ctx, out, dev.p + first, count * sizeof(double));
  });
}

/// validate_plan (src/validate.cpp:53-108): every check on the device
/// (k_validate_plan), the report assembled here in the reference's order
/// and wording.
extern "C" rp_status rp_validate_plan(rp_ctx* ctx, const rp_arm* arm, const rp_grid* g,
                                      const rp_plan* plan, const rp_reach_params* rp,
                                      const rp_path_params* pp, rp_validation* out, char* issues,
                                      int64_t cap) {
  return guarded([&] {
    const PP ppr = resolve_path_params(*pp, *arm, *rp);
    const int n = rp->n_samples;
    const double s4tol = resolved_epsilon(*arm, *rp) + 1e-9;
    std::vector<std::string> msgs;
    int poses_checked = 0, relax_events = 0;
    const size_t m = plan->waypoints.size();
    if (plan->poses.size() != m) {
      msgs.push_back("waypoint and pose counts differ");
    } else if (plan->relax.size() != m) {
      msgs.push_back("relaxation record does not cover every waypoint");
    } else {
      const auto seq = plan->full_sequence();
      const int nseq = static_cast<int>(seq.size());
      cudaStream_t st = ctx->stream;
      std::vector<DevPose> hseq, hposes;
      for (const HostPose* p : seq) hseq.push_back(to_dev(*p));
      for (const HostPose& p : plan->poses) hposes.push_back(to_dev(p));
      const size_t unfold_len = plan->unfold.empty() ? 0 : plan->unfold.size() - 1;
      auto wp_relax = [&](size_t k) {
        if (k < unfold_len) return 1.0;
        const size_t wp = k - unfold_len;
        return wp < plan->relax.size() ? plan->relax[wp] : 1.0;
      };
      std::vector<double> pair_relax;
      for (int k = 0; k + 1 < nseq; ++k) pair_relax.push_back(std::max(wp_relax(k), wp_relax(k + 1)));
      DevBuf<DevPose> dseq(std::max(1, nseq), st), dposes(std::max<size_t>(1, m), st);
      DevBuf<V3> dw(std::max<size_t>(1, m), st);
      DevBuf<double> drelax(std::max<size_t>(1, m), st), dpair(std::max<size_t>(1, pair_relax.size()), st),
          ddist(std::max<size_t>(1, m), st);
      DevBuf<VPose> dout(std::max(1, nseq), st);
      DevBuf<uint8_t> dflags(m + pair_relax.size() + 2, st);
      if (nseq) copy_to_device(ctx, dseq.p, hseq.data(), nseq * sizeof(DevPose));
      if (m) {
        copy_to_device(ctx, dposes.p, hposes.data(), m * sizeof(DevPose));
        copy_to_device(ctx, dw.p, plan->waypoints.data(), m * sizeof(V3));
        copy_to_device(ctx, drelax.p, plan->relax.data(), m * sizeof(double));
      }
      if (!pair_relax.empty())
        copy_to_device(ctx, dpair.p, pair_relax.data(), pair_relax.size() * sizeof(double));
      dflags.zero();
      VArgs a{};
      a.g = g->view();
      a.arm = make_arm_dev(*arm);
      a.seq = dseq.p;
      a.nseq = nseq;
      a.poses = dposes.p;
      a.wps = dw.p;
      a.relax = drelax.p;
      a.pair_relax = dpair.p;
      a.m = static_cast<int>(m);
      a.n = n;
      a.s4tol = s4tol;
      a.eps_wp = ppr.eps_wp;
      a.j1 = ppr.j1;
      a.j2 = ppr.j2;
      a.has_unfold = plan->unfold.empty() ? 0 : 1;
      a.out_pose = dout.p;
      a.out_dist = ddist.p;
      a.out_wp_bad = dflags.p;
      a.out_pair_bad = dflags.p + m;
      a.out_seam_bad = dflags.p + m + pair_relax.size();
      const int items = nseq + static_cast<int>(m) + static_cast<int>(pair_relax.size()) + 1;
      launch(ctx, "validate", k_validate_plan, dim3(nblk(items, 64)), dim3(64), 0, a);
      std::vector<VPose> vp(nseq);
      std::vector<double> dist(m);
      std::vector<uint8_t> flags(m + pair_relax.size() + 2);
      if (nseq) copy_to_host(ctx, vp.data(), dout.p, nseq * sizeof(VPose));
      if (m) copy_to_host(ctx, dist.data(), ddist.p, m * sizeof(double));
      copy_to_host(ctx, flags.data(), dflags.p, flags.size());
      for (int k = 0; k < nseq; ++k) {
        const std::string label = "pose " + std::to_string(k);
        ++poses_checked;
        for (int j = 0; j < seq[k]->nseg; ++j) {
          if (vp[k].len_bad[j])
            msgs.push_back(label + ": segment " + std::to_string(j + 1) + " length off by " +
                           std::to_string(vp[k].len_diff[j]));
          if (seq[k]->has_elbows && vp[k].off_hit[j])
            msgs.push_back(label + ": offset link " + std::to_string(j + 1) + " collides");
          if (vp[k].seg_hit[j])
            msgs.push_back(label + ": segment " + std::to_string(j + 1) + " collides");
        }
        if (vp[k].limits_bad) msgs.push_back(label + ": joint limits violated");
        if (vp[k].self_bad) msgs.push_back(label + ": self-collision");
      }
      for (size_t k = 0; k < m; ++k) {
        if (plan->relax[k] > 1.0) ++relax_events;
        if (flags[k])
          msgs.push_back("waypoint " + std::to_string(k) + ": tracked point off by " +
                         std::to_string(dist[k]));
      }
      for (size_t k = 0; k < pair_relax.size(); ++k)
        if (flags[m + k])
          msgs.push_back("pose pair " + std::to_string(k) + "-" + std::to_string(k + 1) +
                         " exceeds the recorded smoothness bounds");
      if (!plan->unfold.empty() && flags[m + pair_relax.size()])
        msgs.push_back("unfold prefix does not end at the root-waypoint pose");
    }
    std::string all;
    for (size_t k = 0; k < msgs.size(); ++k) all += (k ? "\n" : "") + msgs[k];
    out->ok = msgs.empty() ? 1 : 0;
    out->poses_checked = poses_checked;
    out->relax_events = relax_events;
    out->n_issues = static_cast<int32_t>(msgs.size());
    out->issues_bytes = static_cast<int64_t>(all.size()) + 1;
    if (issues && cap > 0) {
      const size_t c = std::min(all.size(), static_cast<size_t>(cap - 1));
      std::memcpy(issues, all.data(), c);
      issues[c] = 0;
    }
  });
}

extern "C" rp_status rp_exact_refine(rp_ctx* ctx, const rp_arm* arm, const rp_pose* approx,
                                     const double target[3], int32_t variant, rp_pose* out) {
  return guarded([&] {
    HostPose a = from_abi(*approx, nullptr);
    const ArmDev ad = make_arm_dev(*arm);
    const int mode = a.nseg == 4 ? (variant == 1 ? 1 : 0) : 2;
    DevBuf<PoseOpOut> o(1, ctx->stream);
    launch(ctx, "refine", k_refine, dim3(1), dim3(1), 0, ad, to_dev(a),
           V3{target[0], target[1], target[2]}, mode, o.p);
    PoseOpOut r;
    copy_to_host(ctx, &r, o.p, sizeof(r));
    if (r.status) fail(r.status, refine_msg(r.msg));
    to_abi(host_pose_from_dev(r.pose), out, nullptr, 0);
  });
}
