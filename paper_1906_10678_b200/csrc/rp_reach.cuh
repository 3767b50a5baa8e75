// Reach-solver device structures shared by rp_reach.cu and rp_path.cu.
#pragma once

#include "rp_internal.hpp"

namespace rp {

enum Counter {
  C_SEG1_LIMIT = 0,
  C_SEG1_REACH,
  C_SEG1_SURV,
  C_SEG2_LIMIT,
  C_SEG2_CLEAR,
  C_GAP_TESTED,
  C_GAP_PASS,
  C_JOINT_PASS,
  C_V3_CLEAR,
  C_SOLUTIONS,
  C_SHORTCUT_CAND,
  C_COUNT
};

/// Everything a search kernel needs, passed by value.
struct SolveDev {
  rpd::GridView g;
  ArmDev arm;
  int n;       // samples per segment
  int eight;   // 8DOF mode
  int Q;
  int B;
  int scanning;
  int cone_precheck;
  int disable_prune;
  int n_targets;
  double eps, coarse2, budget2, near_r, spacing, L4;
  double band_lo2;  // conservative lower bound of |v3|^2 for the gap band (prefilters)
  double dq_aff;    // floor bracket of rpd::walk_hits_affine for segment-2 walks
  V3 target;
  const double* qx;
  const double* qy;
  const double* qz;
  const V3* bpts;
  const V3* bdirs;
  const int* bcone;
  const uint8_t* walk4_ok;
  const V3* targets;  // reach-precheck targets of segment 1
};

/// Surviving segment-1 hypothesis (Seg1Hypothesis, reach_solver.hpp:49-56).
struct SurvDev {
  int i;
  int has_elbow;
  V3 p1;         // distal end of segment 1
  V3 link_start; // root, or the offset elbow
  rpd::M3 frame; // only filled with limits / offsets
};

struct BestRec {
  double len;
  long long key;
};

/// Shortcut candidate evaluated by k_shortcuts (ShortcutPath fields).
struct ShortcutRec {
  long long key;  // segment-1: i ; segment-2: (1<<62) | pair index
  int valid;
  int segment_index;
  int seg1, seg2;
  int hit;
  int has_bridge;
  int via_direct;
  int n_direct;
  int n_sub;
  V3 origin;
  V3 bridge;
  double path_length;
};

/// Device PoseChain with the recipe of its waypoint samples: waypoint block k
/// is n_wp[k] samples of the walk wp_from[k] -> wp_to[k].
struct DevPose {
  int nseg;
  int has_elbows;
  int no_qidx;  // PoseChain built without quiver indices (joint-space / folded)
  int qidx[4];
  int n_wp_links;
  int n_wp[8];
  double s4dev;
  V3 seg[4];
  V3 joints[5];
  V3 elbows[4];
  V3 wp_from[8];
  V3 wp_to[8];
};

__host__ __device__ inline rpd::V3 qvec(const SolveDev& a, int i) {
  return rpd::V3{a.qx[i], a.qy[i], a.qz[i]};
}

/// chain_from_segments (src/arm_model.cpp:134-161), incl. offset elbows.
__host__ __device__ inline void build_chain(const ArmDev& arm, DevPose& p) {
  p.joints[0] = arm.root;
  p.has_elbows = arm.has_offsets;
  if (!arm.has_offsets) {
    for (int k = 0; k < p.nseg; ++k) p.joints[k + 1] = p.joints[k] + p.seg[k];
    return;
  }
  rpd::M3 frame = arm.base;
  for (int k = 0; k < p.nseg; ++k) {
    const rpd::V3 s = p.seg[k];
    const double len = rpd::norm(s);
    const rpd::FrameStep st = rpd::advance_frame(frame, s / len);
    const rpd::V3 elbow = p.joints[k] + arm.off[k] * rpd::m_col(st.after_azimuth, 0);
    p.elbows[k] = elbow;
    p.joints[k + 1] = elbow + s;
    frame = st.frame;
  }
}

/// self_collision_free over chain_links (src/arm_model.cpp:363-388).
__host__ __device__ inline bool pose_self_free(const DevPose& p, double min_sep) {
  rpd::V3 a[8], b[8];
  int n = 0;
  for (int k = 0; k < p.nseg; ++k) {
    if (p.has_elbows && rpd::sqnorm(p.elbows[k] - p.joints[k]) > 0.0) {
      a[n] = p.joints[k]; b[n++] = p.elbows[k];
      a[n] = p.elbows[k]; b[n++] = p.joints[k + 1];
    } else {
      a[n] = p.joints[k]; b[n++] = p.joints[k + 1];
    }
  }
  for (int i = 0; i + 2 < n; ++i)
    for (int j = i + 2; j < n; ++j)
      if (rpd::seg_seg_distance(a[i], b[i], a[j], b[j]) < min_sep) return false;
  return true;
}

/// joint_limits_ok (src/arm_model.cpp:163-176, 202-212); throws-equivalent
/// zero-length segments report false.
__host__ __device__ inline bool pose_limits_ok(const ArmDev& arm, const DevPose& p) {
  if (!arm.any_limit) return true;
  rpd::M3 frame = arm.base;
  for (int k = 0; k < p.nseg; ++k) {
    const double len = rpd::norm(p.seg[k]);
    if (!(len > 0.0)) return false;
    const rpd::FrameStep st = rpd::advance_frame(frame, p.seg[k] / len);
    if (!rpd::joint_angle_within(st.theta, st.phi, st.degenerate, arm.lim[k])) return false;
    frame = rpd::m_mul(rpd::m_mul(frame, rpd::rot_z(st.theta)), rpd::rot_y(st.phi));
  }
  return true;
}

/// vectors_to_joint_angles (src/arm_model.cpp:163-176)
__host__ __device__ inline bool to_angles(const ArmDev& arm, const DevPose& p, double* az, double* el) {
  rpd::M3 frame = arm.base;
  for (int k = 0; k < p.nseg; ++k) {
    const double len = rpd::norm(p.seg[k]);
    if (!(len > 0.0)) return false;
    const rpd::FrameStep st = rpd::advance_frame(frame, p.seg[k] / len);
    az[k] = st.theta;
    el[k] = st.phi;
    frame = rpd::m_mul(rpd::m_mul(frame, rpd::rot_z(st.theta)), rpd::rot_y(st.phi));
  }
  return true;
}

/// joint_angles_to_vectors (src/arm_model.cpp:178-193)
__host__ __device__ inline DevPose from_angles(const ArmDev& arm, const double* az, const double* el) {
  DevPose p{};
  p.nseg = arm.nseg;
  p.no_qidx = 1;  // joint_angles_to_vectors builds the chain without indices
  rpd::M3 frame = arm.base;
  for (int j = 0; j < arm.nseg; ++j) {
    frame = rpd::m_mul(rpd::m_mul(frame, rpd::rot_z(az[j])), rpd::rot_y(el[j]));
    p.seg[j] = arm.L[j] * rpd::m_col(frame, 2);
    p.qidx[j] = -1;
  }
  build_chain(arm, p);
  return p;
}

HostPose host_pose_from_dev(const DevPose& d);
DevPose to_dev(const HostPose& h);

}  // namespace rp

/// Device-resident SolutionSet (inc/reachplan/reach_solver.hpp:95-101):
/// solutions stay as a bit set over (segment-1 survivor, segment-2 index,
/// backward index) in canonical order; poses are materialised on request.
struct rp_solution_set {
  rp_ctx* ctx = nullptr;
  const rp_quiver* quiver = nullptr;
  rp_arm arm{};
  rp_reach_params rp{};
  rp::SolveDev sd{};
  double target[3] = {0, 0, 0};
  int S1 = 0;
  int part = 0, parts = 1;  // a part of a split solve (solve_reach)
  rp::DevBuf<rp::SurvDev> surv;
  std::vector<int> surv_i;     // segment-1 quiver index per survivor row (read lazily: surv_i_of)
  rp::DevBuf<int> surv_idx_d;  // the same on the device (k_compact_small's list)
  bool surv_i_ready = false;
  int B = 0;
  // backward points, directions, the target, cone indices and walk4 flags
  // (SolveDev bpts / bdirs / targets / bcone / walk4_ok point into it)
  rp::DevBuf<unsigned char> bblock;
  std::vector<rp::V3> h_bpts, h_bdirs;
  std::vector<int> h_bcone;
  int64_t n_pairs = 0;
  rp::DevBuf<uint32_t> sol_bits;
  int64_t n_solutions = 0;
  rp::DevBuf<long long> keys;  // canonical (pair * B + bi), lazily compacted
  bool keys_ready = false;
  std::vector<rp::HostShortcut> shortcuts;
  rp_solve_stats stats{};
  long long best_key = -1;
  double best_len = 0.0;
};

namespace rp {
/// solve_reach into a fresh set (throws Fail).
/// solve_reach (src/reach_solver.cpp:480-546); part / parts > 1 solves the
/// survivor rows [S1 * part / parts, S1 * (part + 1) / parts) only (the
/// reference's worker split, src/reach_solver.cpp:503-516, by rows instead
/// of j so that the parts' keys concatenate in canonical order): segment-1
/// counters are the whole prune's, segment-2 counters, keys, the best
/// solution and the segment-2 shortcuts the part's, and segment-1 shortcuts
/// belong to part 0.
rp_solution_set* solve_reach(rp_ctx* ctx, const rp_arm& arm, const rp_quiver* q, const rp_grid* g,
                             V3 target, const rp_reach_params& rp, int part = 0, int parts = 1);
void ensure_keys(rp_solution_set* s);
/// Materialise solutions by canonical ordinal into device poses.
void materialize_solutions(rp_solution_set* s, const long long* d_ordinals_or_null,
                           const long long* h_keys, int64_t n, DevPose* d_out);
HostPose solution_pose(rp_solution_set* s, int64_t ordinal);
DevPose solution_dev_pose(rp_solution_set* s, int64_t ordinal);
/// select_solution; returns kind and ordinal (throws no_solution on empty).
rp_chosen select(const rp_solution_set* s);
/// revalidate_solution (src/reach_solver.cpp:458-476) over every solution of
/// the set, against `grid` (null: the solve's grid).
struct RevalidateOut {
  int64_t n_bad = 0, first = -1;
  int reason = 0;  // of the first failure: 1 band, 2 limits, 3 self, 4 sample, 5 closure
};
RevalidateOut revalidate(rp_solution_set* s, const rp_grid* grid);
/// The canonical ordinal of a solution key, counted on the device into
/// *d_rank (stream order, no synchronisation).
void launch_rank_of_key(const rp_solution_set* s, long long key, unsigned long long* d_rank);
std::vector<V3> dev_pose_waypoints(const DevPose& p);
}  // namespace rp
