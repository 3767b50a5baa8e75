// Path-planner device structures (src/path_planner.cpp).
#pragma once

#include "rp_reach.cuh"

namespace rp {

/// Resolved PathParams (src/path_planner.cpp:89-102).
struct PP {
  double eps_wp, d_w, slack, j1, j2;
  std::vector<double> relax;
  int unfold_steps;
};
PP resolve_path_params(const rp_path_params& pp, const rp_arm& arm, const rp_reach_params& rp);

/// One waypoint_ik call (src/path_planner.cpp:167-291), passed by value.
struct WikDev {
  rpd::GridView g;
  ArmDev arm;
  int n, Q;
  const double* qx;
  const double* qy;
  const double* qz;
  double spacing;
  V3 wp;
  V3 prev_j1, prev_j2, prev_s2dir;
  double prev_s2len;
  double eps, j1max, j2max;  // relaxed, + 1e-12 as the reference
  double sm1, sm2;           // smoothness bounds (same values)
  int has_bias;
  V3 bias_j1, bias_j2;
  int four;
  int n_opts;
  V3 opt_dir[2];
  double L4;
  int filter_j;  // conservative cone filter for segment 2 (coaxial arms)
  int cond2, cond3;
  double jbound;
  long long* prof;  // RP_PROFILE_PASS section maxima (null otherwise)
};

/// Segment-1 record of the coaxial, limit-free fast path (what the pair
/// tests read): 48 bytes instead of CiData's frame-carrying 152.
struct CiFast {
  int i;
  int ok;
  double move1;
  V3 p1;
};

struct CiData {
  int i;
  int ok;  // walk1 (and offset link) clear
  double move1;
  V3 p1, link1;
  rpd::M3 frame1;
};

struct WikBest {
  double metric;
  long long ord;
  int opt;
  // the candidate itself (fast backward pass: every block rebuilds the
  // winner's pose from these instead of re-reading the candidate arrays)
  int i, j;
  V3 p1;
};

/// A waypoint's winning candidate in the fast backward pass; the poses are
/// rebuilt from these after the pass (pose_from_win), off the serial chain.
struct BpWin {
  int i, j, opt, n_opts;  // i < 0: not published
  V3 p1, wp;
  V3 opt_dir[2];
};

struct WikResult {
  int found;
  int i, j, opt;
  double metric;
  DevPose pose;
};

/// Result of a single-pose device operation (refinement, trail folding).
struct PoseOpOut {
  int status;  // 0 ok, else rp_status
  int msg;
  DevPose pose;
};

/// Persistent backward pass (src/path_planner.cpp:322-400) in one
/// cooperative launch: everything the host loop decides is decided on the
/// device between grid barriers.
constexpr int kBpMaxFactors = 16;
struct BpArgs {
  rpd::GridView g;
  ArmDev arm;
  int n, Q, four, cond2, cond3, filter_j;
  const double* qx;
  const double* qy;
  const double* qz;
  double spacing, L4, pj1, pj2;  // resolved joint1/joint2_max_move
  double eps_wp;                 // resolved epsilon_waypoint
  int m;
  V3* wps;         // [m], cloud substitution writes back
  DevPose* poses;  // [m], poses[m-1] = anchor on entry
  double* relax;   // [m]
  int* kind;       // [m] 0 plain, 1 cloud, 2 fixed junction
  int nf;
  double factors[kBpMaxFactors];
  double cone1[kBpMaxFactors], cone2[kBpMaxFactors];  // host glibc asin, like waypoint_ik
  int cloud;
  double cloud_radius;
  double ring_c[8], ring_s[8];  // cos/sin(2*pi*t/8), host glibc
  int has_fixed, has_bias;
  DevPose fixed_first, bias;
  // scratch
  uint32_t* ibits;
  uint32_t* jbits;
  CiData* ci_by_index;
  CiFast* ci_fast;  // fast-path twin of ci_by_index
  const uint32_t* walk1;  // segment-1 clearance bitmap (fast path)
  BpWin* win;             // [m] fast path: winners, rebuilt into poses at the end
  WikBest* block_best;
  unsigned* bar;  // [2] barrier count + generation
  int* state;     // [4] found, failed_index, ok, cancelled
  const int* cancel;  // device flag set (by a host DMA) to stop the pass early; may be null
  long long* prof;  // optional [8] phase cycle counters (RP_PROFILE_PASS)
  // cluster pass (k_bp_cluster): quiver rings for the candidate cones and
  // the fp32 directions for the pair prefilter
  int nrings;
  const int* ring_off;
  const double* qring_c;  // cos / sin of the ring elevations
  const double* qring_s;
  const float4* qf;
  int list_cap;  // k_bp_cluster: entries of each shared-memory candidate list (<= Q)
};

/// Device scratch reused by every waypoint_ik call of a planner.
struct WikScratch {
  uint32_t* ibits;
  uint32_t* jbits;
  int* cj;
  CiData* ci;
  CiData* ci_by_index;
  int* counts;  // [n_ci, n_cj]
  WikBest* block_best;
  unsigned* done;
  WikResult* result;
  int max_blocks;
};

}  // namespace rp

struct rp_plan {
  std::string kind;
  std::vector<rp::V3> waypoints;
  std::vector<rp::HostPose> poses;
  std::vector<rp::HostPose> unfold;
  std::vector<double> relax;
  std::vector<std::string> notes;
  int switch_index = -1;

  /// PathPlan::full_sequence (src/path_planner.cpp:104-112)
  std::vector<const rp::HostPose*> full_sequence() const {
    std::vector<const rp::HostPose*> s;
    for (const auto& p : unfold) s.push_back(&p);
    for (size_t k = 0; k < poses.size(); ++k) {
      if (k == 0 && !unfold.empty()) continue;
      s.push_back(&poses[k]);
    }
    return s;
  }
};
