// Host orchestration of the path planner over the device kernels.
#pragma once

#include "rp_path.cuh"

#include <optional>
#include <string>
#include <vector>

namespace rp {

/// TrailContext (inc/reachplan/path_planner.hpp:51-54)
struct Trail {
  bool has_back = false, has_fwd = false;
  V3 back{0, 0, 0}, fwd{0, 0, 0};
};

/// Planner state for one (arm, quiver, grid, params) tuple: owns the
/// device scratch reused by every waypoint_ik call.
struct Planner {
  rp_ctx* ctx;
  rp_arm arm;
  const rp_quiver* q;
  const rp_grid* g;
  rp_reach_params rp;
  rp_path_params pp_in;  // as given (workers build their own Planner from it)
  ArmDev ad;
  PP pp;
  int n;
  double spacing;
  int wik_blocks = 0;
  int64_t wik_calls = 0;
  DevBuf<uint32_t> ibits, jbits;
  DevBuf<int> cj, counts;
  DevBuf<CiData> ci, ci_by_index;
  DevBuf<CiFast> ci_fast;
  DevBuf<uint32_t> walk1_bits;  // unused when walk1_device() serves the pass
  bool walk1_ready = false;
  const uint32_t* walk1_ptr = nullptr;
  /// The grid's cached segment-1 verdicts from the root (k_walk1_bits), in
  /// this planner's stream order.
  const uint32_t* walk1_device();
  DevBuf<WikBest> block_best;
  DevBuf<unsigned> done;
  DevBuf<WikResult> result;
  DevBuf<PoseOpOut> opout;
  bool scratch_ready = false;
  void ensure_scratch();
  WikResult* h_result = nullptr;

  Planner(rp_ctx* c, const rp_arm& a, const rp_quiver* qv, const rp_grid* gr,
          const rp_reach_params& r, const rp_path_params& p);
  ~Planner();
  Planner(const Planner&) = delete;
  Planner& operator=(const Planner&) = delete;

  bool waypoint_ik(V3 wp, const HostPose& prev, double relax, const Trail& tr,
                   const HostPose* bias, HostPose* out);
  HostPose refine(const HostPose& approx, V3 target, int mode);
  /// refine split around one read-back: launch on a device pose (result in
  /// opout), then turn the read PoseOpOut into the refined pose (or throw).
  void refine_launch(const DevPose* d_approx, V3 target, int mode);
  HostPose refine_result(const PoseOpOut& r, const HostPose& approx);
  bool append_trail(const HostPose& chain3, const Trail& tr, HostPose* out);
  /// from == nullptr: build_unfold (rotated folded pose); else interpolate_poses.
  std::optional<std::vector<HostPose>> interpolate(const HostPose* from, const HostPose& to,
                                                   int base_steps, bool* rotated_valid = nullptr);
  int first_colliding(const std::vector<HostPose>& poses, const rp_grid* grid);
  /// pose_valid over a batch on the device: first invalid index or -1.
  int valid_poses(const DevPose* poses, int count);

  /// Whole backward pass in one persistent cooperative kernel. Returns
  /// false (nothing done) when the configuration exceeds its limits; then
  /// the caller runs the host-sequenced pass.
  struct BpOut {
    bool ok = false;
    int failed_index = -1;
    std::vector<DevPose> poses;
    std::vector<double> relax;
    std::vector<int> kind;
    std::vector<V3> wps;
    bool cancelled = false;
  };
  bool backward_pass_device(const std::vector<V3>& wps, const HostPose& anchor,
                            const std::vector<double>& factors, bool cloud, double cloud_radius,
                            const HostPose* fixed_first, const HostPose* bias, BpOut* out);
  DevBuf<unsigned char> bp_io;  // a pass's inputs + outputs (backward_pass_device)
  DevBuf<long long> bp_prof;    // RP_PROFILE_PASS counters
  /// backward_pass_device split around the kernel: bp_launch enqueues the
  /// pass on this planner's stream (false: not supported, nothing done),
  /// bp_finish waits for it and reads the result (false: the sequenced pass
  /// must decide). Several planners' passes can be in flight at once.
  struct BpPending {
    bool active = false;
    int m = 0;
    size_t o_wps = 0, o_poses = 0, o_relax = 0, o_kind = 0, o_win = 0;
    bool cluster = false;
  };
  BpPending bp_pend;
  bool bp_launch(const std::vector<V3>& wps, const HostPose& anchor,
                 const std::vector<double>& factors, bool cloud, double cloud_radius,
                 const HostPose* fixed_first, const HostPose* bias);
  bool bp_finish(BpOut* out);
  DevBuf<unsigned> bp_bar;
  DevBuf<WikBest> bp_best;
  int bp_blocks = 0;
  int bp_blocks_cap = 0;  // > 0: at most this many blocks (concurrent passes)
  bool use_device_pass = true;
  /// device flag polled by the cooperative pass (set to stop it; null: never)
  const int* cancel_flag = nullptr;
  std::vector<long long> rank_by_deviation(rp_solution_set* set,
                                           const std::vector<std::vector<V3>>& lists,
                                           const std::vector<V3>& poly, bool lead, V3 lead_pt,
                                           int64_t* total, std::vector<long long>* tail,
                                           int head_n, int tail_n);
};

HostPose folded_pose_host(rp_ctx* ctx, const rp_arm& arm);
double mean_polyline_deviation(rp_ctx* ctx, const std::vector<V3>& pts, const std::vector<V3>& poly);

rp_plan* plan_reach_then_path(rp_ctx* ctx, const rp_arm& arm, const rp_quiver* q, const rp_grid* g,
                              V3 target, const rp_reach_params& rp, const rp_path_params& pp);

}  // namespace rp
