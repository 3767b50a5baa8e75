// TEST INFRASTRUCTURE ONLY — the parity oracle, never the product.
//
// A C-ABI harness over the UNMODIFIED reference reachplan sources, compiled
// in place from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libreachplan_ref.so. It stands in for the reference CLI
// (src/cli.cpp, whose CLI11 dependency is absent) so that tests/, bench.py's
// cpu_baseline / --impl reference legs and __graft_entry__.smoke() can call
// the reference on exactly the inputs the CUDA path gets. POD parameter
// structs are shared with the product header for convenience only.
#include "reachplan_b200.h"

#include "reachplan/io.hpp"
#include "reachplan/motion.hpp"
#include "reachplan/oracle.hpp"
#include "reachplan/path_planner.hpp"
#include "reachplan/pipeline.hpp"
#include "reachplan/reach_solver.hpp"
#include "reachplan/validate.hpp"

#include <chrono>
#include <cstring>
#include <memory>
#include <string>

using namespace reachplan;

namespace {

thread_local std::string g_err;

int status_of(const Error& e) {
  g_err = e.what();
  return static_cast<int>(e.code()) + 1;
}

Vec3 v3(const double* p) { return Vec3(p[0], p[1], p[2]); }
void put3(double* d, const Vec3& v) {
  d[0] = v.x();
  d[1] = v.y();
  d[2] = v.z();
}

ArmSpec to_arm(const rp_arm& a) {
  ArmSpec s;
  s.lengths.assign(a.lengths, a.lengths + a.n_segments);
  s.root = v3(a.root);
  s.arm_radius = a.arm_radius;
  for (int j = 0; j < a.n_limits; ++j)
    s.joint_limits.push_back({a.limits[j].elev_min, a.limits[j].elev_max, a.limits[j].azim_min,
                              a.limits[j].azim_max});
  s.offsets.assign(a.offsets, a.offsets + a.n_offsets);
  s.fold_plane_normal = v3(a.fold_plane_normal);
  s.fold_flex = a.fold_flex;
  s.base_axis = v3(a.base_axis);
  s.base_ref = v3(a.base_ref);
  return s;
}

ReachParams to_rp(const rp_reach_params& r) {
  ReachParams p;
  p.epsilon_gap = r.epsilon_gap;
  p.n_samples_per_segment = r.n_samples;
  p.approach_axis = v3(r.approach_axis);
  p.approach_half_angle = r.approach_half_angle;
  p.near_target_radius = r.near_target_radius;
  p.mode = r.mode == RP_MODE_8DOF ? SolveMode::eight_dof : SolveMode::six_dof;
  p.cone_precheck = r.cone_precheck != 0;
  p.disable_geom_pruning = r.disable_geom_pruning != 0;
  p.refine_triangle_8dof = r.refine_triangle_8dof != 0;
  p.workers = r.workers < 1 ? 1 : r.workers;
  return p;
}

PathParams to_pp(const rp_path_params& r) {
  PathParams p;
  p.epsilon_waypoint = r.epsilon_waypoint;
  p.d_w = r.d_w;
  p.slack = r.slack;
  p.joint1_max_move = r.joint1_max_move;
  p.joint2_max_move = r.joint2_max_move;
  p.relax_schedule.assign(r.relax_schedule, r.relax_schedule + r.n_relax);
  p.unfold_steps = r.unfold_steps;
  return p;
}

SceneObstacle to_obs(const rp_obstacle& o) {
  SceneObstacle s;
  s.shape = o.shape == RP_SHAPE_BOX ? SceneObstacle::Shape::box : SceneObstacle::Shape::cloud;
  s.box_min = v3(o.box_min);
  s.box_max = v3(o.box_max);
  for (int64_t k = 0; k < o.n_points; ++k) s.points.push_back(v3(o.points + 3 * k));
  s.dynamic = o.dynamic != 0;
  s.id = o.id ? o.id : "";
  return s;
}

void to_pose(const PoseChain& p, rp_pose* out, double* wps, int cap) {
  std::memset(out, 0, sizeof(*out));
  out->n_segments = p.segment_count();
  out->has_elbows = p.elbows.empty() ? 0 : 1;
  out->no_indices = p.quiver_indices.empty() ? 1 : 0;
  for (int k = 0; k < RP_MAX_SEGMENTS; ++k)
    out->quiver_indices[k] = k < static_cast<int>(p.quiver_indices.size()) ? p.quiver_indices[k] : -1;
  out->s4_length_dev = p.s4_length_dev;
  for (std::size_t k = 0; k < p.segments.size(); ++k) put3(out->segments[k], p.segments[k]);
  for (std::size_t k = 0; k < p.joints.size(); ++k) put3(out->joints[k], p.joints[k]);
  for (std::size_t k = 0; k < p.elbows.size(); ++k) put3(out->elbows[k], p.elbows[k]);
  out->n_waypoints = static_cast<int>(p.waypoints.size());
  if (wps)
    for (int k = 0; k < out->n_waypoints && k < cap; ++k) put3(wps + 3 * k, p.waypoints[k]);
}

PoseChain from_pose(const rp_pose& p, const double* wps) {
  PoseChain c;
  for (int k = 0; k < p.n_segments; ++k) c.segments.push_back(v3(p.segments[k]));
  for (int k = 0; k <= p.n_segments; ++k) c.joints.push_back(v3(p.joints[k]));
  if (p.has_elbows)
    for (int k = 0; k < p.n_segments; ++k) c.elbows.push_back(v3(p.elbows[k]));
  if (!p.no_indices)
    for (int k = 0; k < p.n_segments; ++k) c.quiver_indices.push_back(p.quiver_indices[k]);
  c.s4_length_dev = p.s4_length_dev;
  if (wps)
    for (int k = 0; k < p.n_waypoints; ++k) c.waypoints.push_back(v3(wps + 3 * k));
  return c;
}

}  // namespace

struct ref_problem {
  ArmSpec arm;
  ReachParams rp;
  Quiver quiver;
  VoxelGrid grid;
  SolutionSet last;
  bool have_last = false;
  double last_ms = 0.0;
};

struct ref_plan {
  PathPlan plan;
};

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

/// Scene grid via build_scene_grid (src/pipeline.cpp:17-34) + quiver
/// (src/quiver.cpp:16-51). dilation < 0 = effective_dilation.
int ref_problem_create(const double* bmin, const double* bmax, double voxel_size, double dilation,
                       const rp_obstacle* obs, int n_obs, const rp_arm* arm,
                       const rp_reach_params* rp, double elev_step, double azim_step,
                       int min_per_ring, ref_problem** out) {
  try {
    auto p = std::make_unique<ref_problem>();
    p->arm = to_arm(*arm);
    p->rp = to_rp(*rp);
    p->quiver = generate_quiver(elev_step, azim_step, min_per_ring);
    Scene scene;
    scene.grid.bounds_min = v3(bmin);
    scene.grid.bounds_max = v3(bmax);
    scene.grid.voxel_size = voxel_size;
    scene.grid.dilation_radius = dilation;
    for (int k = 0; k < n_obs; ++k) scene.obstacles.push_back(to_obs(obs[k]));
    scene.root = p->arm.root;
    p->grid = build_scene_grid(scene, p->arm, p->rp, nullptr);
    *out = p.release();
    return 0;
  } catch (const Error& e) {
    return status_of(e);
  }
}

/// A problem over a caller-supplied occupancy (x fastest, the VoxelGrid
/// layout of inc/reachplan/voxgrid.hpp:28-55) instead of build_scene_grid:
/// lets the 512^3 batched-query parity skip the reference's minutes-long
/// dilation once the grid itself is pinned.
int ref_problem_create_u8(const double* origin, double voxel_size, const int32_t* dims,
                          const uint8_t* occ, double dilation_radius, const rp_arm* arm,
                          const rp_reach_params* rp, double elev_step, double azim_step,
                          int min_per_ring, ref_problem** out) {
  try {
    auto p = std::make_unique<ref_problem>();
    p->arm = to_arm(*arm);
    p->rp = to_rp(*rp);
    p->quiver = generate_quiver(elev_step, azim_step, min_per_ring);
    p->grid.origin = v3(origin);
    p->grid.voxel_size = voxel_size;
    for (int a = 0; a < 3; ++a) p->grid.dims[a] = dims[a];
    const std::size_t n = static_cast<std::size_t>(dims[0]) * dims[1] * dims[2];
    p->grid.occupancy.assign(occ, occ + n);
    p->grid.dilation_radius = dilation_radius;
    *out = p.release();
    return 0;
  } catch (const Error& e) {
    return status_of(e);
  }
}

void ref_problem_destroy(ref_problem* p) { delete p; }

void ref_problem_set_params(ref_problem* p, const rp_reach_params* rp) { p->rp = to_rp(*rp); }

int ref_problem_grid(const ref_problem* p, uint8_t* occ, uint64_t cap, int32_t* dims,
                     double* dilation_radius) {
  for (int a = 0; a < 3; ++a) dims[a] = p->grid.dims[a];
  *dilation_radius = p->grid.dilation_radius;
  if (occ) {
    if (cap < p->grid.occupancy.size()) return RP_E_INVALID_PARAMETER;
    std::memcpy(occ, p->grid.occupancy.data(), p->grid.occupancy.size());
  }
  return 0;
}

int ref_problem_quiver(const ref_problem* p, double* xyz, int cap) {
  const int n = p->quiver.size();
  if (xyz)
    for (int k = 0; k < n && k < cap; ++k) put3(xyz + 3 * k, p->quiver.vectors[k]);
  return n;
}

/// Stand-alone voxel ops for the voxgrid parity tests.
int ref_grid_ops(const double* bmin, const double* bmax, double voxel_size,
                 const rp_obstacle* obs, int n_obs, double radius, uint8_t* occ, uint64_t cap,
                 int32_t* dims) {
  try {
    VoxelGrid g = build_grid(v3(bmin), v3(bmax), voxel_size);
    std::vector<SceneObstacle> list;
    for (int k = 0; k < n_obs; ++k) list.push_back(to_obs(obs[k]));
    mark_obstacles(g, list);
    dilate(g, radius);
    for (int a = 0; a < 3; ++a) dims[a] = g.dims[a];
    if (occ) {
      if (cap < g.occupancy.size()) return RP_E_INVALID_PARAMETER;
      std::memcpy(occ, g.occupancy.data(), g.occupancy.size());
    }
    return 0;
  } catch (const Error& e) {
    return status_of(e);
  }
}

/// Dilate an arbitrary occupancy (dilate, src/voxgrid.cpp:64-92).
int ref_dilate_bytes(const double* origin, double voxel_size, const int32_t* dims, uint8_t* occ,
                     double radius) {
  try {
    VoxelGrid g;
    g.origin = v3(origin);
    g.voxel_size = voxel_size;
    g.dims = {dims[0], dims[1], dims[2]};
    g.occupancy.assign(occ, occ + g.cell_count());
    dilate(g, radius);
    std::memcpy(occ, g.occupancy.data(), g.occupancy.size());
    return 0;
  } catch (const Error& e) {
    return status_of(e);
  }
}

int ref_point_clear(const ref_problem* p, const double* xyz, int64_t n, uint8_t* out) {
  for (int64_t k = 0; k < n; ++k) out[k] = point_clear(p->grid, v3(xyz + 3 * k)) ? 1 : 0;
  return 0;
}

int ref_segment_clear(const ref_problem* p, const double* a, const double* b, int64_t n,
                      int n_samples, uint8_t* out) {
  try {
    for (int64_t k = 0; k < n; ++k)
      out[k] = segment_clear(p->grid, v3(a + 3 * k), v3(b + 3 * k), n_samples).clear ? 1 : 0;
    return 0;
  } catch (const Error& e) {
    return status_of(e);
  }
}

/// Overlay of the replan path (src/path_planner.cpp:1011-1021) as bytes.
int ref_overlay(const ref_problem* p, const rp_obstacle* obs, uint8_t* occ, uint64_t cap) {
  try {
    VoxelGrid aug = p->grid;
    VoxelGrid overlay = build_grid(
        aug.origin,
        aug.origin + Vec3(aug.dims[0] * aug.voxel_size, aug.dims[1] * aug.voxel_size,
                          aug.dims[2] * aug.voxel_size),
        aug.voxel_size);
    mark_obstacles(overlay, {to_obs(*obs)});
    dilate(overlay, p->grid.dilation_radius);
    for (std::size_t c = 0; c < aug.occupancy.size() && c < overlay.occupancy.size(); ++c)
      if (overlay.occupancy[c]) aug.occupancy[c] = 1;
    if (cap < aug.occupancy.size()) return RP_E_INVALID_PARAMETER;
    std::memcpy(occ, aug.occupancy.data(), aug.occupancy.size());
    return 0;
  } catch (const Error& e) {
    return status_of(e);
  }
}

static void put_stats(const SolveStats& s, rp_solve_stats* o) {
  o->seg1_candidates = s.seg1_candidates;
  o->seg1_limit_pass = s.seg1_limit_pass;
  o->seg1_reach_pass = s.seg1_reach_pass;
  o->seg1_survivors = s.seg1_survivors;
  o->pair_candidates = s.pair_candidates;
  o->seg2_limit_pass = s.seg2_limit_pass;
  o->seg2_clear_pass = s.seg2_clear_pass;
  o->gap_tested = s.gap_tested;
  o->gap_pass = s.gap_pass;
  o->joint_pass = s.joint_pass;
  o->v3_clear_pass = s.v3_clear_pass;
  o->solutions = s.solutions;
  o->shortcuts_found = s.shortcuts_found;
  o->wall_ms = s.wall_ms;
}

int ref_prune_segment1(const ref_problem* p, const double* targets, int n_targets,
                       int32_t* out, int cap, int32_t* n_out, rp_solve_stats* stats) {
  try {
    std::vector<Vec3> t;
    for (int k = 0; k < n_targets; ++k) t.push_back(v3(targets + 3 * k));
    SolveStats s;
    auto surv = prune_segment1(p->arm, p->quiver, p->grid, t, p->rp, nullptr, &s, nullptr);
    *n_out = static_cast<int>(surv.size());
    for (int k = 0; k < *n_out && k < cap; ++k) out[k] = surv[k].quiver_index;
    if (stats) put_stats(s, stats);
    return 0;
  } catch (const Error& e) {
    return status_of(e);
  }
}

/// solve_reach (src/reach_solver.cpp:480-546) or, with exhaustive != 0,
/// oracle_solve (src/oracle.cpp:40-98). Result kept in the problem.
int ref_solve_reach(ref_problem* p, const double* target, int exhaustive, int workers,
                    rp_solve_stats* stats, int64_t* n_solutions, int64_t* n_shortcuts) {
  try {
    ReachParams rp = p->rp;
    if (workers > 0) rp.workers = workers;
    const auto t0 = std::chrono::steady_clock::now();
    p->last = exhaustive ? oracle_solve(p->arm, p->quiver, p->grid, v3(target), rp)
                         : solve_reach(p->arm, p->quiver, p->grid, v3(target), rp);
    p->last_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    p->have_last = true;
    if (stats) put_stats(p->last.stats, stats);
    *n_solutions = static_cast<int64_t>(p->last.solutions.size());
    *n_shortcuts = static_cast<int64_t>(p->last.shortcuts.size());
    return 0;
  } catch (const Error& e) {
    return status_of(e);
  }
}

double ref_last_solve_ms(const ref_problem* p) { return p->last_ms; }

int ref_last_keys(const ref_problem* p, int32_t* keys, int64_t cap) {
  const auto& sols = p->last.solutions;
  for (std::size_t k = 0; k < sols.size() && static_cast<int64_t>(k) < cap; ++k) {
    keys[3 * k] = sols[k].quiver_indices[0];
    keys[3 * k + 1] = sols[k].quiver_indices[1];
    keys[3 * k + 2] = sols[k].quiver_indices.size() > 3 ? sols[k].quiver_indices[3] : -1;
  }
  return 0;
}

int ref_last_pose(const ref_problem* p, int64_t k, rp_pose* out, double* wps, int cap) {
  if (k < 0 || k >= static_cast<int64_t>(p->last.solutions.size())) return RP_E_INVALID_PARAMETER;
  to_pose(p->last.solutions[k], out, wps, cap);
  return 0;
}

int ref_last_shortcut(const ref_problem* p, int64_t k, rp_shortcut* out, double* tip, int cap,
                      int32_t* n_tip, const double* target) {
  if (k < 0 || k >= static_cast<int64_t>(p->last.shortcuts.size())) return RP_E_INVALID_PARAMETER;
  const ShortcutPath& s = p->last.shortcuts[k];
  std::memset(out, 0, sizeof(*out));
  out->segment_index = s.segment_index;
  out->hit_sample_index = s.hit_sample_index;
  out->seg1_index = s.seg1_index;
  out->seg2_index = s.seg2_index;
  out->has_bridge = s.bridge ? 1 : 0;
  if (s.bridge) put3(out->bridge, *s.bridge);
  out->via_origin_direct = s.via_origin_direct ? 1 : 0;
  out->n_prefix = static_cast<int>(s.prefix_samples.size());
  out->n_sublength = static_cast<int>(s.sublength_samples.size());
  out->path_length = s.path_length;
  const auto wps = s.tip_waypoints(v3(target));
  *n_tip = static_cast<int>(wps.size());
  for (int q = 0; q < *n_tip && q < cap; ++q) put3(tip + 3 * q, wps[q]);
  return 0;
}

int ref_select(const ref_problem* p, rp_chosen* out) {
  try {
    const ChosenPath c = select_solution(p->last);
    out->kind = c.kind == ChosenPath::Kind::reach_pose ? RP_CHOSEN_REACH_POSE : RP_CHOSEN_SHORTCUT;
    out->path_length = c.path_length;
    out->index = -1;
    if (c.kind == ChosenPath::Kind::reach_pose) {
      for (std::size_t k = 0; k < p->last.solutions.size(); ++k)
        if (p->last.solutions[k].quiver_indices == c.pose.quiver_indices) {
          out->index = static_cast<int64_t>(k);
          break;
        }
    } else {
      for (std::size_t k = 0; k < p->last.shortcuts.size(); ++k) {
        const auto& s = p->last.shortcuts[k];
        if (s.segment_index == c.shortcut.segment_index && s.seg1_index == c.shortcut.seg1_index &&
            s.seg2_index == c.shortcut.seg2_index) {
          out->index = static_cast<int64_t>(k);
          break;
        }
      }
    }
    return 0;
  } catch (const Error& e) {
    return status_of(e);
  }
}

int ref_refine(const ref_problem* p, const rp_pose* approx, const double* target, int triangle,
               rp_pose* out) {
  try {
    const PoseChain a = from_pose(*approx, nullptr);
    PoseChain r = a.segment_count() == 4
                      ? (triangle ? exact_refine_8dof_triangle(p->arm, a, v3(target))
                                  : exact_refine_8dof(p->arm, a, v3(target)))
                      : exact_refine_6dof(p->arm, a, v3(target));
    to_pose(r, out, nullptr, 0);
    return 0;
  } catch (const Error& e) {
    return status_of(e);
  }
}

static int plan_result(PathPlan&& plan, ref_plan** out) {
  auto r = std::make_unique<ref_plan>();
  r->plan = std::move(plan);
  *out = r.release();
  return 0;
}

/// plan_reach_then_path (src/path_planner.cpp:824-829).
int ref_plan_reach_then_path(ref_problem* p, const double* target, const rp_path_params* pp,
                             ref_plan** out) {
  try {
    return plan_result(plan_reach_then_path(p->arm, p->quiver, p->grid, v3(target), p->rp,
                                            to_pp(*pp)),
                       out);
  } catch (const Error& e) {
    return status_of(e);
  }
}

/// plan_from_reach (src/path_planner.cpp:729-738) from a chosen candidate of
/// the last solve: solution `index` (kind 0) or shortcut `index` (kind 1).
int ref_plan_from_chosen(ref_problem* p, int kind, int64_t index, const double* target,
                         const rp_path_params* pp, ref_plan** out) {
  try {
    ChosenPath c;
    if (kind == RP_CHOSEN_REACH_POSE) {
      c.kind = ChosenPath::Kind::reach_pose;
      c.pose = p->last.solutions.at(static_cast<std::size_t>(index));
    } else {
      c.kind = ChosenPath::Kind::shortcut;
      c.shortcut = p->last.shortcuts.at(static_cast<std::size_t>(index));
      c.path_length = c.shortcut.path_length;
    }
    return plan_result(plan_from_reach(p->arm, p->quiver, p->grid, c, p->last, v3(target), p->rp,
                                       to_pp(*pp)),
                       out);
  } catch (const Error& e) {
    return status_of(e);
  }
}

/// The reference's own stage timer, cmd_bench (src/cli.cpp:272-308), on this
/// problem: ms[0] = prune_segment1 alone, ms[1] = solve_reach, ms[2] =
/// select_solution + plan_from_reach (cmd_bench's path-ms excludes the
/// select; ms[3] is that exclusive figure). The plan is returned (or the
/// planner's status) so the caller can chain plan_arbitrary from it.
int ref_bench_stages(ref_problem* p, const double* target, const rp_path_params* pp,
                     int workers, double* ms, int64_t* n_solutions, ref_plan** out) {
  using clk = std::chrono::steady_clock;
  auto dms = [](clk::time_point a, clk::time_point b) {
    return std::chrono::duration<double, std::milli>(b - a).count();
  };
  try {
    ReachParams rp = p->rp;
    if (workers > 0) rp.workers = workers;
    const Vec3 t = v3(target);
    const auto t0 = clk::now();
    SolveStats s1;
    const auto seg1 = prune_segment1(p->arm, p->quiver, p->grid, {t}, rp, nullptr, &s1, nullptr);
    const auto t1 = clk::now();
    SolutionSet set = solve_reach(p->arm, p->quiver, p->grid, t, rp);
    const auto t2 = clk::now();
    ms[0] = dms(t0, t1);
    ms[1] = dms(t1, t2);
    ms[2] = ms[3] = 0.0;
    *n_solutions = static_cast<int64_t>(set.solutions.size());
    (void)seg1;
    const ChosenPath chosen = select_solution(set);
    const auto t3 = clk::now();
    PathPlan plan = plan_from_reach(p->arm, p->quiver, p->grid, chosen, set, t, rp, to_pp(*pp));
    const auto t4 = clk::now();
    ms[2] = dms(t2, t4);
    ms[3] = dms(t3, t4);
    return plan_result(std::move(plan), out);
  } catch (const Error& e) {
    return status_of(e);
  }
}

/// plan_arbitrary (src/path_planner.cpp:906-998) from a start pose.
int ref_plan_arbitrary(ref_problem* p, const rp_pose* start, const double* start_wps,
                       const double* target, const rp_path_params* pp, ref_plan** out) {
  try {
    return plan_result(plan_arbitrary(p->arm, p->quiver, p->grid, from_pose(*start, start_wps),
                                      v3(target), p->rp, to_pp(*pp)),
                       out);
  } catch (const Error& e) {
    return status_of(e);
  }
}

/// replan_dynamic (src/path_planner.cpp:1000-1102) against an active plan.
int ref_replan_dynamic(ref_problem* p, const ref_plan* active, int current_index,
                       const rp_obstacle* obs, double period, double cost,
                       const rp_path_params* pp, ref_plan** out) {
  try {
    const ReplanTiming timing{period, cost};
    return plan_result(replan_dynamic(p->arm, p->quiver, p->grid, active->plan, current_index,
                                      to_obs(*obs), timing, p->rp, to_pp(*pp)),
                       out);
  } catch (const Error& e) {
    return status_of(e);
  }
}

void ref_plan_destroy(ref_plan* p) { delete p; }

int ref_plan_info(const ref_plan* p, rp_plan_info* info) {
  std::memset(info, 0, sizeof(*info));
  info->n_waypoints = static_cast<int>(p->plan.waypoints.size());
  info->n_poses = static_cast<int>(p->plan.poses.size());
  info->n_unfold = static_cast<int>(p->plan.unfold_prefix.size());
  info->n_notes = static_cast<int>(p->plan.provenance.notes.size());
  info->replan_switch_index = p->plan.provenance.replan_switch_index;
  std::strncpy(info->kind, p->plan.provenance.kind.c_str(), sizeof(info->kind) - 1);
  return 0;
}

int ref_plan_waypoints(const ref_plan* p, double* xyz, int cap) {
  for (std::size_t k = 0; k < p->plan.waypoints.size() && static_cast<int>(k) < cap; ++k)
    put3(xyz + 3 * k, p->plan.waypoints[k]);
  return 0;
}

int ref_plan_relax(const ref_plan* p, double* relax, int cap) {
  const auto& r = p->plan.provenance.relax_per_waypoint;
  for (std::size_t k = 0; k < r.size() && static_cast<int>(k) < cap; ++k) relax[k] = r[k];
  return static_cast<int>(r.size());
}

int ref_plan_pose(const ref_plan* p, int which, int k, rp_pose* out, double* wps, int cap) {
  const auto& v = which == 0 ? p->plan.poses : p->plan.unfold_prefix;
  if (k < 0 || k >= static_cast<int>(v.size())) return RP_E_INVALID_PARAMETER;
  to_pose(v[k], out, wps, cap);
  return 0;
}

int ref_plan_note(const ref_plan* p, int k, char* buf, int cap) {
  const auto& n = p->plan.provenance.notes;
  if (k < 0 || k >= static_cast<int>(n.size())) return RP_E_INVALID_PARAMETER;
  std::strncpy(buf, n[k].c_str(), cap - 1);
  buf[cap - 1] = 0;
  return 0;
}

/// waypoint_ik (src/path_planner.cpp:167-291), public in the reference.
int ref_waypoint_ik(const ref_problem* p, const double* wp, const rp_pose* prev, double relax,
                    const double* back, const double* fwd, const rp_pose* bias,
                    const rp_path_params* pp, int32_t* found, rp_pose* out, double* wps, int cap) {
  try {
    TrailContext t;
    if (back) t.back_dir = v3(back);
    if (fwd) t.fwd_dir = v3(fwd);
    const PoseChain pv = from_pose(*prev, nullptr);
    PoseChain pb;
    if (bias) pb = from_pose(*bias, nullptr);
    const PathParams ppr = to_pp(*pp).resolved(p->arm, p->rp);
    auto r = waypoint_ik(p->arm, p->quiver, p->grid, v3(wp), pv, p->rp, ppr, relax, t,
                         bias ? &pb : nullptr);
    *found = r ? 1 : 0;
    if (r) to_pose(*r, out, wps, cap);
    return 0;
  } catch (const Error& e) {
    return status_of(e);
  }
}

double ref_mean_polyline_deviation(const double* pts, int n, const double* poly, int np) {
  std::vector<Vec3> a, b;
  for (int k = 0; k < n; ++k) a.push_back(v3(pts + 3 * k));
  for (int k = 0; k < np; ++k) b.push_back(v3(poly + 3 * k));
  return mean_polyline_deviation(a, b);
}

int ref_folded_pose(const ref_problem* p, rp_pose* out) {
  try {
    to_pose(folded_pose(p->arm), out, nullptr, 0);
    return 0;
  } catch (const Error& e) {
    return status_of(e);
  }
}

/// build_unfold (src/path_planner.cpp:458-484) + interpolate_poses (:405-448)
/// restated from the reference's public pieces (both are file-local there),
/// reporting where it stops: 0 ok, 1 rotated pose invalid, 2 an interpolated
/// pose invalid at *steps_out, 3 never smooth up to 4096 steps.
namespace {
bool h_walk(const VoxelGrid& g, const Vec3& a, const Vec3& b, int n) {
  const Vec3 d = b - a;
  for (int k = 1; k <= n; ++k)
    if (!point_clear(g, a + (static_cast<double>(k) / n) * d)) return false;
  return true;
}
bool h_pose_valid(const ArmSpec& spec, const VoxelGrid& g, const PoseChain& p, int n,
                  double spacing) {
  for (std::size_t j = 0; j < p.segments.size(); ++j) {
    Vec3 from = p.joints[j];
    if (!p.elbows.empty()) {
      const double len = (p.elbows[j] - p.joints[j]).norm();
      if (len != 0.0) {
        const int c = std::max(1, static_cast<int>(std::ceil(len / std::max(spacing, 1e-12))));
        if (!h_walk(g, p.joints[j], p.elbows[j], c)) return false;
      }
      from = p.elbows[j];
    }
    if (!h_walk(g, from, p.joints[j + 1], n)) return false;
  }
  return joint_limits_ok(spec, p) && self_collision_free(spec, p);
}
Vec3 h_perp(const Vec3& dir) {
  const Vec3 seed = std::abs(dir.z()) < 0.9 ? Vec3::UnitZ() : Vec3::UnitX();
  return dir.cross(seed).normalized();
}
Vec3 h_plane_normal(const PoseChain& p) {
  Vec3 n = p.segments[0].cross(p.segments[1]);
  if (n.norm() <= 1e-12) return h_perp(p.segments[0].normalized());
  return n.normalized();
}
}  // namespace

int ref_unfold_debug(const ref_problem* P, const rp_pose* tri_in, const double* tri_wps,
                     const rp_path_params* pp_in, int* steps_out, rp_pose* out, int cap,
                     int* n_out) {
  const ArmSpec& spec = P->arm;
  const VoxelGrid& grid = P->grid;
  const PoseChain tri = from_pose(*tri_in, tri_wps);
  const PathParams pp = to_pp(*pp_in).resolved(spec, P->rp);
  const PoseChain fold = folded_pose(spec);
  const Vec3 u1f = fold.segments[0].normalized(), u1t = tri.segments[0].normalized();
  const Vec3 nf = h_plane_normal(fold), nt = h_plane_normal(tri);
  Mat3 a, b;
  a.col(0) = u1f;
  a.col(1) = nf.cross(u1f);
  a.col(2) = nf;
  b.col(0) = u1t;
  b.col(1) = nt.cross(u1t);
  b.col(2) = nt;
  const Mat3 rot = b * a.transpose();
  std::vector<Vec3> segs;
  for (const Vec3& s : fold.segments) segs.push_back(rot * s);
  const PoseChain rotated = chain_from_segments(spec, segs);
  const int n = P->rp.n_samples_per_segment;
  const double spacing = P->rp.nominal_spacing(spec);
  if (cap > 0) to_pose(rotated, out, nullptr, 0);
  if (!h_pose_valid(spec, grid, rotated, n, spacing)) return 1;
  const JointAngles qa = vectors_to_joint_angles(spec, rotated);
  const JointAngles qb = vectors_to_joint_angles(spec, tri);
  for (int steps = std::max(1, pp.unfold_steps); steps <= 4096; steps *= 2) {
    std::vector<PoseChain> seq{rotated};
    for (int s = 1; s < steps; ++s) {
      const double t = static_cast<double>(s) / steps;
      JointAngles qt;
      for (int j = 0; j < qa.joint_count(); ++j) {
        qt.azimuth.push_back(qa.azimuth[j] + t * wrap_angle(qb.azimuth[j] - qa.azimuth[j]));
        qt.elevation.push_back(qa.elevation[j] + t * (qb.elevation[j] - qa.elevation[j]));
        qt.degenerate.push_back(0);
      }
      PoseChain pose = joint_angles_to_vectors(spec, qt);
      if (!h_pose_valid(spec, grid, pose, n, spacing)) {
        *steps_out = steps;
        *n_out = s;
        if (cap > 1) {
          to_pose(pose, out + 1, nullptr, 0);
          out[1].n_waypoints = (joint_limits_ok(spec, pose) ? 0 : 1) |
                               (self_collision_free(spec, pose) ? 0 : 2);
        }
        return 2;
      }
      seq.push_back(pose);
    }
    seq.push_back(tri);
    bool smooth = true;
    for (std::size_t s = 0; s + 1 < seq.size(); ++s)
      if (!smoothness_ok(seq[s], seq[s + 1], pp, 1.0)) {
        smooth = false;
        break;
      }
    if (smooth) {
      *steps_out = steps;
      *n_out = static_cast<int>(seq.size());
      for (int k = 0; k < *n_out && k < cap; ++k) to_pose(seq[k], out + k, nullptr, 0);
      return 0;
    }
  }
  return 3;
}

/// Independent validate_plan (src/validate.cpp:49-108): number of issues.
int ref_validate_plan(const ref_problem* p, const ref_plan* plan, const rp_path_params* pp) {
  const ValidationReport r = validate_plan(p->arm, p->grid, plan->plan, p->rp, to_pp(*pp));
  return static_cast<int>(r.issues.size());
}

/// validate_plan (src/validate.cpp:53-108) with the whole report: issues
/// joined by '\n' into buf; returns the byte count needed (incl. NUL).
int ref_validate_report(const ref_problem* p, const ref_plan* plan, const rp_path_params* pp,
                        int32_t* ok, int32_t* poses_checked, int32_t* relax_events, char* buf,
                        int cap) {
  const ValidationReport r = validate_plan(p->arm, p->grid, plan->plan, p->rp, to_pp(*pp));
  *ok = r.ok ? 1 : 0;
  *poses_checked = r.poses_checked;
  *relax_events = r.relax_events;
  std::string all;
  for (size_t k = 0; k < r.issues.size(); ++k) all += (k ? "\n" : "") + r.issues[k];
  if (buf && cap > 0) {
    const size_t n = std::min(all.size(), static_cast<size_t>(cap - 1));
    std::memcpy(buf, all.data(), n);
    buf[n] = 0;
  }
  return static_cast<int>(all.size() + 1);
}

/// simulate_execution (src/motion.cpp:62-141): the trace into rp_tick
/// records (caller arrays sized by cap), or the error status + message.
int ref_simulate(const ref_problem* p, const ref_plan* plan, const rp_motion_params* mp,
                 int use_grid, rp_tick* ticks, int64_t cap, int64_t* n_ticks, int32_t* overshoot,
                 int32_t* n_over, int32_t* clamp, int32_t* n_clamp, int32_t* reached, char* msg,
                 int msgcap) {
  MotionParams m;
  m.v_w = mp->v_w;
  m.sample_rate = mp->sample_rate;
  m.max_joint_rate = mp->max_joint_rate;
  m.arrival_tolerance = mp->arrival_tolerance;
  try {
    const ExecutionTrace tr =
        simulate_execution(p->arm, plan->plan, m, use_grid ? &p->grid : nullptr);
    *n_ticks = static_cast<int64_t>(tr.ticks.size());
    for (size_t k = 0; k < tr.ticks.size() && static_cast<int64_t>(k) < cap; ++k) {
      const ExecutionTick& t = tr.ticks[k];
      rp_tick& o = ticks[k];
      std::memset(&o, 0, sizeof(o));
      o.time = t.time;
      o.n_joints = t.q.joint_count();
      for (int j = 0; j < o.n_joints; ++j) {
        o.azimuth[j] = t.q.azimuth[j];
        o.elevation[j] = t.q.elevation[j];
        o.degenerate[j] = t.q.degenerate[j];
      }
      put3(o.tracked, t.tracked_point);
      o.active = t.active_waypoint_index;
      o.n_rates = static_cast<int32_t>(t.commanded.azimuth_rate.size());
      o.clamped = t.commanded.clamped ? 1 : 0;
      for (int j = 0; j < o.n_rates; ++j) {
        o.azimuth_rate[j] = t.commanded.azimuth_rate[j];
        o.elevation_rate[j] = t.commanded.elevation_rate[j];
      }
    }
    *n_over = static_cast<int32_t>(tr.overshoot_events.size());
    *n_clamp = static_cast<int32_t>(tr.clamp_events.size());
    for (size_t k = 0; k < tr.overshoot_events.size() && static_cast<int64_t>(k) < cap; ++k)
      overshoot[k] = tr.overshoot_events[k];
    for (size_t k = 0; k < tr.clamp_events.size() && static_cast<int64_t>(k) < cap; ++k)
      clamp[k] = tr.clamp_events[k];
    *reached = tr.reached_goal ? 1 : 0;
    return 0;
  } catch (const Error& e) {
    if (msg && msgcap > 0) {
      std::strncpy(msg, e.what(), msgcap - 1);
      msg[msgcap - 1] = 0;
    }
    return status_of(e);
  }
}

/// The plan file the reference CLI writes for `plan` (cli.cpp:126-137,
/// 167-185): solve + select + plan_from_reach + emit_plan. Returns the
/// status; the text goes to buf (size needed in *need).
int ref_emit_plan(ref_problem* p, const double* target, double elev_deg, double azim_deg, int mpr,
                  char* buf, int64_t cap, int64_t* need) {
  try {
    const SolutionSet set = solve_reach(p->arm, p->quiver, p->grid, v3(target), p->rp);
    const ChosenPath chosen = select_solution(set);
    const PathParams pp;
    PlanFile pf;
    pf.quiver.elev_step_deg = elev_deg;
    pf.quiver.equator_azim_step_deg = azim_deg;
    pf.quiver.min_per_ring = mpr;
    pf.reach = p->rp;
    pf.path = pp.resolved(p->arm, p->rp);
    pf.arm = p->arm;
    pf.chosen = chosen;
    pf.plan = plan_from_reach(p->arm, p->quiver, p->grid, chosen, set, v3(target), p->rp, pp);
    pf.stats = set.stats;
    pf.stats.wall_ms = 0.0;
    const std::string text = emit_plan(pf);
    *need = static_cast<int64_t>(text.size()) + 1;
    if (buf && cap > 0) {
      const size_t n = std::min(text.size(), static_cast<size_t>(cap - 1));
      std::memcpy(buf, text.data(), n);
      buf[n] = 0;
    }
    return 0;
  } catch (const Error& e) {
    return status_of(e);
  }
}

/// A PathPlan from plain data (plan files / corrupted copies in tests).
ref_plan* ref_plan_create(const char* kind, const double* waypoints, const rp_pose* poses,
                          const double* pose_wps, int wps_per_pose, const double* relax, int n,
                          const rp_pose* unfold, int n_unfold) {
  auto* out = new ref_plan();
  out->plan.provenance.kind = kind ? kind : "";
  for (int k = 0; k < n; ++k) {
    out->plan.waypoints.push_back(v3(waypoints + 3 * k));
    out->plan.poses.push_back(
        from_pose(poses[k], pose_wps ? pose_wps + 3 * static_cast<size_t>(k) * wps_per_pose : nullptr));
    out->plan.provenance.relax_per_waypoint.push_back(relax ? relax[k] : 1.0);
  }
  for (int k = 0; k < n_unfold; ++k) out->plan.unfold_prefix.push_back(from_pose(unfold[k], nullptr));
  return out;
}

}  // extern "C"
