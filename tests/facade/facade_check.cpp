// TEST INFRASTRUCTURE: drives the reachplan C++ API exactly as a reference
// caller would (the reference's own headers, reachplan:: names and types),
// linked against the façade (paper_1906_10678_b200/facade) over
// libreachplan_b200.so instead of the reference's src/*.cpp. Reads a scene
// description, prints the results as JSON for tests/test_facade.py, which
// compares them with the reference run through oracle/_ref.
//
// scene file (whitespace separated):
//   lengths <n> L1 .. Ln   radius <r>   mode <0|1>   samples <n>
//   bounds x0 y0 z0 x1 y1 z1   voxel <vs>   quiver <step_rad> <min_per_ring>
//   target x y z   second x y z   boxes <k> then k lines "x0 y0 z0 x1 y1 z1"
//
// facade_check scene.txt [plan_file]    results as JSON (tests/test_facade.py)
// facade_check scene.txt --bench K      K timed C3-style steps (bench.py)
#include "reachplan/io.hpp"
#include "reachplan/pipeline.hpp"

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>

using namespace reachplan;

namespace {

std::string num(double v) {
  char b[40];
  std::snprintf(b, sizeof(b), "%.17g", v);
  return b;
}
std::string vec(const Vec3& v) { return "[" + num(v.x()) + "," + num(v.y()) + "," + num(v.z()) + "]"; }
template <typename T, typename F>
std::string list(const std::vector<T>& xs, F f) {
  std::string s = "[";
  for (std::size_t k = 0; k < xs.size(); ++k) s += (k ? "," : "") + f(xs[k]);
  return s + "]";
}
std::string pose(const PoseChain& p) {
  return "{\"segments\":" + list(p.segments, vec) + ",\"joints\":" + list(p.joints, vec) +
         ",\"qidx\":" + list(p.quiver_indices, [](int i) { return std::to_string(i); }) +
         ",\"n_waypoints\":" + std::to_string(p.waypoints.size()) +
         ",\"s4dev\":" + num(p.s4_length_dev) + "}";
}
std::string plan(const PathPlan& p) {
  return "{\"kind\":\"" + p.provenance.kind + "\",\"waypoints\":" + list(p.waypoints, vec) +
         ",\"relax\":" + list(p.provenance.relax_per_waypoint, num) +
         ",\"notes\":" + list(p.provenance.notes, [](const std::string& s) { return "\"" + s + "\""; }) +
         ",\"poses\":" + list(p.poses, pose) + ",\"unfold\":" + list(p.unfold_prefix, pose) +
         ",\"switch\":" + std::to_string(p.provenance.replan_switch_index) + "}";
}
std::string stats(const SolveStats& s) {
  const std::vector<long> v{s.seg1_candidates, s.seg1_limit_pass, s.seg1_reach_pass,
                            s.seg1_survivors,  s.pair_candidates, s.seg2_limit_pass,
                            s.seg2_clear_pass, s.gap_tested,      s.gap_pass,
                            s.joint_pass,      s.v3_clear_pass,   s.solutions,
                            s.shortcuts_found};
  return list(v, [](long x) { return std::to_string(x); });
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::cerr << "usage: facade_check scene.txt\n";
    return 2;
  }
  std::ifstream in(argv[1]);
  std::string key;
  ArmSpec arm;
  ReachParams rp;
  Scene scene;
  double qstep = 0.0;
  int mpr = 4;
  Vec3 second = Vec3::Zero();
  while (in >> key) {
    if (key == "lengths") {
      int n;
      in >> n;
      arm.lengths.resize(n);
      for (double& L : arm.lengths) in >> L;
    } else if (key == "radius") {
      in >> arm.arm_radius;
    } else if (key == "mode") {
      int m;
      in >> m;
      rp.mode = m == 0 ? SolveMode::six_dof : SolveMode::eight_dof;
    } else if (key == "samples") {
      in >> rp.n_samples_per_segment;
    } else if (key == "bounds") {
      double a, b, c, d, e, f;
      in >> a >> b >> c >> d >> e >> f;
      scene.grid.bounds_min = Vec3(a, b, c);
      scene.grid.bounds_max = Vec3(d, e, f);
    } else if (key == "voxel") {
      in >> scene.grid.voxel_size;
    } else if (key == "quiver") {
      in >> qstep >> mpr;
    } else if (key == "target") {
      double a, b, c;
      in >> a >> b >> c;
      scene.target = Vec3(a, b, c);
    } else if (key == "second") {
      double a, b, c;
      in >> a >> b >> c;
      second = Vec3(a, b, c);
    } else if (key == "boxes") {
      int k;
      in >> k;
      for (int i = 0; i < k; ++i) {
        SceneObstacle o;
        double a, b, c, d, e, f;
        in >> a >> b >> c >> d >> e >> f;
        o.box_min = Vec3(a, b, c);
        o.box_max = Vec3(d, e, f);
        scene.obstacles.push_back(o);
      }
    }
  }
  if (argc > 3 && std::string(argv[2]) == "--bench") {
    // the C3 step through the reference API, host wall clock per step:
    // build_scene_grid + plan_reach_then_path + plan_arbitrary (from its
    // final pose to `second`); the first step is a warm-up
    const int K = std::atoi(argv[3]);
    try {
      const Quiver q = generate_quiver(qstep, qstep, mpr);
      PathParams pp;
      std::vector<double> ms, parts[3];
      std::size_t wps = 0;
      const auto since = [](auto t) {
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t).count();
      };
      for (int k = 0; k <= K; ++k) {
        const auto t0 = std::chrono::steady_clock::now();
        const VoxelGrid grid = build_scene_grid(scene, arm, rp);
        const double a = since(t0);
        const PathPlan p1 = plan_reach_then_path(arm, q, grid, scene.target, rp, pp);
        const double b = since(t0);
        const PathPlan p2 = plan_arbitrary(arm, q, grid, p1.poses.back(), second, rp, pp);
        const double c = since(t0);
        wps = p1.waypoints.size() + p2.waypoints.size();
        if (k > 0) {
          ms.push_back(c);
          parts[0].push_back(a);
          parts[1].push_back(b - a);
          parts[2].push_back(c - b);
        }
      }
      std::cout << "{\"bench_ms\":" << list(ms, num) << ",\"grid_ms\":" << list(parts[0], num)
                << ",\"reach_path_ms\":" << list(parts[1], num)
                << ",\"arbitrary_ms\":" << list(parts[2], num) << ",\"waypoints\":" << wps
                << "}\n";
    } catch (const Error& e) {
      std::cout << "{\"error\":" << static_cast<int>(e.code()) + 1 << "}\n";
    }
    return 0;
  }
  try {
    const Quiver q = generate_quiver(qstep, qstep, mpr);
    const VoxelGrid grid = build_scene_grid(scene, arm, rp);
    // the same grid again through the primitive calls
    VoxelGrid g2 = build_grid(scene.grid.bounds_min, scene.grid.bounds_max, scene.grid.voxel_size);
    mark_obstacles(g2, scene.obstacles);
    dilate(g2, effective_dilation(scene, arm, rp));
    const SolutionSet set = solve_reach(arm, q, grid, scene.target, rp);
    const ChosenPath chosen = select_solution(set);
    PathParams pp;
    // each planner call reports its own outcome (a plan or the Errc it threw)
    const auto attempt = [](auto&& fn, PathPlan* keep) -> std::string {
      try {
        PathPlan p = fn();
        if (keep) *keep = p;
        return plan(p);
      } catch (const Error& e) {
        return "{\"error\":" + std::to_string(static_cast<int>(e.code()) + 1) + "}";
      }
    };
    PathPlan p1, p3;
    const std::string j1 = attempt([&] { return plan_reach_then_path(arm, q, grid, scene.target, rp, pp); }, &p1);
    const std::string j2 = attempt([&] { return plan_from_reach(arm, q, grid, chosen, set, scene.target, rp, pp); }, nullptr);
    std::string j3 = "null";
    if (!p1.poses.empty())
      j3 = attempt([&] { return plan_arbitrary(arm, q, grid, p1.poses.back(), second, rp, pp); }, &p3);
    const BackwardEndpoints be =
        backward_endpoints(scene.target, arm.lengths.back(), q, rp.approach_axis, 0.0, rp.mode);
    // a reach pose to probe span_gap and the scan with: the chosen one, else
    // (a shortcut was chosen) the first solution, else a straight chain
    PoseChain probe_pose;
    if (chosen.kind == ChosenPath::Kind::reach_pose) {
      probe_pose = chosen.pose;
    } else if (!set.solutions.empty()) {
      probe_pose = set.solutions.front();
    } else {
      probe_pose.segments = {Vec3(arm.length(0), 0, 0), Vec3(arm.length(1), 0, 0)};
      probe_pose.joints = {arm.root, arm.root + probe_pose.segments[0],
                           arm.root + probe_pose.segments[0] + probe_pose.segments[1]};
    }
    const std::vector<GapCandidate> gaps =
        span_gap(probe_pose.joints[2], be.points, arm.length(2), rp.resolved_epsilon(arm));
    const SegmentProbe probe = segment_clear(grid, arm.root, scene.target, 8);
    // backward endpoints of a 0.25 rad approach cone, and span_gap over them
    const BackwardEndpoints cone =
        backward_endpoints(scene.target, arm.lengths.back(), q, rp.approach_axis, 0.25, rp.mode);
    const std::vector<GapCandidate> cone_gaps =
        span_gap(probe_pose.joints[2], cone.points, arm.length(2), rp.resolved_epsilon(arm));
    // prune_segment1 with the near-encounter scan (short_reach_scan) towards
    // a point 0.3 m out along the chosen segment-1 direction
    const Vec3 scan_t = arm.root + 0.3 * probe_pose.segments[0].normalized() + Vec3(0.004, -0.003, 0.002);
    std::vector<ShortcutPath> sink;
    SolveStats s1st;
    const std::vector<Seg1Hypothesis> surv =
        prune_segment1(arm, q, grid, {scene.target}, rp, &sink, &s1st, &scan_t);
    // select_solution on sets this library did not produce: the solutions
    // in reverse order (first 400), and the scan's shortcuts
    SolutionSet rev;
    for (std::size_t k = set.solutions.size(); k-- > 0 && rev.solutions.size() < 400;)
      rev.solutions.push_back(set.solutions[k]);
    const ChosenPath crev = select_solution(rev);
    SolutionSet scs;
    scs.shortcuts = sink;
    std::string csc = "null";
    if (!sink.empty()) {
      const ChosenPath c = select_solution(scs);
      csc = "{\"seg1\":" + std::to_string(c.shortcut.seg1_index) + ",\"path_length\":" +
            num(c.path_length) + "}";
    }
    const auto shortcut = [](const ShortcutPath& sp) {
      return "{\"seg1\":" + std::to_string(sp.seg1_index) + ",\"hit\":" +
             std::to_string(sp.hit_sample_index) + ",\"bridge\":" + (sp.bridge ? "1" : "0") +
             ",\"direct\":" + (sp.via_origin_direct ? "1" : "0") + ",\"n_sub\":" +
             std::to_string(sp.sublength_samples.size()) + ",\"path_length\":" +
             num(sp.path_length) + ",\"tip\":" + list(sp.tip_waypoints(Vec3::Zero()), vec) + "}";
    };
    if (argc > 2) {
      // the plan file the reference CLI writes for `plan` (cli.cpp:126-137,
      // 167-185), from the façade's results and the reference's writer
      try {
        PlanFile pf;
        pf.quiver.elev_step_deg = rad2deg(qstep);
        pf.quiver.equator_azim_step_deg = rad2deg(qstep);
        pf.quiver.min_per_ring = mpr;
        pf.reach = rp;
        pf.path = pp.resolved(arm, rp);
        pf.arm = arm;
        pf.chosen = chosen;
        pf.plan = plan_from_reach(arm, q, grid, chosen, set, scene.target, rp, pp);
        pf.stats = set.stats;
        pf.stats.wall_ms = 0.0;
        std::ofstream(argv[2]) << emit_plan(pf);
      } catch (const Error&) {
      }
    }
    std::cout << "{\"quiver\":" << q.size() << ",\"rings\":" << q.ring_count()
              << ",\"occupied\":" << grid.occupied_count()
              << ",\"grids_equal\":" << (grid.occupancy == g2.occupancy ? "true" : "false")
              << ",\"dilation\":" << num(grid.dilation_radius)
              << ",\"point_clear_target\":" << (point_clear(grid, scene.target) ? 1 : 0)
              << ",\"segment_clear\":" << (probe.clear ? 1 : 0)
              << ",\"stats\":" << stats(set.stats) << ",\"n_solutions\":" << set.solutions.size()
              << ",\"n_shortcuts\":" << set.shortcuts.size()
              << ",\"first_solution\":" << (set.solutions.empty() ? "null" : pose(set.solutions.front()))
              << ",\"last_solution\":" << (set.solutions.empty() ? "null" : pose(set.solutions.back()))
              << ",\"chosen\":{\"kind\":" << (chosen.kind == ChosenPath::Kind::shortcut ? 1 : 0)
              << ",\"path_length\":" << num(chosen.path_length) << ",\"pose\":" << pose(chosen.pose)
              << "},\"span_gap\":" << gaps.size()
              << ",\"cone\":{\"points\":" << list(cone.points, vec)
              << ",\"idx\":" << list(cone.cone_indices, [](int i) { return std::to_string(i); })
              << "},\"cone_gaps\":"
              << list(cone_gaps, [](const GapCandidate& g) {
                   return "[" + std::to_string(g.backward_index) + "," + vec(g.v3) + "]";
                 })
              << ",\"scan\":{\"target\":" << vec(scan_t) << ",\"survivors\":" << surv.size()
              << ",\"stats\":" << stats(s1st) << ",\"shortcuts\":" << list(sink, shortcut)
              << "},\"select_rev\":{\"qidx\":"
              << list(crev.pose.quiver_indices, [](int i) { return std::to_string(i); })
              << ",\"path_length\":" << num(crev.path_length) << "},\"select_sc\":" << csc
              << ",\"mean_dev\":"
              << (p1.waypoints.empty() || p3.waypoints.empty()
                      ? std::string("null")
                      : num(mean_polyline_deviation(p1.waypoints, p3.waypoints)))
              << ",\"plan\":" << j1 << ",\"plan_from_reach\":" << j2 << ",\"arbitrary\":" << j3
              << "}\n";
  } catch (const Error& e) {
    std::cout << "{\"error\":" << static_cast<int>(e.code()) << ",\"what\":\"" << e.what() << "\"}\n";
    return 0;
  }
  return 0;
}
