// Path planner control flow (src/path_planner.cpp) on top of the device
// searches: the sequential backward pass, candidate builds, the fallback
// cascade, arbitrary-pose planning and the dynamic re-plan. Every geometric
// search (waypoint IK, solve_reach, unfold validity, deviation scoring,
// collide scans) runs on the GPU; the host only sequences them.
#include "rp_planner.hpp"

#include <algorithm>
#include <cstdio>
#include <climits>
#include <condition_variable>
#include <mutex>
#include <exception>
#include <thread>
#include <functional>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>

namespace rp {

namespace {

constexpr double kPi = 3.14159265358979323846;

V3 tracked_point(const HostPose& p) { return p.joints[std::min(3, p.nseg)]; }

double total_length(const rp_arm& a) {
  double t = 0.0;
  for (int k = 0; k < a.n_segments; ++k) t += a.lengths[k];
  return t;
}

bool smoothness_ok(const HostPose& prev, const HostPose& cand, const PP& pp, double relax) {
  const double d1 = rpd::norm(cand.joints[1] - prev.joints[1]);
  const double d2 = rpd::norm(cand.joints[2] - prev.joints[2]);
  return d1 <= pp.j1 * relax + 1e-12 && d2 <= pp.j2 * relax + 1e-12;
}

V3 perpendicular_of(V3 dir) {
  const V3 seed = std::abs(dir.z) < 0.9 ? V3{0, 0, 1} : V3{1, 0, 0};
  return rpd::normalized(rpd::cross(dir, seed));
}

Trail trail_context(const std::vector<V3>& wps, size_t k) {
  Trail t;
  if (k > 0) {
    const V3 d = wps[k - 1] - wps[k];
    if (rpd::norm(d) > 1e-12) {
      t.has_back = true;
      t.back = rpd::normalized(d);
    }
  }
  if (k + 1 < wps.size()) {
    const V3 d = wps[k + 1] - wps[k];
    if (rpd::norm(d) > 1e-12) {
      t.has_fwd = true;
      t.fwd = rpd::normalized(d);
    }
  }
  return t;
}

std::vector<double> with_unit_first(const std::vector<double>& s) {
  std::vector<double> f{1.0};
  f.insert(f.end(), s.begin(), s.end());
  return f;
}

/// A reach candidate (ChosenPath) carried through the planner.
struct Cand {
  int kind = RP_CHOSEN_REACH_POSE;
  int64_t ordinal = -1;  // in its solution set (reach) or shortcut list
  HostPose pose;         // unrefined solution pose with its 4n waypoints
  HostShortcut sc;
  // exact_refine of `pose` toward `refined_target` in `refined_mode`,
  // computed in the same device round trip as the selection (select_cand)
  bool has_refined = false;
  int refined_mode = -1;
  V3 refined_target{0, 0, 0};
  PoseOpOut refined{};
};

struct PassOptions {
  std::vector<double> factors{1.0};
  bool cloud = false;
  double cloud_radius = 0.0;
  const HostPose* fixed_first = nullptr;
  const HostPose* junction_bias = nullptr;
};

struct PassResult {
  bool ok = false;
  int failed_index = -1;
  std::vector<HostPose> poses;
  std::vector<double> relax;
  std::vector<V3> waypoints;
  std::vector<std::string> notes;
};

struct Build;
struct Failure {
  Cand candidate;
  std::vector<V3> waypoints;
  int blocked_index = -1;
  std::string reason;
  // the candidate's build (make_candidate_build is a pure function of the
  // candidate, so the cascade's attempts on it reuse this one)
  std::shared_ptr<const Build> build;
};

/// backward_pass's result from a finished device pass.
PassResult pass_from_device(const Planner::BpOut& bo, const std::vector<V3>& waypoints,
                            const HostPose& anchor, const PassOptions& opt) {
  PassResult res;
  const size_t m = waypoints.size();
  res.poses.assign(m, HostPose{});
  res.relax.assign(m, 1.0);
  res.waypoints = waypoints;
  res.poses[m - 1] = anchor;
  {
    res.waypoints = bo.wps;
    res.relax = bo.relax;
    if (!bo.ok) {
      res.failed_index = bo.failed_index;
      return res;
    }
    for (size_t k = m - 1; k-- > 0;) {
      if (bo.kind[k] == 2) {
        res.poses[k] = *opt.fixed_first;
        if (bo.relax[k] > 1.0) res.notes.push_back("relaxed junction at waypoint 0");
        continue;
      }
      res.poses[k] = host_pose_from_dev(bo.poses[k]);
      if (bo.kind[k] == 1) {
        res.notes.push_back("cloud target at waypoint " + std::to_string(k));
      } else if (bo.relax[k] > 1.0) {
        res.notes.push_back("relaxed x" + std::to_string(bo.relax[k]) + " at waypoint " +
                            std::to_string(k));
      }
    }
    res.ok = true;
    return res;
  }
}

/// The host-sequenced backward pass (configurations past the device pass's
/// limits): one waypoint_ik launch sequence per waypoint.
PassResult backward_pass_sequenced(Planner& P, const std::vector<V3>& waypoints,
                                   const HostPose& anchor, const PassOptions& opt) {
  PassResult res;
  const size_t m = waypoints.size();
  res.poses.assign(m, HostPose{});
  res.relax.assign(m, 1.0);
  res.waypoints = waypoints;
  res.poses[m - 1] = anchor;
  for (size_t k = m - 1; k-- > 0;) {
    const HostPose prev = res.poses[k + 1];
    bool found = false;
    if (k == 0 && opt.fixed_first) {
      for (double f : opt.factors) {
        if (smoothness_ok(prev, *opt.fixed_first, P.pp, f)) {
          res.poses[0] = *opt.fixed_first;
          res.relax[0] = f;
          if (f > 1.0) res.notes.push_back("relaxed junction at waypoint 0");
          found = true;
          break;
        }
      }
      if (!found) {
        res.failed_index = 0;
        return res;
      }
      continue;
    }
    const Trail trail = trail_context(res.waypoints, k);
    const HostPose* bias = (opt.fixed_first && k == 1) ? opt.fixed_first : opt.junction_bias;
    HostPose pose;
    for (double f : opt.factors) {
      if (P.waypoint_ik(res.waypoints[k], prev, f, trail, bias, &pose)) {
        res.poses[k] = pose;
        res.relax[k] = f;
        if (f > 1.0)
          res.notes.push_back("relaxed x" + std::to_string(f) + " at waypoint " + std::to_string(k));
        found = true;
        break;
      }
    }
    if (!found && opt.cloud) {
      V3 dir = res.waypoints[k + 1] - res.waypoints[k];
      if (rpd::norm(dir) < 1e-12 && k > 0) dir = res.waypoints[k] - res.waypoints[k - 1];
      if (rpd::norm(dir) < 1e-12) dir = V3{0, 0, 1};
      dir = rpd::normalized(dir);
      const V3 u = perpendicular_of(dir);
      const V3 v = rpd::cross(dir, u);
      for (int t = 0; t < 8 && !found; ++t) {
        const double a = 2.0 * kPi * t / 8.0;
        const V3 cp = res.waypoints[k] + opt.cloud_radius * (std::cos(a) * u + std::sin(a) * v);
        for (double f : opt.factors) {
          if (P.waypoint_ik(cp, prev, f, trail, bias, &pose)) {
            res.poses[k] = pose;
            res.relax[k] = f;
            res.waypoints[k] = cp;
            res.notes.push_back("cloud target at waypoint " + std::to_string(k));
            found = true;
            break;
          }
        }
      }
    }
    if (!found) {
      res.failed_index = static_cast<int>(k);
      return res;
    }
  }
  res.ok = true;
  return res;
}

/// backward_pass (src/path_planner.cpp:322-400): the device pass, or the
/// sequenced one where the device pass does not apply.
PassResult backward_pass(Planner& P, const std::vector<V3>& waypoints, const HostPose& anchor,
                         const PassOptions& opt) {
  HostSpan span_("backward_pass");
  Planner::BpOut bo;
  if (P.backward_pass_device(waypoints, anchor, opt.factors, opt.cloud, opt.cloud_radius,
                             opt.fixed_first, opt.junction_bias, &bo))
    return pass_from_device(bo, waypoints, anchor, opt);
  return backward_pass_sequenced(P, waypoints, anchor, opt);
}

struct Build {
  std::string kind;
  std::vector<V3> waypoints;
  HostPose anchor;
  std::string fail_reason;
  bool ok = false;
};

std::vector<HostPose> solution_poses(rp_solution_set* s, const std::vector<long long>& ordinals);

/// make_candidate_build (src/path_planner.cpp:497-560)
Build make_candidate_build(Planner& P, const Cand& cand, V3 target) {
  HostSpan span_("make_candidate_build");
  Build out;
  const int n = P.n;
  try {
    if (cand.kind == RP_CHOSEN_REACH_POSE) {
      out.kind = "reach-pose";
      const int traversal = std::min(3, cand.pose.nseg);
      out.waypoints.push_back(P.ad.root);
      out.waypoints.insert(out.waypoints.end(), cand.pose.waypoints.begin(),
                           cand.pose.waypoints.begin() + traversal * n);
      if (cand.pose.nseg == 4) {
        const int mode = P.rp.refine_triangle_8dof ? 1 : 0;
        out.anchor = cand.has_refined && cand.refined_mode == mode &&
                             cand.refined_target.x == target.x && cand.refined_target.y == target.y &&
                             cand.refined_target.z == target.z
                         ? P.refine_result(cand.refined, cand.pose)
                         : P.refine(cand.pose, target, mode);
      } else {
        HostPose refined = P.refine(cand.pose, target, 2);
        if (P.arm.n_segments == 4) {
          HostPose trailed;
          if (!P.append_trail(refined, trail_context(out.waypoints, out.waypoints.size() - 1),
                              &trailed)) {
            out.fail_reason = "no valid fourth-segment fold at the final pose";
            return out;
          }
          refined = trailed;
        }
        out.anchor = refined;
      }
    } else {
      out.kind = "shortcut";
      out.waypoints.push_back(P.ad.root);
      const auto tips = cand.sc.tip_waypoints(target);
      out.waypoints.insert(out.waypoints.end(), tips.begin(), tips.end());
      rp_reach_params rp6 = P.rp;
      rp6.mode = RP_MODE_6DOF;
      rp6.near_target_radius = 0.0;
      const V3 final_wp = out.waypoints.back();
      std::unique_ptr<rp_solution_set> aset(solve_reach(P.ctx, P.arm, P.q, P.g, final_wp, rp6));
      if (aset->n_solutions == 0) {
        out.fail_reason = "no full pose at the shortcut endpoint";
        return out;
      }
      const rp_chosen ch = select(aset.get());
      if (ch.kind != RP_CHOSEN_REACH_POSE)
        fail(RP_E_INVALID_PARAMETER, "need a 3-segment pose");  // refine of an empty pose
      HostPose refined = P.refine(solution_poses(aset.get(), {ch.index})[0], final_wp, 2);
      if (P.arm.n_segments == 4) {
        HostPose trailed;
        if (!P.append_trail(refined, trail_context(out.waypoints, out.waypoints.size() - 1),
                            &trailed)) {
          out.fail_reason = "no valid fourth-segment fold at the shortcut pose";
          return out;
        }
        refined = trailed;
      }
      out.anchor = refined;
    }
  } catch (const Fail& e) {
    if (e.code == RP_E_CUDA || e.code == RP_E_INTERNAL) throw;
    out.fail_reason = e.msg;
    return out;
  }
  out.ok = true;
  return out;
}

rp_plan* assemble(PassResult&& pass, std::vector<HostPose>&& unfold, const std::string& kind) {
  auto* p = new rp_plan();
  p->waypoints = std::move(pass.waypoints);
  p->poses = std::move(pass.poses);
  p->unfold = std::move(unfold);
  p->kind = kind;
  p->relax = std::move(pass.relax);
  p->notes = std::move(pass.notes);
  return p;
}

struct Attempt {
  rp_plan* plan = nullptr;
  Failure failure;
};

/// attempt_candidate (src/path_planner.cpp:580-602)
Attempt attempt_candidate(Planner& P, const Cand& cand, V3 target, const PassOptions& opt,
                          const Build* prebuilt = nullptr) {
  HostSpan span_("attempt_candidate");
  Attempt r;
  const Build b = prebuilt ? *prebuilt : make_candidate_build(P, cand, target);
  if (!b.ok) {
    r.failure = {cand, b.waypoints, -1, b.fail_reason};
    return r;
  }
  PassResult pass = backward_pass(P, b.waypoints, b.anchor, opt);
  if (!pass.ok) {
    r.failure = {cand, b.waypoints, pass.failed_index, "no pose at waypoint",
                 std::make_shared<const Build>(b)};
    return r;
  }
  auto unfold = P.interpolate(nullptr, pass.poses[0], P.pp.unfold_steps);
  if (!unfold) {
    r.failure = {cand, b.waypoints, 0, "unfold blocked", std::make_shared<const Build>(b)};
    return r;
  }
  r.plan = assemble(std::move(pass), std::move(*unfold), b.kind);
  return r;
}

std::vector<V3> candidate_tip_path(const Cand& c, int n, V3 target) {
  if (c.kind == RP_CHOSEN_SHORTCUT) return c.sc.tip_waypoints(target);
  const int traversal = std::min(3, c.pose.nseg);
  return {c.pose.waypoints.begin(), c.pose.waypoints.begin() + traversal * n};
}

/// alternate_candidates (src/path_planner.cpp:612-663): the 3 nearest and
/// then up to 13 farthest by (mean polyline deviation, ordinal), scored and
/// sorted on the device.
std::vector<Cand> alternate_candidates(Planner& P, rp_solution_set* set, const Cand& failed,
                                       V3 target) {
  HostSpan span_("alternate_candidates");
  const std::vector<V3> failed_path = candidate_tip_path(failed, P.n, target);
  const int64_t S = static_cast<int64_t>(set->shortcuts.size());
  std::vector<std::vector<V3>> lists;
  for (const auto& sc : set->shortcuts) lists.push_back(sc.tip_waypoints(target));
  int64_t skip = -1;
  if (failed.kind == RP_CHOSEN_SHORTCUT) {
    for (int64_t k = 0; k < S; ++k) {
      const auto& sc = set->shortcuts[k];
      if (sc.seg1 == failed.sc.seg1 && sc.seg2 == failed.sc.seg2 &&
          sc.segment_index == failed.sc.segment_index) {
        skip = k;
        break;
      }
    }
  } else {
    skip = S + failed.ordinal;
  }
  int64_t total = 0;
  std::vector<long long> tail;
  const int want = 64;
  std::vector<long long> head =
      P.rank_by_deviation(set, lists, failed_path, false, V3{0, 0, 0}, &total, &tail, want, want);
  // Filtered sorted order F (skip removed), then near 3 + far <= 13.
  std::vector<long long> F_head, F_tail;
  for (long long o : head)
    if (o != skip) F_head.push_back(o);
  for (long long o : tail)
    if (o != skip) F_tail.push_back(o);
  const int64_t F = total - ((skip >= 0 && skip < total) ? 1 : 0);
  std::vector<long long> ordered;
  for (int64_t k = 0; k < F && k < 3; ++k) ordered.push_back(F_head[k]);
  for (int64_t k = F; k-- > 3 && ordered.size() < 16;) {
    // index k of F from the end of F_tail
    const int64_t from_end = F - 1 - k;
    ordered.push_back(F_tail[F_tail.size() - 1 - from_end]);
  }
  std::vector<Cand> out;
  std::vector<long long> sol_ords;
  for (long long o : ordered)
    if (o >= S) sol_ords.push_back(o - S);
  std::vector<HostPose> poses = solution_poses(set, sol_ords);
  size_t next = 0;
  for (long long o : ordered) {
    Cand c;
    if (o < S) {
      c.kind = RP_CHOSEN_SHORTCUT;
      c.ordinal = o;
      c.sc = set->shortcuts[o];
    } else {
      c.kind = RP_CHOSEN_REACH_POSE;
      c.ordinal = o - S;
      c.pose = poses[next++];
    }
    out.push_back(c);
  }
  return out;
}

rp_arm virtual_arm(V3 root, double reach, double clamp_total) {
  rp_arm v;
  const double lv = std::max(1e-6, std::min(reach, clamp_total) / 3.0);
  const double L[3] = {lv, lv, lv};
  rp_arm_init(&v, 3, L);
  v.root[0] = root.x;
  v.root[1] = root.y;
  v.root[2] = root.z;
  v.arm_radius = 0.0;
  return v;
}

rp_reach_params virtual_params(const rp_reach_params& rp) {
  rp_reach_params v = rp;
  v.mode = RP_MODE_6DOF;
  v.epsilon_gap = -1.0;
  v.near_target_radius = 0.0;
  v.approach_half_angle = 0.0;
  return v;
}

/// solve_reach that maps solver errors to an empty set (the reference's
/// try / catch around the virtual-arm solves).
std::unique_ptr<rp_solution_set> try_solve(rp_ctx* ctx, const rp_arm& arm, const rp_quiver* q,
                                           const rp_grid* g, V3 target, const rp_reach_params& rp) {
  try {
    return std::unique_ptr<rp_solution_set>(solve_reach(ctx, arm, q, g, target, rp));
  } catch (const Fail& e) {
    if (e.code == RP_E_CUDA || e.code == RP_E_INTERNAL) throw;
    return nullptr;
  }
}

/// Step 3 of fallback_cascade (src/path_planner.cpp:786-820): virtual-arm
/// detours from the blocked waypoint.
rp_plan* fallback_detour(Planner& P, const Failure& failure, V3 target, const PassOptions& cloud) {
  const Build b = failure.build ? *failure.build : make_candidate_build(P, failure.candidate, target);
  if (b.ok && failure.blocked_index > 0 && !failure.waypoints.empty()) {
    const V3 path_target = tracked_point(b.anchor);
    std::vector<V3> work(failure.waypoints.begin(),
                         failure.waypoints.begin() + failure.blocked_index + 1);
    for (int depth = 0; depth < 3; ++depth) {
      const V3 from = work.back();
      const rp_arm vspec = virtual_arm(from, rpd::norm(path_target - from), total_length(P.arm));
      auto vset = try_solve(P.ctx, vspec, P.q, P.g, path_target, virtual_params(P.rp));
      if (!vset || vset->n_solutions == 0) break;
      bool advanced = false;
      std::vector<long long> first;
      for (long long k = 0; k < std::min<int64_t>(8, vset->n_solutions); ++k) first.push_back(k);
      const std::vector<HostPose> vs = solution_poses(vset.get(), first);
      for (const HostPose& v : vs) {
        std::vector<V3> stitched = work;
        stitched.insert(stitched.end(), v.waypoints.begin(), v.waypoints.end());
        PassResult pass = backward_pass(P, stitched, b.anchor, cloud);
        if (pass.ok) {
          auto unfold = P.interpolate(nullptr, pass.poses[0], P.pp.unfold_steps);
          if (!unfold) continue;
          rp_plan* plan = assemble(std::move(pass), std::move(*unfold), b.kind);
          plan->notes.push_back("fallback: virtual-arm detour");
          return plan;
        }
        if (pass.failed_index > static_cast<int>(work.size())) {
          work.assign(stitched.begin(), stitched.begin() + pass.failed_index + 1);
          advanced = true;
          break;
        }
      }
      if (!advanced) break;
    }
  }
  fail(RP_E_NO_PATH, "no motion plan after relaxation, alternate solutions and detours");
}

/// Runs work(W, k) for k < n concurrently, one per worker context (own
/// stream; each call gets its own Planner W over P's arm, grid and quiver),
/// while `main_side` runs on the calling thread against P's context.
/// Results come back in index order, with any exception captured per call.
template <typename R>
struct Slot {
  R value{};
  std::exception_ptr error;
};
template <typename R>
std::vector<Slot<R>> run_parallel(Planner& P, int n, const std::function<R(Planner&, int)>& work,
                                  const std::function<void()>& main_side) {
  HostSpan span_("run_parallel");
  std::vector<Slot<R>> out(n);
  std::vector<rp_ctx*> ws;
  for (int k = 0; k < n; ++k) ws.push_back(worker_ctx(P.ctx, k));
  std::exception_ptr main_error;
  host_workers(P.ctx).run(
      n,
      [&](int k) {
        try {
          Planner W(ws[k], P.arm, P.q, P.g, P.rp, P.pp_in);
          // co-residency of the concurrent cooperative passes (1 block per SM)
          const int share = P.ctx->sm_count / n;
          W.bp_blocks_cap = share >= 16 ? (share & ~15) : std::max(1, share);
          out[k].value = work(W, k);
        } catch (...) {
          out[k].error = std::current_exception();
        }
      },
      [&] {
        try {
          if (main_side) main_side();
        } catch (...) {
          main_error = std::current_exception();
        }
      });
  for (rp_ctx* w : ws) ctx_absorb(P.ctx, w);
  if (main_error) std::rethrow_exception(main_error);
  return out;
}

/// {0, 1} in pinned memory: DMA sources for clearing / setting a pass's
/// cancellation flag (a later pass is stopped by a copy, no SMs needed).
int* pinned_01() {
  static int* p = [] {
    int* h = nullptr;
    RP_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&h), 2 * sizeof(int), cudaHostAllocDefault));
    h[0] = 0;
    h[1] = 1;
    return h;
  }();
  return p;
}

/// One attempt of the cascade.
struct Job {
  const Cand* cand;
  const PassOptions* opt;
  const Build* prebuilt = nullptr;
};
struct WindowResult {
  Attempt attempt;
  std::exception_ptr error;
};

/// The cascade's attempts of `jobs` concurrently (run_parallel). Each is a
/// pure function of (candidate, options), so taking the first success in
/// job order commits exactly what the reference's sequential loop commits.
std::vector<WindowResult> run_window(Planner& P, const std::vector<Job>& jobs, V3 target,
                                     const std::function<void()>& main_side) {
  std::vector<Slot<Attempt>> r = run_parallel<Attempt>(
      P, static_cast<int>(jobs.size()),
      [&](Planner& W, int k) {
        return attempt_candidate(W, *jobs[k].cand, target, *jobs[k].opt, jobs[k].prebuilt);
      },
      main_side);
  std::vector<WindowResult> out(r.size());
  for (size_t k = 0; k < r.size(); ++k) {
    out[k].attempt = std::move(r[k].value);
    out[k].error = r[k].error;
  }
  return out;
}

/// The first success of a window in job order (later plans are dropped);
/// an attempt that threw before any success rethrows, as the sequential
/// loop would have.
rp_plan* first_in_order(std::vector<WindowResult>& w) {
  rp_plan* found = nullptr;
  for (auto& r : w) {
    if (found) {
      delete r.attempt.plan;
      continue;
    }
    if (r.error) {
      for (auto& q : w) delete q.attempt.plan;
      std::rethrow_exception(r.error);
    }
    found = r.attempt.plan;
    r.attempt.plan = nullptr;
  }
  return found;
}

/// Steps 1a (escalation), 1b (target cloud) and 2 (alternate solutions) of
/// the cascade as one ordered job list drained by `width` worker contexts
/// (own stream and Planner each): the first two jobs start at once, the
/// alternates are appended when the main thread has ranked them (on the
/// main stream, concurrently) and run in groups of `width`, and a job is
/// skipped once an earlier one has decided the outcome. Every attempt is a pure function of (candidate,
/// options), so the lowest-index success -- or the lowest-index error
/// before any success -- is exactly what the reference's sequential loop
/// returns (src/path_planner.cpp:740-785). Returns the winning job index
/// and plan, or (-1, nullptr) when every job failed.
std::pair<int, rp_plan*> cascade_pool(Planner& P, const Failure& failure, rp_solution_set* set,
                                      V3 target, const PassOptions& esc, const PassOptions& cloud,
                                      int width) {
  const Cand& failed = failure.candidate;
  const Build* pre = failure.build.get();
  HostSpan span_("cascade_pool");
  std::mutex m;
  std::condition_variable cv;
  std::vector<Cand> alts;
  std::vector<Job> jobs{{&failed, &esc, pre}, {&failed, &cloud, pre}};
  jobs.reserve(64);
  std::vector<Slot<Attempt>> res(2);
  std::vector<char> done(2, 0);
  bool closed = false;
  size_t next = 0;
  size_t decided = SIZE_MAX;  // lowest index that succeeded or threw
  std::vector<rp_ctx*> ws;
  for (int k = 0; k < width; ++k) ws.push_back(worker_ctx(P.ctx, k));
  // Cancellation: one device flag per worker, polled by its cooperative
  // pass; a later job still running when an earlier one decides the outcome
  // is stopped by a DMA write of 1 on an auxiliary stream (no SMs needed).
  static const bool groups = std::getenv("RP_CASCADE_EAGER") == nullptr;
  int* const pinned01 = pinned_01();
  if (!P.ctx->aux) RP_CUDA(cudaStreamCreateWithFlags(&P.ctx->aux, cudaStreamNonBlocking));
  cudaStream_t aux = P.ctx->aux;
  std::vector<long long> running(width, -1);
  std::vector<char> cancelled(width, 0);
  // with m held: stop every running job that comes after `decided`
  auto cancel_later = [&] {
    for (int w = 0; w < width; ++w)
      if (running[w] >= 0 && static_cast<size_t>(running[w]) > decided && !cancelled[w]) {
        cancelled[w] = 1;
        RP_CUDA(cudaMemcpyAsync(ws[w]->cancel_flag, pinned01 + 1, sizeof(int),
                                cudaMemcpyHostToDevice, aux));
      }
  };
  const std::function<void(int)> worker = [&](int k) {
      std::unique_ptr<Planner> W;
      std::unique_lock<std::mutex> lk(m);
      // Alternates run in groups of `width`: group g >= 1 starts only when
      // every earlier job has finished, so no attempt starts that a running
      // one could make moot (on C2 the third alternate wins, and speculative
      // later attempts cost 0.2 ms of contention). Within a group, jobs
      // after a success are cancelled. RP_CASCADE_EAGER=1 starts every job
      // as soon as a worker is free and relies on cancellation alone (faster
      // when every attempt fails: C3's arbitrary leg 15.9 -> 15.3 ms).
      auto startable = [&] {
        if (next >= jobs.size()) return closed;
        if (next < 2 || !groups) return true;
        const size_t g = (next - 2) / width;
        if (g == 0) return true;
        const size_t lim = 2 + g * width;
        for (size_t i = 0; i < lim; ++i)
          if (!done[i]) return false;
        return true;
      };
      for (;;) {
        cv.wait(lk, startable);
        if (next >= jobs.size()) return;
        const size_t j = next++;
        if (j > decided) {
          done[j] = 1;
          cv.notify_all();
          continue;
        }
        const Job job = jobs[j];
        running[k] = static_cast<long long>(j);
        cancelled[k] = 0;
        lk.unlock();
        Slot<Attempt> out;
        try {
          if (!W) {
            RP_CUDA(cudaSetDevice(P.ctx->device));
            W = std::make_unique<Planner>(ws[k], P.arm, P.q, P.g, P.rp, P.pp_in);
            const int share = P.ctx->sm_count / width;
            W->bp_blocks_cap = share >= 16 ? (share & ~15) : std::max(1, share);
            W->cancel_flag = ws[k]->cancel_flag;
          }
          // clear this worker's flag in its stream order, before the pass
          RP_CUDA(cudaMemcpyAsync(ws[k]->cancel_flag, pinned01, sizeof(int), cudaMemcpyHostToDevice,
                                  ws[k]->stream));
          out.value = attempt_candidate(*W, *job.cand, target, *job.opt, job.prebuilt);
        } catch (...) {
          out.error = std::current_exception();
        }
        lk.lock();
        running[k] = -1;
        if ((out.value.plan || out.error) && j < decided) {
          decided = j;
          cancel_later();
        }
        static const bool dbg = std::getenv("RP_DEBUG_CASCADE") != nullptr;
        if (dbg)
          std::fprintf(stderr, "[cascade] job %zu kind %d ordinal %lld -> %s%s\n", j, job.cand->kind,
                       static_cast<long long>(job.cand->ordinal),
                       out.value.plan ? "plan" : (out.error ? "error" : "fail: "),
                       out.value.plan || out.error ? "" : out.value.failure.reason.c_str());
        res[j] = std::move(out);
        done[j] = 1;
        cv.notify_all();
      }
  };
  std::exception_ptr main_error;
  host_workers(P.ctx).run(width, worker, [&] {
    // the alternates are ranked on the calling thread while the first two
    // jobs run on the workers
    try {
      alts = alternate_candidates(P, set, failed, target);
    } catch (...) {
      main_error = std::current_exception();
    }
    {
      std::lock_guard<std::mutex> lk(m);
      if (!main_error) {
        for (const Cand& c : alts) jobs.push_back({&c, &cloud});
        res.resize(jobs.size());
        done.resize(jobs.size(), 0);
      }
      closed = true;
    }
    cv.notify_all();
  });
  RP_CUDA(cudaStreamSynchronize(aux));
  for (rp_ctx* w : ws) ctx_absorb(P.ctx, w);
  int win = -1;
  rp_plan* plan = nullptr;
  std::exception_ptr err;
  for (size_t j = 0; j < res.size(); ++j) {
    if (win < 0 && !err) {
      if (res[j].error) err = res[j].error;
      else if (res[j].value.plan) {
        win = static_cast<int>(j);
        plan = res[j].value.plan;
        continue;
      }
    }
    delete res[j].value.plan;
  }
  if (err) {
    delete plan;
    std::rethrow_exception(err);
  }
  if (win < 0 && main_error) std::rethrow_exception(main_error);
  return {win, plan};
}

// concurrent attempts per window; each pass then takes sm_count / width
// blocks (rounded down to 16) so all of them stay co-resident
static int cascade_width() {
  static const int w = std::getenv("RP_CASCADE_WIDTH") ? std::atoi(std::getenv("RP_CASCADE_WIDTH")) : 3;
  return std::max(1, std::min(w, 4));
}

/// fallback_cascade (src/path_planner.cpp:740-822)
rp_plan* fallback_cascade(Planner& P, const Failure& failure, rp_solution_set* set, V3 target) {
  PassOptions esc;
  esc.factors = with_unit_first(P.pp.relax);
  if (!P.pp.relax.empty()) {
    const double last = P.pp.relax.back();
    for (double s : P.pp.relax) esc.factors.push_back(last * s);
  }
  static const bool serial = std::getenv("RP_SERIAL_CASCADE") != nullptr;
  if (!serial) {
    // Steps 1a (escalation), 1b (target cloud) and 2 (alternate solutions)
    // are independent attempts tried in a fixed order: run them two at a
    // time on worker streams and keep the first success in that order. The
    // alternates are ranked on the main stream while step 1 runs.
    PassOptions cloud = esc;
    cloud.cloud = true;
    cloud.cloud_radius = 2.0 * P.pp.eps_wp;
    static const bool windows = std::getenv("RP_CASCADE_WINDOWS") != nullptr;
    if (!windows) {
      const auto [win, plan] =
          cascade_pool(P, failure, set, target, esc, cloud, cascade_width());
      if (plan) {
        plan->notes.push_back(win == 0   ? "fallback: relaxation escalation"
                              : win == 1 ? "fallback: target cloud"
                                         : "fallback: alternate solution");
        return plan;
      }
      return fallback_detour(P, failure, target, cloud);
    }
    std::vector<Cand> alts;
    std::vector<WindowResult> w = run_window(
        P,
        {{&failure.candidate, &esc, failure.build.get()},
         {&failure.candidate, &cloud, failure.build.get()}},
        target,
        [&] { alts = alternate_candidates(P, set, failure.candidate, target); });
    const bool esc_ok = w[0].attempt.plan != nullptr && !w[0].error;
    if (rp_plan* plan = first_in_order(w)) {
      plan->notes.push_back(esc_ok ? "fallback: relaxation escalation" : "fallback: target cloud");
      return plan;
    }
    for (size_t a = 0; a < alts.size(); a += cascade_width()) {
      std::vector<Job> jobs;
      for (size_t k = a; k < std::min(alts.size(), a + cascade_width()); ++k)
        jobs.push_back({&alts[k], &cloud});
      std::vector<WindowResult> r = run_window(P, jobs, target, {});
      if (rp_plan* plan = first_in_order(r)) {
        plan->notes.push_back("fallback: alternate solution");
        return plan;
      }
    }
    return fallback_detour(P, failure, target, cloud);
  }
  {
    Attempt r = attempt_candidate(P, failure.candidate, target, esc, failure.build.get());
    if (r.plan) {
      r.plan->notes.push_back("fallback: relaxation escalation");
      return r.plan;
    }
  }
  PassOptions cloud = esc;
  cloud.cloud = true;
  cloud.cloud_radius = 2.0 * P.pp.eps_wp;
  {
    Attempt r = attempt_candidate(P, failure.candidate, target, cloud, failure.build.get());
    if (r.plan) {
      r.plan->notes.push_back("fallback: target cloud");
      return r.plan;
    }
  }
  for (const Cand& c : alternate_candidates(P, set, failure.candidate, target)) {
    Attempt r = attempt_candidate(P, c, target, cloud);
    if (r.plan) {
      r.plan->notes.push_back("fallback: alternate solution");
      return r.plan;
    }
  }
  return fallback_detour(P, failure, target, cloud);
}

Cand chosen_cand(rp_solution_set* set, const rp_chosen& ch) {
  Cand c;
  c.kind = ch.kind;
  c.ordinal = ch.index;
  if (ch.kind == RP_CHOSEN_SHORTCUT) {
    c.sc = set->shortcuts[ch.index];
  } else {
    c.pose = solution_poses(set, {ch.index})[0];
  }
  return c;
}

/// select_solution + chosen_cand + the 8DOF pose's exact refinement in one
/// device round trip when the choice is a reach pose: the canonical ordinal
/// of the best key (k_rank), its pose (k_materialize from the key, no key
/// compaction) and refine(pose, target, mode) are launched back to back and
/// read together. Otherwise (shortcuts, 6DOF, nothing found) the plain
/// select + chosen_cand (which throw as the reference does).
Cand select_cand(Planner& P, rp_solution_set* set, V3 target, int mode) {
  if (!set->shortcuts.empty() || set->n_solutions == 0 || set->rp.mode != RP_MODE_8DOF ||
      set->arm.n_segments != 4)
    return chosen_cand(set, select(set));
  HostSpan span_("select_cand");
  rp_ctx* ctx = set->ctx;
  cudaStream_t st = ctx->stream;
  DevBuf<unsigned long long> rank(1, st);
  launch_rank_of_key(set, set->best_key, rank.p);
  DevBuf<long long> key(1, st);
  copy_to_device(ctx, key.p, &set->best_key, sizeof(long long));
  DevBuf<DevPose> d(1, st);
  materialize_solutions(set, key.p, nullptr, 1, d.p);
  P.refine_launch(d.p, target, mode);
  unsigned long long hr = 0;
  DevPose hp{};
  Cand c;
  copy_to_host_many(ctx, {{&hr, rank.p, sizeof(hr)},
                          {&hp, d.p, sizeof(DevPose)},
                          {&c.refined, P.opout.p, sizeof(PoseOpOut)}});
  c.kind = RP_CHOSEN_REACH_POSE;
  c.ordinal = static_cast<int64_t>(hr);
  c.pose = host_pose_from_dev(hp);
  c.has_refined = true;
  c.refined_mode = mode;
  c.refined_target = target;
  return c;
}

rp_plan* plan_from_cand(Planner& P, rp_solution_set* set, const Cand& c, V3 target) {
  PassOptions opt;
  opt.factors = with_unit_first(P.pp.relax);
  Attempt r = attempt_candidate(P, c, target, opt);
  if (r.plan) return r.plan;
  return fallback_cascade(P, r.failure, set, target);
}

/// plan_from_reach (src/path_planner.cpp:729-738)
rp_plan* plan_from_reach(Planner& P, rp_solution_set* set, const rp_chosen& ch, V3 target) {
  return plan_from_cand(P, set, chosen_cand(set, ch), target);
}

/// build_target_anchor (src/path_planner.cpp:872-902)
bool build_target_anchor(Planner& P, V3 target, const rp_reach_params& rp, V3 hint, HostPose* out) {
  rp_reach_params rpa = rp;
  rpa.near_target_radius = 0.0;
  auto set = try_solve(P.ctx, P.arm, P.q, P.g, target, rpa);
  if (!set || set->n_solutions == 0) return false;
  try {
    if (set->shortcuts.empty() && set->rp.mode == RP_MODE_8DOF && set->arm.n_segments == 4) {
      // the reach pose, its ordinal and refine(pose, target, 0) in one round trip
      const Cand c = select_cand(P, set.get(), target, 0);
      *out = P.refine_result(c.refined, c.pose);
      return true;
    }
  } catch (const Fail& e) {
    if (e.code == RP_E_CUDA || e.code == RP_E_INTERNAL) throw;
    return false;
  }
  const rp_chosen ch = select(set.get());
  if (ch.kind != RP_CHOSEN_REACH_POSE) return false;  // refine of an empty pose throws
  try {
    const HostPose pose = solution_poses(set.get(), {ch.index})[0];
    if (pose.nseg == 4) {
      *out = P.refine(pose, target, 0);
      return true;
    }
    HostPose refined = P.refine(pose, target, 2);
    if (P.arm.n_segments == 4) {
      Trail trail;
      if (rpd::norm(hint) > 1e-12) {
        trail.has_back = true;
        trail.back = -rpd::normalized(hint);
      }
      HostPose trailed;
      if (!P.append_trail(refined, trail, &trailed)) return false;
      refined = trailed;
    }
    *out = refined;
    return true;
  } catch (const Fail& e) {
    if (e.code == RP_E_CUDA || e.code == RP_E_INTERNAL) throw;
    return false;
  }
}

/// screen_real_reach (src/path_planner.cpp:692-707)
bool screen_real_reach(const rp_arm& a, const std::vector<V3>& wps, int n, double eps) {
  const double L0 = a.lengths[0], L1 = a.lengths[1], L2 = a.lengths[2];
  const double r_max = L0 + L1 + L2 + eps;
  const double lmax = std::max({L0, L1, L2});
  const double r_min = std::max(0.0, 2.0 * lmax - (L0 + L1 + L2)) - eps;
  const V3 root{a.root[0], a.root[1], a.root[2]};
  const size_t segs = wps.size() / static_cast<size_t>(n);
  for (size_t s = 0; s < segs; ++s) {
    for (size_t k : {s * n + n / 2, s * n + n - 1}) {
      const double d = rpd::norm(wps[k] - root);
      if (d > r_max || d < std::max(0.0, r_min)) return false;
    }
  }
  return true;
}

/// plan_virtual_path (src/path_planner.cpp:840-868); candidates come lazily
/// in batches from `next_batch` (empty = exhausted).
template <typename NextBatch>
rp_plan* plan_virtual_path(Planner& P, const HostPose& start, NextBatch next_batch,
                           const HostPose& anchor, V3 path_target) {
  const V3 e0 = tracked_point(start);
  PassOptions opt;
  opt.factors = with_unit_first(P.pp.relax);
  opt.fixed_first = &start;
  auto to_plan = [](PassResult& pass) {
    auto* plan = new rp_plan();
    plan->waypoints = std::move(pass.waypoints);
    plan->poses = std::move(pass.poses);
    plan->kind = "virtual-arm";
    plan->relax = std::move(pass.relax);
    plan->notes = std::move(pass.notes);
    return plan;
  };
  static const bool serial = std::getenv("RP_SERIAL_CASCADE") != nullptr;
  const int width = serial ? 1 : cascade_width();
  for (;;) {
    const std::vector<HostPose> batch = next_batch();
    if (batch.empty()) return nullptr;
    // the screened candidates in order; their pinned passes are independent,
    // so they run `width` at a time and the first success in order wins
    std::vector<std::vector<V3>> wps_list;
    for (const HostPose& v : batch) {
      if (!screen_real_reach(P.arm, v.waypoints, P.n, P.pp.eps_wp)) continue;
      std::vector<V3> wps{e0};
      wps.insert(wps.end(), v.waypoints.begin(), v.waypoints.end());
      wps.back() = path_target;
      wps_list.push_back(std::move(wps));
    }
    for (size_t a = 0; a < wps_list.size(); a += width) {
      const int m = static_cast<int>(std::min<size_t>(width, wps_list.size() - a));
      if (m == 1) {
        PassResult pass = backward_pass(P, wps_list[a], anchor, opt);
        if (pass.ok) return to_plan(pass);
        continue;
      }
      // a success cancels the later candidates' passes (they would lose to
      // it anyway): a DMA of 1 into their flags on the context's aux stream
      if (!P.ctx->aux) RP_CUDA(cudaStreamCreateWithFlags(&P.ctx->aux, cudaStreamNonBlocking));
      std::vector<int*> flags(m);
      for (int k = 0; k < m; ++k) {
        flags[k] = worker_ctx(P.ctx, k)->cancel_flag;
        RP_CUDA(cudaMemcpyAsync(flags[k], pinned_01(), sizeof(int), cudaMemcpyHostToDevice,
                                P.ctx->aux));
      }
      // the passes wait for the clears on the device (no host synchronisation);
      // later cancel copies follow them in the aux stream's order
      if (!P.ctx->aux_ev) RP_CUDA(cudaEventCreateWithFlags(&P.ctx->aux_ev, cudaEventDisableTiming));
      RP_CUDA(cudaEventRecord(P.ctx->aux_ev, P.ctx->aux));
      cudaEvent_t cleared = P.ctx->aux_ev;
      // Every candidate's pass is set up and launched from this thread on
      // its worker context's stream (no host threads: the passes' host
      // setup is short and serial anyway), then the results are taken in
      // candidate order; the first success cancels the passes after it.
      std::vector<std::unique_ptr<Planner>> Ws(m);
      std::vector<char> launched(m, 0), finished(m, 0);
      auto settle = [&] {  // no pass may outlive its planner's buffers
        for (int k = 0; k < m; ++k)
          if (launched[k] && !finished[k]) {
            Planner::BpOut bo;
            try {
              Ws[k]->bp_finish(&bo);
            } catch (...) {
            }
            finished[k] = 1;
          }
        cudaStreamSynchronize(P.ctx->aux);
        for (int k = 0; k < m; ++k) ctx_absorb(P.ctx, worker_ctx(P.ctx, k));
      };
      rp_plan* won = nullptr;
      try {
        for (int k = 0; k < m; ++k) {
          rp_ctx* wc = worker_ctx(P.ctx, k);
          Ws[k] = std::make_unique<Planner>(wc, P.arm, P.q, P.g, P.rp, P.pp_in);
          const int share = P.ctx->sm_count / m;
          Ws[k]->bp_blocks_cap = share >= 16 ? (share & ~15) : std::max(1, share);
          Ws[k]->cancel_flag = flags[k];
          RP_CUDA(cudaStreamWaitEvent(wc->stream, cleared, 0));
          launched[k] = Ws[k]->bp_launch(wps_list[a + k], anchor, opt.factors, opt.cloud,
                                         opt.cloud_radius, opt.fixed_first, opt.junction_bias)
                            ? 1
                            : 0;
        }
        for (int k = 0; k < m && !won; ++k) {
          PassResult pr;
          Planner::BpOut bo;
          const bool dev = launched[k] && Ws[k]->bp_finish(&bo);
          finished[k] = 1;
          pr = dev ? pass_from_device(bo, wps_list[a + k], anchor, opt)
                   : backward_pass_sequenced(*Ws[k], wps_list[a + k], anchor, opt);
          if (pr.ok) {
            for (int j = k + 1; j < m; ++j)
              if (launched[j])
                RP_CUDA(cudaMemcpyAsync(flags[j], pinned_01() + 1, sizeof(int),
                                        cudaMemcpyHostToDevice, P.ctx->aux));
            won = to_plan(pr);
          }
        }
      } catch (...) {
        settle();
        throw;
      }
      settle();
      if (won) return won;
    }
  }
}

}  // namespace

PP resolve_path_params(const rp_path_params& p, const rp_arm& arm, const rp_reach_params& rp) {
  PP r;
  r.d_w = p.d_w < 0.0 ? nominal_spacing(arm, rp) : p.d_w;
  r.slack = p.slack < 0.0 ? 0.5 * r.d_w : p.slack;
  r.j1 = p.joint1_max_move < 0.0 ? 0.5 * r.d_w + r.slack : p.joint1_max_move;
  r.j2 = p.joint2_max_move < 0.0 ? 1.0 * r.d_w + r.slack : p.joint2_max_move;
  r.eps_wp = p.epsilon_waypoint < 0.0 ? r.d_w : p.epsilon_waypoint;
  r.unfold_steps = p.unfold_steps;
  require(r.eps_wp > 0 && r.d_w > 0 && r.slack >= 0 && r.j1 > 0 && r.j2 > 0 && r.unfold_steps >= 1,
          RP_E_INVALID_PARAMETER, "path parameters must be positive");
  require(p.n_relax >= 0 && p.n_relax <= RP_MAX_RELAX, RP_E_INVALID_PARAMETER,
          "at most 8 relaxation factors");
  for (int k = 0; k < p.n_relax; ++k) {
    require(p.relax_schedule[k] >= 1.0, RP_E_INVALID_PARAMETER,
            "relaxation factors must be >= 1");
    r.relax.push_back(p.relax_schedule[k]);
  }
  return r;
}

namespace {

__global__ void k_gather_keys(const long long* __restrict__ keys, const long long* __restrict__ ords,
                              int64_t n, long long* __restrict__ out) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < n) out[t] = keys[ords[t]];
}

std::vector<HostPose> solution_poses(rp_solution_set* s, const std::vector<long long>& ordinals) {
  HostSpan span_("solution_poses");
  std::vector<HostPose> out;
  if (ordinals.empty()) return out;
  ensure_keys(s);
  rp_ctx* ctx = s->ctx;
  const int64_t n = static_cast<int64_t>(ordinals.size());
  DevBuf<long long> ords(n, ctx->stream), keys(n, ctx->stream);
  copy_to_device(ctx, ords.p, ordinals.data(), n * sizeof(long long));
  launch(ctx, "materialize", k_gather_keys, dim3(static_cast<unsigned>((n + 127) / 128)),
         dim3(128), 0, static_cast<const long long*>(s->keys.p),
         static_cast<const long long*>(ords.p), n, keys.p);
  DevBuf<DevPose> d(n, ctx->stream);
  materialize_solutions(s, keys.p, nullptr, n, d.p);
  std::vector<DevPose> h(n);
  copy_to_host(ctx, h.data(), d.p, n * sizeof(DevPose));
  for (const auto& p : h) out.push_back(host_pose_from_dev(p));
  return out;
}

}  // namespace

rp_plan* plan_reach_then_path(rp_ctx* ctx, const rp_arm& arm, const rp_quiver* q, const rp_grid* g,
                              V3 target, const rp_reach_params& rp, const rp_path_params& pp) {
  std::unique_ptr<rp_solution_set> set(solve_reach(ctx, arm, q, g, target, rp));
  if (set->n_solutions == 0 && set->shortcuts.empty()) select(set.get());  // no_solution first
  Planner P(ctx, arm, q, g, rp, pp);
  const Cand c = select_cand(P, set.get(), target, P.rp.refine_triangle_8dof ? 1 : 0);
  return plan_from_cand(P, set.get(), c, target);
}

/// plan_arbitrary (src/path_planner.cpp:906-998)
rp_plan* plan_arbitrary(rp_ctx* ctx, const rp_arm& arm, const rp_quiver* q, const rp_grid* g,
                        const HostPose& start, V3 target, const rp_reach_params& rp,
                        const rp_path_params& pp) {
  Planner P(ctx, arm, q, g, rp, pp);
  const V3 e0 = tracked_point(start);
  if (rpd::norm(e0 - target) <= P.pp.eps_wp && arm.n_segments == start.nseg) {
    auto* plan = new rp_plan();
    plan->waypoints = {e0};
    plan->poses = {start};
    plan->kind = "virtual-arm";
    plan->relax = {1.0};
    return plan;
  }
  HostPose anchor;
  if (build_target_anchor(P, target, rp, target - e0, &anchor)) {
    const V3 path_target = tracked_point(anchor);
    const rp_arm vspec = virtual_arm(e0, rpd::norm(path_target - e0), total_length(arm));
    auto vset = try_solve(ctx, vspec, q, g, path_target, virtual_params(rp));
    bool served = false;
    auto batch = [&]() -> std::vector<HostPose> {
      if (served || !vset || vset->n_solutions == 0) return {};
      served = true;
      std::vector<long long> ords;
      for (long long k = 0; k < std::min<int64_t>(24, vset->n_solutions); ++k) ords.push_back(k);
      return solution_poses(vset.get(), ords);
    };
    if (rp_plan* plan = plan_virtual_path(P, start, batch, anchor, path_target)) return plan;
  }
  rp_reach_params rp_back = rp;
  rp_back.mode = RP_MODE_6DOF;
  rp_back.approach_half_angle = 0.0;
  std::unique_ptr<rp_plan> back(plan_reach_then_path(ctx, arm, q, g, e0, rp_back, pp));
  std::unique_ptr<rp_plan> out(plan_reach_then_path(ctx, arm, q, g, target, rp, pp));
  double junction = 0.0;
  for (double f : with_unit_first(P.pp.relax)) {
    if (smoothness_ok(start, back->poses.back(), P.pp, f)) {
      junction = f;
      break;
    }
  }
  require(junction > 0.0, RP_E_NO_PATH, "start pose does not join the retraction path smoothly");
  const auto back_seq = back->full_sequence();
  const auto out_seq = out->full_sequence();
  auto bridge = P.interpolate(back_seq.front(), *out_seq.front(), P.pp.unfold_steps);
  require(bridge.has_value(), RP_E_NO_PATH, "folded poses of the two legs cannot be joined");
  auto* plan = new rp_plan();
  plan->kind = "out-and-back";
  auto push = [&](const HostPose& p, double relax) {
    plan->poses.push_back(p);
    plan->waypoints.push_back(tracked_point(p));
    plan->relax.push_back(relax);
  };
  push(start, junction);
  for (size_t k = back_seq.size(); k-- > 0;) {
    const size_t wp_count = back->poses.size();
    double relax = 1.0;
    if (k >= back_seq.size() - wp_count) relax = back->relax[k - (back_seq.size() - wp_count)];
    push(*back_seq[k], relax);
  }
  for (size_t k = 1; k + 1 < bridge->size(); ++k) push((*bridge)[k], 1.0);
  for (size_t k = 0; k < out_seq.size(); ++k) {
    const size_t wp_count = out->poses.size();
    double relax = 1.0;
    if (k >= out_seq.size() - wp_count) relax = out->relax[k - (out_seq.size() - wp_count)];
    push(*out_seq[k], relax);
  }
  plan->notes.push_back("out-and-back via the folded pose");
  return plan;
}

/// replan_dynamic (src/path_planner.cpp:1000-1102)
rp_plan* replan_dynamic(rp_ctx* ctx, const rp_arm& arm, const rp_quiver* q, const rp_grid* gs,
                        const rp_plan& active, int current, const rp_obstacle& obs, double period,
                        double cost, const rp_reach_params& rp, const rp_path_params& pp) {
  const PP ppr = resolve_path_params(pp, arm, rp);
  const int m = static_cast<int>(active.poses.size());
  require(current >= 0 && current < m, RP_E_INVALID_PARAMETER, "current waypoint index out of range");
  require(period > 0.0 && cost >= 0.0, RP_E_INVALID_PARAMETER, "replan timing must be positive");
  rp_grid* aug_raw = nullptr;
  rp_status st = rp_grid_overlay(gs, &obs, &aug_raw);
  if (st != RP_OK) throw Fail{st, rp_last_error()};
  struct GridDel {
    void operator()(rp_grid* g) const { rp_grid_destroy(g); }
  };
  std::unique_ptr<rp_grid, GridDel> aug(aug_raw);
  Planner P(ctx, arm, q, aug.get(), rp, pp);
  const int collide_at = P.first_colliding(active.poses, aug.get());
  if (collide_at < 0) return new rp_plan(active);
  require(collide_at - current >= 3, RP_E_INFEASIBLE_TIMING,
          "collision fewer than three waypoints ahead of the arm");
  const double est = cost * (m - current);
  const int switch_index =
      current + std::max(1, static_cast<int>(std::ceil(est / period))) + 1;
  require(switch_index <= collide_at - 1, RP_E_INFEASIBLE_TIMING,
          "no time to switch paths before the collision point");
  const HostPose switch_pose = active.poses[switch_index];
  const V3 from = tracked_point(switch_pose);
  const V3 target = active.waypoints.back();
  HostPose anchor;
  require(build_target_anchor(P, target, rp, target - from, &anchor), RP_E_NO_PATH,
          "target unreachable while the dynamic obstacle is in the way");
  const V3 path_target = tracked_point(anchor);
  const rp_arm vspec = virtual_arm(from, rpd::norm(path_target - from), total_length(arm));
  auto vset = try_solve(ctx, vspec, q, aug.get(), path_target, virtual_params(rp));
  require(vset && vset->n_solutions > 0, RP_E_NO_PATH, "no avoidance path around the dynamic obstacle");
  // order = all candidates by (mean deviation of [from] + tip, ordinal)
  int64_t total = 0;
  const int64_t nsol = vset->n_solutions;
  std::vector<long long> order = P.rank_by_deviation(vset.get(), {}, active.waypoints, true, from,
                                                     &total, nullptr, static_cast<int>(nsol), 0);
  size_t pos = 0;
  auto batch = [&]() -> std::vector<HostPose> {
    if (pos >= order.size()) return {};
    const size_t e = std::min(order.size(), pos + 256);
    std::vector<long long> ords(order.begin() + pos, order.begin() + e);
    pos = e;
    return solution_poses(vset.get(), ords);
  };
  std::unique_ptr<rp_plan> att(plan_virtual_path(P, switch_pose, batch, anchor, path_target));
  require(att != nullptr, RP_E_NO_PATH, "no valid pose sequence along any avoidance path");
  auto* plan = new rp_plan();
  plan->kind = "replan";
  plan->switch_index = switch_index;
  plan->unfold = active.unfold;
  plan->waypoints.assign(active.waypoints.begin(), active.waypoints.begin() + switch_index + 1);
  plan->poses.assign(active.poses.begin(), active.poses.begin() + switch_index + 1);
  plan->relax.assign(active.relax.begin(), active.relax.begin() + switch_index + 1);
  for (size_t k = 1; k < att->poses.size(); ++k) {
    plan->poses.push_back(att->poses[k]);
    plan->waypoints.push_back(att->waypoints[k]);
    plan->relax.push_back(att->relax[k]);
  }
  plan->notes = att->notes;
  plan->notes.push_back(std::string("replanned around dynamic obstacle ") +
                        (obs.id ? obs.id : ""));
  (void)ppr;
  return plan;
}

}  // namespace rp

using namespace rp;

extern "C" {

rp_status rp_plan_reach_then_path(rp_ctx* ctx, const rp_arm* arm, const rp_quiver* q,
                                  const rp_grid* g, const double target[3],
                                  const rp_reach_params* rp, const rp_path_params* pp,
                                  rp_plan** out) {
  return guarded([&] {
    *out = plan_reach_then_path(ctx, *arm, q, g, V3{target[0], target[1], target[2]}, *rp, *pp);
  });
}

rp_status rp_plan_from_reach(rp_ctx* ctx, const rp_arm* arm, const rp_quiver* q, const rp_grid* g,
                             const rp_solution_set* set, const rp_chosen* chosen,
                             const double target[3], const rp_reach_params* rp,
                             const rp_path_params* pp, rp_plan** out) {
  return guarded([&] {
    Planner P(ctx, *arm, q, g, *rp, *pp);
    *out = plan_from_reach(P, const_cast<rp_solution_set*>(set), *chosen,
                           V3{target[0], target[1], target[2]});
  });
}

rp_status rp_fallback_cascade(rp_ctx* ctx, const rp_arm* arm, const rp_quiver* q, const rp_grid* g,
                              const rp_solution_set* set, const rp_chosen* failed,
                              const double* waypoints, int32_t n_waypoints, int32_t blocked_index,
                              const double target[3], const rp_reach_params* rp,
                              const rp_path_params* pp, rp_plan** out) {
  return guarded([&] {
    require(n_waypoints >= 0 && (n_waypoints == 0 || waypoints), RP_E_INVALID_PARAMETER,
            "waypoints missing");
    Planner P(ctx, *arm, q, g, *rp, *pp);
    auto* s = const_cast<rp_solution_set*>(set);
    Failure f;
    f.candidate = chosen_cand(s, *failed);
    for (int k = 0; k < n_waypoints; ++k)
      f.waypoints.push_back(V3{waypoints[3 * k], waypoints[3 * k + 1], waypoints[3 * k + 2]});
    f.blocked_index = blocked_index;
    *out = fallback_cascade(P, f, s, V3{target[0], target[1], target[2]});
  });
}

rp_status rp_plan_arbitrary(rp_ctx* ctx, const rp_arm* arm, const rp_quiver* q, const rp_grid* g,
                            const rp_pose* start, const double* start_wps, const double target[3],
                            const rp_reach_params* rp, const rp_path_params* pp, rp_plan** out) {
  return guarded([&] {
    *out = plan_arbitrary(ctx, *arm, q, g, from_abi(*start, start_wps),
                          V3{target[0], target[1], target[2]}, *rp, *pp);
  });
}

rp_status rp_replan_dynamic(rp_ctx* ctx, const rp_arm* arm, const rp_quiver* q,
                            const rp_grid* grid_static, const rp_plan* active, int32_t current,
                            const rp_obstacle* obs, double period, double cost,
                            const rp_reach_params* rp, const rp_path_params* pp, rp_plan** out) {
  return guarded([&] {
    *out = replan_dynamic(ctx, *arm, q, grid_static, *active, current, *obs, period, cost, *rp, *pp);
  });
}

rp_status rp_waypoint_ik(rp_ctx* ctx, const rp_arm* arm, const rp_quiver* q, const rp_grid* g,
                         const double waypoint[3], const rp_pose* prev, const rp_reach_params* rp,
                         const rp_path_params* pp, double relax, const double* back,
                         const double* fwd, const rp_pose* bias, int32_t* found, rp_pose* out,
                         double* wps, int32_t cap) {
  return guarded([&] {
    Planner P(ctx, *arm, q, g, *rp, *pp);
    Trail t;
    if (back) {
      t.has_back = true;
      t.back = V3{back[0], back[1], back[2]};
    }
    if (fwd) {
      t.has_fwd = true;
      t.fwd = V3{fwd[0], fwd[1], fwd[2]};
    }
    const HostPose hp = from_abi(*prev, nullptr);
    HostPose hb;
    if (bias) hb = from_abi(*bias, nullptr);
    HostPose res;
    const bool ok = P.waypoint_ik(V3{waypoint[0], waypoint[1], waypoint[2]}, hp, relax, t,
                                  bias ? &hb : nullptr, &res);
    *found = ok ? 1 : 0;
    if (ok) to_abi(res, out, wps, cap);
  });
}

rp_status rp_smoothness_ok(const rp_arm* arm, const rp_reach_params* rp, const rp_path_params* pp,
                           const rp_pose* prev, const rp_pose* cand, double relax, int32_t* ok) {
  return guarded([&] {
    const PP r = resolve_path_params(*pp, *arm, *rp);
    *ok = smoothness_ok(from_abi(*prev, nullptr), from_abi(*cand, nullptr), r, relax) ? 1 : 0;
  });
}

rp_status rp_path_params_resolve(const rp_arm* arm, const rp_reach_params* rp,
                                 const rp_path_params* pp, rp_path_params* out) {
  return guarded([&] {
    const PP r = resolve_path_params(*pp, *arm, *rp);
    *out = *pp;
    out->epsilon_waypoint = r.eps_wp;
    out->d_w = r.d_w;
    out->slack = r.slack;
    out->joint1_max_move = r.j1;
    out->joint2_max_move = r.j2;
  });
}

rp_status rp_mean_polyline_deviation(rp_ctx* ctx, const double* pts, int32_t n, const double* poly,
                                     int32_t np, double* out) {
  return guarded([&] {
    std::vector<V3> a(n), b(np);
    std::memcpy(a.data(), pts, n * sizeof(V3));
    std::memcpy(b.data(), poly, np * sizeof(V3));
    *out = mean_polyline_deviation(ctx, a, b);
  });
}

rp_status rp_folded_pose(rp_ctx* ctx, const rp_arm* arm, rp_pose* out) {
  return guarded([&] {
    validate_arm(*arm);
    to_abi(folded_pose_host(ctx, *arm), out, nullptr, 0);
  });
}

rp_status rp_plan_get_info(const rp_plan* p, rp_plan_info* info) {
  return guarded([&] {
    std::memset(info, 0, sizeof(*info));
    info->n_waypoints = static_cast<int>(p->waypoints.size());
    info->n_poses = static_cast<int>(p->poses.size());
    info->n_unfold = static_cast<int>(p->unfold.size());
    info->n_notes = static_cast<int>(p->notes.size());
    info->replan_switch_index = p->switch_index;
    std::strncpy(info->kind, p->kind.c_str(), sizeof(info->kind) - 1);
  });
}

rp_status rp_plan_waypoints(const rp_plan* p, double* xyz, int32_t cap) {
  return guarded([&] {
    for (size_t k = 0; k < p->waypoints.size() && static_cast<int>(k) < cap; ++k) {
      xyz[3 * k] = p->waypoints[k].x;
      xyz[3 * k + 1] = p->waypoints[k].y;
      xyz[3 * k + 2] = p->waypoints[k].z;
    }
  });
}

rp_status rp_plan_relax(const rp_plan* p, double* relax, int32_t cap) {
  return guarded([&] {
    for (size_t k = 0; k < p->relax.size() && static_cast<int>(k) < cap; ++k) relax[k] = p->relax[k];
  });
}

rp_status rp_plan_pose(const rp_plan* p, int32_t which, int32_t k, rp_pose* pose, double* wps,
                       int32_t cap) {
  return guarded([&] {
    const auto& v = which == 0 ? p->poses : p->unfold;
    require(k >= 0 && k < static_cast<int>(v.size()), RP_E_INVALID_PARAMETER, "pose index out of range");
    to_abi(v[k], pose, wps, cap);
  });
}

rp_status rp_plan_poses(const rp_plan* p, int32_t which, int32_t first, int32_t count,
                        rp_pose* poses, double* wps, int32_t wps_per_pose) {
  return guarded([&] {
    const auto& v = which == 0 ? p->poses : p->unfold;
    require(first >= 0 && count >= 0 && first + count <= static_cast<int>(v.size()),
            RP_E_INVALID_PARAMETER, "pose range out of range");
    for (int32_t k = 0; k < count; ++k)
      to_abi(v[first + k], poses + k, wps ? wps + 3 * static_cast<size_t>(wps_per_pose) * k : nullptr,
             wps_per_pose);
  });
}

rp_status rp_plan_note(const rp_plan* p, int32_t k, char* buf, int32_t cap) {
  return guarded([&] {
    require(k >= 0 && k < static_cast<int>(p->notes.size()) && cap > 0, RP_E_INVALID_PARAMETER,
            "note index out of range");
    std::strncpy(buf, p->notes[k].c_str(), cap - 1);
    buf[cap - 1] = 0;
  });
}

rp_status rp_plan_create(const char* kind, const double* waypoints, const rp_pose* poses,
                         const double* relax, int32_t n, const rp_pose* unfold, int32_t n_unfold,
                         rp_plan** out) {
  return guarded([&] {
    auto* p = new rp_plan();
    p->kind = kind ? kind : "";
    for (int k = 0; k < n; ++k) {
      p->waypoints.push_back(V3{waypoints[3 * k], waypoints[3 * k + 1], waypoints[3 * k + 2]});
      p->poses.push_back(from_abi(poses[k], nullptr));
      p->relax.push_back(relax ? relax[k] : 1.0);
    }
    for (int k = 0; k < n_unfold; ++k) p->unfold.push_back(from_abi(unfold[k], nullptr));
    *out = p;
  });
}

rp_status rp_plan_destroy(rp_plan* p) {
  return guarded([&] { delete p; });
}

}  // extern "C"
