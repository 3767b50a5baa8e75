/*
 * reachplan-b200 C ABI: the drop-in boundary for the gMS reach / path hot path.
 *
 * The reference (`reachplan`, /root/reference/proj) exposes this path as plain
 * C++20 free functions in namespace reachplan with value semantics and
 * exceptions. This header replaces them with opaque device-resident handles,
 * plain-old-data parameter structs, caller-owned output buffers and an int
 * status code. Each entry point cites the reference declaration it replaces.
 *
 * Conventions
 *   - Every function returns rp_status: 0 = OK, k+1 = reference Errc ordinal k
 *     (inc/reachplan/types.hpp:34-46), RP_E_CUDA / RP_E_INTERNAL otherwise.
 *     Nothing throws across the ABI. rp_last_error() gives the message,
 *     prefixed with the reference's errc_name (types.hpp:48-63).
 *   - Angles are radians, lengths metres, all arithmetic fp64.
 *   - A context owns one CUDA device + stream; it is not thread-safe, distinct
 *     contexts are. All device work is on the context stream.
 *   - There is no CPU fallback: without a CUDA device every compute entry
 *     point fails with RP_E_CUDA.
 */
#ifndef REACHPLAN_B200_H
#define REACHPLAN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RP_ABI_VERSION 1
#define RP_MAX_SEGMENTS 4
#define RP_MAX_RELAX 8

typedef int32_t rp_status;
enum {
  RP_OK = 0,
  RP_E_INVALID_PARAMETER = 1, /* Errc::invalid_parameter */
  RP_E_CAPACITY_EXCEEDED = 2,
  RP_E_DEGENERATE_INPUT = 3,
  RP_E_UNREACHABLE_TARGET = 4,
  RP_E_EMPTY_CONE = 5,
  RP_E_NO_SOLUTION = 6,
  RP_E_NO_PATH = 7,
  RP_E_INFEASIBLE_TIMING = 8,
  RP_E_EXECUTION_COLLISION = 9,
  RP_E_TIMEOUT = 10,
  RP_E_PARSE_ERROR = 11,
  RP_E_CUDA = 100,
  RP_E_INTERNAL = 101
};

/* ---- plain parameter structs (reference types in brackets) ---------------- */

/* [JointLimit, inc/reachplan/arm_model.hpp:14-21] */
typedef struct rp_joint_limit {
  double elev_min, elev_max, azim_min, azim_max;
} rp_joint_limit;

/* [ArmSpec, inc/reachplan/arm_model.hpp:23-42]; rp_arm_init fills the defaults */
typedef struct rp_arm {
  int32_t n_segments; /* 3 (6DOF) or 4 (8DOF) */
  int32_t n_limits;   /* 0 = unrestricted */
  int32_t n_offsets;  /* 0 = coaxial */
  int32_t _pad;
  double lengths[RP_MAX_SEGMENTS];
  double root[3];
  double arm_radius;
  rp_joint_limit limits[RP_MAX_SEGMENTS];
  double offsets[RP_MAX_SEGMENTS];
  double fold_plane_normal[3];
  double fold_flex;
  double base_axis[3];
  double base_ref[3];
} rp_arm;

enum { RP_MODE_6DOF = 0, RP_MODE_8DOF = 1 };

/* [ReachParams, inc/reachplan/reach_solver.hpp:15-35] negative = derived */
typedef struct rp_reach_params {
  double epsilon_gap;
  double approach_axis[3];
  double approach_half_angle;
  double near_target_radius;
  int32_t n_samples;
  int32_t mode;
  int32_t cone_precheck;
  int32_t disable_geom_pruning;
  int32_t refine_triangle_8dof;
  int32_t workers; /* accepted for API parity; the device decides parallelism */
} rp_reach_params;

/* [PathParams, inc/reachplan/path_planner.hpp:11-22] negative = derived */
typedef struct rp_path_params {
  double epsilon_waypoint, d_w, slack, joint1_max_move, joint2_max_move;
  double relax_schedule[RP_MAX_RELAX];
  int32_t n_relax;
  int32_t unfold_steps;
} rp_path_params;

enum { RP_SHAPE_BOX = 0, RP_SHAPE_CLOUD = 1 };

/* [SceneObstacle, inc/reachplan/voxgrid.hpp:15-23] */
typedef struct rp_obstacle {
  int32_t shape;
  int32_t dynamic;
  double box_min[3], box_max[3];
  const double* points; /* cloud: xyz triples, host memory */
  int64_t n_points;
  const char* id; /* optional label, used in replan provenance notes */
} rp_obstacle;

/* [SolveStats, inc/reachplan/reach_solver.hpp:76-93] */
typedef struct rp_solve_stats {
  int64_t seg1_candidates, seg1_limit_pass, seg1_reach_pass, seg1_survivors;
  int64_t pair_candidates, seg2_limit_pass, seg2_clear_pass;
  int64_t gap_tested, gap_pass, joint_pass, v3_clear_pass;
  int64_t solutions, shortcuts_found;
  double wall_ms; /* informational */
} rp_solve_stats;

/* [PoseChain, inc/reachplan/arm_model.hpp:58-72] waypoints travel separately */
typedef struct rp_pose {
  int32_t n_segments;
  int32_t has_elbows;
  int32_t quiver_indices[RP_MAX_SEGMENTS]; /* -1 = free / refined */
  int32_t n_waypoints;
  int32_t no_indices; /* 1: PoseChain::quiver_indices is empty (joint-space /
                         folded poses), 0: n_segments indices above */
  double s4_length_dev;
  double segments[RP_MAX_SEGMENTS][3];
  double joints[RP_MAX_SEGMENTS + 1][3];
  double elbows[RP_MAX_SEGMENTS][3];
} rp_pose;

/* [ShortcutPath, inc/reachplan/reach_solver.hpp:60-74] */
typedef struct rp_shortcut {
  int32_t segment_index; /* 1 or 2 */
  int32_t hit_sample_index;
  int32_t seg1_index, seg2_index;
  int32_t has_bridge;
  int32_t via_origin_direct;
  int32_t n_prefix, n_sublength; /* sample counts of the tip path pieces */
  double bridge[3];
  double path_length;
} rp_shortcut;

enum { RP_CHOSEN_REACH_POSE = 0, RP_CHOSEN_SHORTCUT = 1 };

/* [ChosenPath, inc/reachplan/reach_solver.hpp:155-161] by index into a set */
typedef struct rp_chosen {
  int32_t kind;
  int32_t _pad;
  int64_t index; /* solution or shortcut index in canonical order */
  double path_length;
} rp_chosen;

/* [PathPlan, inc/reachplan/path_planner.hpp:27-41] sizes + provenance scalars */
typedef struct rp_plan_info {
  int32_t n_waypoints;
  int32_t n_poses;
  int32_t n_unfold;
  int32_t n_notes;
  int32_t replan_switch_index;
  int32_t _pad;
  char kind[32]; /* reach-pose | shortcut | virtual-arm | out-and-back | replan */
} rp_plan_info;

/* ---- opaque handles ---------------------------------------------------------- */
typedef struct rp_ctx rp_ctx;
typedef struct rp_quiver rp_quiver;
typedef struct rp_grid rp_grid;
typedef struct rp_solution_set rp_solution_set;
typedef struct rp_plan rp_plan;

/* ---- context --------------------------------------------------------------- */
int32_t rp_abi_version(void);
const char* rp_last_error(void); /* thread-local message of the last failure */
rp_status rp_ctx_create(int32_t device, rp_ctx** out);
rp_status rp_ctx_destroy(rp_ctx* ctx);
/* Run on a caller stream (cudaStream_t as void*); NULL restores the own stream. */
rp_status rp_ctx_set_stream(rp_ctx* ctx, void* stream);
void* rp_ctx_stream(rp_ctx* ctx);
rp_status rp_ctx_synchronize(rp_ctx* ctx);
/* Per-kernel device timing (CUDA events on the ctx stream): enable, reset,
 * then read totals for a kernel family name ("dilate", "seg2", ...). */
rp_status rp_ctx_enable_timing(rp_ctx* ctx, int32_t enable);
rp_status rp_ctx_kernel_time(rp_ctx* ctx, const char* name, double* total_ms, int64_t* launches);
rp_status rp_ctx_reset_timing(rp_ctx* ctx);
/* Number of this library's kernels launched on ctx since creation. */
int64_t rp_ctx_launch_count(rp_ctx* ctx);

/* ---- defaults (mirror the reference's member initialisers) ----------------- */
void rp_arm_init(rp_arm* arm, int32_t n_segments, const double* lengths);
void rp_reach_params_init(rp_reach_params* rp);
void rp_path_params_init(rp_path_params* pp);
/* [ReachParams::nominal_spacing / resolved_epsilon / resolved_near_radius,
 *  src/reach_solver.cpp:28-43] */
double rp_nominal_spacing(const rp_arm* arm, const rp_reach_params* rp);
double rp_resolved_epsilon(const rp_arm* arm, const rp_reach_params* rp);
double rp_resolved_near_radius(const rp_arm* arm, const rp_reach_params* rp);
/* [ReachParams::validate, src/reach_solver.cpp:45-52] */
rp_status rp_reach_params_validate(const rp_reach_params* rp);
/* [PathParams::resolved, src/path_planner.cpp:89-102] derived fields filled in */
rp_status rp_path_params_resolve(const rp_arm* arm, const rp_reach_params* rp,
                                 const rp_path_params* pp, rp_path_params* out);
/* [effective_dilation, src/pipeline.cpp:8-15]; configured < 0 = derive */
double rp_effective_dilation(const rp_arm* arm, const rp_reach_params* rp, double configured);

/* ---- quiver [inc/reachplan/quiver.hpp:38-49] ---------------------------------- */
/* [generate_quiver, src/quiver.cpp:16-51] */
rp_status rp_quiver_generate(rp_ctx* ctx, double elev_step, double equator_azim_step,
                             int32_t min_per_ring, rp_quiver** out);
/* Upload an existing reference Quiver's vectors (xyz triples). */
rp_status rp_quiver_upload(rp_ctx* ctx, const double* xyz, int32_t n, rp_quiver** out);
int32_t rp_quiver_size(const rp_quiver* q);
rp_status rp_quiver_download(const rp_quiver* q, double* xyz, int32_t cap);
/* [cone_subset, src/quiver.cpp:53-63] indices ascending; *n_out = count */
rp_status rp_cone_subset(rp_ctx* ctx, const rp_quiver* q, const double axis[3],
                         double half_angle, int32_t* idx, int32_t cap, int32_t* n_out);
/* Ring addressing of a generated quiver (Quiver::ring_offsets, ring_elevations,
 * elev_step, equator_azim_step, min_per_ring); *n_rings = 0 for uploads. */
rp_status rp_quiver_rings(const rp_quiver* q, int32_t* ring_offsets, double* ring_elevations,
                          int32_t cap, int32_t* n_rings, double* elev_step,
                          double* equator_azim_step, int32_t* min_per_ring);
rp_status rp_quiver_destroy(rp_quiver* q);

/* ---- voxel grid [inc/reachplan/voxgrid.hpp:60-84] ----------------------------- */
/* [build_grid, src/voxgrid.cpp:12-33] cell_budget 0 = 2^27 (voxgrid.hpp:57) */
rp_status rp_grid_build(rp_ctx* ctx, const double bounds_min[3], const double bounds_max[3],
                        double voxel_size, uint64_t cell_budget, rp_grid** out);
/* [mark_obstacles, src/voxgrid.cpp:35-62] */
rp_status rp_grid_mark(rp_grid* g, const rp_obstacle* obs, int32_t n);
/* [dilate, src/voxgrid.cpp:64-92] */
rp_status rp_grid_dilate(rp_grid* g, double radius);
/* Fused mark + dilate of boxes onto an empty or existing grid: exactly
 * mark_obstacles(boxes) then dilate(radius) when the grid holds no other
 * occupancy; see DESIGN.md. */
rp_status rp_grid_mark_dilate_boxes(rp_grid* g, const rp_obstacle* obs, int32_t n, double radius);
/* z-slab build (multi-GPU grid partitions): planes z0..z1 of the
 * fused mark + dilate of box obstacles, other planes untouched. Each plane
 * depends only on the boxes, so slabs need no halo exchange; the union of
 * slabs equals rp_grid_mark_dilate_boxes on an empty grid bit for bit. */
rp_status rp_grid_mark_dilate_slab(rp_grid* g, const rp_obstacle* obs, int32_t n, double radius,
                                   int32_t z0, int32_t z1);
/* Device pointer of the bit words (for collectives over the grid, e.g. an
 * all-gather of z-slabs); plane z = words [z*words_per_plane, +words_per_plane). */
/* z-slab step of a partitioned dilate (src/voxgrid.cpp:64-92): planes
   z0..z1 are dilated from the current occupancy of planes z0-R..z1+R (R =
   floor(radius/voxel_size + 1e-9): the caller's own slab plus the halo
   planes exchanged with its neighbours); other planes keep their words.
   The grid records dilation_radius = radius. z1 = z0 - 1: no planes. */
rp_status rp_grid_dilate_slab(rp_grid* g, double radius, int32_t z0, int32_t z1);
rp_status rp_grid_device_bits(rp_grid* g, void** bits, uint64_t* n_words,
                              uint64_t* words_per_plane);
/* Benchmark helper: the fused mark + dilate of `obs` onto g (overwriting it)
 * `reps` times back to back on the ctx stream; *ms = device time per pass. */
rp_status rp_grid_mark_dilate_repeat(rp_grid* g, const rp_obstacle* obs, int32_t n, double radius,
                                     int32_t reps, double* ms);
/* Benchmark helper: `reps` passes back to back on the ctx stream, pass r
 * writing grids[r % ng] (same shape, one context); *ms = device time per
 * pass. With ng grids larger than L2 together, every pass's words reach HBM. */
rp_status rp_grid_mark_dilate_rotating(rp_grid* const* grids, int32_t ng, const rp_obstacle* obs,
                                       int32_t n, double radius, int32_t reps, double* ms);
/* Benchmark helper: `ng` same-shape grids of one context, each updated `reps`
 * times on its own stream, all streams concurrently; *ms = device time per
 * update (updates of independent grids overlapping). */
rp_status rp_grid_mark_dilate_concurrent(rp_grid* const* grids, int32_t ng, const rp_obstacle* obs,
                                         int32_t n, double radius, int32_t reps, double* ms);
/* [build_scene_grid, src/pipeline.cpp:17-34] dilation < 0 = effective_dilation */
rp_status rp_build_scene_grid(rp_ctx* ctx, const double bounds_min[3], const double bounds_max[3],
                              double voxel_size, double dilation, const rp_obstacle* obs,
                              int32_t n_obs, const rp_arm* arm, const rp_reach_params* rp,
                              rp_grid** out);
/* Dynamic-obstacle overlay [src/path_planner.cpp:1011-1021]: aug = base OR
 * dilate(mark(new_obstacle), base.dilation_radius). aug may be a fresh handle
 * (*aug == NULL) or an existing same-shape grid that is overwritten. */
rp_status rp_grid_overlay(const rp_grid* base, const rp_obstacle* obs, rp_grid** aug);
rp_status rp_grid_info(const rp_grid* g, int32_t dims[3], double origin[3], double* voxel_size,
                       double* dilation_radius);
/* Reference layout bytes (x fastest, 1 = obstacle). cap in bytes. */
rp_status rp_grid_download_u8(rp_grid* g, uint8_t* dst, uint64_t cap);
/* Device bit words: row-padded, word = (iz*ny + iy)*ceil(nx/64) + ix/64. */
rp_status rp_grid_download_bits(rp_grid* g, uint64_t* dst, uint64_t cap_words);
rp_status rp_grid_upload_u8(rp_ctx* ctx, const double origin[3], double voxel_size,
                            const int32_t dims[3], const uint8_t* occ, double dilation_radius,
                            rp_grid** out);
rp_status rp_grid_occupied_count(rp_grid* g, uint64_t* count);
/* [point_clear, src/voxgrid.cpp:94-98] batched: out[k] = 1 if clear */
rp_status rp_grid_point_clear(rp_grid* g, const double* xyz, int64_t n, uint8_t* out);
/* No reference counterpart (introspection of the solver's free-sample skip):
   out[k] = the cached coarse clearance field's lower bound (m) on the
   distance from xyz[k] to any occupied cell. */
rp_status rp_grid_clearance(rp_grid* g, const double* xyz, int64_t n, double* out);
/* [segment_clear, src/voxgrid.cpp:100-112] batched segments (from,to pairs) */
rp_status rp_grid_segment_clear(rp_grid* g, const double* from_xyz, const double* to_xyz,
                                int64_t n, int32_t n_samples, uint8_t* out);
rp_status rp_grid_copy(const rp_grid* src, rp_grid** out);
rp_status rp_grid_destroy(rp_grid* g);

/* ---- reach solver [inc/reachplan/reach_solver.hpp] ---------------------------- */
/* [prune_segment1, src/reach_solver.cpp:224-300] survivors' quiver indices */
rp_status rp_prune_segment1(rp_ctx* ctx, const rp_arm* arm, const rp_quiver* q, const rp_grid* g,
                            const double* target_points, int32_t n_targets,
                            const rp_reach_params* rp, int32_t* survivors, int32_t cap,
                            int32_t* n_out, rp_solve_stats* stats);
/* [backward_endpoints, src/reach_solver.cpp:54-83] p3 candidates, end-effector
 * directions and cone quiver indices (-1 = exact axis); *n_out = count */
rp_status rp_backward_endpoints(rp_ctx* ctx, const rp_quiver* q, const double target[3], double L4,
                                const rp_reach_params* rp, double* points, double* dirs,
                                int32_t* cone_idx, int32_t cap, int32_t* n_out);
/* [span_gap, src/reach_solver.cpp:85-98] gap vectors p2 -> backward point k
 * passing the coarse + band test, k ascending (v3_out / idx_out hold n slots) */
rp_status rp_span_gap(rp_ctx* ctx, const double p2[3], const double* backward_pts, int32_t n,
                      double L3, double epsilon, double* v3_out, int32_t* idx_out,
                      int32_t* n_out);
/* [short_reach_scan, src/reach_solver.cpp:176-222] one hypothesis scan:
   samples (n x 3) with their clear flags (HypothesisScan::samples /
   sample_clear), prefix (n_prefix x 3, already-cleared segment-1 samples),
   origin (proximal end). *found = 0: no shortcut. Else *sc gets the hit
   index, bridge / direct verdict, n_prefix / n_sublength and path_length,
   and sublength (cap x 3) the sublength samples (the hit prefix of the
   samples, or the direct origin -> target walk). Bridge and direct walks are
   collision-checked on the device. */
/* [select_solution, src/reach_solver.cpp:548-577] on any solution set given
   as data: segments (n x 3 x 3: s1, s2, s3 of each PoseChain, canonical
   order) and the shortcuts' path lengths (n_sc). Any shortcut wins (the
   shortest, first on ties); else the first strict minimum of
   |s1| + |s2| + |s3|. RP_E_NO_SOLUTION when both are empty. */
rp_status rp_select_solution_data(rp_ctx* ctx, const double* segments, int64_t n,
                                  const double* shortcut_lengths, int64_t n_sc, rp_chosen* out);
rp_status rp_short_reach_scan(rp_ctx* ctx, const rp_grid* g, const rp_arm* arm,
                              const rp_reach_params* rp, const double target[3],
                              const double* samples, const uint8_t* sample_clear, int32_t n,
                              const double* prefix, int32_t n_prefix, const double origin[3],
                              int32_t* found, rp_shortcut* sc, double* sublength, int32_t cap);
/* [solve_reach, src/reach_solver.cpp:480-546]; the set stays on the device */
rp_status rp_solve_reach(rp_ctx* ctx, const rp_arm* arm, const rp_quiver* q, const rp_grid* g,
                         const double target[3], const rp_reach_params* rp,
                         rp_solution_set** out);
/* One part of a solve split over devices [solve_reach's worker split,
 * src/reach_solver.cpp:503-535, by segment-1 survivor rows instead of j]:
 * part p of P solves the rows [S1*p/P, S1*(p+1)/P). Its set holds the part's
 * keys (global indices; the parts' key lists concatenate, in part order, to
 * the whole set's canonical list), segment-2 counters and best solution;
 * segment-1 counters are the whole prune's in every part and segment-1
 * shortcuts are part 0's. Merging (paper_1906_10678_b200/shard.py
 * solve_reach_split): counters = part 0's segment-1 fields + the sums of the
 * rest; the chosen solution = the parts' select_solution results compared
 * as the reference does (any shortcut first, by path_length then part;
 * else (length, key)). parts = 1 is rp_solve_reach. */
rp_status rp_solve_reach_part(rp_ctx* ctx, const rp_arm* arm, const rp_quiver* q,
                              const rp_grid* g, const double target[3], const rp_reach_params* rp,
                              int32_t part, int32_t parts, rp_solution_set** out);
/* [revalidate_solution, src/reach_solver.cpp:458-476] the reference's
 * merge-time self-check of every solution of the set (gap band, joint
 * limits, self-collision, every waypoint sample clear, closure on the
 * target) against `grid` (null: the solve's grid): *n_bad failures, the
 * first failing ordinal and its reason (1 band, 2 limits, 3 self-collision,
 * 4 sample in an obstacle, 5 closure). RP_REVALIDATE=1 runs it inside every
 * solve and raises no-solution "internal: ..." as the reference does. */
rp_status rp_solution_set_revalidate(rp_solution_set* s, const rp_grid* grid, int64_t* n_bad,
                                     int64_t* first_bad, int32_t* reason);
rp_status rp_solution_set_stats(const rp_solution_set* s, rp_solve_stats* stats);
rp_status rp_solution_set_sizes(const rp_solution_set* s, int64_t* n_solutions,
                                int64_t* n_shortcuts);
/* keys[3k..3k+2] = (seg1 index, seg2 index, backward index) canonical order */
rp_status rp_solution_set_keys(const rp_solution_set* s, int32_t* keys, int64_t cap_solutions);
/* Materialise solution k (PoseChain incl. waypoints, reach_solver.cpp:434-449). */
rp_status rp_solution_set_pose(const rp_solution_set* s, int64_t k, rp_pose* pose,
                               double* waypoints, int32_t cap_waypoints);
/* Bulk form: solutions [first, first + count) in canonical order; waypoints
 * (nullable) holds wps_per_pose xyz triples per pose. */
rp_status rp_solution_set_poses(const rp_solution_set* s, int64_t first, int64_t count,
                                rp_pose* poses, double* waypoints, int32_t wps_per_pose);
/* Mean polyline deviation (mean_polyline_deviation, src/path_planner.cpp:76-87)
 * of solutions [first, first+count)'s traversal waypoints (segments 1-3, the
 * candidate tip path) from poly[n_poly] -- the score alternate_candidates
 * (src/path_planner.cpp:612-663) ranks by, computed by the same device
 * kernels the planner uses. */
rp_status rp_solution_set_deviations(rp_solution_set* s, const double* poly, int32_t n_poly,
                                     int64_t first, int64_t count, double* out);
/* Shortcut k; tip waypoints (root excluded) into wps (ShortcutPath::tip_waypoints). */
rp_status rp_solution_set_shortcut(const rp_solution_set* s, int64_t k, rp_shortcut* sc,
                                   double* tip_wps, int32_t cap_wps, int32_t* n_wps);
/* ShortcutPath::basis_pose of shortcut k (the hypothesis segments behind it). */
rp_status rp_solution_set_shortcut_basis(const rp_solution_set* s, int64_t k, rp_pose* basis);
rp_status rp_solution_set_destroy(rp_solution_set* s);
/* [select_solution, src/reach_solver.cpp:548-577] */
rp_status rp_select_solution(const rp_solution_set* s, rp_chosen* out);
/* Batched reach queries (BASELINE configs[4]): for each target, exactly
 * solve_reach + select_solution + exact refinement of a chosen reach pose
 * (src/reach_solver.cpp:480-577, src/arm_model.cpp:258-324). The
 * target-independent segment clearance is computed once per call and shared
 * by all targets. */
typedef struct rp_batch_result {
  int32_t status;   /* RP_OK, or RP_E_NO_SOLUTION when the set is empty, or the
                       refinement's error (e.g. RP_E_UNREACHABLE_TARGET) */
  int32_t kind;     /* RP_CHOSEN_REACH_POSE / RP_CHOSEN_SHORTCUT */
  int32_t seg1, seg2, cone; /* chosen key (reach pose) or shortcut indices */
  int32_t _pad;
  int64_t n_solutions, n_shortcuts;
  double path_length;
  rp_pose refined;  /* refined reach pose (kind == REACH_POSE, status == OK) */
  rp_solve_stats stats;
} rp_batch_result;
rp_status rp_solve_reach_batch(rp_ctx* ctx, const rp_arm* arm, const rp_quiver* q,
                               const rp_grid* g, const double* targets, int32_t n_targets,
                               const rp_reach_params* rp, rp_batch_result* out);
/* [exact_refine_8dof / _6dof / _8dof_triangle, src/arm_model.cpp:258-324] */
rp_status rp_exact_refine(rp_ctx* ctx, const rp_arm* arm, const rp_pose* approx,
                          const double target[3], int32_t variant /*0 auto,1 triangle*/,
                          rp_pose* out);

/* ---- path planner [inc/reachplan/path_planner.hpp] ---------------------------- */
/* [plan_reach_then_path, src/path_planner.cpp:824-829] */
rp_status rp_plan_reach_then_path(rp_ctx* ctx, const rp_arm* arm, const rp_quiver* q,
                                  const rp_grid* g, const double target[3],
                                  const rp_reach_params* rp, const rp_path_params* pp,
                                  rp_plan** out);
/* [plan_from_reach, src/path_planner.cpp:729-738] */
rp_status rp_plan_from_reach(rp_ctx* ctx, const rp_arm* arm, const rp_quiver* q, const rp_grid* g,
                             const rp_solution_set* set, const rp_chosen* chosen,
                             const double target[3], const rp_reach_params* rp,
                             const rp_path_params* pp, rp_plan** out);
/* [fallback_cascade, src/path_planner.cpp:740-822] after a failed backward
 * pass of `failed` over `waypoints` (PlanFailure: blocked_index = the
 * waypoint the pass could not place) */
rp_status rp_fallback_cascade(rp_ctx* ctx, const rp_arm* arm, const rp_quiver* q, const rp_grid* g,
                              const rp_solution_set* set, const rp_chosen* failed,
                              const double* waypoints, int32_t n_waypoints, int32_t blocked_index,
                              const double target[3], const rp_reach_params* rp,
                              const rp_path_params* pp, rp_plan** out);
/* [plan_arbitrary, src/path_planner.cpp:906-998]; start_waypoints (nullable)
 * carries start_pose->n_waypoints xyz samples (PoseChain::waypoints) */
rp_status rp_plan_arbitrary(rp_ctx* ctx, const rp_arm* arm, const rp_quiver* q, const rp_grid* g,
                            const rp_pose* start_pose, const double* start_waypoints,
                            const double target[3], const rp_reach_params* rp,
                            const rp_path_params* pp, rp_plan** out);
/* [replan_dynamic, src/path_planner.cpp:1000-1102] */
rp_status rp_replan_dynamic(rp_ctx* ctx, const rp_arm* arm, const rp_quiver* q,
                            const rp_grid* grid_static, const rp_plan* active,
                            int32_t current_index, const rp_obstacle* new_obstacle,
                            double waypoint_period, double replan_per_waypoint,
                            const rp_reach_params* rp, const rp_path_params* pp, rp_plan** out);
/* [waypoint_ik, src/path_planner.cpp:167-291]; trail dirs optional (NULL),
 * bias optional. *found = 0 when no pose qualifies (std::nullopt). */
rp_status rp_waypoint_ik(rp_ctx* ctx, const rp_arm* arm, const rp_quiver* q, const rp_grid* g,
                         const double waypoint[3], const rp_pose* prev, const rp_reach_params* rp,
                         const rp_path_params* pp, double relax, const double* trail_back,
                         const double* trail_fwd, const rp_pose* junction_bias, int32_t* found,
                         rp_pose* out, double* waypoints, int32_t cap_waypoints);
/* [smoothness_ok, src/path_planner.cpp:114-120] with resolved path params */
rp_status rp_smoothness_ok(const rp_arm* arm, const rp_reach_params* rp, const rp_path_params* pp,
                           const rp_pose* prev, const rp_pose* cand, double relax, int32_t* ok);
/* [mean_polyline_deviation, src/path_planner.cpp:76-87] on the device */
rp_status rp_mean_polyline_deviation(rp_ctx* ctx, const double* pts, int32_t n_pts,
                                     const double* poly, int32_t n_poly, double* out);
/* [folded_pose, src/path_planner.cpp:711-727] */
rp_status rp_folded_pose(rp_ctx* ctx, const rp_arm* arm, rp_pose* out);

/* [validate_plan / check_pose, src/validate.cpp:20-108] independent re-check of
 * every pose of a delivered plan on the device (collision, segment lengths,
 * joint limits, self-collision, tracked-point placement, smoothness against
 * the recorded relaxation, unfold seam). The issues (the reference's wording,
 * reference order) are '\n'-joined into `issues` (cap bytes incl. NUL;
 * out->issues_bytes = the size needed). */
typedef struct rp_validation {
  int32_t ok;
  int32_t poses_checked;
  int32_t relax_events;
  int32_t n_issues;
  int64_t issues_bytes;
} rp_validation;
rp_status rp_validate_plan(rp_ctx* ctx, const rp_arm* arm, const rp_grid* g, const rp_plan* plan,
                           const rp_reach_params* rp, const rp_path_params* pp, rp_validation* out,
                           char* issues, int64_t cap);

/* ---- execution simulator [inc/reachplan/motion.hpp] ------------------------- */
/* [MotionParams, motion.hpp:9-19]; objective: 0 time-of-arrival (default) */
typedef struct rp_motion_params {
  double v_w;               /* 0.05 m/s */
  double sample_rate;       /* 100 Hz */
  double max_joint_rate;    /* 30 deg/s in rad/s */
  double arrival_tolerance; /* 0.01 m */
  int32_t objective;
  int32_t _pad;
} rp_motion_params;
/* [ExecutionTick + JointAngles + JointRates, motion.hpp:28-41] */
typedef struct rp_tick {
  double time;
  double azimuth[RP_MAX_SEGMENTS], elevation[RP_MAX_SEGMENTS];
  uint8_t degenerate[RP_MAX_SEGMENTS];
  int32_t n_joints;
  double tracked[3];
  int32_t active;       /* active_waypoint_index */
  int32_t n_rates;      /* 0 for the first tick (no command yet) */
  int32_t clamped;
  int32_t _pad;
  double azimuth_rate[RP_MAX_SEGMENTS], elevation_rate[RP_MAX_SEGMENTS];
} rp_tick;
typedef struct rp_trace rp_trace;
void rp_motion_params_init(rp_motion_params* mp);
/* [simulate_execution, src/motion.cpp:62-141] grid (nullable) = re-check every
 * tick for collision on the device (RP_E_EXECUTION_COLLISION at the first
 * colliding tick); RP_E_TIMEOUT when the tick budget runs out. */
rp_status rp_simulate_execution(rp_ctx* ctx, const rp_arm* arm, const rp_plan* plan,
                                const rp_motion_params* mp, const rp_grid* grid, rp_trace** out);
rp_status rp_trace_info(const rp_trace* t, int64_t* n_ticks, int64_t* n_overshoot,
                        int64_t* n_clamp, int32_t* reached_goal);
rp_status rp_trace_ticks(const rp_trace* t, int64_t first, int64_t count, rp_tick* out);
/* overshoot_events / clamp_events tick indices (sizes from rp_trace_info) */
rp_status rp_trace_events(const rp_trace* t, int32_t* overshoot, int32_t* clamp);
rp_status rp_trace_destroy(rp_trace* t);

rp_status rp_plan_get_info(const rp_plan* p, rp_plan_info* info);
rp_status rp_plan_waypoints(const rp_plan* p, double* xyz, int32_t cap);
rp_status rp_plan_relax(const rp_plan* p, double* relax, int32_t cap);
/* which: 0 = poses (one per waypoint), 1 = unfold prefix */
rp_status rp_plan_pose(const rp_plan* p, int32_t which, int32_t k, rp_pose* pose,
                       double* waypoints, int32_t cap_waypoints);
/* rp_plan_pose for poses [first, first + count) in one call: pose k's
   waypoint samples at waypoints + 3 * wps_per_pose * (k - first) */
rp_status rp_plan_poses(const rp_plan* p, int32_t which, int32_t first, int32_t count,
                        rp_pose* poses, double* waypoints, int32_t wps_per_pose);
rp_status rp_plan_note(const rp_plan* p, int32_t k, char* buf, int32_t cap);
/* Build a plan handle from host data (e.g. a plan file) for rp_replan_dynamic. */
rp_status rp_plan_create(const char* kind, const double* waypoints, const rp_pose* poses,
                         const double* relax, int32_t n, const rp_pose* unfold, int32_t n_unfold,
                         rp_plan** out);
rp_status rp_plan_destroy(rp_plan* p);

#ifdef __cplusplus
}
#endif

#endif /* REACHPLAN_B200_H */
