/*
 * TEST INFRASTRUCTURE ONLY — the parity oracle, never the product.
 *
 * Plain-C restatement of the reference reachplan hot path for the default
 * configuration (coaxial arm, no joint limits, single approach vector):
 * quiver generation, voxel grid build / mark / dilate, point and segment
 * clearance, prune_segment1, seg2_worker and the short-reach scan, with all 13
 * SolveStats counters and the canonical solution key list. Every function
 * cites the reference file:line it restates; arithmetic follows the same
 * operation order (vector dot = (x*x' + y*y') + z*z', no FMA contraction:
 * build with -ffp-contract=off). Only tests/ and __graft_entry__.smoke() load
 * it (oracle/rp_oracle.py); it is pinned against the compiled reference
 * (oracle/_ref) and the golden fixtures under tests/golden/.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct { double x, y, z; } v3;

static v3 vadd(v3 a, v3 b) { v3 r = {a.x + b.x, a.y + b.y, a.z + b.z}; return r; }
static v3 vsub(v3 a, v3 b) { v3 r = {a.x - b.x, a.y - b.y, a.z - b.z}; return r; }
static v3 vscale(double s, v3 v) { v3 r = {s * v.x, s * v.y, s * v.z}; return r; }
static double vdot(v3 a, v3 b) { double xy = a.x * b.x + a.y * b.y; return xy + a.z * b.z; }
static double vnorm(v3 a) { return sqrt(vdot(a, a)); }
static double clampd(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }

static const double kPi = 3.14159265358979323846;

/* generate_quiver, src/quiver.cpp:16-51 */
int rpo_quiver(double elev, double azim, int min_per_ring, double* out, int cap) {
  double rings[4096];
  int nr = 0;
  for (int k = 0;; ++k) {
    const double phi = -kPi / 2.0 + k * elev;
    if (phi >= kPi / 2.0 - 1e-12) { rings[nr++] = kPi / 2.0; break; }
    rings[nr++] = phi;
  }
  const long n_eq = llround(2.0 * kPi / azim);
  int n = 0;
  for (int r = 0; r < nr; ++r) {
    const double phi = rings[r];
    const long by = llround((double)n_eq * cos(phi));
    const int count = (int)(by > min_per_ring ? by : min_per_ring);
    const double cp = cos(phi), sp = sin(phi);
    for (int m = 0; m < count; ++m) {
      const double th = 2.0 * kPi * m / count;
      if (out && n < cap) {
        out[3 * n] = cp * cos(th);
        out[3 * n + 1] = cp * sin(th);
        out[3 * n + 2] = sp;
      }
      ++n;
    }
  }
  return n;
}

typedef struct {
  double o[3], vs;
  int d[3];
  uint8_t* occ;
} grid_t;

/* VoxelGrid::world_to_index, inc/reachplan/voxgrid.hpp:46-50 */
static int w2i(const grid_t* g, double p, int a) { return (int)floor((p - g->o[a]) / g->vs); }

/* point_clear, src/voxgrid.cpp:94-98 */
static int point_clear(const grid_t* g, v3 p) {
  const int ix = w2i(g, p.x, 0), iy = w2i(g, p.y, 1), iz = w2i(g, p.z, 2);
  if (ix < 0 || iy < 0 || iz < 0 || ix >= g->d[0] || iy >= g->d[1] || iz >= g->d[2]) return 1;
  return g->occ[((size_t)iz * g->d[1] + iy) * g->d[0] + ix] == 0;
}

static v3 sample(v3 from, v3 diff, int k, int n) { return vadd(from, vscale((double)k / n, diff)); }

/* walk_segment_into, src/reach_solver.cpp:109-126: first blocked (1-based) or 0 */
static int walk_first_blocked(const grid_t* g, v3 a, v3 b, int n) {
  const v3 d = vsub(b, a);
  for (int k = 1; k <= n; ++k)
    if (!point_clear(g, sample(a, d, k, n))) return k;
  return 0;
}

/* build_grid + mark_obstacles(boxes) + dilate, src/voxgrid.cpp:12-92 */
static int grid_make(grid_t* g, const double* bmin, const double* bmax, double vs,
                     const double* boxes, int nbox, double radius) {
  for (int a = 0; a < 3; ++a) {
    g->o[a] = bmin[a];
    const double ext = bmax[a] - bmin[a];
    const int d = (int)ceil(ext / vs - 1e-9);
    g->d[a] = d > 1 ? d : 1;
  }
  g->vs = vs;
  const size_t cells = (size_t)g->d[0] * g->d[1] * g->d[2];
  if (cells > ((size_t)1 << 27)) return 2;
  g->occ = (uint8_t*)calloc(cells, 1);
  for (int b = 0; b < nbox; ++b) {
    const double* mn = boxes + 6 * b;
    const double* mx = boxes + 6 * b + 3;
    int lo[3], hi[3];
    for (int a = 0; a < 3; ++a) {
      lo[a] = w2i(g, mn[a], a);
      hi[a] = w2i(g, mx[a], a);
      if (lo[a] < 0) lo[a] = 0;
      if (hi[a] > g->d[a] - 1) hi[a] = g->d[a] - 1;
    }
    for (int z = lo[2]; z <= hi[2]; ++z)
      for (int y = lo[1]; y <= hi[1]; ++y)
        for (int x = lo[0]; x <= hi[0]; ++x) {
          const double c[3] = {g->o[0] + vs * (x + 0.5), g->o[1] + vs * (y + 0.5),
                               g->o[2] + vs * (z + 0.5)};
          int in = 1;
          for (int a = 0; a < 3; ++a) in = in && c[a] >= mn[a] && c[a] <= mx[a];
          if (in) g->occ[((size_t)z * g->d[1] + y) * g->d[0] + x] = 1;
        }
  }
  if (radius == 0.0) return 0;
  const double rc = radius / vs;
  const int reach = (int)floor(rc + 1e-9);
  const double r2 = rc * rc + 1e-9;
  uint8_t* before = (uint8_t*)malloc(cells);
  memcpy(before, g->occ, cells);
  for (int z = 0; z < g->d[2]; ++z)
    for (int y = 0; y < g->d[1]; ++y)
      for (int x = 0; x < g->d[0]; ++x) {
        if (!before[((size_t)z * g->d[1] + y) * g->d[0] + x]) continue;
        for (int dz = -reach; dz <= reach; ++dz)
          for (int dy = -reach; dy <= reach; ++dy)
            for (int dx = -reach; dx <= reach; ++dx) {
              if ((double)dx * dx + (double)dy * dy + (double)dz * dz > r2) continue;
              const int X = x + dx, Y = y + dy, Z = z + dz;
              if (X < 0 || Y < 0 || Z < 0 || X >= g->d[0] || Y >= g->d[1] || Z >= g->d[2]) continue;
              g->occ[((size_t)Z * g->d[1] + Y) * g->d[0] + X] = 1;
            }
      }
  free(before);
  return 0;
}

int rpo_grid(const double* bmin, const double* bmax, double vs, const double* boxes, int nbox,
             double radius, uint8_t* occ, int64_t cap, int* dims) {
  grid_t g;
  const int rc = grid_make(&g, bmin, bmax, vs, boxes, nbox, radius);
  if (rc) return rc;
  const size_t cells = (size_t)g.d[0] * g.d[1] * g.d[2];
  for (int a = 0; a < 3; ++a) dims[a] = g.d[a];
  if (occ && (size_t)cap >= cells) memcpy(occ, g.occ, cells);
  free(g.occ);
  return 0;
}

/* point_to_segment, src/reach_solver.cpp:135-141 */
static double point_to_segment(v3 p, v3 a, v3 b) {
  const v3 ab = vsub(b, a);
  const double l2 = vdot(ab, ab);
  if (l2 <= 1e-30) return vnorm(vsub(p, a));
  const double t = clampd(vdot(vsub(p, a), ab) / l2, 0.0, 1.0);
  return vnorm(vsub(p, vadd(a, vscale(t, ab))));
}

/* segment_segment_distance, src/arm_model.cpp:326-361 */
static double seg_seg(v3 a0, v3 a1, v3 b0, v3 b1) {
  const v3 d1 = vsub(a1, a0), d2 = vsub(b1, b0), r = vsub(a0, b0);
  const double a = vdot(d1, d1), e = vdot(d2, d2), f = vdot(d2, r);
  double s = 0.0, t = 0.0;
  if (a <= 1e-30 && e <= 1e-30) return vnorm(r);
  if (a <= 1e-30) {
    t = clampd(f / e, 0.0, 1.0);
  } else {
    const double c = vdot(d1, r);
    if (e <= 1e-30) {
      s = clampd(-c / a, 0.0, 1.0);
    } else {
      const double b = vdot(d1, d2);
      const double den = a * e - b * b;
      if (den > 1e-30) s = clampd((b * f - c * e) / den, 0.0, 1.0);
      t = (b * s + f) / e;
      if (t < 0.0) { t = 0.0; s = clampd(-c / a, 0.0, 1.0); }
      else if (t > 1.0) { t = 1.0; s = clampd((b - c) / a, 0.0, 1.0); }
    }
  }
  return vnorm(vsub(vadd(a0, vscale(s, d1)), vadd(b0, vscale(t, d2))));
}

/* self_collision_free on a coaxial chain, src/arm_model.cpp:376-388 */
static int self_free(const v3* j, int nl, double min_sep) {
  for (int a = 0; a + 2 < nl; ++a)
    for (int b = a + 2; b < nl; ++b)
      if (seg_seg(j[a], j[a + 1], j[b], j[b + 1]) < min_sep) return 0;
  return 1;
}

static int scaled_count(double len, double spacing) {
  const int c = (int)ceil(len / (spacing > 1e-12 ? spacing : 1e-12));
  return c > 1 ? c : 1;
}

/* short_reach_scan, src/reach_solver.cpp:176-222: 1 if a shortcut results */
static int short_reach(const grid_t* g, v3 link, v3 end, int fb, int n, v3 target, v3 origin,
                       double radius, double spacing) {
  const int len = fb ? fb : n;
  const v3 d = vsub(end, link);
  int hit = 0;
  for (int k = 0; k < len; ++k) {
    if (vnorm(vsub(sample(link, d, k + 1, n), target)) <= radius + 1e-12) { hit = k + 1; break; }
    if (fb && k + 1 == fb) break;
  }
  if (!hit) return 0;
  const v3 hp = sample(link, d, hit, n);
  const double dist = vnorm(vsub(hp, target));
  if (dist > 1e-9) {
    if (walk_first_blocked(g, hp, target, scaled_count(dist, spacing)) == 0) return 1;
    const double dl = vnorm(vsub(target, origin));
    if (walk_first_blocked(g, origin, target, scaled_count(dl, spacing)) != 0) return 0;
  }
  return 1;
}

/*
 * solve_reach for a coaxial arm without limits, half-angle-0 approach
 * (src/reach_solver.cpp:224-300 prune_segment1, :316-456 seg2_worker,
 * :480-546 orchestration). counters: the 13 SolveStats fields in order.
 * keys: (i, j, -1) per solution, canonical order. Returns the solution count.
 */
int64_t rpo_solve(const double* bmin, const double* bmax, double vs, const double* boxes, int nbox,
                  double dilation, const double* lengths, int nseg, double arm_radius, int eight,
                  int n, double elev, double azim, int min_per_ring, const double* target_in,
                  const double* axis_in, int32_t* keys, int64_t cap, int64_t* counters) {
  const double L1 = lengths[0], L2 = lengths[1], L3 = lengths[2];
  const double L4 = eight ? lengths[3] : 0.0;
  double dil = dilation;
  if (dil < 0.0) { /* effective_dilation, src/pipeline.cpp:8-15 */
    double m = 0.0;
    for (int j = 0; j < nseg; ++j) m = (lengths[j] / n > m) ? lengths[j] / n : m;
    dil = arm_radius + 1.25 * m;
  }
  grid_t g;
  if (grid_make(&g, bmin, bmax, vs, boxes, nbox, dil)) return -1;
  const int Q = rpo_quiver(elev, azim, min_per_ring, NULL, 0);
  double* q = (double*)malloc(sizeof(double) * 3 * Q);
  rpo_quiver(elev, azim, min_per_ring, q, Q);
  const v3 root = {0, 0, 0};
  const v3 target = {target_in[0], target_in[1], target_in[2]};
  const v3 axis = {axis_in[0], axis_in[1], axis_in[2]};
  /* ReachParams derived values, src/reach_solver.cpp:28-43 */
  const double eps = 0.5 * L3 / n;
  const double spacing = (L1 + L2 + L3) / (3.0 * n);
  const double near = 0.5 * spacing;
  /* backward_endpoints, src/reach_solver.cpp:54-83 */
  const v3 b = eight ? vsub(target, vscale(L4, axis)) : target;
  double budget = L2 + L3 + eps;
  if (eight) budget += L4;
  budget += 1e-9;
  const double budget2 = budget * budget;
  const double coarse2 = (L3 + eps) * (L3 + eps) * (1.0 + 1e-12);
  memset(counters, 0, 13 * sizeof(int64_t));
  int* s_idx = (int*)malloc(sizeof(int) * Q);
  int S1 = 0;
  int64_t shortcuts = 0;
  for (int i = 0; i < Q; ++i) {
    ++counters[0];
    ++counters[1];
    const v3 dir = {q[3 * i], q[3 * i + 1], q[3 * i + 2]};
    const v3 p1 = vadd(root, vscale(L1, dir));
    const v3 dd = vsub(p1, target);
    const int reach = vdot(dd, dd) <= budget2;
    if (reach) ++counters[2];
    const int fb = walk_first_blocked(&g, root, p1, n);
    if (point_to_segment(target, root, p1) <= near + 1e-9 &&
        short_reach(&g, root, p1, fb, n, target, root, near, spacing))
      ++shortcuts;
    if (!reach || fb) continue;
    ++counters[3];
    s_idx[S1++] = i;
  }
  const int walk4 = eight ? walk_first_blocked(&g, b, target, n) == 0 : 1;
  int64_t nsol = 0;
  /* canonical order (i, j): iterate survivors outer, j inner */
  for (int s = 0; s < S1; ++s) {
    const int i = s_idx[s];
    const v3 d1 = {q[3 * i], q[3 * i + 1], q[3 * i + 2]};
    const v3 s1 = vscale(L1, d1);
    const v3 p1 = vadd(root, s1);
    for (int j = 0; j < Q; ++j) {
      ++counters[4];
      ++counters[5];
      const v3 d2 = {q[3 * j], q[3 * j + 1], q[3 * j + 2]};
      const v3 s2 = vscale(L2, d2);
      const v3 p2 = vadd(p1, s2);
      const int fb = walk_first_blocked(&g, p1, p2, n);
      if (point_to_segment(target, p1, p2) <= near + 1e-9 &&
          short_reach(&g, p1, p2, fb, n, target, p1, near, spacing))
        ++shortcuts;
      if (fb) continue;
      ++counters[6];
      ++counters[7];
      const v3 v = vsub(b, p2);
      if (vdot(v, v) > coarse2) continue;
      const double vl = vnorm(v);
      if (fabs(vl - L3) > eps) continue;
      ++counters[8];
      if (vl < 1e-12) continue;
      ++counters[9];
      if (walk_first_blocked(&g, p2, b, n)) continue;
      ++counters[10];
      if (!walk4) continue;
      v3 J[5];
      J[0] = root;
      J[1] = vadd(J[0], s1);
      J[2] = vadd(J[1], s2);
      J[3] = vadd(J[2], v);
      if (eight) J[4] = vadd(J[3], vscale(L4, axis));
      if (!self_free(J, eight ? 4 : 3, 2.0 * arm_radius)) continue;
      if (keys && nsol < cap) {
        keys[3 * nsol] = i;
        keys[3 * nsol + 1] = j;
        keys[3 * nsol + 2] = -1;
      }
      ++nsol;
    }
  }
  counters[11] = nsol;
  counters[12] = shortcuts;
  free(s_idx);
  free(q);
  free(g.occ);
  return nsol;
}
