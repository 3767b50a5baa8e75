// Device geometry for the gMS hot path (sm_100a).
//
// Every decision the reference takes is a threshold on an fp64 expression, so
// these helpers reproduce the reference's IEEE operation sequence exactly:
// the library is compiled with -fmad=false (no FMA contraction, like x86-64
// g++ without -march), double '/' and sqrt are IEEE round-to-nearest, and
// vector reductions follow Eigen's fixed-size-3 order (x*x' + y*y') + z*z'.
// Transcendentals (atan2/hypot/sin/cos) only appear with joint limits,
// offsets or in the unfold interpolation; those results are tolerance-class
// (CUDA libm vs glibc may differ in the last ulp), see DESIGN.md.
#pragma once

#include <cstdint>

namespace rpd {

struct V3 {
  double x, y, z;
};

__host__ __device__ __forceinline__ V3 mk(double x, double y, double z) { return V3{x, y, z}; }
__host__ __device__ __forceinline__ V3 operator+(V3 a, V3 b) { return V3{a.x + b.x, a.y + b.y, a.z + b.z}; }
__host__ __device__ __forceinline__ V3 operator-(V3 a, V3 b) { return V3{a.x - b.x, a.y - b.y, a.z - b.z}; }
__host__ __device__ __forceinline__ V3 operator-(V3 a) { return V3{-a.x, -a.y, -a.z}; }
/// scalar * vector (Eigen: s * v)
__host__ __device__ __forceinline__ V3 operator*(double s, V3 v) { return V3{s * v.x, s * v.y, s * v.z}; }
/// vector * scalar (Eigen: v * s); IEEE multiply commutes, kept for readability
__host__ __device__ __forceinline__ V3 operator*(V3 v, double s) { return V3{v.x * s, v.y * s, v.z * s}; }
__host__ __device__ __forceinline__ V3 operator/(V3 v, double s) { return V3{v.x / s, v.y / s, v.z / s}; }

/// Eigen fixed-size-3 dot: one 2-wide packet then the tail.
__host__ __device__ __forceinline__ double dot(V3 a, V3 b) {
  const double xy = a.x * b.x + a.y * b.y;
  return xy + a.z * b.z;
}
__host__ __device__ __forceinline__ double sqnorm(V3 a) { return dot(a, a); }
__host__ __device__ __forceinline__ double norm(V3 a) { return sqrt(sqnorm(a)); }
__host__ __device__ __forceinline__ V3 normalized(V3 a) {
  const double n2 = sqnorm(a);
  if (n2 > 0.0) {
    const double n = sqrt(n2);
    return V3{a.x / n, a.y / n, a.z / n};
  }
  return a;
}
__host__ __device__ __forceinline__ V3 cross(V3 a, V3 b) {
  return V3{a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
/// std::clamp(v, lo, hi)
__host__ __device__ __forceinline__ double clampd(double v, double lo, double hi) {
  return (v < lo) ? lo : (hi < v) ? hi : v;
}

// ---------------------------------------------------------------------------
// Bit-packed occupancy grid. Rows of x are padded to whole 64-bit words:
// word(ix, iy, iz) = (iz*ny + iy)*wx + ix/64, bit ix%64. 1 = obstacle.
struct GridView {
  const uint64_t* bits;
  int nx, ny, nz, wx;
  double ox, oy, oz;
  double vs;   // voxel_size
  double rvs;  // fl(1/voxel_size), for the exact-floor fast path
  // floor bracket half-width valid for every |q| <= max(n) + 2 (q = a * rvs):
  // beyond that a sample is outside the grid whichever integer it floors to
  double dq;
};

/// floor(a / vs) exactly as the reference (inc/voxgrid.hpp:46-50): the
/// correctly rounded quotient is bracketed by a*fl(1/vs) +- 4u|q|; if no
/// integer lies in the bracket the floor is decided without dividing,
/// otherwise the IEEE division is done. Bit-exact by construction.
__device__ __forceinline__ int vox_floor(double a, double vs, double rvs) {
  const double q = a * rvs;
  const double d = fabs(q) * 8.9e-16 + 1e-300;
  const double lo = floor(q - d);
  // floor(fl(q + d)) == lo  <=>  fl(q + d) < lo + 1, as fl(q + d) >= fl(q - d) >= lo
  if (q + d < lo + 1.0) return static_cast<int>(lo);
  return static_cast<int>(floor(a / vs));
}

/// point_clear (src/voxgrid.cpp:94-98): outside the grid = free.
__device__ __forceinline__ bool point_clear(const GridView& g, V3 p) {
  const int ix = vox_floor(p.x - g.ox, g.vs, g.rvs);
  const int iy = vox_floor(p.y - g.oy, g.vs, g.rvs);
  const int iz = vox_floor(p.z - g.oz, g.vs, g.rvs);
  if (ix < 0 || iy < 0 || iz < 0 || ix >= g.nx || iy >= g.ny || iz >= g.nz) return true;
  const uint64_t w =
      __ldg(g.bits + ((static_cast<size_t>(iz) * g.ny + iy) * g.wx + (ix >> 6)));
  return ((w >> (ix & 63)) & 1ull) == 0ull;
}

/// fl(k / n) for 1 <= n <= kTkMax, 0 <= k <= n, folded at compile time
/// (constant expressions are evaluated with IEEE round-to-nearest, the same
/// result as the run-time division) so the walks skip an fp64 divide per
/// sample.
constexpr int kTkMax = 16;
struct TkTable {
  double v[kTkMax + 1][kTkMax + 1];
};
constexpr TkTable make_tk_table() {
  TkTable t{};
  for (int n = 1; n <= kTkMax; ++n)
    for (int k = 0; k <= n; ++k) t.v[n][k] = static_cast<double>(k) / static_cast<double>(n);
  return t;
}
__constant__ const TkTable c_tk = make_tk_table();

__host__ __device__ __forceinline__ double sample_t(int k, int n) {
#ifdef __CUDA_ARCH__
  if (n <= kTkMax) return c_tk.v[n][k];
#endif
  return static_cast<double>(k) / static_cast<double>(n);
}

/// Sample k of a segment walk: from + (double(k)/n) * (to - from)
/// (src/voxgrid.cpp:105-107, src/reach_solver.cpp:114-116).
__host__ __device__ __forceinline__ V3 walk_sample(V3 from, V3 diff, int k, int n) {
  const double t = sample_t(k, n);
  return from + t * diff;
}

/// Word index and bit of the cell holding p, or -1 outside the grid (free).
__device__ __forceinline__ long long cell_word(const GridView& g, V3 p, int* bit) {
  const int ix = vox_floor(p.x - g.ox, g.vs, g.rvs);
  const int iy = vox_floor(p.y - g.oy, g.vs, g.rvs);
  const int iz = vox_floor(p.z - g.oz, g.vs, g.rvs);
  if (ix < 0 || iy < 0 || iz < 0 || ix >= g.nx || iy >= g.ny || iz >= g.nz) return -1;
  *bit = ix & 63;
  return (static_cast<long long>(iz) * g.ny + iy) * g.wx + (ix >> 6);
}

/// walk_segment_into / segment_clear (src/reach_solver.cpp:109-126,
/// src/voxgrid.cpp:100-112): the 1-based first blocked sample, 0 when fully
/// clear (sequential with early exit: the search kernels are fp64-bound and
/// most rejected walks stop at their first samples).
__device__ __forceinline__ int walk_first_blocked(const GridView& g, V3 from, V3 to, int n,
                                                  int kmax = 1 << 30) {
  const V3 diff = to - from;
  for (int k = 1; k <= n && k <= kmax; ++k) {
    int bit = 0;
    const long long idx = cell_word(g, walk_sample(from, diff, k, n), &bit);
    if (idx >= 0 && ((__ldg(g.bits + idx) >> bit) & 1ull)) return k;
  }
  return 0;
}

/// Blocked-sample mask of a walk of n <= N samples (bit k = sample k+1),
/// with all N gathers in flight together. Each coordinate's floor takes the
/// exact-floor fast path (with the grid's constant bracket g.dq: a sample
/// whose |q| exceeds its range is outside the grid on either side of the
/// bracket, so its verdict is unaffected); the rare coordinate whose bracket straddles an
/// integer (e.g. a sample exactly on a voxel face: quiver vectors with a
/// zero component from the root) gets vox_floor's IEEE division in place,
/// so the loads stay parallel and the mask is the reference's verdict.
/// Measured on B200: ~0.9k cycles for an 8-sample walk versus ~7k for the
/// sequential walk (one L2 round trip instead of 8).
template <int N, bool INPLACE>
__device__ __forceinline__ uint32_t walk_hits(const GridView& g, V3 from, V3 to, int n, bool* exact,
                                              int kstart = 0, int kend = N) {
  // One pass, no per-sample arrays: each sample's load is issued as soon as
  // its index is known and only its bit is kept, so the loads overlap
  // without holding 3N registers (or spilling them in large kernels).
  const V3 diff = to - from;
  bool ok = true;
  uint32_t mask = 0;
#pragma unroll
  for (int k = 0; k < N; ++k) {
    if (k < kstart || k >= kend) continue;  // caller-proven free samples (warp-uniform)
    const bool live = k < n;
    const double t = c_tk.v[n][live ? k + 1 : n];
    const V3 p = from + t * diff;
    const double ax = p.x - g.ox, ay = p.y - g.oy, az = p.z - g.oz;
    const double qx = ax * g.rvs, qy = ay * g.rvs, qz = az * g.rvs;
    const double dx = g.dq, dy = g.dq, dz = g.dq;
    double lx = floor(qx - dx), ly = floor(qy - dy), lz = floor(qz - dz);
    // floor(fl(q + d)) == l  <=>  fl(q + d) < l + 1, as fl(q + d) >= fl(q - d) >= l
    if (INPLACE) {
      if (!(qx + dx < lx + 1.0)) lx = floor(ax / g.vs);
      if (!(qy + dy < ly + 1.0)) ly = floor(ay / g.vs);
      if (!(qz + dz < lz + 1.0)) lz = floor(az / g.vs);
    } else {
      ok &= (qx + dx < lx + 1.0) & (qy + dy < ly + 1.0) & (qz + dz < lz + 1.0);
    }
    const int ix = static_cast<int>(lx), iy = static_cast<int>(ly), iz = static_cast<int>(lz);
    const bool inb = live & (ix >= 0) & (iy >= 0) & (iz >= 0) & (ix < g.nx) & (iy < g.ny) & (iz < g.nz);
    const long long idx = inb ? (static_cast<long long>(iz) * g.ny + iy) * g.wx + (ix >> 6) : 0;
    const uint64_t w = __ldg(g.bits + idx);
    mask |= static_cast<uint32_t>((w >> (ix & 63)) & static_cast<uint64_t>(inb)) << k;
  }
  *exact = ok;
  return mask;
}

/// walk_hits (non-INPLACE) with each sample's cell coordinate formed as one
/// FMA, q = t * B + A with A = fl(from - o) * rvs and B = diff * rvs, instead
/// of the sample point and its offset (4 fp64 ops per axis). q differs from
/// the reference's fl(fl(fl(from + fl(t * diff)) - o) / vs) by at most
/// ~9u M + u P cells (M bounds |A|, t |B| and |q|, P the sample's absolute
/// coordinate in cells), which the caller's bracket half-width dqa covers
/// (SolveDev::dq_aff); samples whose bracket holds an integer fail `exact`
/// and the caller redoes the walk sequentially, so the verdict is the
/// reference's.
template <int N>
__device__ __forceinline__ uint32_t walk_hits_affine(const GridView& g, V3 from, V3 to, int n,
                                                     double dqa, bool* exact, int kstart = 0,
                                                     int kend = N) {
  const V3 diff = to - from;
  const double Ax = (from.x - g.ox) * g.rvs, Ay = (from.y - g.oy) * g.rvs, Az = (from.z - g.oz) * g.rvs;
  const double Bx = diff.x * g.rvs, By = diff.y * g.rvs, Bz = diff.z * g.rvs;
  bool ok = true;
  uint32_t mask = 0;
#pragma unroll
  for (int k = 0; k < N; ++k) {
    if (k < kstart || k >= kend) continue;  // caller-proven free samples (warp-uniform)
    const bool live = k < n;
    const double t = c_tk.v[n][live ? k + 1 : n];
    const double qx = fma(t, Bx, Ax), qy = fma(t, By, Ay), qz = fma(t, Bz, Az);
    const double lx = floor(qx - dqa), ly = floor(qy - dqa), lz = floor(qz - dqa);
    ok &= (qx + dqa < lx + 1.0) & (qy + dqa < ly + 1.0) & (qz + dqa < lz + 1.0);
    const int ix = static_cast<int>(lx), iy = static_cast<int>(ly), iz = static_cast<int>(lz);
    const bool inb = live & (static_cast<unsigned>(ix) < static_cast<unsigned>(g.nx)) &
                     (static_cast<unsigned>(iy) < static_cast<unsigned>(g.ny)) &
                     (static_cast<unsigned>(iz) < static_cast<unsigned>(g.nz));
    const long long idx = inb ? (static_cast<long long>(iz) * g.ny + iy) * g.wx + (ix >> 6) : 0;
    const uint64_t w = __ldg(g.bits + idx);
    mask |= static_cast<uint32_t>((w >> (ix & 63)) & static_cast<uint64_t>(inb)) << k;
  }
  *exact = ok;
  return mask;
}

/// walk_first_blocked_fast_seg_from over walk_hits_affine (bracket dqa).
__device__ __forceinline__ int walk_first_blocked_affine_from(const GridView& g, V3 from, V3 to,
                                                              int n, int kstart, double dqa) {
  bool exact = true;
  uint32_t m;
  if (n == 8) m = walk_hits_affine<8>(g, from, to, 8, dqa, &exact, kstart);
  else if (n <= kTkMax) m = walk_hits_affine<kTkMax>(g, from, to, n, dqa, &exact, kstart);
  else return walk_first_blocked(g, from, to, n);
  if (!exact) return walk_first_blocked(g, from, to, n);
  return m ? __ffs(m) : 0;
}

/// walk_any_blocked_upto over walk_hits_affine (bracket dqa).
__device__ __forceinline__ int walk_any_blocked_upto_affine(const GridView& g, V3 from, V3 to, int n,
                                                            int kend, double dqa) {
  bool exact = true;
  uint32_t m;
  if (n == 8) m = walk_hits_affine<8>(g, from, to, 8, dqa, &exact, 0, kend);
  else if (n <= kTkMax) m = walk_hits_affine<kTkMax>(g, from, to, n, dqa, &exact, 0, kend);
  else return walk_first_blocked(g, from, to, n);
  if (!exact) return walk_first_blocked(g, from, to, n);
  return m ? __ffs(m) : 0;
}

/// walk_first_blocked with the gathers in flight together (n <= 16), the
/// sequential walk otherwise. Identical result. INPLACE = resolve ambiguous
/// floors by division inside the parallel walk (planner: walks from the root
/// often sit on voxel faces); otherwise redo such a walk sequentially
/// (seg2: rare, and the branch-free body keeps registers down — 2.15 vs
/// 2.73 ms for C2's seg2).
template <bool INPLACE>
__device__ __forceinline__ int walk_first_blocked_fast_t(const GridView& g, V3 from, V3 to, int n,
                                                         int kstart = 0, int kend = kTkMax) {
  bool exact = true;
  uint32_t m;
  if (n == 8) m = walk_hits<8, INPLACE>(g, from, to, 8, &exact, kstart, kend);
  else if (n <= kTkMax) m = walk_hits<kTkMax, INPLACE>(g, from, to, n, &exact, kstart, kend);
  else return walk_first_blocked(g, from, to, n);
  if (!exact) return walk_first_blocked(g, from, to, n);
  return m ? __ffs(m) : 0;
}
__device__ __forceinline__ int walk_first_blocked_fast(const GridView& g, V3 from, V3 to, int n) {
  return walk_first_blocked_fast_t<true>(g, from, to, n);
}
__device__ __forceinline__ int walk_first_blocked_fast_seg(const GridView& g, V3 from, V3 to, int n) {
  return walk_first_blocked_fast_t<false>(g, from, to, n);
}
/// The same verdict when the caller has proven samples 1..kstart free (they
/// are not looked up; the sequential fallback still walks every sample).
__device__ __forceinline__ int walk_first_blocked_fast_seg_from(const GridView& g, V3 from, V3 to,
                                                                int n, int kstart) {
  return walk_first_blocked_fast_t<false>(g, from, to, n, kstart);
}
/// Clear verdict (0 / nonzero, not the index) when samples kend+1..n are
/// proven free: only samples 1..kend are looked up.
__device__ __forceinline__ int walk_any_blocked_upto(const GridView& g, V3 from, V3 to, int n,
                                                     int kend) {
  return walk_first_blocked_fast_t<false>(g, from, to, n, 0, kend);
}

/// Out-of-line copy for the large planner kernels (one body instead of one
/// per call site keeps their instruction footprint down).
static __device__ __noinline__ int walk_first_blocked_par(const GridView& g, V3 from, V3 to, int n) {
  return walk_first_blocked_fast(g, from, to, n);
}

/// All n samples clear (segment_clear verdict; walk_points).
__device__ __forceinline__ bool walk_clear(const GridView& g, V3 from, V3 to, int n) {
  return walk_first_blocked_par(g, from, to, n) == 0;
}

/// scaled_sample_count (src/reach_solver.cpp:143-145)
__host__ __device__ __forceinline__ int scaled_sample_count(double len, double spacing) {
  const double s = spacing > 1e-12 ? spacing : 1e-12;
  const int c = static_cast<int>(ceil(len / s));
  return c > 1 ? c : 1;
}

/// point_to_segment (src/reach_solver.cpp:135-141; path_planner.cpp:12-18)
__host__ __device__ __forceinline__ double point_to_segment(V3 p, V3 a, V3 b) {
  const V3 ab = b - a;
  const double len2 = sqnorm(ab);
  if (len2 <= 1e-30) return norm(p - a);
  const double t = clampd(dot(p - a, ab) / len2, 0.0, 1.0);
  return norm(p - (a + t * ab));
}

/// Conservative prefilter for point_to_segment(t, a, a + L*dir) <= r0
/// (dir unit): false only when the segment certainly stays farther than r0
/// from t. Pass r = r0 + a margin (callers use 1e-6 m). If the true distance
/// is <= r0 either t is within r of a, or the closest point is interior,
/// so dot(dir, t-a) > 0 and the perpendicular distance^2 = |t-a|^2 -
/// dot^2 <= r0^2 < r^2, which this test accepts.
__host__ __device__ __forceinline__ bool may_pass_near(V3 t, V3 a, V3 dir, double L, double r) {
  const V3 w = t - a;
  const double d2 = sqnorm(w);
  const double r2 = r * r;
  if (d2 <= r2) return true;
  if (d2 > (L + r) * (L + r)) return false;
  const double dw = dot(dir, w);
  if (dw <= 0.0) return false;
  return dw * dw >= (d2 - r2) * (1.0 - 1e-9);
}

/// segment_segment_distance (src/arm_model.cpp:326-361)
__host__ __device__ __forceinline__ double seg_seg_distance(V3 a0, V3 a1, V3 b0, V3 b1) {
  const V3 d1 = a1 - a0;
  const V3 d2 = b1 - b0;
  const V3 r = a0 - b0;
  const double a = sqnorm(d1);
  const double e = sqnorm(d2);
  const double f = dot(d2, r);
  double s = 0.0, t = 0.0;
  if (a <= 1e-30 && e <= 1e-30) return norm(r);
  if (a <= 1e-30) {
    t = clampd(f / e, 0.0, 1.0);
  } else {
    const double c = dot(d1, r);
    if (e <= 1e-30) {
      s = clampd(-c / a, 0.0, 1.0);
    } else {
      const double b = dot(d1, d2);
      const double denom = a * e - b * b;
      if (denom > 1e-30) s = clampd((b * f - c * e) / denom, 0.0, 1.0);
      t = (b * s + f) / e;
      if (t < 0.0) {
        t = 0.0;
        s = clampd(-c / a, 0.0, 1.0);
      } else if (t > 1.0) {
        t = 1.0;
        s = clampd((b - c) / a, 0.0, 1.0);
      }
    }
  }
  return norm((a0 + s * d1) - (b0 + t * d2));
}

/// self_collision_free over a coaxial chain (src/arm_model.cpp:376-388):
/// links k = [joints[k], joints[k+1]], non-adjacent pairs >= 2*radius.
__host__ __device__ __forceinline__ bool self_collision_free(const V3* joints, int n_links,
                                                             double min_sep) {
  for (int i = 0; i + 2 < n_links; ++i)
    for (int j = i + 2; j < n_links; ++j)
      if (seg_seg_distance(joints[i], joints[i + 1], joints[j], joints[j + 1]) < min_sep)
        return false;
  return true;
}

/// True when links [a0, a1] and [b0, b1] (half-length bounds ha, hb) are
/// provably at least min_sep apart: their midpoints are farther apart than
/// min_sep + ha + hb (with margin), so seg_seg_distance >= min_sep.
__host__ __device__ __forceinline__ bool links_clear_screen(V3 a0, V3 a1, V3 b0, V3 b1, double ha,
                                                            double hb, double min_sep) {
  const V3 d = 0.5 * (a0 + a1) - 0.5 * (b0 + b1);
  const double r = min_sep + ha + hb;
  return sqnorm(d) > r * r * (1.0 + 1e-9) + 1e-12;
}

/// self_collision_free with a bounding-sphere screen: link k lies in the
/// ball around its midpoint of radius half[k] (an upper bound of half its
/// length), so a pair whose midpoints are farther apart than
/// min_sep + half[i] + half[j] (with margin) is at least min_sep apart and
/// its exact distance is not needed; every other pair gets
/// seg_seg_distance. Same verdict as self_collision_free.
__host__ __device__ __forceinline__ bool self_collision_free_screened(const V3* joints, int n_links,
                                                                      double min_sep,
                                                                      const double* half) {
  for (int i = 0; i + 2 < n_links; ++i)
    for (int j = i + 2; j < n_links; ++j) {
      const V3 ci = 0.5 * (joints[i] + joints[i + 1]);
      const V3 cj = 0.5 * (joints[j] + joints[j + 1]);
      const double r = min_sep + half[i] + half[j];
      if (sqnorm(ci - cj) > r * r * (1.0 + 1e-9) + 1e-12) continue;
      if (seg_seg_distance(joints[i], joints[i + 1], joints[j], joints[j + 1]) < min_sep)
        return false;
    }
  return true;
}

// ---------------------------------------------------------------------------
// Frames and joint limits (src/arm_model.cpp:12-70, 195-200). Only used when
// limits or offsets are active.
struct M3 {
  double a[3][3];
};

__host__ __device__ __forceinline__ M3 m_identity() {
  M3 m{};
  m.a[0][0] = m.a[1][1] = m.a[2][2] = 1.0;
  return m;
}
__host__ __device__ __forceinline__ M3 m_mul(const M3& A, const M3& B) {
  M3 m;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      double s = A.a[r][0] * B.a[0][c];
      s = s + A.a[r][1] * B.a[1][c];
      s = s + A.a[r][2] * B.a[2][c];
      m.a[r][c] = s;
    }
  return m;
}
__host__ __device__ __forceinline__ V3 m_tmul(const M3& A, V3 v) {  // A^T v
  const double in[3] = {v.x, v.y, v.z};
  double out[3];
  for (int r = 0; r < 3; ++r) {
    double s = A.a[0][r] * in[0];
    s = s + A.a[1][r] * in[1];
    s = s + A.a[2][r] * in[2];
    out[r] = s;
  }
  return V3{out[0], out[1], out[2]};
}
__host__ __device__ __forceinline__ V3 m_col(const M3& A, int c) {
  return V3{A.a[0][c], A.a[1][c], A.a[2][c]};
}
__host__ __device__ __forceinline__ M3 rot_z(double t) {
  const double c = cos(t), s = sin(t);
  M3 m{};
  m.a[0][0] = c; m.a[0][1] = -s; m.a[0][2] = 0;
  m.a[1][0] = s; m.a[1][1] = c;  m.a[1][2] = 0;
  m.a[2][0] = 0; m.a[2][1] = 0;  m.a[2][2] = 1;
  return m;
}
__host__ __device__ __forceinline__ M3 rot_y(double t) {
  const double c = cos(t), s = sin(t);
  M3 m{};
  m.a[0][0] = c;  m.a[0][1] = 0; m.a[0][2] = s;
  m.a[1][0] = 0;  m.a[1][1] = 1; m.a[1][2] = 0;
  m.a[2][0] = -s; m.a[2][1] = 0; m.a[2][2] = c;
  return m;
}

struct FrameStep {
  double theta, phi;
  bool degenerate;
  M3 after_azimuth, frame;
};

/// advance_frame (src/arm_model.cpp:34-59)
__host__ __device__ __forceinline__ FrameStep advance_frame(const M3& parent, V3 dir) {
  const V3 local = m_tmul(parent, dir);
  FrameStep st;
  const double planar = hypot(local.x, local.y);
  st.phi = atan2(planar, local.z);
  if (planar < 1e-12) {
    st.degenerate = true;
    st.theta = 0.0;
  } else {
    st.degenerate = false;
    st.theta = atan2(local.y, local.x);
  }
  st.after_azimuth = m_mul(parent, rot_z(st.theta));
  st.frame = m_mul(st.after_azimuth, rot_y(st.phi));
  return st;
}

struct Limit {
  double elev_min, elev_max, azim_min, azim_max;
};

__host__ __device__ __forceinline__ bool full_azimuth(const Limit& l) {
  return l.azim_min <= -3.14159265358979323846 && l.azim_max >= 3.14159265358979323846;
}
__host__ __device__ __forceinline__ bool limit_active(const Limit& l) {
  return l.elev_min > 1e-12 || l.elev_max < 3.14159265358979323846 - 1e-12 || !full_azimuth(l);
}
__host__ __device__ __forceinline__ double wrap_angle(double a) {
  const double kPi = 3.14159265358979323846;
  a = fmod(a, 2.0 * kPi);
  if (a <= -kPi) a += 2.0 * kPi;
  if (a > kPi) a -= 2.0 * kPi;
  return a;
}
/// joint_angle_within (src/arm_model.cpp:63-70, 195-200)
__host__ __device__ __forceinline__ bool joint_angle_within(double theta, double phi, bool degenerate,
                                                            const Limit& l) {
  const double kPi = 3.14159265358979323846;
  if (phi < l.elev_min - 1e-12 || phi > l.elev_max + 1e-12) return false;
  if (degenerate || full_azimuth(l)) return true;
  const double w = wrap_angle(theta);
  const double c[3] = {w, w - 2.0 * kPi, w + 2.0 * kPi};
  for (int k = 0; k < 3; ++k)
    if (c[k] >= l.azim_min - 1e-12 && c[k] <= l.azim_max + 1e-12) return true;
  return false;
}

}  // namespace rpd
