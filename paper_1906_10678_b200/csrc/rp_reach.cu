// gMS reach-pose search on the device (src/reach_solver.cpp:224-577).
//
//   k_seg1     prune_segment1 (:224-300): one thread per quiver direction.
//   k_seg2     seg2_worker (:316-456) = the per-segment reachability expansion
//              (p2 = p1 + L2 q_j, swept-segment clearance) fused with the
//              forward/backward intersection (gap band |b - p2| ~ L3, v3 / s4
//              clearance, self-collision). One thread per (survivor, j) pair,
//              grid-stride over warps; solutions are written as a bit set in
//              canonical (i, j, l) order by warp ballot, counters are reduced
//              per thread and flushed with one atomic per warp, the
//              select_solution argmin (:548-577) is reduced per block.
//   k_shortcuts short_reach_scan (:176-222) on the rare near-encounter pairs.
//
// All decisions use rp_device.cuh's reference-order fp64 arithmetic, so the
// solution set, the shortcut set and all 13 SolveStats counters are
// bit-identical to the reference.
#include "rp_reach.cuh"
#include "rp_rings.cuh"
#include "rp_refine.cuh"

#include <cub/cub.cuh>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>

namespace rp {

using rpd::V3;

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr unsigned kShortcutCap = 1u << 20;

__device__ __forceinline__ bool offset_link_clear(const rpd::GridView& g, V3 from, V3 to,
                                                  double spacing) {
  const double len = rpd::norm(to - from);
  if (len == 0.0) return true;
  return rpd::walk_first_blocked(g, from, to, rpd::scaled_sample_count(len, spacing)) == 0;
}

__device__ __forceinline__ void warp_flush(unsigned long long* ctr, int idx, unsigned v) {
  v = __reduce_add_sync(FULL, v);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(ctr + idx, static_cast<unsigned long long>(v));
}

// ---------------------------------------------------------------------------
__global__ void k_walk4(SolveDev a, uint8_t* out) {
  const int bi = blockIdx.x * blockDim.x + threadIdx.x;
  if (bi >= a.B) return;
  out[bi] = rpd::walk_first_blocked(a.g, a.bpts[bi], a.target, a.n) == 0 ? 1 : 0;
}

/// cone_subset membership (src/quiver.cpp:53-63) with an ambiguity flag for
/// angles within 1e-9 rad of the limit (re-decided on the host with glibc).
__global__ void k_cone(const double* qx, const double* qy, const double* qz, int Q, V3 axis,
                       double limit, uint8_t* inside, uint8_t* ambiguous) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= Q) return;
  const V3 v{qx[i], qy[i], qz[i]};
  const double ang = atan2(rpd::norm(rpd::cross(v, axis)), rpd::dot(v, axis));
  inside[i] = ang <= limit ? 1 : 0;
  ambiguous[i] = fabs(ang - limit) < 1e-9 ? 1 : 0;
}

/// prune_segment1 for every quiver direction.
__global__ void __launch_bounds__(256) k_seg1(SolveDev a, uint32_t* __restrict__ surv_bits,
                                              unsigned long long* ctr, long long* sc_list,
                                              unsigned* sc_count) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  bool lim_pass = false, reach = false, surv = false;
  if (i < a.Q) {
    const ArmDev& arm = a.arm;
    const V3 dir = qvec(a, i);
    rpd::FrameStep st{};
    const bool has_elbow = arm.off[0] > 0.0;
    if (arm.lim_active[0] || has_elbow) st = rpd::advance_frame(arm.base, dir);
    lim_pass = !arm.lim_active[0] || rpd::joint_angle_within(st.theta, st.phi, st.degenerate, arm.lim[0]);
    if (lim_pass) {
      V3 link = arm.root, elbow{0, 0, 0};
      if (has_elbow) {
        elbow = arm.root + arm.off[0] * rpd::m_col(st.after_azimuth, 0);
        link = elbow;
      }
      const V3 p1 = link + arm.L[0] * dir;
      reach = a.disable_prune != 0;
      for (int t = 0; !reach && t < a.n_targets; ++t)
        if (rpd::sqnorm(p1 - a.targets[t]) <= a.budget2) reach = true;
      if (reach || a.scanning) {
        if (!has_elbow || offset_link_clear(a.g, arm.root, elbow, a.spacing)) {
          const int fb = rpd::walk_first_blocked(a.g, link, p1, a.n);
          if (a.scanning && rpd::point_to_segment(a.target, link, p1) <= a.near_r + 1e-9) {
            const unsigned pos = atomicAdd(sc_count, 1u);
            if (pos < kShortcutCap) sc_list[pos] = i;
          }
          surv = reach && fb == 0;
        }
      }
    }
  }
  const unsigned m = __ballot_sync(FULL, surv);
  if ((threadIdx.x & 31) == 0 && (i >> 5) < (a.Q + 31) / 32) surv_bits[i >> 5] = m;
  warp_flush(ctr, C_SEG1_LIMIT, lim_pass ? 1u : 0u);
  warp_flush(ctr, C_SEG1_REACH, (lim_pass && reach) ? 1u : 0u);
  warp_flush(ctr, C_SEG1_SURV, surv ? 1u : 0u);
}

/// Ordered compaction of a small bit set in one block (bit k -> out[rank]).
__global__ void k_compact_small(const uint32_t* __restrict__ bits, int nbits, int* __restrict__ out,
                                int* __restrict__ count) {
  typedef cub::BlockScan<int, 1024> Scan;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int nwords = (nbits + 31) / 32;
  for (int w0 = 0; w0 < nwords; w0 += 1024) {
    const int w = w0 + threadIdx.x;
    const uint32_t word = w < nwords ? bits[w] : 0u;
    const int c = __popc(word);
    int off = 0, total = 0;
    Scan(tmp).ExclusiveSum(c, off, total);
    off += carry;
    uint32_t x = word;
    while (x) {
      const int b = __ffs(x) - 1;
      x &= x - 1;
      out[off++] = w * 32 + b;
    }
    __syncthreads();
    if (threadIdx.x == 0) carry += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) *count = carry;
}

__global__ void k_surv_data(SolveDev a, const int* __restrict__ idx, const int* __restrict__ S1p,
                            SurvDev* __restrict__ out) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= *S1p) return;
  const ArmDev& arm = a.arm;
  SurvDev h{};
  h.i = idx[s];
  const V3 dir = qvec(a, h.i);
  V3 link = arm.root;
  if (arm.any_limit || arm.has_offsets) {
    const rpd::FrameStep st = rpd::advance_frame(arm.base, dir);
    h.frame = st.frame;
    if (arm.off[0] > 0.0) {
      link = arm.root + arm.off[0] * rpd::m_col(st.after_azimuth, 0);
      h.has_elbow = 1;
    }
  }
  h.link_start = link;
  h.p1 = link + arm.L[0] * dir;
  out[s] = h;
}

/// seg2_worker over all (survivor, j) pairs; see the file head.
template <bool EIGHT, bool GENERAL, bool B1>
__global__ void __launch_bounds__(256) k_seg2(SolveDev a, const SurvDev* __restrict__ sv,
                                              int64_t p_lo, int64_t npairs,
                                              uint32_t* __restrict__ sol_bits,
                                              unsigned long long* ctr, long long* sc_list,
                                              unsigned* sc_count, BestRec* __restrict__ block_best) {
  unsigned c_lim = 0, c_clear = 0, c_gt = 0, c_gp = 0, c_jp = 0, c_v3 = 0, c_sol = 0;
  double best_len = 1e308;
  long long best_key = LLONG_MAX;
  const int lane = threadIdx.x & 31;
  const int64_t warp_id = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const ArmDev& arm = a.arm;
  const double L1 = arm.L[0], L2 = arm.L[1], L3 = arm.L[2];
  const double min_sep = 2.0 * arm.arm_radius;

  // pairs [p_lo, npairs) (a part of the solve: whole survivor rows); warps
  // start at 32-aligned pair indices so the B == 1 ballot stores whole words
  for (int64_t base = (p_lo & ~int64_t{31}) + warp_id * 32; base < npairs; base += nwarps * 32) {
    const int64_t p = base + lane;
    bool solbit = false;
    if (p >= p_lo && p < npairs) {
      const int s = static_cast<int>(p / a.Q);
      const int j = static_cast<int>(p - static_cast<int64_t>(s) * a.Q);
      const V3 dir2 = qvec(a, j);
      const SurvDev& h = sv[s];
      rpd::FrameStep st2{};
      bool have_st2 = false;
      bool ok = true;
      if (GENERAL && (arm.lim_active[1] || arm.off[1] > 0.0)) {
        st2 = rpd::advance_frame(h.frame, dir2);
        have_st2 = true;
        ok = rpd::joint_angle_within(st2.theta, st2.phi, st2.degenerate, arm.lim[1]);
      }
      if (ok) {
        ++c_lim;
        V3 link = h.p1, e2{0, 0, 0};
        const bool has_e2 = GENERAL && arm.off[1] > 0.0;
        if (has_e2) {
          e2 = h.p1 + arm.off[1] * rpd::m_col(st2.after_azimuth, 0);
          link = e2;
        }
        const V3 p2 = link + L2 * dir2;
        if (GENERAL && EIGHT && a.cone_precheck && !a.disable_prune) {
          const double dist_t = rpd::norm(a.target - p2);
          if (dist_t - a.L4 > L3 + a.eps + 1e-9 || dist_t + a.L4 < L3 - a.eps - 1e-9) ok = false;
        }
        if (ok && has_e2 && !offset_link_clear(a.g, h.p1, e2, a.spacing)) ok = false;
        if (ok) {
          const int fb = rpd::walk_first_blocked(a.g, link, p2, a.n);
          if (rpd::may_pass_near(a.target, link, dir2, L2, a.near_r + 1e-6) &&
              rpd::point_to_segment(a.target, link, p2) <= a.near_r + 1e-9) {
            const unsigned pos = atomicAdd(sc_count, 1u);
            if (pos < kShortcutCap) sc_list[pos] = (1ll << 62) | p;
          }
          if (fb == 0) {
            ++c_clear;
            for (int bi = 0; bi < a.B; ++bi) {
              ++c_gt;
              const V3 b = a.bpts[bi];
              const V3 v3 = b - p2;
              if (rpd::sqnorm(v3) > a.coarse2) continue;
              const double v3_len = rpd::norm(v3);
              if (fabs(v3_len - L3) > a.eps) continue;
              ++c_gp;
              if (v3_len < 1e-12) continue;
              if (GENERAL) {
                const bool l3 = arm.lim_active[2] != 0;
                const bool l4 = EIGHT && arm.lim_active[3] != 0;
                if (l3 || l4) {
                  const V3 v3_hat = v3 / v3_len;
                  if (!have_st2) {
                    st2 = rpd::advance_frame(h.frame, dir2);
                    have_st2 = true;
                  }
                  const rpd::FrameStep st3 = rpd::advance_frame(st2.frame, v3_hat);
                  if (l3 && !rpd::joint_angle_within(st3.theta, st3.phi, st3.degenerate, arm.lim[2]))
                    continue;
                  if (l4) {
                    const rpd::FrameStep st4 = rpd::advance_frame(st3.frame, a.bdirs[bi]);
                    if (!rpd::joint_angle_within(st4.theta, st4.phi, st4.degenerate, arm.lim[3]))
                      continue;
                  }
                }
              }
              ++c_jp;
              if (rpd::walk_first_blocked(a.g, p2, b, a.n) != 0) continue;
              ++c_v3;
              if (EIGHT && !a.walk4_ok[bi]) continue;
              const V3 qi = qvec(a, h.i);
              const V3 s1 = L1 * qi;
              const V3 s2 = L2 * dir2;
              bool free_ok;
              if (!GENERAL || !arm.has_offsets) {
                V3 J[5];
                J[0] = arm.root;
                J[1] = J[0] + s1;
                J[2] = J[1] + s2;
                J[3] = J[2] + v3;
                if (EIGHT) J[4] = J[3] + a.L4 * a.bdirs[bi];
                free_ok = rpd::self_collision_free(J, EIGHT ? 4 : 3, min_sep);
              } else {
                DevPose dp;
                dp.nseg = EIGHT ? 4 : 3;
                dp.seg[0] = s1;
                dp.seg[1] = s2;
                dp.seg[2] = v3;
                if (EIGHT) dp.seg[3] = a.L4 * a.bdirs[bi];
                build_chain(arm, dp);
                free_ok = pose_self_free(dp, min_sep);
              }
              if (!free_ok) continue;
              ++c_sol;
              const long long key = p * a.B + bi;
              if (B1) {
                solbit = true;
              } else {
                atomicOr(sol_bits + (key >> 5), 1u << (key & 31));
              }
              const double len = (rpd::norm(s1) + rpd::norm(s2)) + rpd::norm(v3);
              if (len < best_len || (len == best_len && key < best_key)) {
                best_len = len;
                best_key = key;
              }
            }
          }
        }
      }
    }
    if (B1) {
      const unsigned m = __ballot_sync(FULL, solbit);
      if (lane == 0) sol_bits[base >> 5] = m;
    }
  }
  warp_flush(ctr, C_SEG2_LIMIT, c_lim);
  warp_flush(ctr, C_SEG2_CLEAR, c_clear);
  warp_flush(ctr, C_GAP_TESTED, c_gt);
  warp_flush(ctr, C_GAP_PASS, c_gp);
  warp_flush(ctr, C_JOINT_PASS, c_jp);
  warp_flush(ctr, C_V3_CLEAR, c_v3);
  warp_flush(ctr, C_SOLUTIONS, c_sol);
  // block argmin of (length, canonical key)
  for (int off = 16; off > 0; off >>= 1) {
    const double ol = __shfl_down_sync(FULL, best_len, off);
    const long long ok = __shfl_down_sync(FULL, best_key, off);
    if (ol < best_len || (ol == best_len && ok < best_key)) {
      best_len = ol;
      best_key = ok;
    }
  }
  __shared__ BestRec wb[8];
  if (lane == 0) wb[threadIdx.x >> 5] = BestRec{best_len, best_key};
  __syncthreads();
  if (threadIdx.x == 0) {
    BestRec b = wb[0];
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w)
      if (wb[w].len < b.len || (wb[w].len == b.len && wb[w].key < b.key)) b = wb[w];
    block_best[blockIdx.x] = b;
  }
}

/// k_seg2 for the common case (coaxial arm, no limits, no cone precheck,
/// one backward point): a warp owns survivor rows and sweeps j. Phase 1
/// (every pair, lanes busy) walks segment 2, runs the near-encounter scan
/// and a conservative band prefilter; clear band candidates are queued per
/// warp in shared memory and phase 2 runs the exact gap test, the v3 walk
/// and the self-collision check 32 at a time without divergence. Counters,
/// solution bits (atomicOr into a zeroed set) and the block argmin are the
/// same as k_seg2's.
#ifndef RP_SEG2_PAR_WALK
#define RP_SEG2_PAR_WALK 1
#endif
constexpr bool kSeg2ParWalk = RP_SEG2_PAR_WALK;
#ifndef RP_BQ_MINB
#define RP_BQ_MINB 4
#endif

/// Per end point b: kend = the samples 1..kend of a walk [p2, b] with
/// |b - p2| <= L that are not proven free; sample j lies within
/// (1 - j/n) * L of b, so it is free when that plus sqrt(3) * vs is below
/// the clearance-field lower bound D on the distance from b to any occupied
/// cell (see k_row_skip).
__global__ void k_tail_skip(rpd::GridView g, const V3* __restrict__ pts, int T, double L, int n,
                            ClearanceField f, uint8_t* __restrict__ kend) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const double D = cf_distance(f, g, pts[t]);
  const double Lm = L * (1.0 + 1e-9) + 1e-9;
  const double cell = 1.7320508075688772 * g.vs * (1.0 + 1e-9) + 1e-9;
  int j = n;
  while (j >= 1 && (1.0 - static_cast<double>(j) / n) * Lm + cell < D) --j;
  kend[t] = static_cast<uint8_t>(j);
}

/// Per survivor row: how many leading segment-2 samples are provably free.
/// D = the clearance field's lower bound on the distance from p1 to any
/// occupied cell (grid_clearance_field). Sample k lies within t_k * L2 of p1
/// (|q_j| = 1 up to rounding), and the cell the reference floors it to
/// (off by at most one per axis from the cell holding it) lies within
/// sqrt(3) * vs of it, so samples with t_k * L2 + sqrt(3) * vs < D (with
/// margins) are free. One thread per row.
__global__ void k_row_skip(SolveDev a, const SurvDev* __restrict__ sv, const int* __restrict__ S1p,
                           ClearanceField f, uint8_t* __restrict__ kskip) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= *S1p) return;
  const rpd::GridView& g = a.g;
  const double D = cf_distance(f, g, sv[s].p1);
  const double L2 = a.arm.L[1] * (1.0 + 1e-9) + 1e-9;
  const double cell = 1.7320508075688772 * g.vs * (1.0 + 1e-9) + 1e-9;
  int k = 0;
  while (k < a.n && (static_cast<double>(k + 1) / a.n) * L2 + cell < D) ++k;
  kskip[s] = static_cast<uint8_t>(k);
}

template <bool EIGHT, bool OV>
__global__ void __launch_bounds__(256, 5) k_seg2_rows(SolveDev a, const SurvDev* __restrict__ sv,
                                                   const int* __restrict__ S1p, int part, int parts,
                                                   uint32_t* __restrict__ sol_bits,
                                                   unsigned long long* ctr, long long* sc_list,
                                                   unsigned* sc_count, BestRec* __restrict__ block_best,
                                                   int* unit_ctr, const uint8_t* __restrict__ kskip,
                                                   const uint8_t* __restrict__ kend_b,
                                                   uint32_t* __restrict__ c2bits, uint8_t* c2ok,
                                                   const uint32_t* __restrict__ c2bits_r,
                                                   const uint8_t* __restrict__ c2ok_r, V3 ov_lo,
                                                   V3 ov_hi) {
  unsigned c_lim = 0, c_clear = 0, c_gp = 0, c_jp = 0, c_v3 = 0, c_sol = 0;
  double best_len = 1e308;
  long long best_key = LLONG_MAX;
  const int lane = threadIdx.x & 31;
  const int warp_id = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const ArmDev& arm = a.arm;
  const double L1 = arm.L[0], L2 = arm.L[1], L3 = arm.L[2];
  const double min_sep = 2.0 * arm.arm_radius;
  const V3 b = a.bpts[0];
  const V3 bdir = a.bdirs[0];
  const bool walk4 = !EIGHT || a.walk4_ok[0];
  const double rnear = a.near_r + 1e-6;
  const int kend_bv = *kend_b;  // samples of the v3 walks [p2, b] not proven free
  __shared__ int wqs[8][64];
  int* wq = wqs[threadIdx.x >> 5];
  constexpr int kChunk = 1024;  // j per work unit (balances small S1)
  const int nchunk = (a.Q + kChunk - 1) / kChunk;
  // this part's survivor rows [s_lo, s_hi) of the S1 the prune left on the
  // device (no host read-back between the prune and this kernel)
  const int S1 = *S1p;
  const int s_lo = static_cast<int>(static_cast<int64_t>(S1) * part / parts);
  const int s_hi = static_cast<int>(static_cast<int64_t>(S1) * (part + 1) / parts);
  (void)warp_id;
  (void)nwarps;
  for (;;) {
    // units are taken dynamically: their cost varies with the row's geometry
    int u = 0;
    if (lane == 0) u = atomicAdd(unit_ctr, 1);
    u = __shfl_sync(FULL, u, 0);
    if (u >= (s_hi - s_lo) * nchunk) break;
    const int s = s_lo + u / nchunk;  // survivor rows [s_lo, s_hi): this part's
    const int chunk = u - (s - s_lo) * nchunk;
    const int jbeg = chunk * kChunk;
    const int jend = min(a.Q, jbeg + kChunk);
    const SurvDev& h = sv[s];
    // segment-2 walk verdicts of this row chunk from an earlier solve on
    // the same grid (grid_seg2_cache), or computed here and recorded
    const size_t c2row = static_cast<size_t>(h.i) * ((a.Q + 31) >> 5);
    uint8_t* const c2flag = c2ok ? c2ok + static_cast<size_t>(h.i) * nchunk + chunk : nullptr;
    // an overlay grid reads its base grid's verdicts (c2*_r, never written
    // here): blocked stays blocked, clear is walked again when the segment's
    // box meets the box of the overlay's added cells
    const bool from_base = OV;  // c2ok_r / c2bits_r set
    const bool cached = from_base ? __ldg(c2ok_r + static_cast<size_t>(h.i) * nchunk + chunk) != 0
                                  : (c2flag && __ldcg(c2flag) != 0);
    // a cached chunk's 32 words, one per lane (shuffled out per 32 j)
    const uint32_t c2mine =
        cached && jbeg + 32 * lane < jend
            ? (from_base ? __ldg(c2bits_r + c2row + (jbeg >> 5) + lane)
                         : __ldcg(c2bits + c2row + (jbeg >> 5) + lane))
            : 0u;
    const V3 p1 = h.p1;
    bool row_meets = false;  // some segment of the row may reach the overlay box
    if (OV) {
      const double dx = fmax(fmax(ov_lo.x - p1.x, p1.x - ov_hi.x), 0.0);
      const double dy = fmax(fmax(ov_lo.y - p1.y, p1.y - ov_hi.y), 0.0);
      const double dz = fmax(fmax(ov_lo.z - p1.z, p1.z - ov_hi.z), 0.0);
      row_meets = !(ov_lo.x > ov_hi.x) &&
                  sqrt(dx * dx + dy * dy + dz * dz) <= L2 * (1.0 + 1e-9) + 1e-9;
    }
    const V3 s1 = L1 * qvec(a, h.i);
    const int ks = kskip[s];  // leading samples of every segment-2 walk of this row that are free
    const bool row_near = rpd::sqnorm(a.target - p1) <= (L2 + rnear) * (L2 + rnear);
    const double db = sqrt(rpd::sqnorm(b - p1));
    const bool row_gap = db <= (sqrt(a.coarse2) + L2) * (1.0 + 1e-9) + 1e-12 &&
                         db >= (L3 - a.eps - L2) * (1.0 - 1e-9) - 1e-12;
    const auto heavy = [&](int j) {
      const long long p = static_cast<long long>(s) * a.Q + j;
      const V3 dir2 = qvec(a, j);
      const V3 p2 = p1 + L2 * dir2;
      const V3 v3 = b - p2;
      const double v3_len = rpd::norm(v3);
      if (fabs(v3_len - L3) > a.eps) return;
      ++c_gp;
      if (v3_len < 1e-12) return;
      ++c_jp;
      // |b - p2| passed the gap band, so both ends lie within the arm's reach
      // (the affine bracket's bound); samples past kend_bv are proven free
      if (rpd::walk_any_blocked_upto_affine(a.g, p2, b, a.n, kend_bv, a.dq_aff) != 0) return;
      ++c_v3;
      if (EIGHT && !walk4) return;
      const V3 s2 = L2 * dir2;
      V3 J[5];
      J[0] = arm.root;
      J[1] = J[0] + s1;
      J[2] = J[1] + s2;
      J[3] = J[2] + v3;
      if (EIGHT) J[4] = J[3] + a.L4 * bdir;
      // half-length bounds as in k_bq_tail
      const double w = 1.0 + 1e-9;
      const double half[4] = {0.5 * L1 * w, 0.5 * L2 * w, 0.5 * (L3 + a.eps) * w, 0.5 * a.L4 * w};
      if (!rpd::self_collision_free_screened(J, EIGHT ? 4 : 3, min_sep, half)) return;
      ++c_sol;
      atomicOr(sol_bits + (p >> 5), 1u << (p & 31));
      const double len = (rpd::norm(s1) + rpd::norm(s2)) + rpd::norm(v3);
      if (len < best_len || (len == best_len && p < best_key)) {
        best_len = len;
        best_key = p;
      }
    };
    int qn = 0;
    for (int j0 = jbeg; j0 < jend; j0 += 32) {
      const int j = j0 + lane;
      bool pass = false;
      const uint32_t c2w = __shfl_sync(FULL, c2mine, (j0 - jbeg) >> 5);
      if (j < jend) {
        ++c_lim;
        const V3 dir2 = qvec(a, j);
        const V3 p2 = p1 + L2 * dir2;
        int fb =
            cached ? static_cast<int>(((c2w >> lane) & 1u) ^ 1u)
            : ks >= a.n     ? 0
            : kSeg2ParWalk ? rpd::walk_first_blocked_affine_from(a.g, p1, p2, a.n, ks, a.dq_aff)
                           : rpd::walk_first_blocked(a.g, p1, p2, a.n);
        if (OV && cached && row_meets && fb == 0 &&
            fmin(p1.x, p2.x) <= ov_hi.x + 1e-9 && fmax(p1.x, p2.x) >= ov_lo.x - 1e-9 &&
            fmin(p1.y, p2.y) <= ov_hi.y + 1e-9 && fmax(p1.y, p2.y) >= ov_lo.y - 1e-9 &&
            fmin(p1.z, p2.z) <= ov_hi.z + 1e-9 && fmax(p1.z, p2.z) >= ov_lo.z - 1e-9) {
          // clear on the static grid: only samples inside the box of added
          // cells (it holds every point that floors into one) can block now
          const V3 diff = p2 - p1;
          for (int k = 1; k <= a.n; ++k) {
            const V3 sk = rpd::walk_sample(p1, diff, k, a.n);
            if (sk.x < ov_lo.x - 1e-9 || sk.x > ov_hi.x + 1e-9 || sk.y < ov_lo.y - 1e-9 ||
                sk.y > ov_hi.y + 1e-9 || sk.z < ov_lo.z - 1e-9 || sk.z > ov_hi.z + 1e-9)
              continue;
            int bit = 0;
            const long long w = rpd::cell_word(a.g, sk, &bit);
            if (w >= 0 && ((__ldg(a.g.bits + w) >> bit) & 1ull)) {
              fb = k;
              break;
            }
          }
        }
        if (c2flag && !cached) {
          const unsigned cm = __activemask();
          const unsigned clear = __ballot_sync(cm, fb == 0);
          if (lane == 0) c2bits[c2row + (j >> 5)] = clear;
        }
        if (row_near && rpd::may_pass_near(a.target, p1, dir2, L2, rnear) &&
            rpd::point_to_segment(a.target, p1, p2) <= a.near_r + 1e-9) {
          const unsigned pos = atomicAdd(sc_count, 1u);
          if (pos < kShortcutCap) sc_list[pos] = (1ll << 62) | (static_cast<long long>(s) * a.Q + j);
        }
        if (fb == 0) {
          ++c_clear;
          if (row_gap) {
            const double v2 = rpd::sqnorm(b - p2);
            pass = v2 <= a.coarse2 && v2 >= a.band_lo2;
          }
        }
      }
      const unsigned m = __ballot_sync(FULL, pass);
      if (pass) wq[qn + __popc(m & ((1u << lane) - 1u))] = j;
      qn += __popc(m);
      __syncwarp();
      if (qn >= 32) {
        heavy(wq[lane]);
        __syncwarp();
        if (lane < qn - 32) wq[lane] = wq[32 + lane];
        qn -= 32;
        __syncwarp();
      }
    }
    if (lane < qn) heavy(wq[lane]);
    __syncwarp();
    if (c2flag && !cached) {  // the chunk's words are written: publish it
      __threadfence();
      if (lane == 0) *reinterpret_cast<volatile uint8_t*>(c2flag) = 1;
    }
  }
  warp_flush(ctr, C_SEG2_LIMIT, c_lim);
  warp_flush(ctr, C_SEG2_CLEAR, c_clear);
  warp_flush(ctr, C_GAP_TESTED, c_clear);
  warp_flush(ctr, C_GAP_PASS, c_gp);
  warp_flush(ctr, C_JOINT_PASS, c_jp);
  warp_flush(ctr, C_V3_CLEAR, c_v3);
  warp_flush(ctr, C_SOLUTIONS, c_sol);
  for (int off = 16; off > 0; off >>= 1) {
    const double ol = __shfl_down_sync(FULL, best_len, off);
    const long long ok = __shfl_down_sync(FULL, best_key, off);
    if (ol < best_len || (ol == best_len && ok < best_key)) {
      best_len = ol;
      best_key = ok;
    }
  }
  __shared__ BestRec wb[8];
  if (lane == 0) wb[threadIdx.x >> 5] = BestRec{best_len, best_key};
  __syncthreads();
  if (threadIdx.x == 0) {
    BestRec r = wb[0];
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w)
      if (wb[w].len < r.len || (wb[w].len == r.len && wb[w].key < r.key)) r = wb[w];
    block_best[blockIdx.x] = r;
  }
}

__global__ void k_best_final(const BestRec* __restrict__ in, int n, BestRec* out) {
  __shared__ BestRec sh[256];
  BestRec b{1e308, LLONG_MAX};
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    const BestRec r = in[k];
    if (r.len < b.len || (r.len == b.len && r.key < b.key)) b = r;
  }
  sh[threadIdx.x] = b;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const BestRec r = sh[threadIdx.x + s];
      if (r.len < sh[threadIdx.x].len ||
          (r.len == sh[threadIdx.x].len && r.key < sh[threadIdx.x].key))
        sh[threadIdx.x] = r;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

/// short_reach_scan for one candidate: hypothesis samples along
/// [link, end] (walk truncated at the first blocked sample), origin for the
/// direct completion, prefix length for polyline_length.
__device__ void scan_one(const SolveDev& a, V3 link, V3 end, V3 origin, int fb, ShortcutRec& r,
                         bool has_prefix, V3 prefix_from, V3 prefix_to) {
  const int len = fb ? fb : a.n;
  const V3 diff = end - link;
  int hit = 0;
  for (int k = 0; k < len; ++k) {
    const V3 sk = rpd::walk_sample(link, diff, k + 1, a.n);
    if (rpd::norm(sk - a.target) <= a.near_r + 1e-12) {
      hit = k + 1;
      break;
    }
    const bool clear = !(fb && k + 1 == fb);
    if (!clear) break;
  }
  r.valid = 0;
  if (hit == 0) return;
  r.hit = hit;
  r.n_sub = hit;
  r.origin = origin;
  const V3 hp = rpd::walk_sample(link, diff, hit, a.n);
  const double dist = rpd::norm(hp - a.target);
  r.has_bridge = 0;
  r.via_direct = 0;
  r.n_direct = 0;
  if (dist > 1e-9) {
    const bool bridge_ok =
        rpd::walk_first_blocked(a.g, hp, a.target, rpd::scaled_sample_count(dist, a.spacing)) == 0;
    if (bridge_ok) {
      r.has_bridge = 1;
      r.bridge = a.target - hp;
    } else {
      const double dl = rpd::norm(a.target - origin);
      const int nd = rpd::scaled_sample_count(dl, a.spacing);
      if (rpd::walk_first_blocked(a.g, origin, a.target, nd) != 0) return;
      r.via_direct = 1;
      r.n_direct = nd;
    }
  }
  // polyline_length(root, tip_waypoints) (reach_solver.cpp:157-165, 169-174)
  double acc = 0.0;
  V3 prev = a.arm.root;
  if (has_prefix) {
    const V3 pd = prefix_to - prefix_from;
    for (int k = 1; k <= a.n; ++k) {
      const V3 q = rpd::walk_sample(prefix_from, pd, k, a.n);
      acc += rpd::norm(q - prev);
      prev = q;
    }
  }
  if (r.via_direct) {
    const V3 dd = a.target - origin;
    for (int k = 1; k <= r.n_direct; ++k) {
      const V3 q = rpd::walk_sample(origin, dd, k, r.n_direct);
      acc += rpd::norm(q - prev);
      prev = q;
    }
  } else {
    for (int k = 1; k <= hit; ++k) {
      const V3 q = rpd::walk_sample(link, diff, k, a.n);
      acc += rpd::norm(q - prev);
      prev = q;
    }
  }
  if (r.has_bridge) acc += rpd::norm(a.target - prev);
  r.path_length = acc;
  r.valid = 1;
}

__global__ void k_shortcuts(SolveDev a, const SurvDev* __restrict__ sv, const long long* keys,
                            int n, ShortcutRec* out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const long long key = keys[t];
  ShortcutRec r{};
  r.key = key;
  const ArmDev& arm = a.arm;
  if (!(key >> 62)) {
    const int i = static_cast<int>(key);
    const V3 dir = qvec(a, i);
    V3 link = arm.root;
    if (arm.off[0] > 0.0) {
      const rpd::FrameStep st = rpd::advance_frame(arm.base, dir);
      link = arm.root + arm.off[0] * rpd::m_col(st.after_azimuth, 0);
    }
    const V3 p1 = link + arm.L[0] * dir;
    const int fb = rpd::walk_first_blocked(a.g, link, p1, a.n);
    r.segment_index = 1;
    r.seg1 = i;
    r.seg2 = -1;
    scan_one(a, link, p1, arm.root, fb, r, false, link, link);
  } else {
    const long long p = key & ((1ll << 62) - 1);
    const int s = static_cast<int>(p / a.Q);
    const int j = static_cast<int>(p - static_cast<long long>(s) * a.Q);
    const SurvDev h = sv[s];
    const V3 dir2 = qvec(a, j);
    V3 link = h.p1;
    if (arm.off[1] > 0.0) {
      const rpd::FrameStep st2 = rpd::advance_frame(h.frame, dir2);
      link = h.p1 + arm.off[1] * rpd::m_col(st2.after_azimuth, 0);
    }
    const V3 p2 = link + arm.L[1] * dir2;
    const int fb = rpd::walk_first_blocked(a.g, link, p2, a.n);
    r.segment_index = 2;
    r.seg1 = h.i;
    r.seg2 = j;
    scan_one(a, link, p2, h.p1, fb, r, true, h.link_start, h.p1);
  }
  out[t] = r;
}

__global__ void k_word_popc(const uint32_t* __restrict__ w, int64_t nw, unsigned long long* __restrict__ c) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < nw) c[k] = __popc(w[k]);
}

__global__ void k_scatter_bits(const uint32_t* __restrict__ w, int64_t nw,
                               const unsigned long long* __restrict__ off, long long* __restrict__ keys) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= nw) return;
  uint32_t x = w[k];
  unsigned long long o = off[k];
  while (x) {
    const int b = __ffs(x) - 1;
    x &= x - 1;
    keys[o++] = k * 32 + b;
  }
}

__global__ void k_rank(const uint32_t* __restrict__ w, long long key, unsigned long long* out) {
  unsigned long long c = 0;
  const long long nw = key >> 5;
  for (long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; k < nw;
       k += static_cast<long long>(gridDim.x) * blockDim.x)
    c += __popc(w[k]);
  if (blockIdx.x == 0 && threadIdx.x == 0 && (key & 31))
    c += __popc(w[nw] & ((1u << (key & 31)) - 1u));
  c = __reduce_add_sync(FULL, static_cast<unsigned>(c));
  if ((threadIdx.x & 31) == 0) atomicAdd(out, c);
}

}  // namespace

/// Materialise solution poses from canonical keys (reach_solver.cpp:434-449).
__device__ DevPose materialize_key(const SolveDev& a, const SurvDev* __restrict__ sv, long long key);

__global__ void k_materialize(SolveDev a, const SurvDev* __restrict__ sv,
                              const long long* __restrict__ keys, int64_t n, DevPose* __restrict__ out) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n) return;
  out[t] = materialize_key(a, sv, keys[t]);
}

/// revalidate_solution (src/reach_solver.cpp:458-476) for every solution of
/// a set: the gap band, joint limits, self-collision, every waypoint sample
/// clear of `g`, closure on the target. Counts the failures and keeps the
/// first failing ordinal and its reason (1 band, 2 limits, 3 self, 4 sample,
/// 5 closure).
__global__ void k_revalidate(SolveDev a, const SurvDev* __restrict__ sv,
                             const long long* __restrict__ keys, int64_t n, rpd::GridView g,
                             double total_len, unsigned long long* __restrict__ bad,
                             unsigned long long* __restrict__ first) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const DevPose d = materialize_key(a, sv, keys[t]);
  const ArmDev& arm = a.arm;
  int why = 0;
  if (fabs(rpd::norm(d.seg[2]) - arm.L[2]) > a.eps + 1e-12) why = 1;
  else if (!pose_limits_ok(arm, d)) why = 2;
  else if (!pose_self_free(d, 2.0 * arm.arm_radius)) why = 3;
  if (!why) {
    for (int l = 0; l < d.n_wp_links && !why; ++l) {
      const V3 diff = d.wp_to[l] - d.wp_from[l];
      for (int k = 1; k <= d.n_wp[l]; ++k) {
        int bit = 0;
        const long long w = rpd::cell_word(g, rpd::walk_sample(d.wp_from[l], diff, k, d.n_wp[l]), &bit);
        if (w >= 0 && ((__ldg(g.bits + w) >> bit) & 1ull)) {
          why = 4;
          break;
        }
      }
    }
  }
  if (!why && !(rpd::norm(d.joints[d.nseg] - a.target) <= 1e-9 * fmax(1.0, total_len))) why = 5;
  if (why) {
    atomicAdd(bad, 1ull);
    atomicMin(first, (static_cast<unsigned long long>(t) << 3) | static_cast<unsigned long long>(why));
  }
}

__device__ DevPose materialize_key(const SolveDev& a, const SurvDev* __restrict__ sv, long long key) {
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
  const V3 b = a.bpts[bi];
  DevPose d{};
  d.nseg = a.eight ? 4 : 3;
  d.seg[0] = arm.L[0] * qvec(a, h.i);
  d.seg[1] = arm.L[1] * dir2;
  d.seg[2] = b - p2;
  d.qidx[0] = h.i;
  d.qidx[1] = j;
  d.qidx[2] = -1;
  d.qidx[3] = -1;
  if (a.eight) {
    d.seg[3] = a.L4 * a.bdirs[bi];
    d.qidx[3] = a.bcone[bi];
  }
  build_chain(arm, d);
  d.n_wp_links = a.eight ? 4 : 3;
  d.wp_from[0] = h.link_start; d.wp_to[0] = h.p1;
  d.wp_from[1] = link2;        d.wp_to[1] = p2;
  d.wp_from[2] = p2;           d.wp_to[2] = b;
  d.wp_from[3] = b;            d.wp_to[3] = a.target;
  for (int k = 0; k < 4; ++k) d.n_wp[k] = a.n;
  return d;
}

HostPose host_pose_from_dev(const DevPose& d) {
  HostPose h;
  h.nseg = d.nseg;
  h.has_elbows = d.has_elbows != 0;
  h.no_qidx = d.no_qidx != 0;
  for (int k = 0; k < d.nseg; ++k) {
    h.seg[k] = d.seg[k];
    h.elbows[k] = d.elbows[k];
    h.qidx[k] = d.qidx[k];
  }
  for (int k = 0; k <= d.nseg; ++k) h.joints[k] = d.joints[k];
  h.s4dev = d.s4dev;
  h.waypoints = dev_pose_waypoints(d);
  return h;
}

std::vector<V3> dev_pose_waypoints(const DevPose& d) {
  std::vector<V3> w;
  for (int l = 0; l < d.n_wp_links; ++l) {
    const V3 diff = d.wp_to[l] - d.wp_from[l];
    for (int k = 1; k <= d.n_wp[l]; ++k) w.push_back(rpd::walk_sample(d.wp_from[l], diff, k, d.n_wp[l]));
  }
  return w;
}

static unsigned nblk(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

/// backward_endpoints (src/reach_solver.cpp:54-83).
static void backward_endpoints(rp_ctx* ctx, const rp_quiver* q, V3 target, double L4,
                               const rp_reach_params& rp, std::vector<V3>& pts,
                               std::vector<V3>& dirs, std::vector<int>& cone) {
  const V3 axis{rp.approach_axis[0], rp.approach_axis[1], rp.approach_axis[2]};
  if (rp.mode == RP_MODE_6DOF) {
    pts.push_back(target);
    dirs.push_back(V3{0, 0, 0});
    cone.push_back(-1);
    return;
  }
  if (rp.approach_half_angle == 0.0) {
    require(std::abs(rpd::norm(axis) - 1.0) <= 1e-9, RP_E_INVALID_PARAMETER,
            "approach_axis must be unit");
    pts.push_back(target - L4 * axis);
    dirs.push_back(axis);
    cone.push_back(-1);
    return;
  }
  int32_t cnt = 0;
  std::vector<int32_t> idx(q->n);
  rp_status st = rp_cone_subset(ctx, q, rp.approach_axis, rp.approach_half_angle, idx.data(),
                                q->n, &cnt);
  if (st != RP_OK) throw Fail{st, rp_last_error()};
  require(cnt > 0, RP_E_EMPTY_CONE,
          "no quiver vector inside the approach cone; widen the cone or refine the quiver");
  for (int k = 0; k < cnt; ++k) {
    const int i = idx[k];
    const V3 d{q->host_xyz[3 * i], q->host_xyz[3 * i + 1], q->host_xyz[3 * i + 2]};
    pts.push_back(target - L4 * d);
    dirs.push_back(d);
    cone.push_back(i);
  }
}

/// span_gap (src/reach_solver.cpp:85-98) for one p2 over all backward points:
/// the same coarse + band test k_seg2 inlines.
/// select_solution's argmin over data (rp_select_solution_data): per block
/// the first minimum of its range, then the blocks' in order (strict <, so
/// the lowest index wins ties, as the reference's sequential scan).
__global__ void k_select_data(const V3* __restrict__ segs, int64_t n, const double* __restrict__ scl,
                              int64_t n_sc, BestRec* __restrict__ block_best) {
  double bl = 1e308;
  long long bk = LLONG_MAX;
  const bool sc = n_sc > 0;
  const int64_t count = sc ? n_sc : n;
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < count;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double len = sc ? scl[k]
                          : (rpd::norm(segs[3 * k]) + rpd::norm(segs[3 * k + 1])) +
                                rpd::norm(segs[3 * k + 2]);
    if (len < bl || (len == bl && k < bk)) {
      bl = len;
      bk = k;
    }
  }
  for (int off = 16; off > 0; off >>= 1) {
    const double ol = __shfl_down_sync(FULL, bl, off);
    const long long ok = __shfl_down_sync(FULL, bk, off);
    if (ol < bl || (ol == bl && ok < bk)) {
      bl = ol;
      bk = ok;
    }
  }
  __shared__ BestRec wb[8];
  if ((threadIdx.x & 31) == 0) wb[threadIdx.x >> 5] = BestRec{bl, bk};
  __syncthreads();
  if (threadIdx.x == 0) {
    BestRec r = wb[0];
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w)
      if (wb[w].len < r.len || (wb[w].len == r.len && wb[w].key < r.key)) r = wb[w];
    block_best[blockIdx.x] = r;
  }
}

/// short_reach_scan on one HypothesisScan (src/reach_solver.cpp:176-222):
/// the first sample within near_target_radius + 1e-12 of the target behind a
/// clear prefix, completed by a collision-checked bridge, else by the direct
/// origin -> target segment; path_length = polyline_length(root, prefix +
/// sublength (+ target)) (:157-165). One thread: a scalar chain.
struct ScanArgs {
  rpd::GridView g;
  V3 root, target, origin;
  double near_r, spacing;
  const V3* samples;
  const uint8_t* clear;
  int n;
  const V3* prefix;
  int n_prefix;
  V3* sub;  // out: sublength samples
  int sub_cap;
};
struct ScanOut {
  int found, status, hit, has_bridge, via_direct, n_sub;
  V3 bridge;
  double path_length;
};

__global__ void k_short_reach_scan(ScanArgs a, ScanOut* out) {
  ScanOut r{};
  int hit = 0;
  for (int k = 0; k < a.n; ++k) {
    // loop invariant: samples proximal to k are collision-free
    if (rpd::norm(a.samples[k] - a.target) <= a.near_r + 1e-12) {
      hit = k + 1;
      break;
    }
    if (!a.clear[k]) break;
  }
  if (hit == 0) {
    *out = r;
    return;
  }
  r.hit = hit;
  r.n_sub = hit;
  for (int k = 0; k < hit; ++k) a.sub[k] = a.samples[k];
  const V3 hp = a.samples[hit - 1];
  const double dist = rpd::norm(hp - a.target);
  if (dist > 1e-9) {
    const bool bridge_ok =
        rpd::walk_first_blocked(a.g, hp, a.target, rpd::scaled_sample_count(dist, a.spacing)) == 0;
    if (bridge_ok) {
      r.has_bridge = 1;
      r.bridge = a.target - hp;
    } else {
      const double dl = rpd::norm(a.target - a.origin);
      const int nd = rpd::scaled_sample_count(dl, a.spacing);
      if (nd > a.sub_cap) {
        r.status = 1;
        *out = r;
        return;
      }
      if (rpd::walk_first_blocked(a.g, a.origin, a.target, nd) != 0) {
        *out = r;  // found = 0
        return;
      }
      r.via_direct = 1;
      r.n_sub = nd;
      const V3 dd = a.target - a.origin;
      for (int k = 1; k <= nd; ++k) a.sub[k - 1] = rpd::walk_sample(a.origin, dd, k, nd);
    }
  }
  double acc = 0.0;
  V3 prev = a.root;
  for (int k = 0; k < a.n_prefix; ++k) {
    acc += rpd::norm(a.prefix[k] - prev);
    prev = a.prefix[k];
  }
  for (int k = 0; k < r.n_sub; ++k) {
    acc += rpd::norm(a.sub[k] - prev);
    prev = a.sub[k];
  }
  if (r.has_bridge) acc += rpd::norm(a.target - prev);
  r.path_length = acc;
  r.found = 1;
  *out = r;
}

__global__ void k_span_gap(V3 p2, const V3* __restrict__ bpts, int n, double L3, double eps,
                           V3* __restrict__ v3_out, uint8_t* __restrict__ pass) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const V3 v3 = bpts[k] - p2;
  bool ok = rpd::sqnorm(v3) <= (L3 + eps) * (L3 + eps) * (1.0 + 1e-12);
  if (ok) ok = !(fabs(rpd::norm(v3) - L3) > eps);
  v3_out[k] = v3;
  pass[k] = ok ? 1 : 0;
}

static HostShortcut host_shortcut(const rp_solution_set* s, const ShortcutRec& r) {
  const SolveDev& a = s->sd;
  const ArmDev& arm = a.arm;
  const std::vector<double>& qx = s->quiver->host_xyz;
  auto q = [&](int i) { return V3{qx[3 * i], qx[3 * i + 1], qx[3 * i + 2]}; };
  HostShortcut h;
  h.segment_index = r.segment_index;
  h.seg1 = r.seg1;
  h.seg2 = r.seg2;
  h.hit = r.hit;
  h.has_bridge = r.has_bridge != 0;
  h.via_direct = r.via_direct != 0;
  h.bridge = r.bridge;
  h.path_length = r.path_length;
  const V3 d1 = q(r.seg1);
  V3 link1 = arm.root;
  rpd::FrameStep st{};
  if (arm.any_limit || arm.has_offsets) st = rpd::advance_frame(arm.base, d1);
  if (arm.off[0] > 0.0) link1 = arm.root + arm.off[0] * rpd::m_col(st.after_azimuth, 0);
  const V3 p1 = link1 + arm.L[0] * d1;
  V3 link = link1, end = p1;
  DevPose basis{};
  basis.seg[0] = arm.L[0] * d1;
  basis.qidx[0] = r.seg1;
  basis.nseg = 1;
  if (r.segment_index == 2) {
    const V3 d2 = q(r.seg2);
    link = p1;
    if (arm.off[1] > 0.0) {
      const rpd::FrameStep st2 = rpd::advance_frame(st.frame, d2);
      link = p1 + arm.off[1] * rpd::m_col(st2.after_azimuth, 0);
    }
    end = link + arm.L[1] * d2;
    const V3 pd = p1 - link1;
    for (int k = 1; k <= a.n; ++k) h.prefix.push_back(rpd::walk_sample(link1, pd, k, a.n));
    basis.seg[1] = arm.L[1] * d2;
    basis.qidx[1] = r.seg2;
    basis.nseg = 2;
  }
  if (h.via_direct) {
    const V3 dd = a.target - r.origin;
    for (int k = 1; k <= r.n_direct; ++k)
      h.sublength.push_back(rpd::walk_sample(r.origin, dd, k, r.n_direct));
  } else {
    const V3 diff = end - link;
    for (int k = 1; k <= r.hit; ++k) h.sublength.push_back(rpd::walk_sample(link, diff, k, a.n));
  }
  build_chain(arm, basis);
  basis.n_wp_links = 0;
  h.basis = host_pose_from_dev(basis);
  return h;
}

/// Bracket half-width (cells) of rpd::walk_hits_affine for walks between
/// points the arm reaches: every such point lies within Rw = max |root - o|
/// + sum(L) + sum(|off|) of the grid origin per axis, so M = 2 Rw / vs bounds
/// |A|, t |B| and |q| and P = (max |o| + 2 Rw) / vs the absolute coordinate;
/// the error bound ~9u M + u P is covered 8x, plus the grid's own dq.
double affine_bracket(const rpd::GridView& g, const rp_arm& arm) {
  double rw = std::max({std::fabs(arm.root[0] - g.ox), std::fabs(arm.root[1] - g.oy),
                        std::fabs(arm.root[2] - g.oz)});
  for (int k = 0; k < arm.n_segments && k < RP_MAX_SEGMENTS; ++k)
    rw += std::fabs(arm.lengths[k]) + (k < arm.n_offsets ? std::fabs(arm.offsets[k]) : 0.0);
  const double M = 2.0 * rw / g.vs;
  const double P = (std::max({std::fabs(g.ox), std::fabs(g.oy), std::fabs(g.oz)}) + 2.0 * rw) / g.vs;
  const double u = 1.1102230246251565e-16;
  return 8.0 * u * (9.0 * M + P + 4.0) + g.dq;
}

rp_solution_set* solve_reach(rp_ctx* ctx, const rp_arm& arm, const rp_quiver* q, const rp_grid* g,
                             V3 target, const rp_reach_params& rp, int part, int parts) {
  HostSpan span_("solve_reach");
  require(parts >= 1 && part >= 0 && part < parts, RP_E_INVALID_PARAMETER,
          "part must be in [0, parts)");
  validate_arm(arm);
  validate_reach(rp);
  if (rp.mode == RP_MODE_8DOF) {
    require(arm.n_segments == 4, RP_E_INVALID_PARAMETER, "8DOF solve needs 4 segments");
  } else {
    require(arm.n_segments >= 3, RP_E_INVALID_PARAMETER, "6DOF solve needs 3 segments");
  }
  const double off2 = arm.n_offsets > 2 ? arm.offsets[2] : 0.0;
  const double off3 = arm.n_offsets > 3 ? arm.offsets[3] : 0.0;
  require(off2 == 0.0 && off3 == 0.0, RP_E_INVALID_PARAMETER,
          "reach solving supports joint offsets at joints 1 and 2 only");
  require(q && g && ctx_shares(ctx, q->ctx) && ctx_shares(ctx, g->ctx), RP_E_INVALID_PARAMETER,
          "quiver / grid belong to another context");

  auto* s = new rp_solution_set();
  try {
    s->ctx = ctx;
    s->quiver = q;
    s->arm = arm;
    s->rp = rp;
    s->target[0] = target.x;
    s->target[1] = target.y;
    s->target[2] = target.z;
    cudaStream_t st = ctx->stream;
    const bool eight = rp.mode == RP_MODE_8DOF;
    const double L4 = eight ? arm.lengths[3] : 0.0;
    backward_endpoints(ctx, q, target, L4, rp, s->h_bpts, s->h_bdirs, s->h_bcone);
    s->B = static_cast<int>(s->h_bpts.size());

    SolveDev& a = s->sd;
    a.g = g->view();
    a.arm = make_arm_dev(arm);
    a.n = rp.n_samples;
    a.eight = eight ? 1 : 0;
    a.Q = q->n;
    a.B = s->B;
    a.scanning = 1;
    a.cone_precheck = rp.cone_precheck;
    a.disable_prune = rp.disable_geom_pruning;
    const double eps = resolved_epsilon(arm, rp);
    const double L3 = arm.lengths[2];
    a.eps = eps;
    a.coarse2 = (L3 + eps) * (L3 + eps) * (1.0 + 1e-12);
    a.band_lo2 = L3 - eps > 0.0 ? (L3 - eps) * (L3 - eps) * (1.0 - 1e-9) : 0.0;
    a.dq_aff = affine_bracket(a.g, arm);
    double budget = arm.lengths[1] + arm.lengths[2] + eps;
    if (eight) budget += arm.lengths[3];
    budget += 1e-9;
    a.budget2 = budget * budget;
    a.near_r = resolved_near_radius(arm, rp);
    a.spacing = nominal_spacing(arm, rp);
    a.L4 = L4;
    a.target = target;
    a.qx = q->d_soa;
    a.qy = q->d_soa + q->n;
    a.qz = q->d_soa + 2 * static_cast<size_t>(q->n);
    {
      // the backward points, directions, cone indices and the target in one
      // device block and one upload: [bpts][bdirs][target][bcone][walk4]
      const size_t nb = s->B + 1;
      const size_t o_dirs = nb * sizeof(V3), o_tg = 2 * nb * sizeof(V3);
      const size_t o_cone = o_tg + sizeof(V3), o_w4 = o_cone + nb * sizeof(int);
      const size_t bytes = o_w4 + nb;
      s->bblock.alloc(bytes, st);
      std::vector<unsigned char> h(o_w4, 0);
      std::memcpy(h.data(), s->h_bpts.data(), s->B * sizeof(V3));
      std::memcpy(h.data() + o_dirs, s->h_bdirs.data(), s->B * sizeof(V3));
      std::memcpy(h.data() + o_tg, &target, sizeof(V3));
      std::memcpy(h.data() + o_cone, s->h_bcone.data(), s->B * sizeof(int));
      copy_to_device(ctx, s->bblock.p, h.data(), o_w4);
      a.bpts = reinterpret_cast<V3*>(s->bblock.p);
      a.bdirs = reinterpret_cast<V3*>(s->bblock.p + o_dirs);
      a.targets = reinterpret_cast<V3*>(s->bblock.p + o_tg);
      a.bcone = reinterpret_cast<int*>(s->bblock.p + o_cone);
      a.walk4_ok = s->bblock.p + o_w4;
    }
    a.n_targets = 1;
    if (eight)
      launch(ctx, "walk4", k_walk4, dim3(nblk(s->B, 128)), dim3(128), 0, a,
             const_cast<uint8_t*>(a.walk4_ok));

    // the solve's temporaries in the context's scratch block (one
    // allocation kept across solves; stream order protects reuse): counters
    // and flags first, zeroed by one memset
    const int qwords = (q->n + 31) / 32;
    ScratchCarver sk;
    const size_t o_ctr = sk.reserve<unsigned long long>(C_COUNT);
    const size_t o_scc = sk.reserve<unsigned>(1);
    const size_t o_uc = sk.reserve<int>(1);
    const size_t o_sv = sk.reserve<int>(1);
    const size_t zero_bytes = sk.off;
    const size_t o_scl = sk.reserve<long long>(kShortcutCap);
    const size_t o_sb = sk.reserve<uint32_t>(qwords);
    const size_t o_bb = sk.reserve<BestRec>(static_cast<size_t>(ctx->sm_count) * 8);
    const size_t o_best = sk.reserve<BestRec>(1);
    const size_t o_ks = sk.reserve<uint8_t>(std::max(1, q->n));
    const size_t o_ke = sk.reserve<uint8_t>(1);
    sk.bind(ctx_scratch(ctx, sk.off));
    auto* ctr = sk.at<unsigned long long>(o_ctr);
    auto* sc_count = sk.at<unsigned>(o_scc);
    auto* unit_ctr = sk.at<int>(o_uc);
    auto* surv_cnt = sk.at<int>(o_sv);
    auto* sc_list = sk.at<long long>(o_scl);
    auto* surv_bits = sk.at<uint32_t>(o_sb);
    auto* bb = sk.at<BestRec>(o_bb);
    auto* best = sk.at<BestRec>(o_best);
    auto* kskip = sk.at<uint8_t>(o_ks);
    auto* kend_b = sk.at<uint8_t>(o_ke);
    RP_CUDA(cudaMemsetAsync(sk.base, 0, zero_bytes, st));
    launch(ctx, "seg1", k_seg1, dim3(nblk(q->n, 256)), dim3(256), 0, a, surv_bits, ctr,
           sc_list, sc_count);
    DevBuf<int> surv_idx(q->n + 1, st);
    launch(ctx, "compact", k_compact_small, dim3(1), dim3(1024), 0,
           static_cast<const uint32_t*>(surv_bits), q->n, surv_idx.p, surv_cnt);
    const bool B1 = s->B == 1;
    const bool general = a.arm.any_limit || a.arm.has_offsets || (rp.cone_precheck && eight);
    static const bool flat = std::getenv("RP_SEG2_FLAT") != nullptr;
    // The row kernel (default arms, one backward point) runs without a host
    // read-back between the prune and segment 2: buffers are sized for
    // S1 <= Q and the kernels read S1 on the device; the count and the
    // survivor list come back with the solve's counters. The flat kernel
    // (limits, offsets, cones) and quivers past 16384 directions (whose Q^2
    // bit set would be large) read S1 first.
    const bool rows_kernel = !general && B1 && !flat;
    const bool sync_free = rows_kernel && q->n <= 16384;
    int S1 = 0;
    std::vector<int> surv_all(q->n);
    if (!sync_free)
      copy_to_host_many(ctx, {{&S1, surv_cnt, sizeof(int)},
                              {surv_all.data(), surv_idx.p, q->n * sizeof(int)}});
    const int cap_rows = sync_free ? q->n : S1;
    s->surv.alloc(cap_rows + 1, st);
    if (cap_rows > 0)
      launch(ctx, "seg1", k_surv_data, dim3(nblk(cap_rows, 128)), dim3(128), 0, a,
             static_cast<const int*>(surv_idx.p), static_cast<const int*>(surv_cnt), s->surv.p);
    // this part's survivor rows (the whole set for parts == 1); the pair and
    // key indices stay global, so parts' keys concatenate in canonical order
    int s_lo = static_cast<int>(static_cast<int64_t>(S1) * part / parts);
    int s_hi = static_cast<int>(static_cast<int64_t>(S1) * (part + 1) / parts);
    s->part = part;
    s->parts = parts;
    if (part != 0)  // segment-1 hypotheses belong to part 0
      RP_CUDA(cudaMemsetAsync(sc_count, 0, sizeof(unsigned), st));

    s->n_pairs = static_cast<int64_t>(cap_rows) * q->n;  // exact once S1 is known
    const int64_t nbits = s->n_pairs * s->B;
    const int64_t nwords = (nbits + 31) / 32 + 1;
    s->sol_bits.alloc(nwords, st);
    if (!B1 || parts > 1) s->sol_bits.zero();
    const int threads = 256;
    int blocks = ctx->sm_count * 8;
    const int64_t p_lo = static_cast<int64_t>(s_lo) * q->n, p_hi = static_cast<int64_t>(s_hi) * q->n;
    const int64_t need = (p_hi - p_lo + threads - 1) / threads;
    if (!rows_kernel && need < blocks) blocks = static_cast<int>(std::max<int64_t>(1, need));
    if (sync_free || p_hi > p_lo) {
      auto run = [&](auto kern) {
        launch(ctx, "seg2", kern, dim3(blocks), dim3(threads), 0, a,
               static_cast<const SurvDev*>(s->surv.p), p_lo, p_hi, s->sol_bits.p, ctr,
               sc_list, sc_count, bb);
      };
      if (rows_kernel) {
        s->sol_bits.zero();
        const int64_t units = static_cast<int64_t>(cap_rows) * ((q->n + 1023) / 1024);
        const int rblocks = static_cast<int>(
            std::max<int64_t>(1, std::min<int64_t>(ctx->sm_count * 8, (units + 7) / 8)));
        // free leading samples per row (k_row_skip) and trailing samples of
        // the v3 walks (k_tail_skip) from the grid's cached clearance field
        static const bool no_skip = std::getenv("RP_NO_ROW_SKIP") != nullptr;
        if (no_skip) {
          RP_CUDA(cudaMemsetAsync(kskip, 0, std::max(1, cap_rows), st));
          RP_CUDA(cudaMemsetAsync(kend_b, rp.n_samples, 1, st));
        } else {
          const ClearanceField cf = grid_clearance_field(g, ctx);
          launch(ctx, "seg2", k_row_skip, dim3(nblk(std::max(1, cap_rows), 128)), dim3(128), 0, a,
                 static_cast<const SurvDev*>(s->surv.p), static_cast<const int*>(surv_cnt), cf,
                 kskip);
          launch(ctx, "seg2", k_tail_skip, dim3(1), dim3(32), 0, a.g,
                 static_cast<const V3*>(a.bpts), 1, L3 + eps, rp.n_samples, cf, kend_b);
        }
        uint32_t* c2bits = nullptr;
        uint8_t* c2ok = nullptr;
        const uint32_t* c2bits_r = nullptr;
        const uint8_t* c2ok_r = nullptr;
        V3 ov_lo{1, 1, 1}, ov_hi{-1, -1, -1};
        if (!grid_seg2_base_cache(g, q, arm, rp.n_samples, &c2bits_r, &c2ok_r, &ov_lo, &ov_hi) &&
            !grid_seg2_cache(g, q, arm, rp.n_samples, &c2bits, &c2ok))
          c2bits = nullptr, c2ok = nullptr;
        auto runr = [&](auto kern) {
          launch(ctx, "seg2", kern, dim3(rblocks), dim3(threads), 0, a,
                 static_cast<const SurvDev*>(s->surv.p), static_cast<const int*>(surv_cnt), part,
                 parts, s->sol_bits.p, ctr, sc_list,
                 sc_count, bb, unit_ctr, static_cast<const uint8_t*>(kskip),
                 static_cast<const uint8_t*>(kend_b), c2bits, c2ok, c2bits_r, c2ok_r, ov_lo,
                 ov_hi);
        };
        if (c2ok_r)
          eight ? runr(k_seg2_rows<true, true>) : runr(k_seg2_rows<false, true>);
        else
          eight ? runr(k_seg2_rows<true, false>) : runr(k_seg2_rows<false, false>);
        blocks = rblocks;
      } else if (eight) {
        if (general) B1 ? run(k_seg2<true, true, true>) : run(k_seg2<true, true, false>);
        else B1 ? run(k_seg2<true, false, true>) : run(k_seg2<true, false, false>);
      } else {
        if (general) B1 ? run(k_seg2<false, true, true>) : run(k_seg2<false, true, false>);
        else B1 ? run(k_seg2<false, false, true>) : run(k_seg2<false, false, false>);
      }
      launch(ctx, "select", k_best_final, dim3(1), dim3(256), 0,
             static_cast<const BestRec*>(bb), blocks, best);
    }
    unsigned long long hc[C_COUNT];
    unsigned nsc = 0;
    BestRec hb{0.0, -1};
    if (sync_free) {
      // the solve's one read-back: counters, shortcut count, best, S1 and
      // the survivor list
      // (the survivor list stays on the device until rp_solution_set_keys)
      copy_to_host_many(ctx, {{hc, ctr, sizeof(hc)},
                              {&nsc, sc_count, sizeof(unsigned)},
                              {&hb, best, sizeof(BestRec)},
                              {&S1, surv_cnt, sizeof(int)}});
      s_lo = static_cast<int>(static_cast<int64_t>(S1) * part / parts);
      s_hi = static_cast<int>(static_cast<int64_t>(S1) * (part + 1) / parts);
      s->n_pairs = static_cast<int64_t>(S1) * q->n;
    } else {
      copy_to_host_many(ctx, {{hc, ctr, sizeof(hc)},
                              {&nsc, sc_count, sizeof(unsigned)},
                              {&hb, best, p_hi > p_lo ? sizeof(BestRec) : 0}});
    }
    s->S1 = S1;
    if (!sync_free) {
      s->surv_i.assign(surv_all.begin(), surv_all.begin() + S1);
      s->surv_i_ready = true;
    }
    s->surv_idx_d = std::move(surv_idx);
    require(nsc <= kShortcutCap, RP_E_CAPACITY_EXCEEDED, "too many near-encounter hypotheses");

    rp_solve_stats& S = s->stats;
    std::memset(&S, 0, sizeof(S));
    S.seg1_candidates = q->n;
    S.seg1_limit_pass = hc[C_SEG1_LIMIT];
    S.seg1_reach_pass = hc[C_SEG1_REACH];
    S.seg1_survivors = hc[C_SEG1_SURV];
    S.pair_candidates = static_cast<int64_t>(s_hi - s_lo) * q->n;
    S.seg2_limit_pass = hc[C_SEG2_LIMIT];
    S.seg2_clear_pass = hc[C_SEG2_CLEAR];
    S.gap_tested = hc[C_GAP_TESTED];
    S.gap_pass = hc[C_GAP_PASS];
    S.joint_pass = hc[C_JOINT_PASS];
    S.v3_clear_pass = hc[C_V3_CLEAR];
    S.solutions = hc[C_SOLUTIONS];
    s->n_solutions = S.solutions;
    s->best_key = S.solutions > 0 ? hb.key : -1;
    s->best_len = hb.len;

    if (nsc > 0) {
      DevBuf<long long> sorted(nsc, st);
      size_t tmp_bytes = 0;
      cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, sc_list, sorted.p, static_cast<int>(nsc),
                                     0, 64, st);
      DevBuf<unsigned char> tmp(tmp_bytes, st);
      RP_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tmp_bytes, sc_list, sorted.p,
                                             static_cast<int>(nsc), 0, 64, st));
      DevBuf<ShortcutRec> recs(nsc, st);
      launch(ctx, "shortcuts", k_shortcuts, dim3(nblk(nsc, 128)), dim3(128), 0, a,
             static_cast<const SurvDev*>(s->surv.p), static_cast<const long long*>(sorted.p),
             static_cast<int>(nsc), recs.p);
      std::vector<ShortcutRec> h(nsc);
      copy_to_host(ctx, h.data(), recs.p, nsc * sizeof(ShortcutRec));
      for (const auto& r : h)
        if (r.valid) s->shortcuts.push_back(host_shortcut(s, r));
    }
    S.shortcuts_found = static_cast<int64_t>(s->shortcuts.size());
    // RP_REVALIDATE=1: the reference's merge-time self-check of every
    // solution (src/reach_solver.cpp:537-540), raising as it does
    static const bool reval = std::getenv("RP_REVALIDATE") != nullptr;
    if (reval) {
      static const char* what[] = {"", "internal: solution violates the gap band",
                                   "internal: solution violates joint limits",
                                   "internal: solution self-collides",
                                   "internal: solution sample inside an obstacle",
                                   "internal: solution does not close on the target"};
      const RevalidateOut r = revalidate(s, nullptr);
      if (r.n_bad) fail(RP_E_NO_SOLUTION, what[r.reason]);
    }
  } catch (...) {
    delete s;
    throw;
  }
  return s;
}

void ensure_keys(rp_solution_set* s) {
  HostSpan span_("ensure_keys");
  if (s->keys_ready) return;
  rp_ctx* ctx = s->ctx;
  cudaStream_t st = ctx->stream;
  s->keys.alloc(s->n_solutions + 1, st);
  if (s->n_solutions > 0) {
    const int64_t nw = (s->n_pairs * s->B + 31) / 32;
    DevBuf<unsigned long long> cnt(nw, st), off(nw, st);
    launch(ctx, "compact", k_word_popc, dim3(nblk(nw, 256)), dim3(256), 0,
           static_cast<const uint32_t*>(s->sol_bits.p), nw, cnt.p);
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.p, off.p, nw, st);
    DevBuf<unsigned char> tmp(tb, st);
    RP_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, cnt.p, off.p, nw, st));
    launch(ctx, "compact", k_scatter_bits, dim3(nblk(nw, 256)), dim3(256), 0,
           static_cast<const uint32_t*>(s->sol_bits.p), nw,
           static_cast<const unsigned long long*>(off.p), s->keys.p);
  }
  s->keys_ready = true;
}

void materialize_solutions(rp_solution_set* s, const long long* d_keys, const long long* h_keys,
                           int64_t n, DevPose* d_out) {
  if (n <= 0) return;
  DevBuf<long long> tmp;
  const long long* keys = d_keys;
  if (!keys) {
    tmp.alloc(n, s->ctx->stream);
    copy_to_device(s->ctx, tmp.p, h_keys, n * sizeof(long long));
    keys = tmp.p;
  }
  launch(s->ctx, "materialize", k_materialize, dim3(nblk(n, 128)), dim3(128), 0, s->sd,
         static_cast<const SurvDev*>(s->surv.p), keys, n, d_out);
}

static long long key_of_ordinal(rp_solution_set* s, int64_t ordinal) {
  ensure_keys(s);
  long long key = 0;
  copy_to_host(s->ctx, &key, s->keys.p + ordinal, sizeof(long long));
  return key;
}

DevPose solution_dev_pose_by_key(rp_solution_set* s, long long key) {
  DevBuf<DevPose> d(1, s->ctx->stream);
  materialize_solutions(s, nullptr, &key, 1, d.p);
  DevPose h;
  copy_to_host(s->ctx, &h, d.p, sizeof(DevPose));
  return h;
}

DevPose solution_dev_pose(rp_solution_set* s, int64_t ordinal) {
  return solution_dev_pose_by_key(s, key_of_ordinal(s, ordinal));
}

HostPose solution_pose(rp_solution_set* s, int64_t ordinal) {
  return host_pose_from_dev(solution_dev_pose(s, ordinal));
}

void launch_rank_of_key(const rp_solution_set* s, long long key, unsigned long long* d_rank) {
  RP_CUDA(cudaMemsetAsync(d_rank, 0, sizeof(unsigned long long), s->ctx->stream));
  launch(s->ctx, "select", k_rank, dim3(s->ctx->sm_count), dim3(256), 0,
         static_cast<const uint32_t*>(s->sol_bits.p), key, d_rank);
}

static int64_t rank_of_key(const rp_solution_set* s, long long key) {
  DevBuf<unsigned long long> c(1, s->ctx->stream);
  c.zero();
  launch(s->ctx, "select", k_rank, dim3(s->ctx->sm_count), dim3(256), 0,
         static_cast<const uint32_t*>(s->sol_bits.p), key, c.p);
  unsigned long long h = 0;
  copy_to_host(s->ctx, &h, c.p, sizeof(h));
  return static_cast<int64_t>(h);
}

RevalidateOut revalidate(rp_solution_set* s, const rp_grid* grid) {
  HostSpan span_("revalidate");
  RevalidateOut r;
  if (s->n_solutions == 0) return r;
  ensure_keys(s);
  rp_ctx* ctx = s->ctx;
  DevBuf<unsigned long long> out(2, ctx->stream);
  const unsigned long long init[2] = {0ull, ~0ull};
  copy_to_device(ctx, out.p, init, sizeof(init));
  double total = 0.0;
  for (int k = 0; k < s->arm.n_segments; ++k) total += s->arm.lengths[k];
  launch(ctx, "revalidate", k_revalidate, dim3(static_cast<unsigned>((s->n_solutions + 127) / 128)),
         dim3(128), 0, s->sd, static_cast<const SurvDev*>(s->surv.p),
         static_cast<const long long*>(s->keys.p), s->n_solutions,
         grid ? grid->view() : s->sd.g, total, out.p, out.p + 1);
  unsigned long long h[2];
  copy_to_host(ctx, h, out.p, sizeof(h));
  r.n_bad = static_cast<int64_t>(h[0]);
  if (h[0]) {
    r.first = static_cast<int64_t>(h[1] >> 3);
    r.reason = static_cast<int>(h[1] & 7);
  }
  return r;
}

rp_chosen select(const rp_solution_set* s) {
  require(s->n_solutions > 0 || !s->shortcuts.empty(), RP_E_NO_SOLUTION,
          "no reach solution under the given constraints");
  rp_chosen c{};
  if (!s->shortcuts.empty()) {
    size_t best = 0;
    for (size_t k = 1; k < s->shortcuts.size(); ++k)
      if (s->shortcuts[k].path_length < s->shortcuts[best].path_length) best = k;
    c.kind = RP_CHOSEN_SHORTCUT;
    c.index = static_cast<int64_t>(best);
    c.path_length = s->shortcuts[best].path_length;
    return c;
  }
  c.kind = RP_CHOSEN_REACH_POSE;
  c.index = rank_of_key(s, s->best_key);
  c.path_length = s->best_len;
  return c;
}

}  // namespace rp

using namespace rp;

extern "C" {

rp_status rp_cone_subset(rp_ctx* ctx, const rp_quiver* q, const double axis[3], double half,
                         int32_t* idx, int32_t cap, int32_t* n_out) {
  return guarded([&] {
    const V3 ax{axis[0], axis[1], axis[2]};
    require(std::abs(rpd::norm(ax) - 1.0) <= 1e-9, RP_E_INVALID_PARAMETER,
            "cone axis must be unit");
    require(half >= 0.0 && half <= 3.14159265358979323846, RP_E_INVALID_PARAMETER,
            "half_angle must be in [0, pi]");
    const double limit = half + 1e-12;
    DevBuf<uint8_t> in(q->n, ctx->stream), amb(q->n, ctx->stream);
    launch(ctx, "cone", k_cone, dim3(nblk(q->n, 256)), dim3(256), 0,
           static_cast<const double*>(q->d_soa), static_cast<const double*>(q->d_soa + q->n),
           static_cast<const double*>(q->d_soa + 2 * static_cast<size_t>(q->n)), q->n, ax, limit,
           in.p, amb.p);
    std::vector<uint8_t> hin(q->n), hamb(q->n);
    copy_to_host(ctx, hin.data(), in.p, q->n);
    copy_to_host(ctx, hamb.data(), amb.p, q->n);
    int32_t cnt = 0;
    for (int i = 0; i < q->n; ++i) {
      bool inside = hin[i] != 0;
      if (hamb[i]) {  // within 1e-9 rad of the boundary: decide with glibc atan2
        const V3 v{q->host_xyz[3 * i], q->host_xyz[3 * i + 1], q->host_xyz[3 * i + 2]};
        inside = std::atan2(rpd::norm(rpd::cross(v, ax)), rpd::dot(v, ax)) <= limit;
      }
      if (inside) {
        if (cnt < cap) idx[cnt] = i;
        ++cnt;
      }
    }
    *n_out = cnt;
  });
}

rp_status rp_prune_segment1(rp_ctx* ctx, const rp_arm* arm, const rp_quiver* q, const rp_grid* g,
                            const double* targets, int32_t n_targets, const rp_reach_params* rp,
                            int32_t* survivors, int32_t cap, int32_t* n_out,
                            rp_solve_stats* stats) {
  return guarded([&] {
    cudaStream_t st = ctx->stream;
    SolveDev a{};
    a.g = g->view();
    a.arm = make_arm_dev(*arm);
    a.n = rp->n_samples;
    a.eight = rp->mode == RP_MODE_8DOF;
    a.Q = q->n;
    a.disable_prune = rp->disable_geom_pruning;
    const double eps = resolved_epsilon(*arm, *rp);
    double budget = arm->lengths[1] + arm->lengths[2] + eps;
    if (a.eight) budget += arm->lengths[3];
    budget += 1e-9;
    a.budget2 = budget * budget;
    a.spacing = nominal_spacing(*arm, *rp);
    a.near_r = resolved_near_radius(*arm, *rp);
    a.qx = q->d_soa;
    a.qy = q->d_soa + q->n;
    a.qz = q->d_soa + 2 * static_cast<size_t>(q->n);
    DevBuf<V3> tg(std::max(1, n_targets), st);
    copy_to_device(ctx, tg.p, targets, n_targets * sizeof(V3));
    a.targets = tg.p;
    a.n_targets = n_targets;
    a.scanning = 0;
    DevBuf<unsigned long long> ctr(C_COUNT, st);
    ctr.zero();
    DevBuf<unsigned> scc(1, st);
    scc.zero();
    DevBuf<long long> scl(1, st);
    DevBuf<uint32_t> bits((q->n + 31) / 32, st);
    launch(ctx, "seg1", k_seg1, dim3(nblk(q->n, 256)), dim3(256), 0, a, bits.p, ctr.p, scl.p,
           scc.p);
    DevBuf<int> idx(q->n + 1, st), cnt(1, st);
    launch(ctx, "compact", k_compact_small, dim3(1), dim3(1024), 0,
           static_cast<const uint32_t*>(bits.p), q->n, idx.p, cnt.p);
    int S1 = 0;
    copy_to_host(ctx, &S1, cnt.p, sizeof(int));
    std::vector<int> h(S1);
    copy_to_host(ctx, h.data(), idx.p, S1 * sizeof(int));
    for (int k = 0; k < S1 && k < cap; ++k) survivors[k] = h[k];
    *n_out = S1;
    if (stats) {
      unsigned long long hc[C_COUNT];
      copy_to_host(ctx, hc, ctr.p, sizeof(hc));
      std::memset(stats, 0, sizeof(*stats));
      stats->seg1_candidates = q->n;
      stats->seg1_limit_pass = hc[C_SEG1_LIMIT];
      stats->seg1_reach_pass = hc[C_SEG1_REACH];
      stats->seg1_survivors = hc[C_SEG1_SURV];
    }
  });
}

rp_status rp_solve_reach(rp_ctx* ctx, const rp_arm* arm, const rp_quiver* q, const rp_grid* g,
                         const double target[3], const rp_reach_params* rp, rp_solution_set** out) {
  return guarded([&] {
    *out = solve_reach(ctx, *arm, q, g, V3{target[0], target[1], target[2]}, *rp);
  });
}

rp_status rp_solve_reach_part(rp_ctx* ctx, const rp_arm* arm, const rp_quiver* q,
                              const rp_grid* g, const double target[3], const rp_reach_params* rp,
                              int32_t part, int32_t parts, rp_solution_set** out) {
  return guarded([&] {
    *out = solve_reach(ctx, *arm, q, g, V3{target[0], target[1], target[2]}, *rp, part, parts);
  });
}

rp_status rp_solution_set_revalidate(rp_solution_set* s, const rp_grid* grid, int64_t* n_bad,
                                     int64_t* first_bad, int32_t* reason) {
  return guarded([&] {
    const RevalidateOut r = revalidate(s, grid);
    if (n_bad) *n_bad = r.n_bad;
    if (first_bad) *first_bad = r.first;
    if (reason) *reason = r.reason;
  });
}

rp_status rp_solution_set_stats(const rp_solution_set* s, rp_solve_stats* stats) {
  return guarded([&] { *stats = s->stats; });
}

rp_status rp_solution_set_sizes(const rp_solution_set* s, int64_t* ns, int64_t* nc) {
  return guarded([&] {
    if (ns) *ns = s->n_solutions;
    if (nc) *nc = static_cast<int64_t>(s->shortcuts.size());
  });
}

/// The segment-1 quiver index of every survivor row (read back on first use).
static const std::vector<int>& surv_i_of(rp_solution_set* s) {
  if (!s->surv_i_ready) {
    s->surv_i.assign(s->S1, 0);
    if (s->S1 > 0) copy_to_host(s->ctx, s->surv_i.data(), s->surv_idx_d.p, s->S1 * sizeof(int));
    s->surv_i_ready = true;
  }
  return s->surv_i;
}

rp_status rp_solution_set_keys(const rp_solution_set* cs, int32_t* keys, int64_t cap) {
  return guarded([&] {
    auto* s = const_cast<rp_solution_set*>(cs);
    ensure_keys(s);
    const int64_t n = std::min<int64_t>(cap, s->n_solutions);
    std::vector<long long> k(n);
    copy_to_host(s->ctx, k.data(), s->keys.p, n * sizeof(long long));
    for (int64_t t = 0; t < n; ++t) {
      const long long p = k[t] / s->B;
      const int bi = static_cast<int>(k[t] - p * s->B);
      const int sidx = static_cast<int>(p / s->sd.Q);
      keys[3 * t] = surv_i_of(s)[sidx];
      keys[3 * t + 1] = static_cast<int>(p - static_cast<long long>(sidx) * s->sd.Q);
      keys[3 * t + 2] = s->sd.eight ? s->h_bcone[bi] : -1;
    }
  });
}

rp_status rp_solution_set_pose(const rp_solution_set* cs, int64_t k, rp_pose* pose, double* wps,
                               int32_t cap) {
  return guarded([&] {
    auto* s = const_cast<rp_solution_set*>(cs);
    require(k >= 0 && k < s->n_solutions, RP_E_INVALID_PARAMETER, "solution index out of range");
    to_abi(solution_pose(s, k), pose, wps, cap);
  });
}

rp_status rp_solution_set_poses(const rp_solution_set* cs, int64_t first, int64_t count,
                                rp_pose* poses, double* wps, int32_t wps_per_pose) {
  return guarded([&] {
    auto* s = const_cast<rp_solution_set*>(cs);
    require(first >= 0 && count >= 0 && first + count <= s->n_solutions, RP_E_INVALID_PARAMETER,
            "solution range out of bounds");
    if (count == 0) return;
    ensure_keys(s);
    constexpr int64_t kChunk = 1 << 16;
    DevBuf<DevPose> d(std::min(count, kChunk), s->ctx->stream);
    std::vector<DevPose> h(std::min(count, kChunk));
    for (int64_t c0 = 0; c0 < count; c0 += kChunk) {
      const int64_t n = std::min(kChunk, count - c0);
      materialize_solutions(s, s->keys.p + first + c0, nullptr, n, d.p);
      copy_to_host(s->ctx, h.data(), d.p, n * sizeof(DevPose));
      for (int64_t k = 0; k < n; ++k)
        to_abi(host_pose_from_dev(h[k]), poses + c0 + k,
               wps ? wps + (c0 + k) * 3 * static_cast<int64_t>(wps_per_pose) : nullptr,
               wps ? wps_per_pose : 0);
    }
  });
}

rp_status rp_backward_endpoints(rp_ctx* ctx, const rp_quiver* q, const double target[3], double L4,
                                const rp_reach_params* rp, double* points, double* dirs,
                                int32_t* cone_idx, int32_t cap, int32_t* n_out) {
  return guarded([&] {
    std::vector<V3> pts, ds;
    std::vector<int> cone;
    backward_endpoints(ctx, q, V3{target[0], target[1], target[2]}, L4, *rp, pts, ds, cone);
    require(static_cast<int>(pts.size()) <= cap, RP_E_CAPACITY_EXCEEDED,
            "backward endpoint buffer too small");
    *n_out = static_cast<int32_t>(pts.size());
    for (size_t k = 0; k < pts.size(); ++k) {
      std::memcpy(points + 3 * k, &pts[k], sizeof(V3));
      if (dirs) std::memcpy(dirs + 3 * k, &ds[k], sizeof(V3));
      if (cone_idx) cone_idx[k] = cone[k];
    }
  });
}

rp_status rp_select_solution_data(rp_ctx* ctx, const double* segments, int64_t n,
                                  const double* shortcut_lengths, int64_t n_sc, rp_chosen* out) {
  return guarded([&] {
    require(n >= 0 && n_sc >= 0, RP_E_INVALID_PARAMETER, "negative count");
    require(n + n_sc > 0, RP_E_NO_SOLUTION, "no reach solution under the given constraints");
    cudaStream_t st = ctx->stream;
    const int64_t count = n_sc > 0 ? n_sc : n;
    const int blocks = static_cast<int>(std::min<int64_t>(nblk(count, 256), 4 * ctx->sm_count));
    DevBuf<V3> ds(n_sc > 0 ? 1 : 3 * n, st);
    DevBuf<double> dl(std::max<int64_t>(1, n_sc), st);
    DevBuf<BestRec> bb(blocks, st), best(1, st);
    if (n_sc > 0)
      copy_to_device(ctx, dl.p, shortcut_lengths, n_sc * sizeof(double));
    else
      copy_to_device(ctx, ds.p, segments, 3 * n * sizeof(V3));
    launch(ctx, "select", k_select_data, dim3(blocks), dim3(256), 0, static_cast<const V3*>(ds.p), n,
           static_cast<const double*>(dl.p), n_sc, bb.p);
    launch(ctx, "select", k_best_final, dim3(1), dim3(256), 0, static_cast<const BestRec*>(bb.p),
           blocks, best.p);
    BestRec h{};
    copy_to_host(ctx, &h, best.p, sizeof(h));
    out->kind = n_sc > 0 ? RP_CHOSEN_SHORTCUT : RP_CHOSEN_REACH_POSE;
    out->index = h.key;
    out->path_length = h.len;
  });
}

rp_status rp_short_reach_scan(rp_ctx* ctx, const rp_grid* g, const rp_arm* arm,
                              const rp_reach_params* rp, const double target[3],
                              const double* samples, const uint8_t* sample_clear, int32_t n,
                              const double* prefix, int32_t n_prefix, const double origin[3],
                              int32_t* found, rp_shortcut* sc, double* sublength, int32_t cap) {
  return guarded([&] {
    require(n >= 0 && n_prefix >= 0, RP_E_INVALID_PARAMETER, "negative sample count");
    require(g->ctx == ctx, RP_E_INVALID_PARAMETER, "grid belongs to another context");
    *found = 0;
    if (n == 0) return;
    cudaStream_t st = ctx->stream;
    const int nd_max = 1 << 16;  // direct walks: scaled_sample_count(|target - origin|, spacing)
    DevBuf<V3> ds(n, st), dp(std::max(1, n_prefix), st), sub(std::max(n, 1) + nd_max, st);
    DevBuf<uint8_t> dc(n, st);
    DevBuf<ScanOut> out(1, st);
    copy_to_device(ctx, ds.p, samples, n * sizeof(V3));
    copy_to_device(ctx, dc.p, sample_clear, n);
    if (n_prefix) copy_to_device(ctx, dp.p, prefix, n_prefix * sizeof(V3));
    ScanArgs a{};
    a.g = g->view();
    a.root = V3{arm->root[0], arm->root[1], arm->root[2]};
    a.target = V3{target[0], target[1], target[2]};
    a.origin = V3{origin[0], origin[1], origin[2]};
    a.near_r = resolved_near_radius(*arm, *rp);
    a.spacing = nominal_spacing(*arm, *rp);
    a.samples = ds.p;
    a.clear = dc.p;
    a.n = n;
    a.prefix = dp.p;
    a.n_prefix = n_prefix;
    a.sub = sub.p;
    a.sub_cap = std::max(n, 1) + nd_max;
    launch(ctx, "shortcuts", k_short_reach_scan, dim3(1), dim3(1), 0, a, out.p);
    ScanOut h{};
    copy_to_host(ctx, &h, out.p, sizeof(h));
    if (h.status) fail(RP_E_CAPACITY_EXCEEDED, "short_reach_scan: direct walk too long");
    if (!h.found) return;
    require(h.n_sub <= cap, RP_E_CAPACITY_EXCEEDED, "sublength buffer too small");
    copy_to_host(ctx, sublength, sub.p, h.n_sub * sizeof(V3));
    sc->segment_index = 1;
    sc->hit_sample_index = h.hit;
    sc->seg1_index = sc->seg2_index = -1;
    sc->has_bridge = h.has_bridge;
    sc->via_origin_direct = h.via_direct;
    sc->n_prefix = n_prefix;
    sc->n_sublength = h.n_sub;
    std::memcpy(sc->bridge, &h.bridge, sizeof(V3));
    sc->path_length = h.path_length;
    *found = 1;
  });
}

rp_status rp_span_gap(rp_ctx* ctx, const double p2[3], const double* backward_pts, int32_t n,
                      double L3, double epsilon, double* v3_out, int32_t* idx_out,
                      int32_t* n_out) {
  return guarded([&] {
    require(n >= 0, RP_E_INVALID_PARAMETER, "negative point count");
    *n_out = 0;
    if (n == 0) return;
    cudaStream_t st = ctx->stream;
    DevBuf<V3> b(n, st), v(n, st);
    DevBuf<uint8_t> pass(n, st);
    copy_to_device(ctx, b.p, backward_pts, n * sizeof(V3));
    launch(ctx, "span_gap", k_span_gap, dim3(nblk(n, 128)), dim3(128), 0, V3{p2[0], p2[1], p2[2]},
           static_cast<const V3*>(b.p), n, L3, epsilon, v.p, pass.p);
    std::vector<V3> hv(n);
    std::vector<uint8_t> hp(n);
    copy_to_host(ctx, hv.data(), v.p, n * sizeof(V3));
    copy_to_host(ctx, hp.data(), pass.p, n);
    for (int k = 0; k < n; ++k) {
      if (!hp[k]) continue;
      std::memcpy(v3_out + 3 * *n_out, &hv[k], sizeof(V3));
      idx_out[*n_out] = k;
      ++*n_out;
    }
  });
}

rp_status rp_solution_set_shortcut_basis(const rp_solution_set* s, int64_t k, rp_pose* basis) {
  return guarded([&] {
    require(k >= 0 && k < static_cast<int64_t>(s->shortcuts.size()), RP_E_INVALID_PARAMETER,
            "shortcut index out of range");
    to_abi(s->shortcuts[k].basis, basis, nullptr, 0);
  });
}

rp_status rp_solution_set_shortcut(const rp_solution_set* s, int64_t k, rp_shortcut* sc,
                                   double* tip, int32_t cap, int32_t* n_tip) {
  return guarded([&] {
    require(k >= 0 && k < static_cast<int64_t>(s->shortcuts.size()), RP_E_INVALID_PARAMETER,
            "shortcut index out of range");
    const HostShortcut& h = s->shortcuts[k];
    std::memset(sc, 0, sizeof(*sc));
    sc->segment_index = h.segment_index;
    sc->hit_sample_index = h.hit;
    sc->seg1_index = h.seg1;
    sc->seg2_index = h.seg2;
    sc->has_bridge = h.has_bridge;
    sc->via_origin_direct = h.via_direct;
    sc->n_prefix = static_cast<int>(h.prefix.size());
    sc->n_sublength = static_cast<int>(h.sublength.size());
    sc->bridge[0] = h.bridge.x;
    sc->bridge[1] = h.bridge.y;
    sc->bridge[2] = h.bridge.z;
    sc->path_length = h.path_length;
    const auto w = h.tip_waypoints(V3{s->target[0], s->target[1], s->target[2]});
    if (n_tip) *n_tip = static_cast<int>(w.size());
    if (tip)
      for (int q = 0; q < static_cast<int>(w.size()) && q < cap; ++q) {
        tip[3 * q] = w[q].x;
        tip[3 * q + 1] = w[q].y;
        tip[3 * q + 2] = w[q].z;
      }
  });
}

rp_status rp_solution_set_destroy(rp_solution_set* s) {
  return guarded([&] {
    if (!s) return;
    cudaStreamSynchronize(s->ctx->stream);
    delete s;
  });
}

rp_status rp_select_solution(const rp_solution_set* s, rp_chosen* out) {
  return guarded([&] { *out = select(s); });
}

}  // extern "C"

// ===========================================================================
// Batched reach queries (BASELINE configs[4]).
//
// Segment-1 and segment-2 clearance depend only on (i, j), not on the target
// (src/reach_solver.cpp:278, 368): one target-independent bitmap
// clear2[i][j] (Q^2 bits, 13 MB at 2 deg) is built once per call and every
// query's segment-2 expansion tests a bit instead of walking 8 samples. The
// target-dependent tests (reach precheck, gap band, v3 / s4 walks,
// self-collision, near-encounter scans) run per query exactly as in k_seg2,
// so every counter and the chosen solution equal solve_reach's.
namespace rp {
namespace {

/// Row-wise clearance of segment 2 for every (i, j) with a clear segment 1.
__global__ void __launch_bounds__(256, 4) k_clear2(SolveDev a, const uint32_t* __restrict__ walk1_bits,
                                                int W, uint32_t* __restrict__ clear2) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int64_t total = static_cast<int64_t>(a.Q) * W;
  for (int64_t wd = warp; wd < total; wd += nwarps) {
    const int i = static_cast<int>(wd / W);
    const int j = static_cast<int>(wd - static_cast<int64_t>(i) * W) * 32 + lane;
    bool clear = false;
    if (j < a.Q && ((walk1_bits[i >> 5] >> (i & 31)) & 1u)) {
      const V3 p1 = a.arm.root + a.arm.L[0] * qvec(a, i);
      const V3 p2 = p1 + a.arm.L[1] * qvec(a, j);
      clear = (kSeg2ParWalk ? rpd::walk_first_blocked_affine_from(a.g, p1, p2, a.n, 0, a.dq_aff)
                            : rpd::walk_first_blocked(a.g, p1, p2, a.n)) == 0;
    }
    const unsigned m = __ballot_sync(FULL, clear);
    if (lane == 0) clear2[wd] = m;
  }
}

/// Segment-1 walk verdicts (target independent).
__global__ void k_walk1(SolveDev a, uint32_t* __restrict__ bits) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  bool clear = false;
  if (i < a.Q) {
    const V3 p1 = a.arm.root + a.arm.L[0] * qvec(a, i);
    clear = rpd::walk_first_blocked(a.g, a.arm.root, p1, a.n) == 0;
  }
  const unsigned m = __ballot_sync(FULL, clear);
  if ((threadIdx.x & 31) == 0 && (i >> 5) < (a.Q + 31) / 32) bits[i >> 5] = m;
}

// ---- multi-query pipeline: every stage covers all targets of a chunk ------

constexpr unsigned kBatchShortcutCap = 1u << 24;  // near-encounter candidates per chunk
// gap-passing pairs are queued for k_bq_tail in target-tagged blocks of
// kTailBlock entries taken from a fixed pool (overflow: evaluated in place)
constexpr int kTailBlock = 256;

struct BatchDev {
  SolveDev a;  // shared constants (target fields unused)
  int T, W, BPT, eight;
  const V3* targets;
  const V3* bpts;
  const uint8_t* walk4_ok;
  const uint32_t* walk1;
  const uint32_t* clear2;
  uint32_t* surv_bits;  // [T*W]
  int* surv_idx;        // [T*Q]
  int* surv_cnt;        // [T]
  unsigned long long* ctr;  // [T*C_COUNT]
  long long* sc_list;       // (t << 40) | (seg2 << 39) | payload
  unsigned* sc_count;
  BestRec* bb;    // [T*BPT]
  BestRec* best;  // [T]
  // quiver rings (generated quivers): ring r = directions
  // ring_off[r] .. ring_off[r+1]-1 at elevation (cos, sin) = (ring_c, ring_s),
  // azimuth 2*pi*m/count; nrings == 0 -> sweep every direction
  int* row_ctr;  // [T] next survivor row (dynamic row assignment in k_bq_seg2)
  // tail queue: pool[tail_cap * kTailBlock] pair keys s*Q + j, per block its
  // target and length; tail_ctr = blocks taken (tail_cap == 0: no queue)
  uint32_t* tail_pool;
  int* tail_tgt;
  int* tail_len;
  unsigned* tail_ctr;
  int tail_cap;
  BestRec* tail_best;  // [T] argmin over the queued pairs
  const uint8_t* kend_b;  // [T] samples of the v3 walks [p2, b] not proven free (k_tail_skip)
  int nrings;
  const int* ring_off;
  const double* ring_c;
  const double* ring_s;
};

__device__ __forceinline__ void warp_flush_t(unsigned long long* ctr, int idx, unsigned v) {
  v = __reduce_add_sync(FULL, v);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(ctr + idx, static_cast<unsigned long long>(v));
}

__global__ void k_bq_walk4(BatchDev d, uint8_t* walk4) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= d.T) return;
  walk4[t] = (!d.eight || rpd::walk_first_blocked(d.a.g, d.bpts[t], d.targets[t], d.a.n) == 0) ? 1 : 0;
}

/// prune_segment1 for every (target, direction): blockIdx.y = target.
__global__ void __launch_bounds__(256) k_bq_seg1(BatchDev d) {
  const int t = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const SolveDev& a = d.a;
  const V3 target = d.targets[t];
  bool valid = i < a.Q, reach = false, surv = false;
  if (valid) {
    const V3 p1 = a.arm.root + a.arm.L[0] * qvec(a, i);
    reach = a.disable_prune != 0 || rpd::sqnorm(p1 - target) <= a.budget2;
    if (rpd::point_to_segment(target, a.arm.root, p1) <= a.near_r + 1e-9) {
      const unsigned pos = atomicAdd(d.sc_count, 1u);
      if (pos < kBatchShortcutCap) d.sc_list[pos] = (static_cast<long long>(t) << 40) | i;
    }
    surv = reach && ((d.walk1[i >> 5] >> (i & 31)) & 1u);
  }
  const unsigned m = __ballot_sync(FULL, surv);
  if ((threadIdx.x & 31) == 0 && (i >> 5) < d.W) d.surv_bits[static_cast<size_t>(t) * d.W + (i >> 5)] = m;
  unsigned long long* c = d.ctr + static_cast<size_t>(t) * C_COUNT;
  warp_flush_t(c, C_SEG1_LIMIT, valid ? 1u : 0u);
  warp_flush_t(c, C_SEG1_REACH, reach ? 1u : 0u);
  warp_flush_t(c, C_SEG1_SURV, surv ? 1u : 0u);
}

/// Ordered survivor compaction, one block per target.
__global__ void __launch_bounds__(1024) k_bq_compact(BatchDev d) {
  typedef cub::BlockScan<int, 1024> Scan;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int carry;
  const int t = blockIdx.x;
  const uint32_t* bits = d.surv_bits + static_cast<size_t>(t) * d.W;
  int* out = d.surv_idx + static_cast<size_t>(t) * d.a.Q;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int w0 = 0; w0 < d.W; w0 += 1024) {
    const int w = w0 + threadIdx.x;
    const uint32_t word = w < d.W ? bits[w] : 0u;
    int off = 0, total = 0;
    Scan(tmp).ExclusiveSum(__popc(word), off, total);
    off += carry;
    uint32_t x = word;
    while (x) {
      const int b = __ffs(x) - 1;
      x &= x - 1;
      out[off++] = w * 32 + b;
    }
    __syncthreads();
    if (threadIdx.x == 0) carry += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) d.surv_cnt[t] = carry;
}

/// k_seg2_cached for every target of the chunk: blockIdx.y = target,
/// blockIdx.x strides over that target's (survivor, j) pairs.
template <bool EIGHT>
__global__ void __launch_bounds__(256, RP_BQ_MINB) k_bq_seg2(BatchDev d) {
  const int t = blockIdx.y;
  const SolveDev& a = d.a;
  const ArmDev& arm = a.arm;
  const double L1 = arm.L[0], L2 = arm.L[1], L3 = arm.L[2];
  const double min_sep = 2.0 * arm.arm_radius;
  const V3 target = d.targets[t];
  const V3 b = d.bpts[t];
  const V3 bdir = a.bdirs[0];
  const bool walk4 = !EIGHT || d.walk4_ok[t];
  const int S1 = d.surv_cnt[t];
  const int* sidx = d.surv_idx + static_cast<size_t>(t) * a.Q;
  const int64_t npairs = static_cast<int64_t>(S1) * a.Q;
  unsigned c_clear = 0, c_gp = 0, c_jp = 0, c_v3 = 0, c_sol = 0;
  double best_len = 1e308;
  long long best_key = LLONG_MAX;
  const int lane = threadIdx.x & 31;
  const int warp_id = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const double rnear = a.near_r + 1e-6;
  (void)npairs;
  // the warp's current tail-queue block (uniform): -2 none taken yet, -1
  // no pool (or exhausted): evaluate in place
  int tb = d.tail_cap > 0 ? -2 : -1, tf = 0;
  __shared__ int wiv[8][32 * 8], wive[8][32 * 8];  // per warp: 32 rings x 8 intervals
  __shared__ signed char wniv[8][32];
  __shared__ int wbase[8][32];
  // a warp owns whole survivor rows (s) and sweeps j; row constants hoisted
  (void)warp_id;
  (void)nwarps;
  // rows are taken dynamically (per-target counter): row costs differ by
  // orders of magnitude (rows that cannot reach the gap shell are skipped)
  for (;;) {
    int s = 0;
    if (lane == 0) s = atomicAdd(d.row_ctr + t, 1);
    s = __shfl_sync(FULL, s, 0);
    if (s >= S1) break;
    const int i = sidx[s];
    const V3 s1 = L1 * qvec(a, i);
    const V3 p1 = arm.root + s1;
    const uint32_t* crow = d.clear2 + static_cast<int64_t>(i) * d.W;
    const double dt2 = rpd::sqnorm(target - p1);
    const bool row_near = dt2 <= (L2 + rnear) * (L2 + rnear);  // else no pair can be near
    // segment-2 clear count of the row = popcount of its clearance bits
    for (int w = lane; w < d.W; w += 32) {
      uint32_t bits = __ldg(crow + w);
      const int rem = a.Q - w * 32;
      if (rem < 32) bits &= (1u << rem) - 1u;
      c_clear += __popc(bits);
    }
    // no j can pass the coarse gap test when b lies outside the shell
    // |b - p1| in [L3 - eps - L2, sqrt(coarse2) + L2] (margins absorb rounding)
    const double db = sqrt(rpd::sqnorm(b - p1));
    const bool row_gap = db <= (sqrt(a.coarse2) + L2) * (1.0 + 1e-9) + 1e-12 &&
                         db >= (L3 - a.eps - L2) * (1.0 - 1e-9) - 1e-12;
    if (!row_near && !row_gap) continue;
    // Phase 1 (all lanes busy): near-encounter scan and a conservative
    // band + clearance prefilter; passers are queued per warp in shared
    // memory. Phase 2 runs the exact gap test, the v3 walk and the
    // self-collision check 32 queued pairs at a time, so the heavy tail
    // (a few % of pairs) executes without divergence.
    const auto heavy = [&](int j) {
      const int64_t p = static_cast<int64_t>(i) * a.Q + j;  // key i * Q + j (see k_bq_tail)
      const V3 dir2 = qvec(a, j);
      const V3 p2 = p1 + L2 * dir2;
      const V3 v3 = b - p2;
      const double v3_len = rpd::norm(v3);
      (void)v3_len;  // gap and length tests already passed in visit
      if (rpd::walk_first_blocked(a.g, p2, b, a.n, d.kend_b[t]) != 0) return;
      ++c_v3;
      if (!walk4) return;
      const V3 s2 = L2 * dir2;
      V3 J[5];
      J[0] = arm.root;
      J[1] = J[0] + s1;
      J[2] = J[1] + s2;
      J[3] = J[2] + v3;
      if (EIGHT) J[4] = J[3] + a.L4 * bdir;
      if (!rpd::self_collision_free(J, EIGHT ? 4 : 3, min_sep)) return;
      ++c_sol;
      const double len = (rpd::norm(s1) + rpd::norm(s2)) + rpd::norm(v3);
      if (len < best_len || (len == best_len && p < best_key)) {
        best_len = len;
        best_key = p;
      }
    };
    // every lane calls this with its own j (valid or not) in lockstep.
    // Band + clearance passers get the exact gap test here; the pairs that
    // reach the v3 walk are appended to the warp's block of the tail queue
    // (k_bq_tail evaluates them with a small code footprint -- ncu showed
    // instruction-fetch stalls dominating when the tail ran inline) or, if
    // the pool is exhausted, evaluated in place.
    const auto visit = [&](int j, bool valid) {
      bool pass = false;
      if (valid) {
        const V3 dir2 = qvec(a, j);
        const V3 p2 = p1 + L2 * dir2;
        if (row_near && rpd::may_pass_near(target, p1, dir2, L2, rnear) &&
            rpd::point_to_segment(target, p1, p2) <= a.near_r + 1e-9) {
          const unsigned pos = atomicAdd(d.sc_count, 1u);
          if (pos < kBatchShortcutCap)
            d.sc_list[pos] = (static_cast<long long>(t) << 40) | (1ll << 39) |
                             (static_cast<int64_t>(s) * a.Q + j);
        }
        if (row_gap) {
          const double v2 = rpd::sqnorm(b - p2);
          pass = v2 <= a.coarse2 && v2 >= a.band_lo2 &&
                 ((__ldg(crow + (j >> 5)) >> (j & 31)) & 1u);
          if (pass) {
            // heavy()'s first tests: v3 = b - p2, |v3| = sqrt(v2)
            const double v3_len = sqrt(v2);
            if (fabs(v3_len - L3) > a.eps) {
              pass = false;
            } else {
              ++c_gp;
              if (v3_len < 1e-12) pass = false;
              else ++c_jp;
            }
          }
        }
      }
      const unsigned m = __ballot_sync(FULL, pass);
      if (!m) return;
      const int n = __popc(m);
      if (tb == -2 || (tb >= 0 && tf + n > kTailBlock)) {  // close the block, take the next
        int nb = 0;
        if (lane == 0) {
          if (tb >= 0) d.tail_len[tb] = tf;
          nb = static_cast<int>(atomicAdd(d.tail_ctr, 1u));
          if (nb < d.tail_cap) d.tail_tgt[nb] = t;
        }
        nb = __shfl_sync(FULL, nb, 0);
        tb = nb < d.tail_cap ? nb : -1;
        tf = 0;
      }
      if (tb >= 0) {
        if (pass)
          d.tail_pool[static_cast<size_t>(tb) * kTailBlock + tf + __popc(m & ((1u << lane) - 1u))] =
              static_cast<uint32_t>(static_cast<int64_t>(i) * a.Q + j);
        tf += n;
      } else if (pass) {
        heavy(j);
      }
    };
    // Directions visited: with quiver rings, only those that can pass the
    // gap band (q.u_b within the band's cosine range around
    // u_b = (b - p1)/|b - p1|) or pass near the target (q.u_t >= cos of the
    // near cone around u_t): per ring at most four azimuth arcs, found by
    // lanes in parallel 32 rings at a time and packed densely. Skipped
    // directions fail both tests outright, so counters, shortcuts and the
    // argmin are unchanged; the exact tests run on every visited pair.
    // Without ring data the whole quiver is one "ring".
    const double L2sq = L2 * L2;
    double blo = 2.0, bhi = -2.0, clo = 2.0;
    V3 ub{0, 0, 1}, ut{0, 0, 1};
    bool band_all = false, cap_all = false;
    if (row_gap) {
      if (db > 1e-9) {
        ub = (b - p1) / db;
        blo = (db * db + L2sq - a.coarse2) / (2.0 * L2 * db) - 1e-9;
        bhi = (db * db + L2sq - a.band_lo2) / (2.0 * L2 * db) + 1e-9;
      } else {
        band_all = true;
      }
    }
    if (row_near) {
      const double dt = sqrt(dt2);
      if (dt > rnear * (1.0 + 1e-9) + 1e-12) {
        ut = (target - p1) / dt;
        const double sr = rnear / dt;
        clo = sqrt(fmax(0.0, 1.0 - sr * sr)) - 1e-9;
      } else {
        cap_all = true;
      }
    }
    int* ivs = wiv[threadIdx.x >> 5];
    int* ive = wive[threadIdx.x >> 5];
    signed char* niv = wniv[threadIdx.x >> 5];
    const int nrt = d.nrings > 0 ? d.nrings : 1;
    for (int r0 = 0; r0 < nrt; r0 += 32) {
      const int r = r0 + lane;
      niv[lane] = 0;
      if (r < nrt) {
        const int off = d.nrings ? d.ring_off[r] : 0;
        const int cnt = d.nrings ? d.ring_off[r + 1] - off : a.Q;
        int a0[4], ln[4], na = 0;
        if (d.nrings == 0 || band_all || cap_all) {
          a0[0] = 0;
          ln[0] = cnt;
          na = 1;
        } else {
          if (row_gap) na += ring_arcs(d.ring_c[r], d.ring_s[r], cnt, ub, blo, bhi, a0, ln);
          if (row_near)
            na += ring_arcs(d.ring_c[r], d.ring_s[r], cnt, ut, clo, 2.0, a0 + na, ln + na);
        }
        int m = ring_intervals(cnt, a0, ln, na, ivs + lane * 8, ive + lane * 8);
        if (m < 0) {
          ivs[lane * 8] = 0;
          ive[lane * 8] = cnt;
          m = 1;
        }
        niv[lane] = static_cast<signed char>(m);
      }
      // pack the rings' intervals densely: exclusive scan of the per-ring
      // direction counts, then each lane maps its slot of the packed range
      // back to (ring, interval, offset)
      int mine = 0;
      for (int k = 0; k < niv[lane]; ++k) mine += ive[lane * 8 + k] - ivs[lane * 8 + k];
      int incl = mine;
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += v;
      }
      wbase[threadIdx.x >> 5][lane] = incl - mine;
      const int total = __shfl_sync(FULL, incl, 31);
      __syncwarp();
      const int* base = wbase[threadIdx.x >> 5];
      for (int t0 = 0; t0 < total; t0 += 32) {
        const int tt = t0 + lane;
        int j = 0;
        if (tt < total) {
          int lo = 0, hi = 31;  // last ring whose base <= tt
          while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (base[mid] <= tt) lo = mid; else hi = mid - 1;
          }
          int rem = tt - base[lo];
          int k = 0;
          while (rem >= ive[lo * 8 + k] - ivs[lo * 8 + k]) {
            rem -= ive[lo * 8 + k] - ivs[lo * 8 + k];
            ++k;
          }
          j = (d.nrings ? d.ring_off[r0 + lo] : 0) + ivs[lo * 8 + k] + rem;
        }
        visit(j, tt < total);
      }
      __syncwarp();
    }
  }
  if (tb >= 0 && lane == 0) d.tail_len[tb] = tf;
  unsigned long long* c = d.ctr + static_cast<size_t>(t) * C_COUNT;
  warp_flush_t(c, C_SEG2_CLEAR, c_clear);
  warp_flush_t(c, C_GAP_PASS, c_gp);
  warp_flush_t(c, C_JOINT_PASS, c_jp);
  warp_flush_t(c, C_V3_CLEAR, c_v3);
  warp_flush_t(c, C_SOLUTIONS, c_sol);
  for (int off = 16; off > 0; off >>= 1) {
    const double ol = __shfl_down_sync(FULL, best_len, off);
    const long long ok = __shfl_down_sync(FULL, best_key, off);
    if (ol < best_len || (ol == best_len && ok < best_key)) {
      best_len = ol;
      best_key = ok;
    }
  }
  __shared__ BestRec wb[8];
  if (lane == 0) wb[threadIdx.x >> 5] = BestRec{best_len, best_key};
  __syncthreads();
  if (threadIdx.x == 0) {
    BestRec r = wb[0];
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w)
      if (wb[w].len < r.len || (wb[w].len == r.len && wb[w].key < r.key)) r = wb[w];
    d.bb[static_cast<size_t>(t) * d.BPT + blockIdx.x] = r;
  }
}

/// 16-byte compare-and-swap (atom.cas.b128, sm_90+); returns the old value.
__device__ __forceinline__ BestRec cas_best(BestRec* addr, BestRec cmp, BestRec val) {
  unsigned long long o0, o1;
  asm volatile(
      "{\n\t.reg .b128 c, v, o;\n\t"
      "mov.b128 c, {%2, %3};\n\t"
      "mov.b128 v, {%4, %5};\n\t"
      "atom.global.cas.b128 o, [%6], c, v;\n\t"
      "mov.b128 {%0, %1}, o;\n\t}"
      : "=l"(o0), "=l"(o1)
      : "l"(__double_as_longlong(cmp.len)), "l"(cmp.key), "l"(__double_as_longlong(val.len)),
        "l"(val.key), "l"(addr)
      : "memory");
  return BestRec{__longlong_as_double(static_cast<long long>(o0)), static_cast<long long>(o1)};
}

__device__ __forceinline__ bool best_less(const BestRec& x, const BestRec& y) {
  return x.len < y.len || (x.len == y.len && x.key < y.key);
}

/// The tail of k_bq_seg2's pair test for the queued pairs, one block per
/// queue block (all of one target): the v3 walk (gathers in flight
/// together), the fourth-segment verdict and the self-collision check, the
/// v3-clear / solution counters and the (length, key) argmin -- the same
/// arithmetic heavy() performs in place.
template <bool EIGHT>
__global__ void __launch_bounds__(kTailBlock, 5) k_bq_tail(BatchDev d) {
  const int c = blockIdx.x;
  const int t = d.tail_tgt[c];
  const int len = d.tail_len[c];
  const SolveDev& a = d.a;
  const ArmDev& arm = a.arm;
  const double L1 = arm.L[0], L2 = arm.L[1];
  const V3 b = d.bpts[t];
  unsigned c_v3 = 0, c_sol = 0;
  BestRec best{1e308, LLONG_MAX};
  if (static_cast<int>(threadIdx.x) < len) {
    // queued key i * Q + j (ordered as the canonical (s, j): i ascends with s)
    const uint32_t p = d.tail_pool[static_cast<size_t>(c) * kTailBlock + threadIdx.x];
    const int i = static_cast<int>(p / static_cast<uint32_t>(a.Q));
    const int j = static_cast<int>(p - static_cast<uint32_t>(i) * static_cast<uint32_t>(a.Q));
    const V3 s1 = L1 * qvec(a, i);
    const V3 p1 = arm.root + s1;
    const V3 dir2 = qvec(a, j);
    const V3 p2 = p1 + L2 * dir2;
    const V3 v3 = b - p2;
    if (rpd::walk_any_blocked_upto_affine(a.g, p2, b, a.n, d.kend_b[t], a.dq_aff) == 0) {
      ++c_v3;
      if (!EIGHT || d.walk4_ok[t]) {
        const V3 s2 = L2 * dir2;
        V3 J[5];
        J[0] = arm.root;
        J[1] = J[0] + s1;
        J[2] = J[1] + s2;
        J[3] = J[2] + v3;
        if (EIGHT) J[4] = J[3] + a.L4 * a.bdirs[0];
        // half-length bounds: |s1| = L1, |s2| = L2 (unit quiver vectors,
        // widened for rounding), |v3| <= L3 + eps (gap band), |s4| = L4
        const double w = 1.0 + 1e-9;
        const double half[4] = {0.5 * L1 * w, 0.5 * L2 * w, 0.5 * (arm.L[2] + a.eps) * w,
                                0.5 * a.L4 * w};
        if (rpd::self_collision_free_screened(J, EIGHT ? 4 : 3, 2.0 * arm.arm_radius, half)) {
          ++c_sol;
          best = BestRec{(rpd::norm(s1) + rpd::norm(s2)) + rpd::norm(v3), static_cast<long long>(p)};
        }
      }
    }
  }
  c_v3 = __reduce_add_sync(FULL, c_v3);
  c_sol = __reduce_add_sync(FULL, c_sol);
  for (int off = 16; off > 0; off >>= 1) {
    const BestRec o{__shfl_down_sync(FULL, best.len, off), __shfl_down_sync(FULL, best.key, off)};
    if (best_less(o, best)) best = o;
  }
  __shared__ unsigned sv3[kTailBlock / 32], ssol[kTailBlock / 32];
  __shared__ BestRec sb[kTailBlock / 32];
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sv3[w] = c_v3;
    ssol[w] = c_sol;
    sb[w] = best;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned tv = 0, ts = 0;
    BestRec bb = sb[0];
    for (int k = 0; k < kTailBlock / 32; ++k) {
      tv += sv3[k];
      ts += ssol[k];
      if (best_less(sb[k], bb)) bb = sb[k];
    }
    unsigned long long* ctr = d.ctr + static_cast<size_t>(t) * C_COUNT;
    if (tv) atomicAdd(ctr + C_V3_CLEAR, static_cast<unsigned long long>(tv));
    if (ts) atomicAdd(ctr + C_SOLUTIONS, static_cast<unsigned long long>(ts));
    if (ts) {
      BestRec* dst = d.tail_best + t;
      const volatile long long* vp = reinterpret_cast<const volatile long long*>(dst);
      BestRec cur{__longlong_as_double(vp[0]), vp[1]};  // a torn read only fails the CAS
      while (best_less(bb, cur)) {
        const BestRec old = cas_best(dst, cur, bb);
        if (__double_as_longlong(old.len) == __double_as_longlong(cur.len) && old.key == cur.key)
          break;
        cur = old;
      }
    }
  }
}

__global__ void k_bq_best(BatchDev d) {
  const int t = blockIdx.x;
  BestRec b = d.tail_cap > 0 ? d.tail_best[t] : BestRec{1e308, LLONG_MAX};
  for (int k = threadIdx.x; k < d.BPT; k += blockDim.x) {
    const BestRec r = d.bb[static_cast<size_t>(t) * d.BPT + k];
    if (r.len < b.len || (r.len == b.len && r.key < b.key)) b = r;
  }
  for (int off = 16; off > 0; off >>= 1) {
    const double ol = __shfl_down_sync(FULL, b.len, off);
    const long long ok = __shfl_down_sync(FULL, b.key, off);
    if (ol < b.len || (ol == b.len && ok < b.key)) b = BestRec{ol, ok};
  }
  __shared__ BestRec wb[32];
  if ((threadIdx.x & 31) == 0) wb[threadIdx.x >> 5] = b;
  __syncthreads();
  if (threadIdx.x == 0) {
    b = wb[0];
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w)
      if (wb[w].len < b.len || (wb[w].len == b.len && wb[w].key < b.key)) b = wb[w];
    d.best[t] = b;
  }
}

/// short_reach_scan for near-encounter candidates of any target.
__global__ void k_bq_shortcuts(BatchDev d, const long long* keys, int n, ShortcutRec* out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const long long key = keys[k];
  const int t = static_cast<int>(key >> 40);
  const bool seg2 = (key >> 39) & 1;
  const long long payload = key & ((1ll << 39) - 1);
  SolveDev a = d.a;
  a.target = d.targets[t];
  const ArmDev& arm = a.arm;
  ShortcutRec r{};
  r.key = key;
  if (!seg2) {
    const int i = static_cast<int>(payload);
    const V3 p1 = arm.root + arm.L[0] * qvec(a, i);
    const int fb = rpd::walk_first_blocked(a.g, arm.root, p1, a.n);
    r.segment_index = 1;
    r.seg1 = i;
    r.seg2 = -1;
    scan_one(a, arm.root, p1, arm.root, fb, r, false, arm.root, arm.root);
  } else {
    const int s = static_cast<int>(payload / a.Q);
    const int j = static_cast<int>(payload - static_cast<long long>(s) * a.Q);
    const int i = d.surv_idx[static_cast<size_t>(t) * a.Q + s];
    const V3 p1 = arm.root + arm.L[0] * qvec(a, i);
    const V3 p2 = p1 + arm.L[1] * qvec(a, j);
    const int fb = rpd::walk_first_blocked(a.g, p1, p2, a.n);
    r.segment_index = 2;
    r.seg1 = i;
    r.seg2 = j;
    scan_one(a, p1, p2, p1, fb, r, true, arm.root, p1);
  }
  out[k] = r;
}

/// Per-target shortcut summary: count and select_solution's pick (shortest,
/// first in canonical order).
struct ScBest {
  int count, seg1, seg2, _pad;
  double path_length;
};

/// One block per target over its (key-sorted) shortcut records.
__global__ void __launch_bounds__(1024) k_bq_sc_reduce(const long long* __restrict__ keys, const ShortcutRec* __restrict__ recs,
                               int n, ScBest* __restrict__ out, uint8_t* __restrict__ has_sc) {
  const long long t = blockIdx.x;
  // [lo, hi) of keys with target t (keys sorted ascending)
  auto lower = [&](long long v) {
    int a = 0, b = n;
    while (a < b) {
      const int m = (a + b) >> 1;
      if (keys[m] < v) a = m + 1; else b = m;
    }
    return a;
  };
  const int lo = lower(t << 40), hi = lower((t + 1) << 40);
  int cnt = 0;
  double bl = 1e308;
  int bp = INT_MAX;
  for (int k = lo + threadIdx.x; k < hi; k += blockDim.x) {
    if (!recs[k].valid) continue;
    ++cnt;
    if (recs[k].path_length < bl || (recs[k].path_length == bl && k < bp)) {
      bl = recs[k].path_length;
      bp = k;
    }
  }
  cnt = __reduce_add_sync(FULL, cnt);
  for (int off = 16; off > 0; off >>= 1) {
    const double ol = __shfl_down_sync(FULL, bl, off);
    const int op = __shfl_down_sync(FULL, bp, off);
    if (ol < bl || (ol == bl && op < bp)) {
      bl = ol;
      bp = op;
    }
  }
  __shared__ int sc[32], sp[32];
  __shared__ double sl[32];
  if ((threadIdx.x & 31) == 0) {
    sc[threadIdx.x >> 5] = cnt;
    sl[threadIdx.x >> 5] = bl;
    sp[threadIdx.x >> 5] = bp;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    ScBest r{0, -1, -1, 0, 0.0};
    double l = 1e308;
    int p = INT_MAX;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) {
      r.count += sc[w];
      if (sl[w] < l || (sl[w] == l && sp[w] < p)) {
        l = sl[w];
        p = sp[w];
      }
    }
    if (r.count > 0) {
      r.seg1 = recs[p].seg1;
      r.seg2 = recs[p].seg2;
      r.path_length = recs[p].path_length;
    }
    out[t] = r;
    has_sc[t] = r.count > 0 ? 1 : 0;
  }
}

struct BatchPose {
  int status, msg;
  int i, j;  // chosen key (refinement clears the free segments' indices)
  DevPose pose;
};

/// Materialise each target's chosen reach pose (k_materialize arithmetic)
/// and refine it exactly (rp_refine.cuh).
__global__ void k_bq_finish(BatchDev d, const uint8_t* has_shortcut, int refine_mode,
                            BatchPose* out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= d.T) return;
  BatchPose r{};
  const BestRec b = d.best[t];
  if (has_shortcut[t] || b.key == LLONG_MAX) {
    r.status = -1;
    out[t] = r;
    return;
  }
  const SolveDev& a = d.a;
  const ArmDev& arm = a.arm;
  const int i = static_cast<int>(b.key / a.Q);  // batch keys are i * Q + j
  const int j = static_cast<int>(b.key - static_cast<long long>(i) * a.Q);
  const V3 p1 = arm.root + arm.L[0] * qvec(a, i);
  const V3 p2 = p1 + arm.L[1] * qvec(a, j);
  DevPose p{};
  p.nseg = d.eight ? 4 : 3;
  p.seg[0] = arm.L[0] * qvec(a, i);
  p.seg[1] = arm.L[1] * qvec(a, j);
  p.seg[2] = d.bpts[t] - p2;
  p.qidx[0] = i;
  p.qidx[1] = j;
  p.qidx[2] = -1;
  p.qidx[3] = -1;
  if (d.eight) p.seg[3] = a.L4 * a.bdirs[0];
  build_chain(arm, p);
  r.i = i;
  r.j = j;
  r.status = refine_pose(arm, p, d.targets[t], refine_mode, &r.msg);
  r.pose = p;
  out[t] = r;
}

}  // namespace
}  // namespace rp

extern "C" rp_status rp_solve_reach_batch(rp_ctx* ctx, const rp_arm* arm, const rp_quiver* q,
                                          const rp_grid* g, const double* targets,
                                          int32_t n_targets, const rp_reach_params* rp,
                                          rp_batch_result* out) {
  return guarded([&] {
    HostSpan span_("solve_reach_batch");
    validate_arm(*arm);
    validate_reach(*rp);
    const bool eight = rp->mode == RP_MODE_8DOF;
    const ArmDev ad = make_arm_dev(*arm);
    const bool fast = !ad.any_limit && !ad.has_offsets && (!eight || rp->approach_half_angle == 0.0) &&
                      !(rp->cone_precheck && eight);
    auto finish = [&](int t, rp_solution_set* s) {
      rp_batch_result& r = out[t];
      std::memset(&r, 0, sizeof(r));
      r.stats = s->stats;
      r.n_solutions = s->n_solutions;
      r.n_shortcuts = static_cast<int64_t>(s->shortcuts.size());
      r.seg1 = r.seg2 = r.cone = -1;
      if (r.n_solutions + r.n_shortcuts == 0) {
        r.status = RP_E_NO_SOLUTION;
        return;
      }
      // select_solution (src/reach_solver.cpp:548-577) from the set's
      // shortcut records and its device argmin (no ordinal needed here)
      if (!s->shortcuts.empty()) {
        size_t bi = 0;
        for (size_t k = 1; k < s->shortcuts.size(); ++k)
          if (s->shortcuts[k].path_length < s->shortcuts[bi].path_length) bi = k;
        r.kind = RP_CHOSEN_SHORTCUT;
        r.path_length = s->shortcuts[bi].path_length;
        r.seg1 = s->shortcuts[bi].seg1;
        r.seg2 = s->shortcuts[bi].seg2;
        return;
      }
      r.kind = RP_CHOSEN_REACH_POSE;
      r.path_length = s->best_len;
      const DevPose dp = solution_dev_pose_by_key(s, s->best_key);
      r.seg1 = dp.qidx[0];
      r.seg2 = dp.qidx[1];
      r.cone = dp.nseg == 4 ? dp.qidx[3] : -1;
      rp_pose approx;
      to_abi(host_pose_from_dev(dp), &approx, nullptr, 0);
      r.status = rp_exact_refine(ctx, arm, &approx, targets + 3 * t,
                                 rp->refine_triangle_8dof ? 1 : 0, &r.refined);
      if (r.status == RP_E_CUDA || r.status == RP_E_INTERNAL) fail(r.status, rp_last_error());
    };
    if (!fast) {  // general configurations: one full solve per query
      for (int t = 0; t < n_targets; ++t) {
        std::unique_ptr<rp_solution_set> s(
            solve_reach(ctx, *arm, q, g, V3{targets[3 * t], targets[3 * t + 1], targets[3 * t + 2]}, *rp));
        finish(t, s.get());
      }
      return;
    }
    cudaStream_t st = ctx->stream;
    // ---- target-independent clearance
    rp_solution_set proto;
    proto.ctx = ctx;
    proto.quiver = q;
    proto.arm = *arm;
    proto.rp = *rp;
    SolveDev& a = proto.sd;
    a.g = g->view();
    a.arm = ad;
    a.n = rp->n_samples;
    a.eight = eight ? 1 : 0;
    a.Q = q->n;
    a.B = 1;
    a.scanning = 1;
    const double eps = resolved_epsilon(*arm, *rp);
    const double L3 = arm->lengths[2];
    const double L4 = eight ? arm->lengths[3] : 0.0;
    a.eps = eps;
    a.coarse2 = (L3 + eps) * (L3 + eps) * (1.0 + 1e-12);
    a.band_lo2 = L3 - eps > 0.0 ? (L3 - eps) * (L3 - eps) * (1.0 - 1e-9) : 0.0;
    a.dq_aff = affine_bracket(a.g, *arm);
    double budget = arm->lengths[1] + arm->lengths[2] + eps;
    if (eight) budget += arm->lengths[3];
    budget += 1e-9;
    a.budget2 = budget * budget;
    a.near_r = resolved_near_radius(*arm, *rp);
    a.spacing = nominal_spacing(*arm, *rp);
    a.L4 = L4;
    a.qx = q->d_soa;
    a.qy = q->d_soa + q->n;
    a.qz = q->d_soa + 2 * static_cast<size_t>(q->n);
    const int W = (q->n + 31) / 32;
    DevBuf<uint32_t> walk1(W, st), clear2(static_cast<size_t>(q->n) * W, st);
    launch(ctx, "clear2", k_walk1, dim3(nblk(q->n, 256)), dim3(256), 0, a, walk1.p);
    launch(ctx, "clear2", k_clear2, dim3(ctx->sm_count * 8), dim3(256), 0, a,
           static_cast<const uint32_t*>(walk1.p), W, clear2.p);
    // ---- all targets of a chunk go through each stage together
    const V3 axis{rp->approach_axis[0], rp->approach_axis[1], rp->approach_axis[2]};
    const V3 bdir = eight ? axis : V3{0, 0, 0};
    proto.bblock.alloc(sizeof(V3), st);
    copy_to_device(ctx, proto.bblock.p, &bdir, sizeof(V3));
    a.bdirs = reinterpret_cast<const V3*>(proto.bblock.p);
    static const int CH = std::getenv("RP_BATCH_CHUNK") ? std::atoi(std::getenv("RP_BATCH_CHUNK")) : 128;
    const int BPT = 64;
    const int refine_mode = eight ? (rp->refine_triangle_8dof ? 1 : 0) : 2;
    DevBuf<V3> d_t(CH, st), d_b(CH, st);
    DevBuf<uint8_t> d_w4(CH, st), d_hs(CH, st);
    DevBuf<uint32_t> d_sbits(static_cast<size_t>(CH) * W, st);
    DevBuf<int> d_sidx(static_cast<size_t>(CH) * q->n, st), d_scnt(CH, st);
    DevBuf<unsigned long long> d_ctr(static_cast<size_t>(CH) * C_COUNT, st);
    DevBuf<unsigned> d_scc(2, st);  // [0] near-encounter keys, [1] tail-queue blocks taken
    // tail queue (k_bq_tail): RP_TAIL_POOL_MB of pair keys (0: evaluate in place)
    const char* tail_env = std::getenv("RP_TAIL_POOL_MB");  // read per call (tests vary it)
    const long tail_mb = tail_env ? std::atol(tail_env) : 1024;
    const bool keys_fit = static_cast<double>(q->n) * q->n < 4294967296.0;
    int tail_cap = keys_fit ? static_cast<int>(std::max(0L, tail_mb) * (1L << 20) /
                                               (kTailBlock * static_cast<long>(sizeof(uint32_t))))
                            : 0;
    DevBuf<uint32_t> d_tpool;
    try {
      d_tpool.alloc(static_cast<size_t>(std::max(1, tail_cap)) * kTailBlock, st);
    } catch (const Fail&) {
      // short on device memory: evaluate every pair in place (tail_cap = 0)
      cudaGetLastError();
      tail_cap = 0;
      d_tpool.alloc(kTailBlock, st);
    }
    DevBuf<int> d_ttgt(std::max(1, tail_cap), st), d_tlen(std::max(1, tail_cap), st);
    DevBuf<BestRec> d_tbest(CH, st);
    const std::vector<BestRec> tbest_init(CH, BestRec{1e308, LLONG_MAX});
    // the grid's clearance field (cached) for k_tail_skip
    static const bool no_skip = std::getenv("RP_NO_ROW_SKIP") != nullptr;
    const ClearanceField cf = no_skip ? ClearanceField{} : grid_clearance_field(g, ctx);
    DevBuf<uint8_t> d_kend(CH, st);
    DevBuf<long long> d_scl(kBatchShortcutCap, st);
    DevBuf<BestRec> d_bb(static_cast<size_t>(CH) * BPT, st), d_best(CH, st);
    DevBuf<BatchPose> d_pose(CH, st);
    DevBuf<ScBest> d_scb(CH, st);
    // quiver rings for the batched seg2's arc culling (generated quivers)
    static const bool no_cull = std::getenv("RP_BATCH_NO_CULL") != nullptr;
    const int ring_n = no_cull ? 0 : static_cast<int>(q->ring_offsets.size());
    DevBuf<int> d_roff(ring_n + 1, st);
    DevBuf<double> d_rc(std::max(1, ring_n), st), d_rs(std::max(1, ring_n), st);
    if (ring_n > 0) {
      std::vector<int> ro(q->ring_offsets);
      ro.push_back(q->n);
      std::vector<double> rc(ring_n), rs(ring_n);
      for (int r = 0; r < ring_n; ++r) {
        rc[r] = std::cos(q->ring_elevations[r]);
        rs[r] = std::sin(q->ring_elevations[r]);
      }
      copy_to_device(ctx, d_roff.p, ro.data(), ro.size() * sizeof(int));
      copy_to_device(ctx, d_rc.p, rc.data(), ring_n * sizeof(double));
      copy_to_device(ctx, d_rs.p, rs.data(), ring_n * sizeof(double));
    }
    DevBuf<int> d_rowc(CH, st);
    std::vector<V3> ht, hb;
    for (int c0 = 0; c0 < n_targets; c0 += CH) {
      const int T = std::min(CH, n_targets - c0);
      ht.resize(T);
      hb.resize(T);
      for (int k = 0; k < T; ++k) {
        ht[k] = V3{targets[3 * (c0 + k)], targets[3 * (c0 + k) + 1], targets[3 * (c0 + k) + 2]};
        hb[k] = eight ? ht[k] - L4 * axis : ht[k];  // backward_endpoints, half-angle 0
      }
      copy_to_device(ctx, d_t.p, ht.data(), T * sizeof(V3));
      copy_to_device(ctx, d_b.p, hb.data(), T * sizeof(V3));
      RP_CUDA(cudaMemsetAsync(d_ctr.p, 0, static_cast<size_t>(T) * C_COUNT * sizeof(unsigned long long), st));
      d_scc.zero();
      d_hs.zero();
      BatchDev d{};
      d.a = a;
      d.T = T;
      d.W = W;
      d.BPT = BPT;
      d.eight = eight ? 1 : 0;
      d.targets = d_t.p;
      d.bpts = d_b.p;
      d.walk4_ok = d_w4.p;
      d.walk1 = walk1.p;
      d.clear2 = clear2.p;
      d.surv_bits = d_sbits.p;
      d.surv_idx = d_sidx.p;
      d.surv_cnt = d_scnt.p;
      d.ctr = d_ctr.p;
      d.sc_list = d_scl.p;
      d.sc_count = d_scc.p;
      d.bb = d_bb.p;
      d.best = d_best.p;
      d.nrings = ring_n;
      d.row_ctr = d_rowc.p;
      RP_CUDA(cudaMemsetAsync(d_rowc.p, 0, T * sizeof(int), st));
      d.ring_off = d_roff.p;
      d.ring_c = d_rc.p;
      d.ring_s = d_rs.p;
      d.tail_pool = d_tpool.p;
      d.tail_tgt = d_ttgt.p;
      d.tail_len = d_tlen.p;
      d.tail_ctr = d_scc.p + 1;
      d.tail_cap = tail_cap;
      d.tail_best = d_tbest.p;
      copy_to_device(ctx, d_tbest.p, tbest_init.data(), T * sizeof(BestRec));
      if (no_skip) {
        RP_CUDA(cudaMemsetAsync(d_kend.p, rp->n_samples, T, st));
      } else {
        launch(ctx, "seg2", k_tail_skip, dim3(nblk(T, 128)), dim3(128), 0, a.g,
               static_cast<const V3*>(d_b.p), T, L3 + eps, rp->n_samples, cf, d_kend.p);
      }
      d.kend_b = d_kend.p;
      launch(ctx, "walk4", k_bq_walk4, dim3(nblk(T, 128)), dim3(128), 0, d, d_w4.p);
      launch(ctx, "seg1", k_bq_seg1, dim3(nblk(q->n, 256), T), dim3(256), 0, d);
      launch(ctx, "compact", k_bq_compact, dim3(T), dim3(1024), 0, d);
      if (eight)
        launch(ctx, "seg2", k_bq_seg2<true>, dim3(BPT, T), dim3(256), 0, d);
      else
        launch(ctx, "seg2", k_bq_seg2<false>, dim3(BPT, T), dim3(256), 0, d);
      unsigned hcc[2] = {0, 0};
      copy_to_host(ctx, hcc, d_scc.p, sizeof(hcc));
      const unsigned nsc = hcc[0];
      const int ntail = static_cast<int>(std::min<unsigned>(hcc[1], static_cast<unsigned>(tail_cap)));
      if (ntail > 0) {
        if (eight)
          launch(ctx, "tail", k_bq_tail<true>, dim3(ntail), dim3(kTailBlock), 0, d);
        else
          launch(ctx, "tail", k_bq_tail<false>, dim3(ntail), dim3(kTailBlock), 0, d);
      }
      launch(ctx, "select", k_bq_best, dim3(T), dim3(64), 0, d);
      require(nsc <= kBatchShortcutCap, RP_E_CAPACITY_EXCEEDED,
              "too many near-encounter hypotheses");
      // shortcuts: sorted keys = (target, segment, canonical index), scanned
      // and reduced per target on the device
      RP_CUDA(cudaMemsetAsync(d_scb.p, 0, T * sizeof(ScBest), st));
      if (nsc > 0) {
        DevBuf<long long> sorted(nsc, st);
        size_t tb = 0;
        cub::DeviceRadixSort::SortKeys(nullptr, tb, d_scl.p, sorted.p, static_cast<int>(nsc), 0,
                                       64, st);
        DevBuf<unsigned char> tmp(tb, st);
        RP_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tb, d_scl.p, sorted.p,
                                               static_cast<int>(nsc), 0, 64, st));
        DevBuf<ShortcutRec> recs(nsc, st);
        launch(ctx, "shortcuts", k_bq_shortcuts, dim3(nblk(nsc, 128)), dim3(128), 0, d,
               static_cast<const long long*>(sorted.p), static_cast<int>(nsc), recs.p);
        launch(ctx, "shortcuts", k_bq_sc_reduce, dim3(T), dim3(1024), 0,
               static_cast<const long long*>(sorted.p), static_cast<const ShortcutRec*>(recs.p),
               static_cast<int>(nsc), d_scb.p, d_hs.p);
      }
      std::vector<ScBest> hscb(T);
      copy_to_host(ctx, hscb.data(), d_scb.p, T * sizeof(ScBest));
      launch(ctx, "finish", k_bq_finish, dim3(nblk(T, 64)), dim3(64), 0, d,
             static_cast<const uint8_t*>(d_hs.p), refine_mode, d_pose.p);
      std::vector<unsigned long long> hc(static_cast<size_t>(T) * C_COUNT);
      std::vector<int> hcnt(T);
      std::vector<BestRec> hbest(T);
      std::vector<BatchPose> hpose(T);
      copy_to_host(ctx, hc.data(), d_ctr.p, hc.size() * sizeof(unsigned long long));
      copy_to_host(ctx, hcnt.data(), d_scnt.p, T * sizeof(int));
      copy_to_host(ctx, hbest.data(), d_best.p, T * sizeof(BestRec));
      copy_to_host(ctx, hpose.data(), d_pose.p, T * sizeof(BatchPose));
      for (int k = 0; k < T; ++k) {
        rp_batch_result& r = out[c0 + k];
        std::memset(&r, 0, sizeof(r));
        const unsigned long long* c = hc.data() + static_cast<size_t>(k) * C_COUNT;
        const int64_t pairs = static_cast<int64_t>(hcnt[k]) * q->n;
        rp_solve_stats& S = r.stats;
        S.seg1_candidates = q->n;
        S.seg1_limit_pass = c[C_SEG1_LIMIT];
        S.seg1_reach_pass = c[C_SEG1_REACH];
        S.seg1_survivors = c[C_SEG1_SURV];
        S.pair_candidates = pairs;
        S.seg2_limit_pass = pairs;
        S.seg2_clear_pass = c[C_SEG2_CLEAR];
        S.gap_tested = c[C_SEG2_CLEAR];
        S.gap_pass = c[C_GAP_PASS];
        S.joint_pass = c[C_JOINT_PASS];
        S.v3_clear_pass = c[C_V3_CLEAR];
        S.solutions = c[C_SOLUTIONS];
        S.shortcuts_found = hscb[k].count;
        r.n_solutions = S.solutions;
        r.n_shortcuts = S.shortcuts_found;
        r.seg1 = r.seg2 = r.cone = -1;
        if (hscb[k].count > 0) {  // select_solution: shortest shortcut, first on ties
          r.kind = RP_CHOSEN_SHORTCUT;
          r.path_length = hscb[k].path_length;
          r.seg1 = hscb[k].seg1;
          r.seg2 = hscb[k].seg2;
          continue;
        }
        if (r.n_solutions == 0) {
          r.status = RP_E_NO_SOLUTION;
          continue;
        }
        r.kind = RP_CHOSEN_REACH_POSE;
        r.path_length = hbest[k].len;
        r.seg1 = hpose[k].i;
        r.seg2 = hpose[k].j;
        r.status = hpose[k].status;
        if (r.status == 0) {
          HostPose hp = host_pose_from_dev(hpose[k].pose);
          hp.waypoints.clear();
          to_abi(hp, &r.refined, nullptr, 0);
        }
      }
    }
  });
}
