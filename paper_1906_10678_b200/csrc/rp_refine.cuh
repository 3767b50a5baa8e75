// Exact refinement of a discretised reach pose (src/arm_model.cpp:214-324),
// shared by the planner (rp_path.cu) and the batched queries (rp_reach.cu).
#pragma once

#include "rp_reach.cuh"

namespace rp {

/// triangle_vertex (src/arm_model.cpp:219-238); returns 0 or an rp_status
/// with *msg the message id of refine_msg().
__host__ __device__ inline int triangle_vertex(V3 a, V3 b, double la, double lb, V3 n, V3 hint,
                                               V3* out, int* msg) {
  const V3 ab = b - a;
  const double c = rpd::norm(ab);
  if (!(c <= (la + lb) * (1.0 + 1e-12))) { *msg = 1; return RP_E_UNREACHABLE_TARGET; }
  if (!(c >= fabs(la - lb) * (1.0 - 1e-12) - 1e-15)) { *msg = 2; return RP_E_UNREACHABLE_TARGET; }
  const V3 c_hat = ab / c;
  V3 m_hat = rpd::cross(n, c_hat);
  const double m_norm = rpd::norm(m_hat);
  if (!(m_norm > 1e-12)) { *msg = 3; return RP_E_DEGENERATE_INPUT; }
  m_hat = m_hat / m_norm;
  const double along = (c * c + la * la - lb * lb) / (2.0 * c);
  const double h2 = la * la - along * along;
  const double h = sqrt(h2 > 0.0 ? h2 : 0.0);
  const V3 base = a + along * c_hat;
  const V3 pp = base + h * m_hat;
  const V3 pm = base - h * m_hat;
  *out = rpd::sqnorm(pp - hint) <= rpd::sqnorm(pm - hint) ? pp : pm;
  return 0;
}

/// plane_normal_for_refine (src/arm_model.cpp:240-254)
__host__ __device__ inline V3 plane_normal_for_refine(const DevPose& p, V3 anchor, V3 target,
                                                      int sa, int sb) {
  V3 n = rpd::cross(p.seg[sa], p.seg[sb]);
  if (rpd::norm(n) > 1e-12 * rpd::norm(p.seg[sa]) * rpd::norm(p.seg[sb])) return rpd::normalized(n);
  n = rpd::cross(target - anchor, p.joints[sa + 1] - anchor);
  if (rpd::norm(n) > 1e-12) return rpd::normalized(n);
  const V3 chord = rpd::normalized(target - anchor);
  const V3 seed = fabs(chord.z) < 0.9 ? V3{0, 0, 1} : V3{1, 0, 0};
  return rpd::normalized(rpd::cross(chord, seed));
}

/// mode 0: exact_refine_8dof, 1: _8dof_triangle, 2: exact_refine_6dof
/// (src/arm_model.cpp:258-324). Refines `p` in place; returns 0 or an
/// rp_status (msg id for the message).
__host__ __device__ inline int refine_pose(const ArmDev& arm, DevPose& p, V3 target, int mode,
                                           int* msg) {
  if (mode == 2) {
    if (p.nseg < 3) { *msg = 4; return RP_E_INVALID_PARAMETER; }
    if (arm.off[1] != 0.0 || arm.off[2] != 0.0) { *msg = 5; return RP_E_INVALID_PARAMETER; }
    const V3 p1 = p.joints[1];
    const V3 n = plane_normal_for_refine(p, p1, target, 1, 2);
    V3 p2;
    const int st = triangle_vertex(p1, target, arm.L[1], arm.L[2], n, p.joints[2], &p2, msg);
    if (st) return st;
    p.seg[1] = p2 - p1;
    p.seg[2] = target - p2;
    p.joints[2] = p2;
    p.joints[3] = target;
    p.qidx[1] = -1;
    p.qidx[2] = -1;
    return 0;
  }
  if (p.nseg != 4) { *msg = 6; return RP_E_INVALID_PARAMETER; }
  if (arm.off[2] != 0.0 || arm.off[3] != 0.0) { *msg = 7; return RP_E_INVALID_PARAMETER; }
  if (mode == 0) {
    const V3 v3 = p.seg[2];
    const double v3_len = rpd::norm(v3);
    if (!(v3_len >= 1e-9)) { *msg = 8; return RP_E_DEGENERATE_INPUT; }
    const V3 p2 = p.joints[2];
    const V3 d3 = target - p2;
    const V3 s3 = v3 * (arm.L[2] / v3_len);
    const V3 s4 = d3 - s3;
    p.seg[2] = s3;
    p.seg[3] = s4;
    p.joints[3] = p2 + s3;
    p.joints[4] = p.joints[3] + s4;
    p.s4dev = fabs(rpd::norm(s4) - arm.L[3]);
  } else {
    const V3 p2 = p.joints[2];
    const V3 n = plane_normal_for_refine(p, p2, target, 2, 3);
    V3 p3;
    const int st = triangle_vertex(p2, target, arm.L[2], arm.L[3], n, p.joints[3], &p3, msg);
    if (st) return st;
    p.seg[2] = p3 - p2;
    p.seg[3] = target - p3;
    p.joints[3] = p3;
    p.joints[4] = target;
    p.s4dev = fabs(rpd::norm(p.seg[3]) - arm.L[3]);
  }
  p.qidx[2] = -1;
  p.qidx[3] = -1;
  return 0;
}

inline const char* refine_msg(int m) {
  switch (m) {
    case 1: return "target beyond combined segment lengths";
    case 2: return "target inside the unreachable inner sphere";
    case 3: return "solution plane normal parallel to chord";
    case 4: return "need a 3-segment pose";
    case 5: return "triangle refinement requires coaxial joints 2 and 3";
    case 6: return "need a 4-segment pose";
    case 7: return "8DOF refinement requires coaxial joints 3 and 4";
    case 8: return "gap vector is numerically zero";
  }
  return "refinement failed";
}

}  // namespace rp
