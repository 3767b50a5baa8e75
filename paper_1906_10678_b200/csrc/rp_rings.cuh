// Quiver ring geometry shared by the direction-culling kernels (the batched
// segment-2 expansion and the backward pass's candidate cones).
//
// A generated quiver (src/quiver.cpp:16-51) is a set of latitude rings: ring
// r holds directions ring_off[r] .. ring_off[r+1]-1 at elevation phi_r with
// azimuths 2*pi*m/count. The directions q with lo <= q.u <= hi form at most
// two azimuth arcs per ring, so a cone or a band around u is enumerated by
// visiting a few arcs instead of every direction.
#pragma once

#include "rp_device.cuh"

namespace rp {

using rpd::V3;

/// Azimuth index arcs of ring (cphi, sphi, cnt) whose directions q satisfy
/// lo <= q.u <= hi (u unit), widened by 1.5 azimuth steps so that rounding
/// in the generator or here can only add directions, never drop one. Writes
/// up to 2 arcs as (first index, length) and returns their number; a full
/// ring is one arc (0, cnt).
static __device__ __noinline__ int ring_arcs(double cphi_d, double sphi_d, int cnt, V3 u, double lo_d,
                                     double hi_d, int* a0, int* len) {
  // Evaluated in fp32: the arcs only choose which directions are visited
  // (every visited pair gets the exact tests), so they need to be a
  // superset, not exact. The band is widened by 1e-5 for the fp32 dot
  // product and the angular margin by 2e-3 rad for fp32 acos/atan2 (its
  // error near |x| = 1 is below 4e-4 rad) on top of the 1.5-step margin.
  const float cphi = static_cast<float>(cphi_d), sphi = static_cast<float>(sphi_d);
  const float ux = static_cast<float>(u.x), uy = static_cast<float>(u.y), uz = static_cast<float>(u.z);
  const float lo = static_cast<float>(lo_d) - 1e-5f, hi = static_cast<float>(hi_d) + 1e-5f;
  const float rho = sqrtf(ux * ux + uy * uy);
  const float A = cphi * rho, B = sphi * uz;
  if (!(A > 1e-5f)) {  // q.u is B +- A over the whole ring
    if (B + A + 1e-5f >= lo && B - A - 1e-5f <= hi) {
      a0[0] = 0;
      len[0] = cnt;
      return 1;
    }
    return 0;
  }
  const float x_hi = (hi - B) / A, x_lo = (lo - B) / A;
  if (x_lo > 1.0f || x_hi < -1.0f) return 0;
  const float kPiF = 3.14159265358979323846f;
  const float step = 2.0f * kPiF / cnt;
  const float marg = 1.5f * step + 2e-3f;
  const float d_lo = fmaxf(0.0f, (x_hi >= 1.0f ? 0.0f : acosf(fmaxf(-1.0f, x_hi))) - marg);
  const float d_hi = fminf(kPiF, (x_lo <= -1.0f ? kPiF : acosf(fminf(1.0f, x_lo))) + marg);
  if (d_lo <= 0.0f && d_hi >= kPiF) {
    a0[0] = 0;
    len[0] = cnt;
    return 1;
  }
  const float thu = atan2f(uy, ux);
  int n = 0;
  auto arc = [&](float t0, float t1) {
    const int m0 = static_cast<int>(ceilf(t0 / step)), m1 = static_cast<int>(floorf(t1 / step));
    const int c = m1 - m0 + 1;
    if (c <= 0) return;
    if (c >= cnt) {
      a0[n] = 0;
      len[n++] = cnt;
      return;
    }
    int s0 = m0 % cnt;
    if (s0 < 0) s0 += cnt;
    a0[n] = s0;
    len[n++] = c;
  };
  if (d_lo <= 0.0f) {
    arc(thu - d_hi, thu + d_hi);
  } else {
    arc(thu + d_lo, thu + d_hi);
    arc(thu - d_hi, thu - d_lo);
  }
  return n;
}

/// Merged index intervals [s, e) (ring-local, ascending, disjoint) of up to
/// four arcs; returns the count (<= 8) or -1 for "whole ring".
static __device__ __noinline__ int ring_intervals(int cnt, const int* a0, const int* len, int na, int* is, int* ie) {
  int s[8], e[8], n = 0;
  for (int k = 0; k < na; ++k) {
    if (len[k] >= cnt) return -1;
    const int st = a0[k], en = a0[k] + len[k];
    if (en <= cnt) {
      s[n] = st;
      e[n++] = en;
    } else {  // wraps past the last azimuth
      s[n] = st;
      e[n++] = cnt;
      s[n] = 0;
      e[n++] = en - cnt;
    }
  }
  for (int i = 1; i < n; ++i)  // insertion sort by start
    for (int j = i; j > 0 && s[j] < s[j - 1]; --j) {
      const int ts = s[j], te = e[j];
      s[j] = s[j - 1];
      e[j] = e[j - 1];
      s[j - 1] = ts;
      e[j - 1] = te;
    }
  int m = 0;
  for (int i = 0; i < n; ++i) {
    if (m > 0 && s[i] <= ie[m - 1]) {
      if (e[i] > ie[m - 1]) ie[m - 1] = e[i];
    } else {
      is[m] = s[i];
      ie[m++] = e[i];
    }
  }
  return m;
}


}  // namespace rp
