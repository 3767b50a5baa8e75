// Scratch A/B of the 512^3 fused mark+dilate pass (not part of the product).
// Variants timed as 200 PDL launches in one CUDA graph:
//   k_cur   : replica of k_mark_dilate_rowwise<8,32,256,1> (block-staged prims, 3 block syncs)
//   k_floor : same launch shape, writes zeros through the same bulk-store path (no prims)
//   k_warp  : prims in the kernel-parameter bank, warp-ballot culling, per-warp staging and
//             bulk store, no block barriers
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o dil_floor dil_floor.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <vector>
#include <random>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

struct Prim { int a[3], b[3]; };
struct GridView { int nx, ny, nz, wx; };
constexpr int kMaxP = 64;
struct PrimParams { int np; Prim p[kMaxP]; };

__device__ __forceinline__ uint64_t range_mask(int lo, int hi, int base) {
  const int l = lo - base, h = hi - base;
  if (h < 0 || l > 63) return 0ull;
  const int l2 = l < 0 ? 0 : l, h2 = h > 63 ? 63 : h;
  const uint64_t upto = (h2 == 63) ? ~0ull : ((1ull << (h2 + 1)) - 1ull);
  return upto & ~((1ull << l2) - 1ull);
}

template <int WX>
__global__ void __launch_bounds__(256) k_cur(uint64_t* __restrict__ bits, GridView g,
                                             const Prim* __restrict__ prims, int np,
                                             const int* __restrict__ wtab, int reach) {
  extern __shared__ Prim sp_all[];
  Prim* sp = sp_all + np;
  int* swt = reinterpret_cast<int*>(sp_all + 2 * np);
  __shared__ int ns;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  constexpr int TY = 32, NT = 256, TZ = 8;
  const int yt = blockIdx.x * TY, zt = blockIdx.y * TZ;
  if (threadIdx.x == 0) ns = 0;
  {
    const int* src = reinterpret_cast<const int*>(prims);
    int* dst = reinterpret_cast<int*>(sp_all);
    for (int k = threadIdx.x; k < 6 * np; k += blockDim.x) dst[k] = __ldg(src + k);
    const int nw = 2 * reach * reach + 1;
    for (int k = threadIdx.x; k < nw; k += blockDim.x) swt[k] = __ldg(wtab + k);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < np; k += blockDim.x) {
    const Prim p = sp_all[k];
    if (p.a[2] - reach > zt + TZ - 1 || p.b[2] + reach < zt) continue;
    if (p.a[1] - reach > yt + TY - 1 || p.b[1] + reach < yt) continue;
    sp[atomicAdd(&ns, 1)] = p;
  }
  __syncthreads();
  const int y = yt + threadIdx.x % TY, z = zt + threadIdx.x / TY;
  uint64_t m[WX];
#pragma unroll
  for (int w = 0; w < WX; ++w) m[w] = 0;
  const int n_here = ns;
  for (int k = 0; k < n_here; ++k) {
    const Prim p = sp[k];
    const int dy = y < p.a[1] ? p.a[1] - y : (y > p.b[1] ? y - p.b[1] : 0);
    const int dz = z < p.a[2] ? p.a[2] - z : (z > p.b[2] ? z - p.b[2] : 0);
    if (dy > reach || dz > reach) continue;
    const int wd = swt[dy * dy + dz * dz];
    if (wd < 0) continue;
    int lo = p.a[0] - wd, hi = p.b[0] + wd;
    lo = lo < 0 ? 0 : lo;
    hi = hi > g.nx - 1 ? g.nx - 1 : hi;
#pragma unroll
    for (int w = 0; w < WX; ++w) m[w] |= range_mask(lo, hi, 64 * w);
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __shared__ __align__(128) uint64_t tile[NT * WX];
#pragma unroll
  for (int w = 0; w < WX; ++w) tile[threadIdx.x * WX + w] = m[w];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < TZ) {
    const int zz = zt + threadIdx.x;
    uint64_t* gdst = bits + ((size_t)zz * g.ny + yt) * WX;
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(&tile[threadIdx.x * TY * WX]);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(sa),
                 "r"((uint32_t)(TY * WX * 8)) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
}

template <int WX>
__global__ void __launch_bounds__(256) k_floor(uint64_t* __restrict__ bits, GridView g) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  constexpr int TY = 32, NT = 256, TZ = 8;
  const int yt = blockIdx.x * TY, zt = blockIdx.y * TZ;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __shared__ __align__(128) uint64_t tile[NT * WX];
#pragma unroll
  for (int w = 0; w < WX; ++w) tile[threadIdx.x * WX + w] = threadIdx.x;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < TZ) {
    const int zz = zt + threadIdx.x;
    uint64_t* gdst = bits + ((size_t)zz * g.ny + yt) * WX;
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(&tile[threadIdx.x * TY * WX]);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(sa),
                 "r"((uint32_t)(TY * WX * 8)) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
}

// plain 16-byte coalesced stores, no smem
__global__ void __launch_bounds__(256) k_floor_st(uint64_t* __restrict__ bits, size_t nwords) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const size_t i = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 8;
  if (i + 8 <= nwords) {
    ulonglong2* d = reinterpret_cast<ulonglong2*>(bits + i);
    ulonglong2 v = make_ulonglong2(i, i);
#pragma unroll
    for (int k = 0; k < 4; ++k) d[k] = v;
  }
}

// warp-level: each warp = 32 rows (y) of one plane z; prims from the param bank;
// widths from a global table (L1); warp staging + one bulk store per warp.
template <int WX, int WPB>
__global__ void __launch_bounds__(32 * WPB) k_warp(uint64_t* __restrict__ bits, GridView g,
                                                   const __grid_constant__ PrimParams P,
                                                   const int* __restrict__ wtab, int reach) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  __shared__ __align__(128) uint64_t tile[WPB][32 * WX];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int yt = blockIdx.x * 32;
  const int z = blockIdx.y * WPB + warp;
  const int y = yt + lane;
  uint64_t m[WX];
#pragma unroll
  for (int w = 0; w < WX; ++w) m[w] = 0;
  for (int k0 = 0; k0 < P.np; k0 += 32) {
    bool hit = false;
    const int k = k0 + lane;
    if (k < P.np) {
      const Prim p = P.p[k];
      hit = !(p.a[2] - reach > z || p.b[2] + reach < z || p.a[1] - reach > yt + 31 ||
              p.b[1] + reach < yt);
    }
    unsigned bal = __ballot_sync(0xffffffffu, hit);
    while (bal) {
      const int kk = k0 + __ffs(bal) - 1;
      bal &= bal - 1;
      const Prim p = P.p[kk];
      const int dy = y < p.a[1] ? p.a[1] - y : (y > p.b[1] ? y - p.b[1] : 0);
      const int dz = z < p.a[2] ? p.a[2] - z : (z > p.b[2] ? z - p.b[2] : 0);
      if (dy > reach || dz > reach) continue;
      const int wd = __ldg(wtab + dy * dy + dz * dz);
      if (wd < 0) continue;
      int lo = p.a[0] - wd, hi = p.b[0] + wd;
      lo = lo < 0 ? 0 : lo;
      hi = hi > g.nx - 1 ? g.nx - 1 : hi;
#pragma unroll
      for (int w = 0; w < WX; ++w) m[w] |= range_mask(lo, hi, 64 * w);
    }
  }
#pragma unroll
  for (int w = 0; w < WX; ++w) tile[warp][lane * WX + w] = m[w];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (lane == 0) {
    uint64_t* gdst = bits + ((size_t)z * g.ny + yt) * WX;
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(&tile[warp][0]);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(sa),
                 "r"((uint32_t)(32 * WX * 8)) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
}

// warp-level with direct 16B stores from registers (each lane owns a 64 B row):
// 4 store instructions per warp cover the 2 KB run fully.
template <int WX, int WPB>
__global__ void __launch_bounds__(32 * WPB) k_warp_st(uint64_t* __restrict__ bits, GridView g,
                                                      const __grid_constant__ PrimParams P,
                                                      const int* __restrict__ wtab, int reach) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int yt = blockIdx.x * 32;
  const int z = blockIdx.y * WPB + warp;
  const int y = yt + lane;
  uint64_t m[WX];
#pragma unroll
  for (int w = 0; w < WX; ++w) m[w] = 0;
  for (int k0 = 0; k0 < P.np; k0 += 32) {
    bool hit = false;
    const int k = k0 + lane;
    if (k < P.np) {
      const Prim p = P.p[k];
      hit = !(p.a[2] - reach > z || p.b[2] + reach < z || p.a[1] - reach > yt + 31 ||
              p.b[1] + reach < yt);
    }
    unsigned bal = __ballot_sync(0xffffffffu, hit);
    while (bal) {
      const int kk = k0 + __ffs(bal) - 1;
      bal &= bal - 1;
      const Prim p = P.p[kk];
      const int dy = y < p.a[1] ? p.a[1] - y : (y > p.b[1] ? y - p.b[1] : 0);
      const int dz = z < p.a[2] ? p.a[2] - z : (z > p.b[2] ? z - p.b[2] : 0);
      if (dy > reach || dz > reach) continue;
      const int wd = __ldg(wtab + dy * dy + dz * dz);
      if (wd < 0) continue;
      int lo = p.a[0] - wd, hi = p.b[0] + wd;
      lo = lo < 0 ? 0 : lo;
      hi = hi > g.nx - 1 ? g.nx - 1 : hi;
#pragma unroll
      for (int w = 0; w < WX; ++w) m[w] |= range_mask(lo, hi, 64 * w);
    }
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  ulonglong2* row = reinterpret_cast<ulonglong2*>(bits + ((size_t)z * g.ny + y) * WX);
#pragma unroll
  for (int w = 0; w < WX / 2; ++w) row[w] = make_ulonglong2(m[2 * w], m[2 * w + 1]);
}

struct BigParams { int np; int nw; Prim p[kMaxP]; int w[512]; };

__device__ __forceinline__ uint64_t range_mask2(int lo, int hi, int base) {
  // branch-free: bits [lo, hi] of the word starting at base (shift amounts clamped to [0, 64])
  int l = lo - base, h = hi - base + 1;  // [l, h)
  l = min(max(l, 0), 64);
  h = min(max(h, 0), 64);
  const uint64_t a = l >= 64 ? 0ull : (~0ull << l);
  const uint64_t b = h >= 64 ? ~0ull : ((1ull << h) - 1ull);
  return a & b;
}

template <int WX, int ROWS, bool PARAM, bool RM2>
__global__ void __launch_bounds__(ROWS) k_plane(uint64_t* __restrict__ bits, GridView g,
                                                const Prim* __restrict__ prims, int np,
                                                const int* __restrict__ wtab, int reach,
                                                const __grid_constant__ BigParams P) {
  extern __shared__ Prim sp_all[];
  Prim* sp = sp_all + np;
  int* swt = reinterpret_cast<int*>(sp_all + 2 * np);
  __shared__ int ns;
  __shared__ __align__(128) uint64_t tile[ROWS * WX];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int row0 = blockIdx.x * ROWS;  // flat row index z*ny + y
  const int z = row0 / g.ny, yt = row0 % g.ny;
  if (threadIdx.x == 0) ns = 0;
  const int nw = 2 * reach * reach + 1;
  if (PARAM) {
    for (int k = threadIdx.x; k < np; k += blockDim.x) sp_all[k] = P.p[k];
    for (int k = threadIdx.x; k < nw; k += blockDim.x) swt[k] = P.w[k];
  } else {
    const int* src = reinterpret_cast<const int*>(prims);
    int* dst = reinterpret_cast<int*>(sp_all);
    for (int k = threadIdx.x; k < 6 * np; k += blockDim.x) dst[k] = __ldg(src + k);
    for (int k = threadIdx.x; k < nw; k += blockDim.x) swt[k] = __ldg(wtab + k);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < np; k += blockDim.x) {
    const Prim p = sp_all[k];
    if (p.a[2] - reach > z || p.b[2] + reach < z) continue;
    if (p.a[1] - reach > yt + ROWS - 1 || p.b[1] + reach < yt) continue;
    sp[atomicAdd(&ns, 1)] = p;
  }
  __syncthreads();
  const int y = yt + threadIdx.x;
  uint64_t m[WX];
#pragma unroll
  for (int w = 0; w < WX; ++w) m[w] = 0;
  const int n_here = ns;
  for (int k = 0; k < n_here; ++k) {
    const Prim p = sp[k];
    const int dy = y < p.a[1] ? p.a[1] - y : (y > p.b[1] ? y - p.b[1] : 0);
    const int dz = z < p.a[2] ? p.a[2] - z : (z > p.b[2] ? z - p.b[2] : 0);
    if (dy > reach || dz > reach) continue;
    const int wd = swt[dy * dy + dz * dz];
    if (wd < 0) continue;
    int lo = p.a[0] - wd, hi = p.b[0] + wd;
    lo = lo < 0 ? 0 : lo;
    hi = hi > g.nx - 1 ? g.nx - 1 : hi;
#pragma unroll
    for (int w = 0; w < WX; ++w) m[w] |= RM2 ? range_mask2(lo, hi, 64 * w) : range_mask(lo, hi, 64 * w);
  }
#pragma unroll
  for (int w = 0; w < WX; ++w) tile[threadIdx.x * WX + w] = m[w];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) {
    uint64_t* gdst = bits + (size_t)row0 * WX;
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(&tile[0]);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(sa),
                 "r"((uint32_t)(ROWS * WX * 8)) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
}

template <int WX, int ROWS>
__global__ void __launch_bounds__(ROWS) k_floor_plane(uint64_t* __restrict__ bits, GridView g) {
  __shared__ __align__(128) uint64_t tile[ROWS * WX];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#pragma unroll
  for (int w = 0; w < WX; ++w) tile[threadIdx.x * WX + w] = threadIdx.x;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) {
    uint64_t* gdst = bits + (size_t)blockIdx.x * ROWS * WX;
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(&tile[0]);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(sa),
                 "r"((uint32_t)(ROWS * WX * 8)) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
}

// k_cur with branch-free masks
template <int WX>
__global__ void __launch_bounds__(256) k_cur2(uint64_t* __restrict__ bits, GridView g,
                                             const Prim* __restrict__ prims, int np,
                                             const int* __restrict__ wtab, int reach) {
  extern __shared__ Prim sp_all[];
  Prim* sp = sp_all + np;
  int* swt = reinterpret_cast<int*>(sp_all + 2 * np);
  __shared__ int ns;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  constexpr int TY = 32, NT = 256, TZ = 8;
  const int yt = blockIdx.x * TY, zt = blockIdx.y * TZ;
  if (threadIdx.x == 0) ns = 0;
  {
    const int* src = reinterpret_cast<const int*>(prims);
    int* dst = reinterpret_cast<int*>(sp_all);
    for (int k = threadIdx.x; k < 6 * np; k += blockDim.x) dst[k] = __ldg(src + k);
    const int nw = 2 * reach * reach + 1;
    for (int k = threadIdx.x; k < nw; k += blockDim.x) swt[k] = __ldg(wtab + k);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < np; k += blockDim.x) {
    const Prim p = sp_all[k];
    if (p.a[2] - reach > zt + TZ - 1 || p.b[2] + reach < zt) continue;
    if (p.a[1] - reach > yt + TY - 1 || p.b[1] + reach < yt) continue;
    sp[atomicAdd(&ns, 1)] = p;
  }
  __syncthreads();
  const int y = yt + threadIdx.x % TY, z = zt + threadIdx.x / TY;
  uint64_t m[WX];
#pragma unroll
  for (int w = 0; w < WX; ++w) m[w] = 0;
  const int n_here = ns;
  for (int k = 0; k < n_here; ++k) {
    const Prim p = sp[k];
    const int dy = y < p.a[1] ? p.a[1] - y : (y > p.b[1] ? y - p.b[1] : 0);
    const int dz = z < p.a[2] ? p.a[2] - z : (z > p.b[2] ? z - p.b[2] : 0);
    if (dy > reach || dz > reach) continue;
    const int wd = swt[dy * dy + dz * dz];
    if (wd < 0) continue;
    int lo = p.a[0] - wd, hi = p.b[0] + wd;
    lo = lo < 0 ? 0 : lo;
    hi = hi > g.nx - 1 ? g.nx - 1 : hi;
#pragma unroll
    for (int w = 0; w < WX; ++w) m[w] |= range_mask2(lo, hi, 64 * w);
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __shared__ __align__(128) uint64_t tile[NT * WX];
#pragma unroll
  for (int w = 0; w < WX; ++w) tile[threadIdx.x * WX + w] = m[w];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < TZ) {
    const int zz = zt + threadIdx.x;
    uint64_t* gdst = bits + ((size_t)zz * g.ny + yt) * WX;
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(&tile[threadIdx.x * TY * WX]);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(sa),
                 "r"((uint32_t)(TY * WX * 8)) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
}

// plane tile, block-staged prims, warp-level ballot culling (no atomics, one block barrier
// before compute); U32: build the row as 32-bit words
template <int WX, int ROWS, bool U32>
__global__ void __launch_bounds__(ROWS) k_plane_w(uint64_t* __restrict__ bits, GridView g,
                                                  const Prim* __restrict__ prims, int np,
                                                  const int* __restrict__ wtab, int reach) {
  extern __shared__ Prim sp_all[];
  int* swt = reinterpret_cast<int*>(sp_all + 2 * np);
  __shared__ __align__(128) uint64_t tile[ROWS * WX];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int row0 = blockIdx.x * ROWS;
  const int z = row0 / g.ny, yt = row0 % g.ny;
  const int nw = 2 * reach * reach + 1;
  {
    const int* src = reinterpret_cast<const int*>(prims);
    int* dst = reinterpret_cast<int*>(sp_all);
    for (int k = threadIdx.x; k < 6 * np; k += blockDim.x) dst[k] = __ldg(src + k);
    for (int k = threadIdx.x; k < nw; k += blockDim.x) swt[k] = __ldg(wtab + k);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int yw = yt + (threadIdx.x & ~31);
  const int y = yt + threadIdx.x;
  uint64_t m[WX];
  uint32_t m32[2 * WX];
#pragma unroll
  for (int w = 0; w < WX; ++w) m[w] = 0;
#pragma unroll
  for (int w = 0; w < 2 * WX; ++w) m32[w] = 0;
  for (int k0 = 0; k0 < np; k0 += 32) {
    bool hit = false;
    if (k0 + lane < np) {
      const Prim p = sp_all[k0 + lane];
      hit = !(p.a[2] - reach > z || p.b[2] + reach < z || p.a[1] - reach > yw + 31 ||
              p.b[1] + reach < yw);
    }
    unsigned bal = __ballot_sync(0xffffffffu, hit);
    while (bal) {
      const int kk = k0 + __ffs(bal) - 1;
      bal &= bal - 1;
      const Prim p = sp_all[kk];
      const int dy = y < p.a[1] ? p.a[1] - y : (y > p.b[1] ? y - p.b[1] : 0);
      const int dz = z < p.a[2] ? p.a[2] - z : (z > p.b[2] ? z - p.b[2] : 0);
      if (dy > reach || dz > reach) continue;
      const int wd = swt[dy * dy + dz * dz];
      if (wd < 0) continue;
      int lo = p.a[0] - wd, hi = p.b[0] + wd;
      lo = lo < 0 ? 0 : lo;
      hi = hi > g.nx - 1 ? g.nx - 1 : hi;
      if (U32) {
        const uint32_t A = ~0u << (lo & 31), B = ~0u >> (31 - (hi & 31));
        const int wl = lo >> 5, wh = hi >> 5;
#pragma unroll
        for (int w = 0; w < 2 * WX; ++w) {
          uint32_t mk = (w == wl ? A : ~0u) & (w == wh ? B : ~0u);
          m32[w] |= (w >= wl && w <= wh) ? mk : 0u;
        }
      } else {
#pragma unroll
        for (int w = 0; w < WX; ++w) m[w] |= range_mask(lo, hi, 64 * w);
      }
    }
  }
  if (U32) {
#pragma unroll
    for (int w = 0; w < WX; ++w) m[w] = (uint64_t)m32[2 * w] | ((uint64_t)m32[2 * w + 1] << 32);
  }
  // stage: a barrier is needed only because smem prims are shared; tile rows are per thread
#pragma unroll
  for (int w = 0; w < WX; ++w) tile[threadIdx.x * WX + w] = m[w];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) {
    uint64_t* gdst = bits + (size_t)row0 * WX;
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(&tile[0]);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(sa),
                 "r"((uint32_t)(ROWS * WX * 8)) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
}

// plane tile of ROWS rows, NT threads, ROWS/NT rows per thread (strided by NT)
template <int WX, int ROWS, int NT>
__global__ void __launch_bounds__(NT) k_plane_r(uint64_t* __restrict__ bits, GridView g,
                                                const Prim* __restrict__ prims, int np,
                                                const int* __restrict__ wtab, int reach) {
  extern __shared__ Prim sp_all[];
  Prim* sp = sp_all + np;
  int* swt = reinterpret_cast<int*>(sp_all + 2 * np);
  __shared__ int ns;
  __shared__ __align__(128) uint64_t tile[ROWS * WX];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int row0 = blockIdx.x * ROWS;
  const int z = row0 / g.ny, yt = row0 % g.ny;
  if (threadIdx.x == 0) ns = 0;
  const int nw = 2 * reach * reach + 1;
  {
    const int* src = reinterpret_cast<const int*>(prims);
    int* dst = reinterpret_cast<int*>(sp_all);
    for (int k = threadIdx.x; k < 6 * np; k += blockDim.x) dst[k] = __ldg(src + k);
    for (int k = threadIdx.x; k < nw; k += blockDim.x) swt[k] = __ldg(wtab + k);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < np; k += blockDim.x) {
    const Prim p = sp_all[k];
    if (p.a[2] - reach > z || p.b[2] + reach < z) continue;
    if (p.a[1] - reach > yt + ROWS - 1 || p.b[1] + reach < yt) continue;
    sp[atomicAdd(&ns, 1)] = p;
  }
  __syncthreads();
  const int n_here = ns;
#pragma unroll
  for (int r = 0; r < ROWS / NT; ++r) {
    const int y = yt + threadIdx.x + r * NT;
    uint64_t m[WX];
#pragma unroll
    for (int w = 0; w < WX; ++w) m[w] = 0;
    for (int k = 0; k < n_here; ++k) {
      const Prim p = sp[k];
      const int dy = y < p.a[1] ? p.a[1] - y : (y > p.b[1] ? y - p.b[1] : 0);
      const int dz = z < p.a[2] ? p.a[2] - z : (z > p.b[2] ? z - p.b[2] : 0);
      if (dy > reach || dz > reach) continue;
      const int wd = swt[dy * dy + dz * dz];
      if (wd < 0) continue;
      int lo = p.a[0] - wd, hi = p.b[0] + wd;
      lo = lo < 0 ? 0 : lo;
      hi = hi > g.nx - 1 ? g.nx - 1 : hi;
#pragma unroll
      for (int w = 0; w < WX; ++w) m[w] |= range_mask(lo, hi, 64 * w);
    }
#pragma unroll
    for (int w = 0; w < WX; ++w) tile[(threadIdx.x + r * NT) * WX + w] = m[w];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) {
    uint64_t* gdst = bits + (size_t)row0 * WX;
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(&tile[0]);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(sa),
                 "r"((uint32_t)(ROWS * WX * 8)) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
}

// plane tile of ROWS rows, SPLIT threads per row (each WX/SPLIT words)
template <int WX, int ROWS, int SPLIT>
__global__ void __launch_bounds__(ROWS * SPLIT) k_plane_s(uint64_t* __restrict__ bits, GridView g,
                                                const Prim* __restrict__ prims, int np,
                                                const int* __restrict__ wtab, int reach) {
  extern __shared__ Prim sp_all[];
  Prim* sp = sp_all + np;
  int* swt = reinterpret_cast<int*>(sp_all + 2 * np);
  __shared__ int ns;
  __shared__ __align__(128) uint64_t tile[ROWS * WX];
  constexpr int WS = WX / SPLIT;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int row0 = blockIdx.x * ROWS;
  const int z = row0 / g.ny, yt = row0 % g.ny;
  if (threadIdx.x == 0) ns = 0;
  const int nw = 2 * reach * reach + 1;
  {
    const int* src = reinterpret_cast<const int*>(prims);
    int* dst = reinterpret_cast<int*>(sp_all);
    for (int k = threadIdx.x; k < 6 * np; k += blockDim.x) dst[k] = __ldg(src + k);
    for (int k = threadIdx.x; k < nw; k += blockDim.x) swt[k] = __ldg(wtab + k);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < np; k += blockDim.x) {
    const Prim p = sp_all[k];
    if (p.a[2] - reach > z || p.b[2] + reach < z) continue;
    if (p.a[1] - reach > yt + ROWS - 1 || p.b[1] + reach < yt) continue;
    sp[atomicAdd(&ns, 1)] = p;
  }
  __syncthreads();
  const int n_here = ns;
  const int rr = threadIdx.x / SPLIT, part = threadIdx.x % SPLIT;
  const int y = yt + rr;
  const int base = part * WS * 64;
  uint64_t m[WS];
#pragma unroll
  for (int w = 0; w < WS; ++w) m[w] = 0;
  for (int k = 0; k < n_here; ++k) {
    const Prim p = sp[k];
    const int dy = y < p.a[1] ? p.a[1] - y : (y > p.b[1] ? y - p.b[1] : 0);
    const int dz = z < p.a[2] ? p.a[2] - z : (z > p.b[2] ? z - p.b[2] : 0);
    if (dy > reach || dz > reach) continue;
    const int wd = swt[dy * dy + dz * dz];
    if (wd < 0) continue;
    int lo = p.a[0] - wd, hi = p.b[0] + wd;
    lo = lo < 0 ? 0 : lo;
    hi = hi > g.nx - 1 ? g.nx - 1 : hi;
#pragma unroll
    for (int w = 0; w < WS; ++w) m[w] |= range_mask(lo, hi, base + 64 * w);
  }
#pragma unroll
  for (int w = 0; w < WS; ++w) tile[rr * WX + part * WS + w] = m[w];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) {
    uint64_t* gdst = bits + (size_t)row0 * WX;
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(&tile[0]);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(sa),
                 "r"((uint32_t)(ROWS * WX * 8)) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
}

// floor with conflict-free (transposed, wrong-order) staging: timing bound only
template <int WX, int ROWS>
__global__ void __launch_bounds__(ROWS) k_floor_nc(uint64_t* __restrict__ bits, GridView g) {
  __shared__ __align__(128) uint64_t tile[ROWS * WX];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#pragma unroll
  for (int w = 0; w < WX; ++w) tile[w * ROWS + threadIdx.x] = threadIdx.x;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) {
    uint64_t* gdst = bits + (size_t)blockIdx.x * ROWS * WX;
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(&tile[0]);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(sa),
                 "r"((uint32_t)(ROWS * WX * 8)) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
}

// k_plane with rotated staging: store j of lane l writes word (j + l) & 7 of its row
// (register array rotated by l & 7 first: 3 select stages); 2-way bank conflicts instead of 16
template <int ROWS, int MODE>
__global__ void __launch_bounds__(ROWS) k_plane_rot(uint64_t* __restrict__ bits, GridView g,
                                                const Prim* __restrict__ prims, int np,
                                                const int* __restrict__ wtab, int reach) {
  constexpr int WX = 8;
  extern __shared__ Prim sp_all[];
  Prim* sp = sp_all + np;
  int* swt = reinterpret_cast<int*>(sp_all + 2 * np);
  __shared__ int ns;
  __shared__ __align__(128) uint64_t tile[ROWS * WX];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int row0 = blockIdx.x * ROWS;
  const int z = row0 / g.ny, yt = row0 % g.ny;
  if (threadIdx.x == 0) ns = 0;
  const int nw = 2 * reach * reach + 1;
  {
    const int* src = reinterpret_cast<const int*>(prims);
    int* dst = reinterpret_cast<int*>(sp_all);
    for (int k = threadIdx.x; k < 6 * np; k += blockDim.x) dst[k] = __ldg(src + k);
    for (int k = threadIdx.x; k < nw; k += blockDim.x) swt[k] = __ldg(wtab + k);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < np; k += blockDim.x) {
    const Prim p = sp_all[k];
    if (p.a[2] - reach > z || p.b[2] + reach < z) continue;
    if (p.a[1] - reach > yt + ROWS - 1 || p.b[1] + reach < yt) continue;
    sp[atomicAdd(&ns, 1)] = p;
  }
  __syncthreads();
  const int y = yt + threadIdx.x;
  uint64_t m[WX];
#pragma unroll
  for (int w = 0; w < WX; ++w) m[w] = 0;
  const int n_here = ns;
  for (int k = 0; k < n_here; ++k) {
    const Prim p = sp[k];
    const int dy = y < p.a[1] ? p.a[1] - y : (y > p.b[1] ? y - p.b[1] : 0);
    const int dz = z < p.a[2] ? p.a[2] - z : (z > p.b[2] ? z - p.b[2] : 0);
    if (dy > reach || dz > reach) continue;
    const int wd = swt[dy * dy + dz * dz];
    if (wd < 0) continue;
    int lo = p.a[0] - wd, hi = p.b[0] + wd;
    lo = lo < 0 ? 0 : lo;
    hi = hi > g.nx - 1 ? g.nx - 1 : hi;
    if (MODE == 2) {
      const int rot = (threadIdx.x >> 1) & 7;
#pragma unroll
      for (int j = 0; j < WX; ++j) m[j] |= range_mask(lo, hi, 64 * ((j + rot) & 7));
    } else {
#pragma unroll
    for (int w = 0; w < WX; ++w) m[w] |= range_mask(lo, hi, 64 * w);
    }
  }
  if (MODE == 2) {
    // word slot j holds word (j + rot) & 7: conflict-free 8-byte staging stores
    const int rot = (threadIdx.x >> 1) & 7;
    uint64_t* row = &tile[threadIdx.x * WX];
#pragma unroll
    for (int j = 0; j < WX; ++j) row[(j + rot) & 7] = m[j];
  } else if (MODE == 0) {  // wrong order, conflict-free: timing bound
#pragma unroll
    for (int w = 0; w < WX; ++w) tile[w * ROWS + threadIdx.x] = m[w];
  } else {
    const int rot = threadIdx.x & 7;
    // r[j] = m[(j + rot) & 7]
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      const bool b = (rot >> s) & 1;
      uint64_t t[WX];
#pragma unroll
      for (int j = 0; j < WX; ++j) t[j] = b ? m[(j + (1 << s)) & 7] : m[j];
#pragma unroll
      for (int j = 0; j < WX; ++j) m[j] = t[j];
    }
    uint64_t* row = &tile[threadIdx.x * WX];
#pragma unroll
    for (int j = 0; j < WX; ++j) row[(j + rot) & 7] = m[j];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) {
    uint64_t* gdst = bits + (size_t)row0 * WX;
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(&tile[0]);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(sa),
                 "r"((uint32_t)(ROWS * WX * 8)) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
}

template <typename F>
float time_graph(cudaStream_t s, int reps, F launch_one) {
  cudaGraph_t graph;
  cudaGraphExec_t exec;
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  for (int r = 0; r < reps; ++r) launch_one();
  CK(cudaStreamEndCapture(s, &graph));
  CK(cudaGraphInstantiate(&exec, graph, 0));
  CK(cudaGraphLaunch(exec, s));
  CK(cudaStreamSynchronize(s));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int it = 0; it < 5; ++it) {
    cudaEventRecord(e0, s);
    CK(cudaGraphLaunch(exec, s));
    cudaEventRecord(e1, s);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  cudaGraphExecDestroy(exec);
  cudaGraphDestroy(graph);
  return best * 1000.f / reps;  // us per launch
}

template <typename... KArgs, typename... Args>
void pdl(cudaStream_t s, void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...));
}

int main() {
  const int N = 512, WX = 8;
  GridView g{N, N, N, WX};
  const size_t nwords = (size_t)N * N * WX;
  const double r_cells = 15.7;
  const int reach = (int)std::floor(r_cells + 1e-9);
  const double r2 = r_cells * r_cells + 1e-9;
  std::vector<int> w(2 * reach * reach + 1, -1);
  for (int s = 0; s < (int)w.size(); ++s)
    for (int dx = 0; dx <= reach; ++dx)
      if (double(dx) * dx + double(s) <= r2) w[s] = dx;
  std::mt19937 rng(1240);
  std::vector<Prim> prims(40);
  for (auto& p : prims)
    for (int ax = 0; ax < 3; ++ax) {
      int c = rng() % N, h = 4 + rng() % 28;
      p.a[ax] = std::max(0, c - h);
      p.b[ax] = std::min(N - 1, c + h);
    }
  if (FILE* f = fopen("scratch/c5_prims.txt", "r")) {
    prims.clear();
    Prim p;
    while (fscanf(f, "%d %d %d %d %d %d", &p.a[0], &p.b[0], &p.a[1], &p.b[1], &p.a[2], &p.b[2]) == 6) prims.push_back(p);
    fclose(f);
    printf("C5 prims: %zu\n", prims.size());
  }
  const int np = (int)prims.size();
  PrimParams P{};
  P.np = np;
  memcpy(P.p, prims.data(), np * sizeof(Prim));
  uint64_t *d0, *d1, *d2;
  Prim* dp;
  int* dw;
  CK(cudaMalloc(&d0, nwords * 8));
  CK(cudaMalloc(&d1, nwords * 8));
  CK(cudaMalloc(&d2, nwords * 8));
  CK(cudaMalloc(&dp, np * sizeof(Prim)));
  CK(cudaMalloc(&dw, w.size() * 4));
  CK(cudaMemcpy(dp, prims.data(), np * sizeof(Prim), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dw, w.data(), w.size() * 4, cudaMemcpyHostToDevice));
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  const size_t smem = 2 * np * sizeof(Prim) + w.size() * 4;
  const int reps = 200;
  const double mb = nwords * 8.0;
  auto rep = [&](const char* name, float us) {
    printf("%-28s %7.3f us/pass  %7.1f GB/s  frac %.3f\n", name, us, mb / (us * 1e-6) / 1e9,
           mb / (us * 1e-6) / 1e9 / 6558.1);
  };
  rep("k_cur", time_graph(s, reps, [&] { pdl(s, k_cur<8>, dim3(N / 32, N / 8), dim3(256), smem, d0, g, (const Prim*)dp, np, (const int*)dw, reach); }));
  rep("k_floor (bulk, no work)", time_graph(s, reps, [&] { pdl(s, k_floor<8>, dim3(N / 32, N / 8), dim3(256), 0, d2, g); }));
  rep("k_floor_st (16B stores)", time_graph(s, reps, [&] { pdl(s, k_floor_st, dim3((unsigned)(nwords / 8 / 256)), dim3(256), 0, d2, nwords); }));
  rep("memsetAsync", time_graph(s, reps, [&] { CK(cudaMemsetAsync(d2, 0, nwords * 8, s)); }));
  std::vector<uint64_t> h0(nwords), h1(nwords);
  CK(cudaMemcpy(h0.data(), d0, nwords * 8, cudaMemcpyDeviceToHost));
  BigParams BP{};
  BP.np = np; BP.nw = (int)w.size();
  memcpy(BP.p, prims.data(), np * sizeof(Prim));
  memcpy(BP.w, w.data(), w.size() * 4);
  auto check = [&](const char* n) {
    CK(cudaMemcpy(h1.data(), d1, nwords * 8, cudaMemcpyDeviceToHost));
    printf("   %s == k_cur: %d\n", n, (int)(h0 == h1));
    CK(cudaMemset(d1, 0, nwords * 8));
  };
#define PL(R, PA, M2) rep("k_plane<" #R "," #PA "," #M2 ">", time_graph(s, reps, [&] { pdl(s, k_plane<8, R, PA, M2>, dim3(N * N / R), dim3(R), smem, d1, g, (const Prim*)dp, np, (const int*)dw, reach, BP); })); check("k_plane");
#define PW(R, U) rep("k_plane_w<" #R "," #U ">", time_graph(s, reps, [&] { pdl(s, k_plane_w<8, R, U>, dim3(N * N / R), dim3(R), smem, d1, g, (const Prim*)dp, np, (const int*)dw, reach); })); check("k_plane_w");
#define PR(R, T) rep("k_plane_r<" #R "," #T ">", time_graph(s, reps, [&] { pdl(s, k_plane_r<8, R, T>, dim3(N * N / R), dim3(T), smem, d1, g, (const Prim*)dp, np, (const int*)dw, reach); })); check("k_plane_r");
#define PS(R, S) rep("k_plane_s<" #R "," #S ">", time_graph(s, reps, [&] { pdl(s, k_plane_s<8, R, S>, dim3(N * N / R), dim3(R * S), smem, d1, g, (const Prim*)dp, np, (const int*)dw, reach); })); check("k_plane_s");
  rep("k_floor_plane<256>", time_graph(s, reps, [&] { pdl(s, k_floor_plane<8, 256>, dim3(N * N / 256), dim3(256), 0, d2, g); }));
  rep("k_floor_nc<256>", time_graph(s, reps, [&] { pdl(s, k_floor_nc<8, 256>, dim3(N * N / 256), dim3(256), 0, d2, g); }));
  rep("k_floor_nc<128>", time_graph(s, reps, [&] { pdl(s, k_floor_nc<8, 128>, dim3(N * N / 128), dim3(128), 0, d2, g); }));
#define PT(R, M) rep("k_plane_rot<" #R "," #M ">", time_graph(s, reps, [&] { pdl(s, k_plane_rot<R, M>, dim3(N * N / R), dim3(R), smem, d1, g, (const Prim*)dp, np, (const int*)dw, reach); })); check("k_plane_rot");
  PL(256, false, false)
  PT(256, 0)
  PT(256, 1)
  PT(256, 2)
  PT(128, 2)
  PT(512, 2)
  PT(128, 0)
  PT(128, 1)
  PL(256, false, false)
  size_t occ = 0;
  for (auto v : h0) occ += __builtin_popcountll(v);
  printf("occupied %zu of %zu\n", occ, nwords * 64);
  return 0;
}
