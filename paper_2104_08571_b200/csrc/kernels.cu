// kernels.cu -- sm_100a kernels of the split FORCE step.
//
//   k_sweep   (K-A)  one sweep along d, one thread per cell: the paper's
//                    update_state_x / update_state_y node (Listing 8).
//   k_step2d  (K-B)  all sweeps of a 2-D step in one HBM pass.
//   k_fill           set_boundary + halo for every ghost of a partition.
//   k_maxws          max |u| + c over the interior (Listing 8 set_wavespeeds +
//                    then_reduce(Max)).
// All step kernels write the ghost images of the cells they produce (scheme.cuh),
// so no separate boundary or halo kernel runs between steps on one rank.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "async.cuh"
#include "kernels.hpp"
#include "scheme.cuh"

namespace rpl {

constexpr unsigned kFull = 0xffffffffu;

template <typename T>
struct Vec2;
template <>
struct Vec2<double> {
  using type = double2;
};
template <>
struct Vec2<float> {
  using type = float2;
};

template <int D, int L, typename T>
__device__ __forceinline__ void load_cell(const Geom& g, const T* __restrict__ buf, int64_t x,
                                          int64_t y, int64_t z, T* v) {
#pragma unroll
  for (int c = 0; c < D + 2; ++c) v[c] = buf[g.at(c, x, y, z)];
}

// Cold path: ghost images of one boundary cell.  Values travel in registers,
// the launch arguments are read in place (__grid_constant__).
template <int D, int L, typename T>
__device__ __noinline__ void images_nl(const KArgs<T>* a, int64_t x, int64_t y, int64_t z, T v0,
                                       T v1, T v2, T v3, T v4) {
  const T v[5] = {v0, v1, v2, v3, v4};
  write_images<D, L>(a->g, a->outs, a->lo, x, y, z, v);
}

template <int D, int L, typename T>
__device__ __forceinline__ void images(const KArgs<T>& a, int64_t x, int64_t y, int64_t z,
                                       const T* v) {
  if (L == 0 && a.g.img_fast) {
    images_single<D>(a.g, a.out, (int)x, (int)y, (int)z, v);
    return;
  }
  images_nl<D, L, T>(&a, x, y, z, v[0], v[1], v[2], v[3], D > 2 ? v[4] : T(0));
}

// ---------------------------------------------------------------------------
// K-A: one sweep along d.  Thread per interior cell; both faces of the cell are
// evaluated (the simple, unfused baseline: 3 flux evaluations + 2 faces).
// ---------------------------------------------------------------------------
template <typename T, int D, int d, int L>
__global__ void __launch_bounds__(256) k_sweep(const __grid_constant__ KArgs<T> a) {
  constexpr int C = D + 2;
  const Geom& g = a.g;
  const int64_t n = g.cells();
  Coef<T> k;
  if (!step_coef(a, k)) return;
  const bool ws = a.cf.dev != nullptr && a.cf.last;
  const T gam = (T)a.cf.gamma;
  T wmax = T(0);
  int bad = 0, nan = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = i % g.S[0];
    const int64_t y = (i / g.S[0]) % g.S[1];
    const int64_t z = i / (g.S[0] * g.S[1]);
    const int64_t dm[3] = {d == 0 ? 1 : 0, d == 1 ? 1 : 0, d == 2 ? 1 : 0};
    T Um[C], U0[C], Up[C], Fm[C], F0[C], Fp[C];
    load_cell<D, L>(g, a.in, x - dm[0], y - dm[1], z - dm[2], Um);
    load_cell<D, L>(g, a.in, x, y, z, U0);
    load_cell<D, L>(g, a.in, x + dm[0], y + dm[1], z + dm[2], Up);
    phys_flux<D, d>(Um, Fm, a.gm1);
    bad |= phys_flux<D, d>(U0, F0, a.gm1);
    phys_flux<D, d>(Up, Fp, a.gm1);
    T PL[C], PR[C], o[C];
    force_face<D, d>(Um, Fm, U0, F0, PL, k.q[d], k.nq2[d], a.gm1);
    force_face<D, d>(U0, F0, Up, Fp, PR, k.q[d], k.nq2[d], a.gm1);
#pragma unroll
    for (int c = 0; c < C; ++c) o[c] = U0[c] - (PR[c] - PL[c]);
    nan = max(nan, max(naninf(o[0]), naninf(o[C - 1])));
    store_cell<D, L>(g, a.out, x, y, z, o);
    if (ws) wmax = fmax(wmax, wavespeed<D>(o, a.gm1, gam));
    if (near_face<D>(g, x, y, z)) images<D, L>(a, x, y, z, o);
  }
  if (bad < 0 || nan >= kExpMask<T>) atomicOr(a.flag, 1u);
  if (ws) publish_max(a, wmax);
}

// ---------------------------------------------------------------------------
// K-A, order 2: one sweep along d with MUSCL-Hancock + FORCE.  Thread
// per interior cell: loads U_{i-2..i+2}, evolves the boundary values of cells
// i-1, i, i+1 (hancock), FORCE at faces i-1/2 and i+1/2, update.
// ---------------------------------------------------------------------------
template <typename T, int D, int d, int L>
__global__ void __launch_bounds__(256) k_sweep2(const __grid_constant__ KArgs<T> a) {
  constexpr int C = D + 2;
  const Geom& g = a.g;
  const int64_t n = g.cells();
  Coef<T> k;
  if (!step_coef(a, k)) return;
  const bool ws = a.cf.dev != nullptr && a.cf.last;
  const T gam = (T)a.cf.gamma;
  T wmax = T(0);
  int bad = 0, nan = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = i % g.S[0];
    const int64_t y = (i / g.S[0]) % g.S[1];
    const int64_t z = i / (g.S[0] * g.S[1]);
    const int64_t dm[3] = {d == 0 ? 1 : 0, d == 1 ? 1 : 0, d == 2 ? 1 : 0};
    T U[5][C];
#pragma unroll
    for (int j = 0; j < 5; ++j)
      load_cell<D, L>(g, a.in, x + (j - 2) * dm[0], y + (j - 2) * dm[1], z + (j - 2) * dm[2], U[j]);
    T bL[3][C], FbL[3][C], bR[3][C], FbR[3][C];
#pragma unroll
    for (int j = 0; j < 3; ++j)
      bad |= hancock<D, d>(U[j], U[j + 1], U[j + 2], k.h2[d], a.gm1, bL[j], FbL[j], bR[j], FbR[j]);
    T PL[C], PR[C], o[C];
    force_face<D, d>(bR[0], FbR[0], bL[1], FbL[1], PL, k.q[d], k.nq2[d], a.gm1);
    force_face<D, d>(bR[1], FbR[1], bL[2], FbL[2], PR, k.q[d], k.nq2[d], a.gm1);
#pragma unroll
    for (int c = 0; c < C; ++c) o[c] = U[2][c] - (PR[c] - PL[c]);
    nan = max(nan, max(naninf(o[0]), naninf(o[C - 1])));
    store_cell<D, L>(g, a.out, x, y, z, o);
    if (ws) wmax = fmax(wmax, wavespeed<D>(o, a.gm1, gam));
    if (near_face<D>(g, x, y, z)) images<D, L>(a, x, y, z, o);
  }
  if (bad < 0 || nan >= kExpMask<T>) atomicOr(a.flag, 1u);
  if (ws) publish_max(a, wmax);
}

// ---------------------------------------------------------------------------
// K-B (2-D): x-sweep and y-sweep of one step fused into a single pass.
//
// A warp owns a 64-slot window of one row (lane l holds slots 2l, 2l+1 as one
// 128-bit (fp64) / 64-bit (fp32) vector; slot s <-> x = 62 w - 1 + s) and marches
// down a chunk of `rows` rows.  For each row: vector-load U (prefetched one row
// ahead), x-sweep in registers (face values shared across lanes with warp
// shuffles; slots 0 and 63 are the window's halo), then the y-face between this
// row and the previous one from the march state (previous U*, F_y(U*), previous
// y-face), update and store the previous row.  HBM traffic per cell: one read of
// U^n, one write of U^{n+1}; the window's x-halo (2 of 64 slots) and the chunk's
// 2 halo rows are recomputed, not re-stored.  Vector loads are aligned because
// the layout puts x = -1 on an even element offset (geometry.hpp).
// ---------------------------------------------------------------------------
template <typename T>
struct Vert {  // y-march state of the lane's two cells (a, b)
  T us[2][4];  // U* of the previous row
  T fy[2][4];  // F_y(U*) of the previous row
  T ph[2][4];  // previous y-face (scaled flux)
};

template <typename T>
struct Ctx2 {  // loop-invariant per-lane data of k_step2d
  const T* src;
  T* dst;
  int64_t rs, cp;
  bool va, vb, ina, inb, xa_face, xb_face;
  int64_t xa;
  T gm1, qx, nqx, qy, nqy;
  int pad, sy;
};

// x-sweep of the row held in u (lane's 2 cells), then F_y of the result.
template <typename T>
__device__ __forceinline__ void xsweep2(const Ctx2<T>& k, const typename Vec2<T>::type* u,
                                        T (&S)[2][4], T (&G)[2][4], int& bad) {
  constexpr int D = 2, C = 4;
  T Ua[C], Ub[C], Fa[C], Fb[C], Pab[C], Pbn[C], Un[C], Fn[C];
#pragma unroll
  for (int c = 0; c < C; ++c) {
    Ua[c] = u[c].x;
    Ub[c] = u[c].y;
  }
  const int ba = phys_flux<D, 0>(Ua, Fa, k.gm1);
  const int bb = phys_flux<D, 0>(Ub, Fb, k.gm1);
  bad |= (k.ina ? ba : 0) | (k.inb ? bb : 0);
  force_face<D, 0>(Ua, Fa, Ub, Fb, Pab, k.qx, k.nqx, k.gm1);
#pragma unroll
  for (int c = 0; c < C; ++c) {
    Un[c] = __shfl_down_sync(kFull, Ua[c], 1);
    Fn[c] = __shfl_down_sync(kFull, Fa[c], 1);
  }
  force_face<D, 0>(Ub, Fb, Un, Fn, Pbn, k.qx, k.nqx, k.gm1);
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const T Ppa = __shfl_up_sync(kFull, Pbn[c], 1);
    S[0][c] = Ua[c] - (Pab[c] - Ppa);
    S[1][c] = Ub[c] - (Pbn[c] - Pab[c]);
  }
  const int ya = phys_flux<D, 1>(S[0], G[0], k.gm1);
  const int yb = phys_flux<D, 1>(S[1], G[1], k.gm1);
  bad |= (k.va ? ya : 0) | (k.vb ? yb : 0);
}

// One march step at row y (>= y0+1): x-sweep row y (already fetched into `cur`),
// y-face y-1/2, update and store row y-1.
template <typename T>
__device__ __forceinline__ void march2(const KArgs<T>& a, const Ctx2<T>& k, int y, T* dst,
                                       const typename Vec2<T>::type* cur, const Vert<T>& in,
                                       Vert<T>& out, int& bad, int& nan) {
  constexpr int D = 2, C = 4;
  using V = typename Vec2<T>::type;
  xsweep2(k, cur, out.us, out.fy, bad);
#pragma unroll
  for (int h = 0; h < 2; ++h)
    force_face<D, 1>(in.us[h], in.fy[h], out.us[h], out.fy[h], out.ph[h], k.qy, k.nqy, k.gm1);
  T o[2][C];
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int c = 0; c < C; ++c) o[h][c] = in.us[h][c] - (out.ph[h][c] - in.ph[h][c]);
  nan = max(nan, max(max(k.va ? naninf(o[0][0]) : 0, k.va ? naninf(o[0][3]) : 0),
                     max(k.vb ? naninf(o[1][0]) : 0, k.vb ? naninf(o[1][3]) : 0)));
  if (k.va & k.vb) {
#pragma unroll
    for (int c = 0; c < C; ++c) {
      V w;
      w.x = o[0][c];
      w.y = o[1][c];
      *reinterpret_cast<V*>(dst + c * k.cp) = w;
    }
  } else {
    if (k.va) {
#pragma unroll
      for (int c = 0; c < C; ++c) dst[c * k.cp] = o[0][c];
    }
    if (k.vb) {
#pragma unroll
      for (int c = 0; c < C; ++c) dst[c * k.cp + 1] = o[1][c];
    }
  }
  const bool yface = (y - 1 < k.pad) | (y - 1 >= k.sy - k.pad);
  if (k.va && (k.xa_face || yface)) images<D, 0>(a, k.xa, y - 1, 0, o[0]);
  if (k.vb && (k.xb_face || yface)) images<D, 0>(a, k.xa + 1, y - 1, 0, o[1]);
}

// Per-warp ring of kNS row buffers filled by TMA bulk copies (cp.async.bulk):
// each stage holds the window's 4 component sub-rows of one grid row; lane 0
// refills a stage as soon as the warp has consumed it, so kNS-1 rows are in
// flight while the warp computes (no prefetch registers).
constexpr int kNS = 3;

template <typename T>
struct Ring2 {
  static constexpr int RB = 64 * (int)sizeof(T) + 16;  // bytes per component sub-row
  static constexpr int SB = 4 * RB;                    // bytes per stage
  static constexpr int WB = kNS * SB + 64;             // bytes per warp (+ barriers)
  unsigned char* buf;
  uint64_t* bar;
  const char* src0;  // 16-byte aligned global address of row y0-1, component 0
  int64_t rowb, compb;  // bytes between rows / components
  unsigned bytes;       // bytes per component copy
  int shift;            // elements between the aligned start and slot 0
  int krow_end;         // last row counter to fetch

  __device__ __forceinline__ void issue(int kr) {  // lane 0 only
    if (kr > krow_end) return;
    const int s = kr % kNS;
    const char* src = src0 + kr * rowb;
    mbar_arrive_expect_tx(&bar[s], 4 * bytes);
#pragma unroll
    for (int c = 0; c < 4; ++c) bulk_g2s(buf + s * SB + c * RB, src + c * compb, bytes, &bar[s]);
  }
  __device__ __forceinline__ void fetch(int kr, int lane, typename Vec2<T>::type* u) {
    using V = typename Vec2<T>::type;
    const int s = kr % kNS;
    mbar_wait(&bar[s], (kr / kNS) & 1);
    const unsigned char* b = buf + s * SB + (shift + 2 * lane) * (int)sizeof(T);
#pragma unroll
    for (int c = 0; c < 4; ++c) u[c] = *reinterpret_cast<const V*>(b + c * RB);
    __syncwarp();
    if (lane == 0) {
      fence_proxy_async();
      issue(kr + kNS);
    }
  }
};

template <typename T, int MINB>
__global__ void __launch_bounds__(128, MINB) k_step2d(const __grid_constant__ KArgs<T> a, int nwin,
                                                      int ntask) {
  constexpr int D = 2, C = 4;
  using V = typename Vec2<T>::type;
  extern __shared__ __align__(128) unsigned char smem[];
  const Geom& g = a.g;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int wid = blockIdx.x * (blockDim.x >> 5) + wib;
  if (wid >= ntask) return;
  const int win = wid % nwin;
  const int chunk = wid / nwin;
  Ctx2<T> k;
  const int64_t xw = (int64_t)win * kWinOut - 1;  // x of slot 0
  k.xa = xw + 2 * lane;
  const int y0 = chunk * a.rows;
  const int y1 = min(y0 + a.rows, (int)g.S[1]);
  k.rs = g.rstride;
  k.cp = g.cstride;
  k.va = (lane >= 1) & (k.xa < g.S[0]);
  k.vb = (lane <= 30) & (k.xa + 1 < g.S[0]);
  k.ina = (k.xa >= -1) & (k.xa <= g.S[0]);
  k.inb = (k.xa + 1 >= -1) & (k.xa + 1 <= g.S[0]);
  k.xa_face = k.va & ((k.xa < g.pad) | (k.xa >= g.S[0] - g.pad));
  k.xb_face = k.vb & ((k.xa + 1 < g.pad) | (k.xa + 1 >= g.S[0] - g.pad));
  k.gm1 = a.gm1;
  k.qx = a.q[0];
  k.nqx = a.nq2[0];
  k.qy = a.q[1];
  k.nqy = a.nq2[1];
  k.pad = g.pad;
  k.sy = (int)g.S[1];

  Ring2<T> ring;
  ring.buf = smem + wib * Ring2<T>::WB;
  ring.bar = reinterpret_cast<uint64_t*>(ring.buf + kNS * Ring2<T>::SB);
  const T* w0 = a.in + g.row(y0 - 1, 0) * k.rs + g.xo + xw;
  const uintptr_t mis = reinterpret_cast<uintptr_t>(w0) & 15;
  ring.src0 = reinterpret_cast<const char*>(w0) - mis;
  ring.shift = (int)(mis / sizeof(T));
  ring.bytes = 64 * sizeof(T) + (mis ? 16 : 0);
  ring.rowb = k.rs * (int64_t)sizeof(T);
  ring.compb = k.cp * (int64_t)sizeof(T);
  ring.krow_end = y1 - (y0 - 1);
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < kNS; ++s) mbar_init(&ring.bar[s], 1);
    fence_barrier_init();
#pragma unroll
    for (int s = 0; s < kNS; ++s) ring.issue(s);
  }
  __syncwarp();

  T* dst = a.out + g.row(y0, 0) * k.rs + g.xo + k.xa;
  int bad = 0, nan = 0;
  // prologue: rows y0-1 and y0 (no update yet)
  Vert<T> s0, s1;
  V r[C];
  ring.fetch(0, lane, r);
  xsweep2(k, r, s0.us, s0.fy, bad);
  ring.fetch(1, lane, r);
  xsweep2(k, r, s1.us, s1.fy, bad);
#pragma unroll
  for (int h = 0; h < 2; ++h)
    force_face<D, 1>(s0.us[h], s0.fy[h], s1.us[h], s1.fy[h], s1.ph[h], k.qy, k.nqy, k.gm1);
  // steady state, two rows per iteration (state ping-pongs s1 -> s0 -> s1)
  int y = y0 + 1;
  for (; y + 1 <= y1; y += 2) {
    ring.fetch(y - (y0 - 1), lane, r);
    march2(a, k, y, dst, r, s1, s0, bad, nan);
    dst += k.rs;
    ring.fetch(y + 1 - (y0 - 1), lane, r);
    march2(a, k, y + 1, dst, r, s0, s1, bad, nan);
    dst += k.rs;
  }
  if (y <= y1) {
    ring.fetch(y - (y0 - 1), lane, r);
    march2(a, k, y, dst, r, s1, s0, bad, nan);
  }
  if (__any_sync(kFull, bad < 0 || nan >= kExpMask<T>) && lane == 0) atomicOr(a.flag, 1u);
}

// ---------------------------------------------------------------------------
// K-B (2-D), tile form: one CTA = one x-window (W = 32V slots, W-2 outputs) x
// NW-2 output rows; warp j owns row y0-1+j (warps 0 and NW-1 are the y-halo).
//   X  each warp loads its row (coalesced 64/128-bit vectors), x-sweeps it in
//      registers (shuffles share faces), evaluates F_y and publishes (U*, F_y)
//      in shared memory;
//   Y  warp j >= 1 computes the y-face between rows j-1 and j once, publishes it;
//      warps 1..NW-2 update and store.
// No per-warp march: every warp does one row, so the SM holds many short,
// independent warps (the fused step is latency-bound on long dependency chains
// otherwise).  Recompute: the 2 halo rows per NW-2 rows and
// the 2 halo slots per window.
// ---------------------------------------------------------------------------
template <typename T, int V>
struct VecV;
template <typename T>
struct VecV<T, 1> {
  using type = T;
};
template <typename T>
struct VecV<T, 2> {
  using type = typename Vec2<T>::type;
};

template <typename T, int V, int NW>
__global__ void __launch_bounds__(32 * NW) k_step2d_tile(const __grid_constant__ KArgs<T> a,
                                                         int nwin) {
  constexpr int D = 2, C = 4, W = 32 * V;
  using VT = typename VecV<T, V>::type;
  __shared__ T xy[NW][2 * C][W];
  __shared__ T fy[NW - 1][C][W];
  const Geom& g = a.g;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int win = blockIdx.x % nwin;
  const int yb = blockIdx.x / nwin;
  const int xw = win * (W - 2) - 1;
  const int y0 = yb * (NW - 2);
  const int yr = y0 - 1 + warp;
  const int SX = (int)g.S[0], SY = (int)g.S[1];
  const bool row_in = yr <= SY;  // rows -1..SY hold interior/ghost data
  const bool row_out = (warp >= 1) & (warp <= NW - 2) & (yr < SY);
  const T gm1 = a.gm1;
  int xs[V];
  bool out_ok[V], in_ok[V], xface[V];
#pragma unroll
  for (int v = 0; v < V; ++v) {
    xs[v] = xw + V * lane + v;
    const int slot = V * lane + v;
    out_ok[v] = (slot >= 1) & (slot <= W - 2) & (xs[v] < SX);
    in_ok[v] = (xs[v] >= -1) & (xs[v] <= SX);
    xface[v] = (xs[v] < g.pad) | (xs[v] >= SX - g.pad);
  }
  int bad = 0, nan = 0;
  // ---- X
  T U[V][C], F[V][C], S_[V][C], G[V][C];
  if (row_in) {
    const T* src = a.in + g.row(yr, 0) * g.rstride + g.xo + xw + V * lane;
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const VT u = *reinterpret_cast<const VT*>(src + c * g.cstride);
      if constexpr (V == 1) {
        U[0][c] = u;
      } else {
        U[0][c] = u.x;
        U[1][c] = u.y;
      }
    }
  } else {
#pragma unroll
    for (int v = 0; v < V; ++v)
#pragma unroll
      for (int c = 0; c < C; ++c) U[v][c] = (c == 0 || c == C - 1) ? T(1) : T(0);
  }
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const int b = phys_flux<D, 0>(U[v], F[v], gm1);
    bad |= (in_ok[v] & row_in) ? b : 0;
  }
  {
    T Pin[C], Pnx[C], Un[C], Fn[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
      Un[c] = __shfl_down_sync(kFull, U[0][c], 1);
      Fn[c] = __shfl_down_sync(kFull, F[0][c], 1);
    }
    force_face<D, 0>(U[V - 1], F[V - 1], Un, Fn, Pnx, a.q[0], a.nq2[0], gm1);
    if constexpr (V == 2) force_face<D, 0>(U[0], F[0], U[1], F[1], Pin, a.q[0], a.nq2[0], gm1);
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const T Ppv = __shfl_up_sync(kFull, Pnx[c], 1);
      if constexpr (V == 2) {
        S_[0][c] = U[0][c] - (Pin[c] - Ppv);
        S_[1][c] = U[1][c] - (Pnx[c] - Pin[c]);
      } else {
        S_[0][c] = U[0][c] - (Pnx[c] - Ppv);
      }
    }
  }
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const int b = phys_flux<D, 1>(S_[v], G[v], gm1);
    bad |= (out_ok[v] & row_in) ? b : 0;
  }
#pragma unroll
  for (int c = 0; c < C; ++c)
#pragma unroll
    for (int v = 0; v < V; ++v) {
      xy[warp][c][V * lane + v] = S_[v][c];
      xy[warp][C + c][V * lane + v] = G[v][c];
    }
  __syncthreads();
  // ---- Y face between rows warp-1 and warp
  T Py[V][C];
  if (warp >= 1) {
#pragma unroll
    for (int v = 0; v < V; ++v) {
      T Sp[C], Gp[C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        Sp[c] = xy[warp - 1][c][V * lane + v];
        Gp[c] = xy[warp - 1][C + c][V * lane + v];
      }
      force_face<D, 1>(Sp, Gp, S_[v], G[v], Py[v], a.q[1], a.nq2[1], gm1);
#pragma unroll
      for (int c = 0; c < C; ++c) fy[warp - 1][c][V * lane + v] = Py[v][c];
    }
  }
  __syncthreads();
  // ---- update + store
  if (row_out) {
    T* dst = a.out + g.row(yr, 0) * g.rstride + g.xo + xw + V * lane;
    T o[V][C];
#pragma unroll
    for (int v = 0; v < V; ++v)
#pragma unroll
      for (int c = 0; c < C; ++c) o[v][c] = S_[v][c] - (fy[warp][c][V * lane + v] - Py[v][c]);
    const bool yface = (yr < g.pad) | (yr >= SY - g.pad);
    if constexpr (V == 2) {
      if (out_ok[0] & out_ok[1]) {
#pragma unroll
        for (int c = 0; c < C; ++c) {
          VT w;
          w.x = o[0][c];
          w.y = o[1][c];
          *reinterpret_cast<VT*>(dst + c * g.cstride) = w;
        }
      } else {
#pragma unroll
        for (int v = 0; v < V; ++v)
          if (out_ok[v])
#pragma unroll
            for (int c = 0; c < C; ++c) dst[c * g.cstride + v] = o[v][c];
      }
    } else {
      if (out_ok[0])
#pragma unroll
        for (int c = 0; c < C; ++c) dst[c * g.cstride] = o[0][c];
    }
#pragma unroll
    for (int v = 0; v < V; ++v) {
      if (out_ok[v]) {
        nan = max(nan, max(naninf(o[v][0]), naninf(o[v][C - 1])));
        if (xface[v] | yface) images<D, 0>(a, xs[v], yr, 0, o[v]);
      }
    }
  }
  if (__any_sync(kFull, bad < 0 || nan >= kExpMask<T>) && lane == 0) atomicOr(a.flag, 1u);
}

template <typename T, int V, int NW>
static void launch_tile2d(const KArgs<T>& a, cudaStream_t s) {
  constexpr int W = 32 * V;
  const int nwin = (int)((a.g.S[0] + (W - 2) - 1) / (W - 2));
  const int nyb = (int)((a.g.S[1] + (NW - 2) - 1) / (NW - 2));
  k_step2d_tile<T, V, NW><<<nwin * nyb, 32 * NW, 0, s>>>(a, nwin);
}

// ---------------------------------------------------------------------------
// K-B (2-D), persistent TMA form (the default).  Same tile work as
// k_step2d_tile, but each CTA loops over tiles and one elected thread streams
// the next tiles' input boxes [NW rows][C comps][W slots] into a 2-stage
// shared-memory ring with cp.async.bulk.tensor (TMA, mbarrier completion), so
// HBM latency overlaps the previous tile's compute.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void tma_load_box(void* dst, const CUtensorMap* map, uint64_t* bar,
                                             int x, int c, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(c), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

template <typename T, int V, int NW>
struct SmemPT {
  static constexpr int W = 32 * V, C = 4;
  // TMA boxes must start 16-byte aligned in x: load AL extra elements from the
  // aligned-down coordinate and skip `shift` of them when reading
  static constexpr int AL = 16 / (int)sizeof(T);
  static constexpr int WB = W + AL;
  static constexpr int STAGE = NW * C * WB;
  static constexpr int XY = NW * 2 * C * W;
  static constexpr int FY = (NW - 1) * C * W;
  static constexpr size_t bytes() { return (size_t)(2 * STAGE + XY + FY) * sizeof(T) + 64; }
};

template <typename T, int V, int NW, int MB>
__global__ void __launch_bounds__(32 * NW, MB)
    k_step2d_pt(const __grid_constant__ KArgs<T> a, const __grid_constant__ CUtensorMap tmap,
                int nwin, int ntiles) {
  constexpr int D = 2, C = 4, W = 32 * V;
  using SM = SmemPT<T, V, NW>;
  using VT = typename VecV<T, V>::type;
  extern __shared__ __align__(1024) unsigned char smem[];
  T* stage = reinterpret_cast<T*>(smem);
  T* xy = stage + 2 * SM::STAGE;
  T* fy = xy + SM::XY;
  uint64_t* bar = reinterpret_cast<uint64_t*>(fy + SM::FY);
  const Geom& g = a.g;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int SX = (int)g.S[0], SY = (int)g.S[1];
  const int G = gridDim.x;
  Coef<T> kc;
  if (!step_coef(a, kc)) return;
  const bool ws = a.cf.dev != nullptr;
  const T gam = (T)a.cf.gamma;
  T wmax = T(0);
  const T gm1 = a.gm1, qx = kc.q[0], nqx = kc.nq2[0], qy = kc.q[1], nqy = kc.nq2[1];
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
  }
  __syncthreads();
  auto issue = [&](int i) {
    const int tile = blockIdx.x + i * G;
    if (tile >= ntiles) return;
    const int s = i & 1;
    const int w = tile % nwin, yb = tile / nwin;
    mbar_arrive_expect_tx(&bar[s], SM::STAGE * (unsigned)sizeof(T));
    const int x0 = (int)g.xo + w * (W - 2) - 1;
    tma_load_box(stage + s * SM::STAGE, &tmap, &bar[s], x0 - x0 % SM::AL, 0,
                 (int)g.off[1] + yb * (NW - 2) - 1, 0);
  };
  if (threadIdx.x == 0) {
    issue(0);
    issue(1);
  }
  int bad = 0, nan = 0;
  // tile t = blockIdx.x + i G  <->  (win, yb) = (t % nwin, t / nwin), advanced
  // incrementally (no per-tile integer division)
  const int Gq = G / nwin, Gr = G - (G / nwin) * nwin;
  int win = (int)blockIdx.x % nwin, yb = (int)blockIdx.x / nwin;
  const int nyb = ntiles / nwin;
  const int64_t cs = g.cstride;
  for (int i = 0;; ++i) {
    if (yb >= nyb) break;
    const int xw = win * (W - 2) - 1;
    const int yr = yb * (NW - 2) - 1 + warp;
    const bool row_in = yr <= SY;
    const bool row_out = (warp >= 1) & (warp <= NW - 2) & (yr < SY);
    const int s = i & 1;
    mbar_wait(&bar[s], (i >> 1) & 1);
    // ---- X
    T U[V][C], F[V][C], S_[V][C], G_[V][C];
    {
      const int sh = ((int)g.xo + xw) % SM::AL;
      const T* st = stage + s * SM::STAGE + warp * C * SM::WB + sh + V * lane;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const VT u = *reinterpret_cast<const VT*>(st + c * SM::WB);
        if constexpr (V == 1) {
          U[0][c] = u;
        } else {
          U[0][c] = u.x;
          U[1][c] = u.y;
        }
      }
    }
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int xv = xw + V * lane + v;
      const int b = phys_flux<D, 0>(U[v], F[v], gm1);
      bad |= ((xv >= -1) & (xv <= SX) & row_in) ? b : 0;
    }
    {
      T Pin[C], Pnx[C], Un[C], Fn[C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        Un[c] = __shfl_down_sync(kFull, U[0][c], 1);
        Fn[c] = __shfl_down_sync(kFull, F[0][c], 1);
      }
      force_face<D, 0>(U[V - 1], F[V - 1], Un, Fn, Pnx, qx, nqx, gm1);
      if constexpr (V == 2) force_face<D, 0>(U[0], F[0], U[1], F[1], Pin, qx, nqx, gm1);
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const T Ppv = __shfl_up_sync(kFull, Pnx[c], 1);
        if constexpr (V == 2) {
          S_[0][c] = U[0][c] - (Pin[c] - Ppv);
          S_[1][c] = U[1][c] - (Pnx[c] - Pin[c]);
        } else {
          S_[0][c] = U[0][c] - (Pnx[c] - Ppv);
        }
      }
    }
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int xv = xw + V * lane + v;
      const int slot = V * lane + v;
      const int b = phys_flux<D, 1>(S_[v], G_[v], gm1);
      bad |= ((slot >= 1) & (slot <= W - 2) & (xv < SX) & row_in) ? b : 0;
    }
    {
      T* xr = xy + warp * 2 * C * W + V * lane;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        VT sv, gv;
        if constexpr (V == 1) {
          sv = S_[0][c];
          gv = G_[0][c];
        } else {
          sv.x = S_[0][c];
          sv.y = S_[1][c];
          gv.x = G_[0][c];
          gv.y = G_[1][c];
        }
        *reinterpret_cast<VT*>(xr + c * W) = sv;
        *reinterpret_cast<VT*>(xr + (C + c) * W) = gv;
      }
    }
    __syncthreads();  // (A) stage s consumed; (U*, F_y) published
    if (threadIdx.x == 0) {
      fence_proxy_async();
      issue(i + 2);
    }
    // ---- Y face between rows warp-1 and warp
    T Py[V][C];
    if (warp >= 1) {
      const T* pr = xy + (warp - 1) * 2 * C * W + V * lane;
      T Sp[V][C], Gp[V][C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const VT sv = *reinterpret_cast<const VT*>(pr + c * W);
        const VT gv = *reinterpret_cast<const VT*>(pr + (C + c) * W);
        if constexpr (V == 1) {
          Sp[0][c] = sv;
          Gp[0][c] = gv;
        } else {
          Sp[0][c] = sv.x;
          Sp[1][c] = sv.y;
          Gp[0][c] = gv.x;
          Gp[1][c] = gv.y;
        }
      }
#pragma unroll
      for (int v = 0; v < V; ++v) force_face<D, 1>(Sp[v], Gp[v], S_[v], G_[v], Py[v], qy, nqy, gm1);
      T* fw = fy + (warp - 1) * C * W + V * lane;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        VT pv;
        if constexpr (V == 1) {
          pv = Py[0][c];
        } else {
          pv.x = Py[0][c];
          pv.y = Py[1][c];
        }
        *reinterpret_cast<VT*>(fw + c * W) = pv;
      }
    }
    __syncthreads();  // (B) y-faces published
    // ---- update + store
    if (row_out) {
      T* dst = a.out + ((int64_t)((int)g.off[1] + yr) * g.rstride + (int)g.xo + xw + V * lane);
      const T* fu = fy + warp * C * W + V * lane;
      T o[V][C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const VT pv = *reinterpret_cast<const VT*>(fu + c * W);
        if constexpr (V == 1) {
          o[0][c] = S_[0][c] - (pv - Py[0][c]);
        } else {
          o[0][c] = S_[0][c] - (pv.x - Py[0][c]);
          o[1][c] = S_[1][c] - (pv.y - Py[1][c]);
        }
      }
      bool ok[V];
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const int slot = V * lane + v;
        ok[v] = (slot >= 1) & (slot <= W - 2) & (xw + slot < SX);
      }
      if constexpr (V == 2) {
        if (ok[0] & ok[1]) {
#pragma unroll
          for (int c = 0; c < C; ++c) {
            VT w;
            w.x = o[0][c];
            w.y = o[1][c];
            *reinterpret_cast<VT*>(dst + c * cs) = w;
          }
        } else {
#pragma unroll
          for (int v = 0; v < V; ++v)
            if (ok[v])
#pragma unroll
              for (int c = 0; c < C; ++c) dst[c * cs + v] = o[v][c];
        }
      } else {
        if (ok[0]) {
          T* p = dst;
#pragma unroll
          for (int c = 0; c < C; ++c) {
            *p = o[0][c];
            p += cs;
          }
        }
      }
      const bool yface = (yr < g.pad) | (yr >= SY - g.pad);
#pragma unroll
      for (int v = 0; v < V; ++v) {
        if (ok[v]) {
          nan = max(nan, max(naninf(o[v][0]), naninf(o[v][C - 1])));
          if (ws) wmax = fmax(wmax, wavespeed<D>(o[v], gm1, gam));
          const int xv = xw + V * lane + v;
          if (yface | (xv < g.pad) | (xv >= SX - g.pad)) images<D, 0>(a, xv, yr, 0, o[v]);
        }
      }
    }
    win += Gr;
    yb += Gq;
    if (win >= nwin) {
      win -= nwin;
      ++yb;
    }
  }
  if (__any_sync(kFull, bad < 0 || nan >= kExpMask<T>) && lane == 0) atomicOr(a.flag, 1u);
  if (ws) publish_max(a, wmax);
}

// ---------------------------------------------------------------------------
// K-B (2-D), low-register form of k_step2d_pt (V = 1): no value stays in
// registers across a CTA barrier -- the Y phase re-reads the row's own (U*, F_y)
// and the update re-reads U* and both y-faces from shared memory -- so each
// phase's live set is its own, for 64-register builds (32 warps / SM).  Same
// arithmetic as k_step2d_pt, bitwise identical results.
// ---------------------------------------------------------------------------
template <typename T, int NW, int MB>
__global__ void __launch_bounds__(32 * NW, MB)
    k_step2d_lr(const __grid_constant__ KArgs<T> a, const __grid_constant__ CUtensorMap tmap,
                int nwin, int ntiles) {
  constexpr int D = 2, C = 4, W = 32;
  using SM = SmemPT<T, 1, NW>;
  extern __shared__ __align__(1024) unsigned char smem[];
  T* stage = reinterpret_cast<T*>(smem);
  T* xy = stage + 2 * SM::STAGE;
  T* fy = xy + SM::XY;
  uint64_t* bar = reinterpret_cast<uint64_t*>(fy + SM::FY);
  const Geom& g = a.g;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int SX = (int)g.S[0], SY = (int)g.S[1];
  const int G = gridDim.x;
  Coef<T> kc;
  if (!step_coef(a, kc)) return;
  const bool ws = a.cf.dev != nullptr;
  const T gam = (T)a.cf.gamma;
  T wmax = T(0);
  const T gm1 = a.gm1;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
  }
  __syncthreads();
  auto issue = [&](int i) {
    const int tile = blockIdx.x + i * G;
    if (tile >= ntiles) return;
    const int s = i & 1;
    const int w = tile % nwin, yb = tile / nwin;
    mbar_arrive_expect_tx(&bar[s], SM::STAGE * (unsigned)sizeof(T));
    const int x0 = (int)g.xo + w * (W - 2) - 1;
    tma_load_box(stage + s * SM::STAGE, &tmap, &bar[s], x0 - x0 % SM::AL, 0,
                 (int)g.off[1] + yb * (NW - 2) - 1, 0);
  };
  if (threadIdx.x == 0) {
    issue(0);
    issue(1);
  }
  int bad = 0, nan = 0;
  const int Gq = G / nwin, Gr = G - (G / nwin) * nwin;
  int win = (int)blockIdx.x % nwin, yb = (int)blockIdx.x / nwin;
  const int nyb = ntiles / nwin;
  const int64_t cs = g.cstride;
  T* const xr = xy + warp * 2 * C * W + lane;  // this row's (U*, F_y)
  for (int i = 0;; ++i) {
    if (yb >= nyb) break;
    const int xw = win * (W - 2) - 1;
    const int yr = yb * (NW - 2) - 1 + warp;
    const int xv = xw + lane;
    const bool row_in = yr <= SY;
    const int s = i & 1;
    mbar_wait(&bar[s], (i >> 1) & 1);
    // ---- X
    {
      T U[C], F[C];
      const int sh = ((int)g.xo + xw) % SM::AL;
      const T* st = stage + s * SM::STAGE + warp * C * SM::WB + sh + lane;
#pragma unroll
      for (int c = 0; c < C; ++c) U[c] = st[c * SM::WB];
      const int b0 = phys_flux<D, 0>(U, F, gm1);
      bad |= ((xv >= -1) & (xv <= SX) & row_in) ? b0 : 0;
      T Pnx[C];
      {
        T Un[C], Fn[C];
#pragma unroll
        for (int c = 0; c < C; ++c) {
          Un[c] = __shfl_down_sync(kFull, U[c], 1);
          Fn[c] = __shfl_down_sync(kFull, F[c], 1);
        }
        force_face<D, 0>(U, F, Un, Fn, Pnx, kc.q[0], kc.nq2[0], gm1);
      }
      T S_[C], G_[C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const T Ppv = __shfl_up_sync(kFull, Pnx[c], 1);
        S_[c] = U[c] - (Pnx[c] - Ppv);
      }
      const int b1 = phys_flux<D, 1>(S_, G_, gm1);
      bad |= ((lane >= 1) & (lane <= W - 2) & (xv < SX) & row_in) ? b1 : 0;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        xr[c * W] = S_[c];
        xr[(C + c) * W] = G_[c];
      }
    }
    __syncthreads();  // (A) stage s consumed; (U*, F_y) published
    if (threadIdx.x == 0) {
      fence_proxy_async();
      issue(i + 2);
    }
    // ---- Y face between rows warp-1 and warp
    if (warp >= 1) {
      T Sp[C], Gp[C], S_[C], G_[C], Py[C];
      const T* pr = xr - 2 * C * W;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        Sp[c] = pr[c * W];
        Gp[c] = pr[(C + c) * W];
        S_[c] = xr[c * W];
        G_[c] = xr[(C + c) * W];
      }
      force_face<D, 1>(Sp, Gp, S_, G_, Py, kc.q[1], kc.nq2[1], gm1);
      T* fw = fy + (warp - 1) * C * W + lane;
#pragma unroll
      for (int c = 0; c < C; ++c) fw[c * W] = Py[c];
    }
    __syncthreads();  // (B) y-faces published
    // ---- update + store
    if ((warp >= 1) & (warp <= NW - 2) & (yr < SY) & (lane >= 1) & (lane <= W - 2) & (xv < SX)) {
      const T* fd = fy + (warp - 1) * C * W + lane;  // face below (j - 1/2)
      T o[C];
#pragma unroll
      for (int c = 0; c < C; ++c) o[c] = xr[c * W] - (fd[(c + C) * W] - fd[c * W]);
      T* dst = a.out + ((int64_t)((int)g.off[1] + yr) * g.rstride + (int)g.xo + xv);
#pragma unroll
      for (int c = 0; c < C; ++c) {
        *dst = o[c];
        dst += cs;
      }
      nan = max(nan, max(naninf(o[0]), naninf(o[C - 1])));
      if (ws) wmax = fmax(wmax, wavespeed<D>(o, gm1, gam));
      if ((yr < g.pad) | (yr >= SY - g.pad) | (xv < g.pad) | (xv >= SX - g.pad))
        images<D, 0>(a, xv, yr, 0, o);
    }
    win += Gr;
    yb += Gq;
    if (win >= nwin) {
      win -= nwin;
      ++yb;
    }
  }
  if (__any_sync(kFull, bad < 0 || nan >= kExpMask<T>) && lane == 0) atomicOr(a.flag, 1u);
  if (ws) publish_max(a, wmax);
}

template <typename T, int NW, int MB>
static void launch_lr2d(const KArgs<T>& a, const void* tmap, cudaStream_t s) {
  constexpr int W = 32;
  using SM = SmemPT<T, 1, NW>;
  const int nwin = (int)((a.g.S[0] + (W - 2) - 1) / (W - 2));
  const int nyb = (int)((a.g.S[1] + (NW - 2) - 1) / (NW - 2));
  const int ntiles = nwin * nyb;
  static int per_sm = 0;
  if (!per_sm) {
    cudaFuncSetAttribute(k_step2d_lr<T, NW, MB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)SM::bytes());
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_step2d_lr<T, NW, MB>, 32 * NW,
                                                  SM::bytes());
    if (per_sm < 1) per_sm = 1;
  }
  int nsm = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  int grid = per_sm * nsm;
  if (grid > ntiles) grid = ntiles;
  k_step2d_lr<T, NW, MB><<<grid, 32 * NW, SM::bytes(), s>>>(
      a, *reinterpret_cast<const CUtensorMap*>(tmap), nwin, ntiles);
}

// ---------------------------------------------------------------------------
// K-B (2-D), warp-march form: no CTA barriers, no shared-memory hand-offs.
// Each warp independently owns tasks = (32-slot x-window, chunk of R rows) and
// marches down the chunk's rows y0-1 .. y1 (y1 = min(y0+R, SY)): per row it
// x-sweeps in registers (shuffles), forms the y-face with the previous row's
// (U*, F_y) held in registers, and updates + stores the previous row.  Rows
// arrive through a per-warp DEPTH-slot TMA ring (box = one row, C components),
// prefetched DEPTH rows ahead across task boundaries.  Same arithmetic as
// k_step2d_pt (bitwise identical results).
// ---------------------------------------------------------------------------
template <typename T>
struct WMRow {
  static constexpr int W = 32, C = 4, AL = 16 / (int)sizeof(T), WB = W + AL;
  static constexpr int ELEMS = C * WB;  // one TMA row box
  // slot stride: TMA tensor destinations must be 128-byte aligned
  static constexpr int SLOT = ((ELEMS * (int)sizeof(T) + 127) / 128) * 128 / (int)sizeof(T);
};

template <typename T, int DEPTH, int NWB, int MB>
__global__ void __launch_bounds__(32 * NWB, MB)
    k_step2d_wm(const __grid_constant__ KArgs<T> a, const __grid_constant__ CUtensorMap tmap,
                int nwin, int R, int ntask) {
  constexpr int D = 2, C = 4, W = 32;
  using RW = WMRow<T>;
  extern __shared__ __align__(1024) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  T* ring = reinterpret_cast<T*>(smem) + warp * DEPTH * RW::SLOT;
  uint64_t* bar = reinterpret_cast<uint64_t*>(reinterpret_cast<T*>(smem) + NWB * DEPTH * RW::SLOT) +
                  warp * DEPTH;
  const Geom& g = a.g;
  const int SX = (int)g.S[0], SY = (int)g.S[1];
  Coef<T> kc;
  if (!step_coef(a, kc)) return;
  const bool ws = a.cf.dev != nullptr;
  const T gam = (T)a.cf.gamma;
  T wmax = T(0);
  const T gm1 = a.gm1;
  const int gw = blockIdx.x * NWB + warp, nw = gridDim.x * NWB;
  if (gw >= ntask) return;  // warp-uniform; no CTA-wide synchronisation below
  if (lane == 0) {
    for (int j = 0; j < DEPTH; ++j) mbar_init(&bar[j], 1);
    fence_barrier_init();
  }
  __syncwarp();
  // producer cursor (lane 0): task pt, row index pr within it
  int pt = gw, pr = 0;
  auto task_rows = [&](int t) {
    const int y0 = (t / nwin) * R;
    return min(y0 + R, SY) - y0 + 2;  // rows y0-1 .. y1
  };
  auto produce = [&](int slot) {  // lane 0: next row of the stream into slot
    if (pt >= ntask) return;
    const int win = pt % nwin, y0 = (pt / nwin) * R;
    const int x0 = (int)g.xo + win * (W - 2) - 1;
    mbar_arrive_expect_tx(&bar[slot], RW::ELEMS * (unsigned)sizeof(T));
    tma_load_box(ring + slot * RW::SLOT, &tmap, &bar[slot], x0 - x0 % RW::AL, 0,
                 (int)g.off[1] + y0 - 1 + pr, 0);
    if (++pr == task_rows(pt)) {
      pr = 0;
      pt += nw;
    }
  };
  if (lane == 0)
    for (int j = 0; j < DEPTH; ++j) produce(j);
  int bad = 0, nan = 0;
  const int64_t cs = g.cstride;
  unsigned k = 0;  // stream position (row counter of this warp)
  for (int t = gw; t < ntask; t += nw) {
    const int win = t % nwin, y0 = (t / nwin) * R;
    const int y1 = min(y0 + R, SY);
    const int xw = win * (W - 2) - 1;
    const int xv = xw + lane;
    const bool x_in = (xv >= -1) & (xv <= SX);
    const bool x_out = (lane >= 1) & (lane <= W - 2) & (xv < SX);
    const int sh = ((int)g.xo + xw) % RW::AL;
    T Sp[C], Gp[C], Pp[C];  // previous row: U*, F_y(U*), face below it
    for (int yr = y0 - 1; yr <= y1; ++yr, ++k) {
      const int slot = k % DEPTH;
      mbar_wait(&bar[slot], (k / DEPTH) & 1);
      T U[C], F[C], S_[C], G_[C];
      {
        const T* st = ring + slot * RW::SLOT + sh + lane;
#pragma unroll
        for (int c = 0; c < C; ++c) U[c] = st[c * RW::WB];
      }
      __syncwarp();
      if (lane == 0) {
        fence_proxy_async();
        produce(slot);
      }
      const int b0 = phys_flux<D, 0>(U, F, gm1);
      bad |= x_in ? b0 : 0;
      {
        T Pnx[C], Un[C], Fn[C];
#pragma unroll
        for (int c = 0; c < C; ++c) {
          Un[c] = __shfl_down_sync(kFull, U[c], 1);
          Fn[c] = __shfl_down_sync(kFull, F[c], 1);
        }
        force_face<D, 0>(U, F, Un, Fn, Pnx, kc.q[0], kc.nq2[0], gm1);
#pragma unroll
        for (int c = 0; c < C; ++c) {
          const T Ppv = __shfl_up_sync(kFull, Pnx[c], 1);
          S_[c] = U[c] - (Pnx[c] - Ppv);
        }
      }
      const int b1 = phys_flux<D, 1>(S_, G_, gm1);
      bad |= x_out ? b1 : 0;
      if (yr >= y0) {
        T Py[C];  // face between rows yr-1 and yr
        force_face<D, 1>(Sp, Gp, S_, G_, Py, kc.q[1], kc.nq2[1], gm1);
        if (yr >= y0 + 1 && x_out) {  // update and store row yr-1
          const int yo = yr - 1;
          T o[C];
#pragma unroll
          for (int c = 0; c < C; ++c) o[c] = Sp[c] - (Py[c] - Pp[c]);
          T* dst = a.out + ((int64_t)((int)g.off[1] + yo) * g.rstride + (int)g.xo + xv);
#pragma unroll
          for (int c = 0; c < C; ++c) {
            *dst = o[c];
            dst += cs;
          }
          nan = max(nan, max(naninf(o[0]), naninf(o[C - 1])));
          if (ws) wmax = fmax(wmax, wavespeed<D>(o, gm1, gam));
          if ((yo < g.pad) | (yo >= SY - g.pad) | (xv < g.pad) | (xv >= SX - g.pad))
            images<D, 0>(a, xv, yo, 0, o);
        }
#pragma unroll
        for (int c = 0; c < C; ++c) Pp[c] = Py[c];
      }
#pragma unroll
      for (int c = 0; c < C; ++c) {
        Sp[c] = S_[c];
        Gp[c] = G_[c];
      }
    }
  }
  if (__any_sync(kFull, bad < 0 || nan >= kExpMask<T>) && lane == 0) atomicOr(a.flag, 1u);
  if (ws) publish_max(a, wmax);
}

// rows per task: one round of tasks over all warp slots when the grid allows
static int wm_rows(const Geom& g, int warp_slots) {
  const int nwin = (int)((g.S[0] + 29) / 30);
  int nc = warp_slots / nwin;
  if (nc < 1) nc = 1;
  int R = (int)((g.S[1] + nc - 1) / nc);
  if (R < 4) R = 4;
  return R;
}

template <typename T, int DEPTH, int NWB, int MB>
static void launch_wm2d(const KArgs<T>& a, const void* tmap, cudaStream_t s) {
  using RW = WMRow<T>;
  const size_t sm = (size_t)NWB * DEPTH * (RW::SLOT * sizeof(T) + 8) + 64;
  static int per_sm = 0;
  if (!per_sm) {
    cudaFuncSetAttribute(k_step2d_wm<T, DEPTH, NWB, MB>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_step2d_wm<T, DEPTH, NWB, MB>,
                                                  32 * NWB, sm);
    if (per_sm < 1) per_sm = 1;
  }
  int nsm = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int slots = per_sm * nsm * NWB;
  const int nwin = (int)((a.g.S[0] + 29) / 30);
  const int R = a.rows > 0 ? a.rows : wm_rows(a.g, slots);
  const int ntask = nwin * (int)((a.g.S[1] + R - 1) / R);
  int grid = (ntask + NWB - 1) / NWB;
  if (grid > per_sm * nsm) grid = per_sm * nsm;
  k_step2d_wm<T, DEPTH, NWB, MB><<<grid, 32 * NWB, sm, s>>>(
      a, *reinterpret_cast<const CUtensorMap*>(tmap), nwin, R, ntask);
}

template <typename T, int V, int NW, int MB = (V == 1 ? 2 : 1)>
static void launch_pt2d(const KArgs<T>& a, const void* tmap, cudaStream_t s) {
  constexpr int W = 32 * V;
  using SM = SmemPT<T, V, NW>;
  const int nwin = (int)((a.g.S[0] + (W - 2) - 1) / (W - 2));
  const int nyb = (int)((a.g.S[1] + (NW - 2) - 1) / (NW - 2));
  const int ntiles = nwin * nyb;
  static int per_sm = 0;
  if (!per_sm) {
    cudaFuncSetAttribute(k_step2d_pt<T, V, NW, MB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)SM::bytes());
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_step2d_pt<T, V, NW, MB>, 32 * NW,
                                                  SM::bytes());
    if (per_sm < 1) per_sm = 1;
  }
  int nsm = 148;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  int grid = per_sm * nsm;
  if (grid > ntiles) grid = ntiles;
  k_step2d_pt<T, V, NW, MB><<<grid, 32 * NW, SM::bytes(), s>>>(
      a, *reinterpret_cast<const CUtensorMap*>(tmap), nwin, ntiles);
}

// ---------------------------------------------------------------------------
// K-B (2-D), order 2: MUSCL-Hancock + FORCE, both sweeps of a step
// in one HBM pass.  Persistent CTAs of NW warps; a tile is 28 x-cells x (NW-4)
// rows (stencil radius 2 in both directions), TMA streams the tiles' [NW rows]
// [C][32+AL] input boxes into a 2-stage ring.  Per tile, warp j owns row
// yr = y0 - 2 + j:
//   X   lane = x slot: slopes from shuffled neighbours, evolved boundary values
//       (hancock), face l+1/2 = FORCE(Ubar^R_l, Ubar^L_{l+1}) (shuffle), update
//       -> U* (valid on slots 2..29), published to shared memory;
//   Y1  rows 1..NW-2: y-slopes from the rows above/below, evolved y boundary
//       values; Ubar^R and F_y(Ubar^R) published;
//   Y2  rows 2..NW-2: y-face between rows j-1 and j, published;
//   upd rows 2..NW-3: U^{n+1} = U* - (Phi_{j+1/2} - Phi_{j-1/2}), store + images.
// ---------------------------------------------------------------------------
template <typename T, int NW>
struct SmemO2 {
  static constexpr int W = 32, C = 4;
  static constexpr int AL = 16 / (int)sizeof(T);
  static constexpr int WB = W + AL;
  static constexpr int STAGE = NW * C * WB;
  static constexpr int SX = NW * C * W;
  static constexpr int BR = NW * 2 * C * W;
  static constexpr int FY = NW * C * W;
  static constexpr size_t bytes() { return (size_t)(2 * STAGE + SX + BR + FY) * sizeof(T) + 64; }
};

template <typename T, int NW, int MB>
__global__ void __launch_bounds__(32 * NW, MB)
    k_step2d_o2(const __grid_constant__ KArgs<T> a, const __grid_constant__ CUtensorMap tmap,
                int nwin, int ntiles) {
  constexpr int D = 2, C = 4, W = 32;
  using SM = SmemO2<T, NW>;
  extern __shared__ __align__(1024) unsigned char smem[];
  T* stage = reinterpret_cast<T*>(smem);
  T* sx = stage + 2 * SM::STAGE;
  T* br = sx + SM::SX;
  T* fyb = br + SM::BR;
  uint64_t* bar = reinterpret_cast<uint64_t*>(fyb + SM::FY);
  const Geom& g = a.g;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int SX = (int)g.S[0], SY = (int)g.S[1];
  const int G = gridDim.x;
  Coef<T> kc;
  if (!step_coef(a, kc)) return;
  const bool ws = a.cf.dev != nullptr;
  const T gam = (T)a.cf.gamma;
  T wmax = T(0);
  const T gm1 = a.gm1;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
  }
  __syncthreads();
  auto issue = [&](int i) {
    const int tile = blockIdx.x + i * G;
    if (tile >= ntiles) return;
    const int s = i & 1;
    const int w = tile % nwin, yb = tile / nwin;
    mbar_arrive_expect_tx(&bar[s], SM::STAGE * (unsigned)sizeof(T));
    const int x0 = (int)g.xo + w * (W - 4) - 2;
    tma_load_box(stage + s * SM::STAGE, &tmap, &bar[s], x0 - x0 % SM::AL, 0,
                 (int)g.off[1] + yb * (NW - 4) - 2, 0);
  };
  if (threadIdx.x == 0) {
    issue(0);
    issue(1);
  }
  int bad = 0, nan = 0;
  const bool lane_in = (lane >= 1) & (lane <= 30);   // has both x-neighbours
  const bool lane_out = (lane >= 2) & (lane <= 29);  // U* valid
  const int Gq = G / nwin, Gr = G - (G / nwin) * nwin;
  int win = (int)blockIdx.x % nwin, yb = (int)blockIdx.x / nwin;
  const int nyb = ntiles / nwin;
  for (int i = 0;; ++i) {
    if (yb >= nyb) break;
    const int xw = win * (W - 4) - 2;
    const int yr = yb * (NW - 4) - 2 + warp;
    const int xv = xw + lane;
    const bool row_in = yr <= SY + 1;
    const int s = i & 1;
    mbar_wait(&bar[s], (i >> 1) & 1);
    // ---- X
    T S_[C];
    {
      T U[C], Um[C], Up[C];
      const int sh = ((int)g.xo + xw) % SM::AL;
      const T* st = stage + s * SM::STAGE + warp * C * SM::WB + sh + lane;
#pragma unroll
      for (int c = 0; c < C; ++c) U[c] = st[c * SM::WB];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        Um[c] = __shfl_up_sync(kFull, U[c], 1);
        Up[c] = __shfl_down_sync(kFull, U[c], 1);
      }
      T bL[C], FbL[C], bR[C], FbR[C];
      const int b = hancock<D, 0>(Um, U, Up, kc.h2[0], gm1, bL, FbL, bR, FbR);
      bad |= (lane_in & (xv >= -1) & (xv <= SX) & row_in) ? b : 0;
      T Pnx[C];
      {
        T bLn[C], FbLn[C];
#pragma unroll
        for (int c = 0; c < C; ++c) {
          bLn[c] = __shfl_down_sync(kFull, bL[c], 1);
          FbLn[c] = __shfl_down_sync(kFull, FbL[c], 1);
        }
        force_face<D, 0>(bR, FbR, bLn, FbLn, Pnx, kc.q[0], kc.nq2[0], gm1);
      }
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const T Ppv = __shfl_up_sync(kFull, Pnx[c], 1);
        S_[c] = U[c] - (Pnx[c] - Ppv);
      }
      T* xr = sx + warp * C * W + lane;
#pragma unroll
      for (int c = 0; c < C; ++c) xr[c * W] = S_[c];
    }
    __syncthreads();  // (A) stage s consumed; U* published
    if (threadIdx.x == 0) {
      fence_proxy_async();
      issue(i + 2);
    }
    // ---- Y1: evolved y boundary values of this row
    T byL[C], FbyL[C];
    if (warp >= 1 && warp <= NW - 2) {
      T Sm[C], Sp[C], byR[C], FbyR[C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        Sm[c] = sx[(warp - 1) * C * W + c * W + lane];
        Sp[c] = sx[(warp + 1) * C * W + c * W + lane];
      }
      const int b = hancock<D, 1>(Sm, S_, Sp, kc.h2[1], gm1, byL, FbyL, byR, FbyR);
      bad |= (lane_out & (xv < SX) & (yr >= -1) & (yr <= SY)) ? b : 0;
      T* w = br + warp * 2 * C * W + lane;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        w[c * W] = byR[c];
        w[(C + c) * W] = FbyR[c];
      }
    }
    __syncthreads();  // (B) Ubar^R_y published
    // ---- Y2: face between rows warp-1 and warp
    T Py[C];
    if (warp >= 2 && warp <= NW - 2) {
      T pR[C], pF[C];
      const T* r = br + (warp - 1) * 2 * C * W + lane;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        pR[c] = r[c * W];
        pF[c] = r[(C + c) * W];
      }
      force_face<D, 1>(pR, pF, byL, FbyL, Py, kc.q[1], kc.nq2[1], gm1);
      T* fw = fyb + warp * C * W + lane;
#pragma unroll
      for (int c = 0; c < C; ++c) fw[c * W] = Py[c];
    }
    __syncthreads();  // (C) y-faces published
    // ---- update + store
    if (warp >= 2 && warp <= NW - 3 && yr < SY && lane_out && xv < SX) {
      const T* fu = fyb + (warp + 1) * C * W + lane;
      T o[C];
#pragma unroll
      for (int c = 0; c < C; ++c) o[c] = S_[c] - (fu[c * W] - Py[c]);
      T* dst = a.out + ((int64_t)((int)g.off[1] + yr) * g.rstride + (int)g.xo + xv);
      const int64_t cs = g.cstride;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        *dst = o[c];
        dst += cs;
      }
      nan = max(nan, max(naninf(o[0]), naninf(o[C - 1])));
      if (ws) wmax = fmax(wmax, wavespeed<D>(o, gm1, gam));
      if ((yr < g.pad) | (yr >= SY - g.pad) | (xv < g.pad) | (xv >= SX - g.pad))
        images<D, 0>(a, xv, yr, 0, o);
    }
    win += Gr;
    yb += Gq;
    if (win >= nwin) {
      win -= nwin;
      ++yb;
    }
  }
  if (__any_sync(kFull, bad < 0 || nan >= kExpMask<T>) && lane == 0) atomicOr(a.flag, 1u);
  if (ws) publish_max(a, wmax);
}

template <typename T, int NW, int MB>
static void launch_o2(const KArgs<T>& a, const void* tmap, cudaStream_t s) {
  constexpr int W = 32;
  using SM = SmemO2<T, NW>;
  const int nwin = (int)((a.g.S[0] + (W - 4) - 1) / (W - 4));
  const int nyb = (int)((a.g.S[1] + (NW - 4) - 1) / (NW - 4));
  const int ntiles = nwin * nyb;
  static int per_sm = 0;
  if (!per_sm) {
    cudaFuncSetAttribute(k_step2d_o2<T, NW, MB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)SM::bytes());
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_step2d_o2<T, NW, MB>, 32 * NW,
                                                  SM::bytes());
    if (per_sm < 1) per_sm = 1;
  }
  int nsm = 148;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  int grid = per_sm * nsm;
  if (grid > ntiles) grid = ntiles;
  k_step2d_o2<T, NW, MB><<<grid, 32 * NW, SM::bytes(), s>>>(
      a, *reinterpret_cast<const CUtensorMap*>(tmap), nwin, ntiles);
}

// order-2 variants (RPL_VARIANT; box rows = NW)
static int o2_rows(int variant) {
  switch (variant) {
    case 71: return 12;
    case 72: return 12;
    case 73: return 24;
    default: return 16;
  }
}

int tmap2d_box_o2(const Geom& g, int variant, int* box_w, int* box_rows) {
  *box_w = 32 + 16 / g.elem;
  *box_rows = o2_rows(variant);
  return 1;
}

template <typename T>
static void launch_step2d_o2(const KArgs<T>& a, const void* tmap, cudaStream_t s) {
  switch (a.variant) {
    case 71: return launch_o2<T, 12, 2>(a, tmap, s);
    case 72: return launch_o2<T, 12, 1>(a, tmap, s);
    case 73: return launch_o2<T, 24, 1>(a, tmap, s);
    default: return launch_o2<T, 16, 1>(a, tmap, s);
  }
}

// ---------------------------------------------------------------------------
// K-B (2-D), column-march form.  A work item is one x-window (W-2 outputs) x a
// chunk of rows; the CTA marches down the chunk NW rows per step:
//   X      warp j x-sweeps row k = NW t + j of the chunk (k = 0 is the row above
//          the chunk) and publishes (U*, F_y) into a 2NW-row shared ring;
//   Y      warp j computes the y-face between rows k-1 and k (row k-1 comes from
//          the ring: the previous warp, or the previous step's last warp);
//   update warp j updates row k with faces k (own) and k+1 (warp j+1); the last
//          warp's update waits for the next step's first face (read back from
//          the rings), so every row is x-swept once and every face computed once.
// TMA streams the step boxes [NW rows][C][W+AL] into an NS-stage ring, NS
// steps ahead, continuously across the CTA's work items (persistent grid).
// ---------------------------------------------------------------------------
template <typename T, int V, int NW>
struct SmemCM {
  static constexpr int W = 32 * V, C = 4, NS = 2;
  static constexpr int AL = 16 / (int)sizeof(T);
  static constexpr int WB = W + AL;
  static constexpr int STAGE = NW * C * WB;
  // ring depths (rows): U* of row k-1 is read again by the deferred update one
  // step later -> 3 NW; F_y and faces are dead one step later -> 2 NW
  static constexpr int RS = 3 * NW, RG = 2 * NW, RF = 2 * NW;
  static constexpr int SR = RS * C * W, GR = RG * C * W, FR = RF * C * W;
  static constexpr size_t bytes() { return (size_t)(NS * STAGE + SR + GR + FR) * sizeof(T) + 64; }
};

struct CMCursor {  // (work item, step) walker over this CTA's items
  int i, t, nst, item;
  __device__ __forceinline__ void set(int i_, int nwin, int chunk, int SY, int NW, int G,
                                      int nwork) {
    i = i_;
    t = 0;
    item = blockIdx.x + i * G;
    nst = 0;
    if (item < nwork) {
      const int c = item / nwin;
      const int y0 = c * chunk;
      const int y1 = min(y0 + chunk, SY);
      nst = (y1 - y0 + 2 + NW - 1) / NW;
    }
  }
  __device__ __forceinline__ void next(int nwin, int chunk, int SY, int NW, int G, int nwork) {
    if (++t >= nst) set(i + 1, nwin, chunk, SY, NW, G, nwork);
  }
};

template <typename T, int V, int NW, int MB>
__global__ void __launch_bounds__(32 * NW, MB)
    k_step2d_cm(const __grid_constant__ KArgs<T> a, const __grid_constant__ CUtensorMap tmap,
                int nwin, int chunk, int nwork) {
  constexpr int D = 2, C = 4, W = 32 * V;
  using SM = SmemCM<T, V, NW>;
  using VT = typename VecV<T, V>::type;
  extern __shared__ __align__(1024) unsigned char smem[];
  T* stage = reinterpret_cast<T*>(smem);
  T* sr = stage + SM::NS * SM::STAGE;
  T* gr = sr + SM::SR;
  T* fy = gr + SM::GR;
  uint64_t* bar = reinterpret_cast<uint64_t*>(fy + SM::FR);
  const Geom& g = a.g;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int SX = (int)g.S[0], SY = (int)g.S[1];
  const int G = gridDim.x;
  const T gm1 = a.gm1, qx = a.q[0], nqx = a.nq2[0], qy = a.q[1], nqy = a.nq2[1];
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < SM::NS; ++s) mbar_init(&bar[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  // producer cursor (thread 0) runs NS steps ahead of the consumers: a stage is
  // refilled right after barrier A of the step that consumed it
  CMCursor pc;
  int pseq = 0;
  auto issue_one = [&]() {
    if (pc.item >= nwork) return;
    const int s = pseq % SM::NS;
    const int win = pc.item % nwin, c = pc.item / nwin;
    const int x0 = (int)g.xo + win * (W - 2) - 1;
    mbar_arrive_expect_tx(&bar[s], SM::STAGE * (unsigned)sizeof(T));
    tma_load_box(stage + s * SM::STAGE, &tmap, &bar[s], x0 - x0 % SM::AL, 0,
                 (int)g.off[1] + c * chunk - 1 + NW * pc.t, 0);
    ++pseq;
    pc.next(nwin, chunk, SY, NW, G, nwork);
  };
  if (threadIdx.x == 0) {
    pc.set(0, nwin, chunk, SY, NW, G, nwork);
    for (int s = 0; s < SM::NS; ++s) issue_one();
  }
  CMCursor cc;
  cc.set(0, nwin, chunk, SY, NW, G, nwork);
  int cseq = 0;
  int bad = 0, nan = 0;
  while (cc.item < nwork) {
    const int win = cc.item % nwin, ch = cc.item / nwin;
    const int y0 = ch * chunk;
    const int y1 = min(y0 + chunk, SY);
    const int xw = win * (W - 2) - 1;
    const int sh = ((int)g.xo + xw) % SM::AL;
    const int t = cc.t;
    const int k = NW * t + warp;     // chunk-local row index, grid row y0 - 1 + k
    // ring row: keeps increasing across work items, so ring slots are only
    // reused after the barriers that order their last reads (NW * cseq + warp)
    const int kr = NW * cseq + warp;
    const int yr = y0 - 1 + k;
    const bool row_in = yr <= SY;
    const int s = cseq % SM::NS;
    mbar_wait(&bar[s], (cseq / SM::NS) & 1);
    // ---- X
    T U[V][C], F[V][C], S_[V][C], G_[V][C];
    {
      const T* st = stage + s * SM::STAGE + warp * C * SM::WB + sh + V * lane;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const VT u = *reinterpret_cast<const VT*>(st + c * SM::WB);
        if constexpr (V == 1) {
          U[0][c] = u;
        } else {
          U[0][c] = u.x;
          U[1][c] = u.y;
        }
      }
    }
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int xv = xw + V * lane + v;
      const int b = phys_flux<D, 0>(U[v], F[v], gm1);
      bad |= ((xv >= -1) & (xv <= SX) & row_in) ? b : 0;
    }
    {
      T Pin[C], Pnx[C], Un[C], Fn[C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        Un[c] = __shfl_down_sync(kFull, U[0][c], 1);
        Fn[c] = __shfl_down_sync(kFull, F[0][c], 1);
      }
      force_face<D, 0>(U[V - 1], F[V - 1], Un, Fn, Pnx, qx, nqx, gm1);
      if constexpr (V == 2) force_face<D, 0>(U[0], F[0], U[1], F[1], Pin, qx, nqx, gm1);
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const T Ppv = __shfl_up_sync(kFull, Pnx[c], 1);
        if constexpr (V == 2) {
          S_[0][c] = U[0][c] - (Pin[c] - Ppv);
          S_[1][c] = U[1][c] - (Pnx[c] - Pin[c]);
        } else {
          S_[0][c] = U[0][c] - (Pnx[c] - Ppv);
        }
      }
    }
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int xv = xw + V * lane + v;
      const int slot = V * lane + v;
      const int b = phys_flux<D, 1>(S_[v], G_[v], gm1);
      bad |= ((slot >= 1) & (slot <= W - 2) & (xv < SX) & row_in) ? b : 0;
    }
    {
      T* sw = sr + (kr % SM::RS) * C * W + V * lane;
      T* gw = gr + (kr % SM::RG) * C * W + V * lane;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        VT sv, gv;
        if constexpr (V == 1) {
          sv = S_[0][c];
          gv = G_[0][c];
        } else {
          sv.x = S_[0][c];
          sv.y = S_[1][c];
          gv.x = G_[0][c];
          gv.y = G_[1][c];
        }
        *reinterpret_cast<VT*>(sw + c * W) = sv;
        *reinterpret_cast<VT*>(gw + c * W) = gv;
      }
    }
    __syncthreads();  // (A): stage consumed, (U*, F_y) of this step published
    if (threadIdx.x == 0) {
      fence_proxy_async();
      issue_one();
    }
    // ---- Y: face k between rows k-1 and k
    T Py[V][C];
    if (k >= 1) {
      const T* ps = sr + ((kr - 1) % SM::RS) * C * W + V * lane;
      const T* pg = gr + ((kr - 1) % SM::RG) * C * W + V * lane;
      T Sp[V][C], Gp[V][C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const VT sv = *reinterpret_cast<const VT*>(ps + c * W);
        const VT gv = *reinterpret_cast<const VT*>(pg + c * W);
        if constexpr (V == 1) {
          Sp[0][c] = sv;
          Gp[0][c] = gv;
        } else {
          Sp[0][c] = sv.x;
          Sp[1][c] = sv.y;
          Gp[0][c] = gv.x;
          Gp[1][c] = gv.y;
        }
      }
#pragma unroll
      for (int v = 0; v < V; ++v) force_face<D, 1>(Sp[v], Gp[v], S_[v], G_[v], Py[v], qy, nqy, gm1);
      T* fw = fy + (kr % SM::RF) * C * W + V * lane;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        VT pv;
        if constexpr (V == 1) {
          pv = Py[0][c];
        } else {
          pv.x = Py[0][c];
          pv.y = Py[1][c];
        }
        *reinterpret_cast<VT*>(fw + c * W) = pv;
      }
    }
    __syncthreads();  // (B): faces of this step published
    // ---- updates: warp j < NW-1 updates its own row k (faces k and k+1);
    // warp 0 also completes the previous step's last row (k-1) from the rings.
    auto update_store = [&](int kk, const T (*Sv)[C], const T (*Pl)[C], const T* fup) {
      const int yy = y0 - 1 + kk;
      if (kk < 1 || yy >= y1) return;
      T* dst = a.out + g.row(yy, 0) * g.rstride + g.xo + xw + V * lane;
      T o[V][C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const VT pv = *reinterpret_cast<const VT*>(fup + c * W);
        if constexpr (V == 1) {
          o[0][c] = Sv[0][c] - (pv - Pl[0][c]);
        } else {
          o[0][c] = Sv[0][c] - (pv.x - Pl[0][c]);
          o[1][c] = Sv[1][c] - (pv.y - Pl[1][c]);
        }
      }
      bool ok[V];
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const int slot = V * lane + v;
        ok[v] = (slot >= 1) & (slot <= W - 2) & (xw + slot < SX);
      }
      if constexpr (V == 2) {
        if (ok[0] & ok[1]) {
#pragma unroll
          for (int c = 0; c < C; ++c) {
            VT w;
            w.x = o[0][c];
            w.y = o[1][c];
            *reinterpret_cast<VT*>(dst + c * g.cstride) = w;
          }
        } else {
#pragma unroll
          for (int v = 0; v < V; ++v)
            if (ok[v])
#pragma unroll
              for (int c = 0; c < C; ++c) dst[c * g.cstride + v] = o[v][c];
        }
      } else {
        if (ok[0])
#pragma unroll
          for (int c = 0; c < C; ++c) dst[c * g.cstride] = o[0][c];
      }
      const bool yface = (yy < g.pad) | (yy >= SY - g.pad);
#pragma unroll
      for (int v = 0; v < V; ++v) {
        if (ok[v]) {
          nan = max(nan, max(naninf(o[v][0]), naninf(o[v][C - 1])));
          const int xv = xw + V * lane + v;
          if (yface | (xv < g.pad) | (xv >= SX - g.pad)) images<D, 0>(a, xv, yy, 0, o[v]);
        }
      }
    };
    // (the last warp's row of a chunk's final step is never an output row)
    if (warp < NW - 1) update_store(k, S_, Py, fy + ((kr + 1) % SM::RF) * C * W + V * lane);
    if (warp == 0 && t >= 1) {
      // previous step's last row kp = k - 1 (warp NW-1 of step t-1): U* and its lower
      // face from the rings, upper face = this warp's face k
      const int kp = k - 1;
      const T* pr = sr + ((kr - 1) % SM::RS) * C * W + V * lane;
      const T* pl = fy + ((kr - 1) % SM::RF) * C * W + V * lane;
      T Sv[V][C], Pl[V][C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const VT sv = *reinterpret_cast<const VT*>(pr + c * W);
        const VT lv = *reinterpret_cast<const VT*>(pl + c * W);
        if constexpr (V == 1) {
          Sv[0][c] = sv;
          Pl[0][c] = lv;
        } else {
          Sv[0][c] = sv.x;
          Sv[1][c] = sv.y;
          Pl[0][c] = lv.x;
          Pl[1][c] = lv.y;
        }
      }
      update_store(kp, Sv, Pl, fy + (kr % SM::RF) * C * W + V * lane);
    }
    ++cseq;
    cc.next(nwin, chunk, SY, NW, G, nwork);
  }
  if (__any_sync(kFull, bad < 0 || nan >= kExpMask<T>) && lane == 0) atomicOr(a.flag, 1u);
}

template <typename T, int V, int NW, int MB>
static void launch_cm2d(const KArgs<T>& a, const void* tmap, cudaStream_t s) {
  constexpr int W = 32 * V;
  using SM = SmemCM<T, V, NW>;
  const int nwin = (int)((a.g.S[0] + (W - 2) - 1) / (W - 2));
  static int per_sm = 0;
  if (!per_sm) {
    cudaFuncSetAttribute(k_step2d_cm<T, V, NW, MB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)SM::bytes());
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_step2d_cm<T, V, NW, MB>, 32 * NW,
                                                  SM::bytes());
    if (per_sm < 1) per_sm = 1;
  }
  int nsm = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int resident = per_sm * nsm;
  // chunk rows: ~2 work items per resident CTA, a multiple of NW, >= 2 NW
  const int64_t SY = a.g.S[1];
  int64_t chunk = (SY * nwin + 2 * resident - 1) / (2 * resident);
  chunk = (chunk + NW - 1) / NW * NW;
  if (chunk < 2 * NW) chunk = 2 * NW;
  if (a.rows > 0) chunk = a.rows;
  const int nchunk = (int)((SY + chunk - 1) / chunk);
  const int nwork = nwin * nchunk;
  const int grid = nwork < resident ? nwork : resident;
  k_step2d_cm<T, V, NW, MB><<<grid, 32 * NW, SM::bytes(), s>>>(
      a, *reinterpret_cast<const CUtensorMap*>(tmap), nwin, (int)chunk, nwork);
}

// ---------------------------------------------------------------------------
// K-B (2-D), point-to-point form: the tile work of k_step2d_pt without CTA-wide
// barriers.  A producer warp issues the TMA boxes (full/empty mbarrier ring);
// compute warp j only waits for the rows it actually needs -- row j-1's
// (U*, F_y) (xyReady), the face computed by warp j+1 (fyReady) -- and signals
// when it is done reading a neighbour's slot (xyFree / fyFree), so warps drift
// across tiles instead of meeting at __syncthreads (the publish buffers are
// double-buffered by tile parity).
// ---------------------------------------------------------------------------
template <typename T, int V, int NW>
struct SmemPP {
  static constexpr int W = 32 * V, C = 4, NS = 3;
  static constexpr int AL = 16 / (int)sizeof(T);
  static constexpr int WB = W + AL;
  static constexpr int STAGE = NW * C * WB;
  static constexpr int XY = 2 * NW * 2 * C * W;
  static constexpr int FY = 2 * (NW - 1) * C * W;
  static constexpr int NBAR = 2 * NS + 2 * NW + 2 * (NW - 1) + 2 * NW + 2 * (NW - 1);
  static constexpr size_t bytes() {
    return (size_t)(NS * STAGE + XY + FY) * sizeof(T) + NBAR * 8 + 64;
  }
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <typename T, int V, int NW, int MB>
__global__ void __launch_bounds__(32 * (NW + 1), MB)
    k_step2d_pp(const __grid_constant__ KArgs<T> a, const __grid_constant__ CUtensorMap tmap,
                int nwin, int ntiles) {
  constexpr int D = 2, C = 4, W = 32 * V;
  using SM = SmemPP<T, V, NW>;
  using VT = typename VecV<T, V>::type;
  extern __shared__ __align__(1024) unsigned char smem[];
  T* stage = reinterpret_cast<T*>(smem);
  T* xy = stage + SM::NS * SM::STAGE;  // [2][NW][2C][W]
  T* fy = xy + SM::XY;                 // [2][NW-1][C][W]
  uint64_t* bars = reinterpret_cast<uint64_t*>(fy + SM::FY);
  uint64_t* full = bars;                       // [NS]
  uint64_t* empty = full + SM::NS;             // [NS]
  uint64_t* xyReady = empty + SM::NS;          // [2][NW]
  uint64_t* fyReady = xyReady + 2 * NW;        // [2][NW-1]
  uint64_t* xyFree = fyReady + 2 * (NW - 1);   // [2][NW]
  uint64_t* fyFree = xyFree + 2 * NW;          // [2][NW-1]
  const Geom& g = a.g;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int SX = (int)g.S[0], SY = (int)g.S[1];
  const int G = gridDim.x;
  if (threadIdx.x == 0) {
    for (int i = 0; i < SM::NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], NW);
    }
    for (int i = 0; i < 2 * NW; ++i) {
      mbar_init(&xyReady[i], 1);
      mbar_init(&xyFree[i], 1);
    }
    for (int i = 0; i < 2 * (NW - 1); ++i) {
      mbar_init(&fyReady[i], 1);
      mbar_init(&fyFree[i], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  if (warp == NW) {  // ---------------- producer warp
    if (lane == 0) {
      for (int it = 0;; ++it) {
        const int tile = blockIdx.x + it * G;
        if (tile >= ntiles) break;
        const int s = it % SM::NS;
        if (it >= SM::NS) mbar_wait(&empty[s], ((it / SM::NS) - 1) & 1);
        const int w = tile % nwin, yb = tile / nwin;
        const int x0 = (int)g.xo + w * (W - 2) - 1;
        mbar_arrive_expect_tx(&full[s], SM::STAGE * (unsigned)sizeof(T));
        tma_load_box(stage + s * SM::STAGE, &tmap, &full[s], x0 - x0 % SM::AL, 0,
                     (int)g.off[1] + yb * (NW - 2) - 1, 0);
      }
    }
    return;
  }
  // ---------------- compute warps
  const T gm1 = a.gm1, qx = a.q[0], nqx = a.nq2[0], qy = a.q[1], nqy = a.nq2[1];
  int bad = 0, nan = 0;
  for (int it = 0;; ++it) {
    const int tile = blockIdx.x + it * G;
    if (tile >= ntiles) break;
    const int p = it & 1, u = it >> 1;
    const int win = tile % nwin, yb = tile / nwin;
    const int xw = win * (W - 2) - 1;
    const int yr = yb * (NW - 2) - 1 + warp;
    const bool row_in = yr <= SY;
    const int s = it % SM::NS;
    mbar_wait(&full[s], (it / SM::NS) & 1);
    T U[V][C], F[V][C], S_[V][C], G_[V][C];
    {
      const int sh = ((int)g.xo + xw) % SM::AL;
      const T* st = stage + s * SM::STAGE + warp * C * SM::WB + sh + V * lane;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const VT uu = *reinterpret_cast<const VT*>(st + c * SM::WB);
        if constexpr (V == 1) {
          U[0][c] = uu;
        } else {
          U[0][c] = uu.x;
          U[1][c] = uu.y;
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int xv = xw + V * lane + v;
      const int b = phys_flux<D, 0>(U[v], F[v], gm1);
      bad |= ((xv >= -1) & (xv <= SX) & row_in) ? b : 0;
    }
    {
      T Pin[C], Pnx[C], Un[C], Fn[C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        Un[c] = __shfl_down_sync(kFull, U[0][c], 1);
        Fn[c] = __shfl_down_sync(kFull, F[0][c], 1);
      }
      force_face<D, 0>(U[V - 1], F[V - 1], Un, Fn, Pnx, qx, nqx, gm1);
      if constexpr (V == 2) force_face<D, 0>(U[0], F[0], U[1], F[1], Pin, qx, nqx, gm1);
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const T Ppv = __shfl_up_sync(kFull, Pnx[c], 1);
        if constexpr (V == 2) {
          S_[0][c] = U[0][c] - (Pin[c] - Ppv);
          S_[1][c] = U[1][c] - (Pnx[c] - Pin[c]);
        } else {
          S_[0][c] = U[0][c] - (Pnx[c] - Ppv);
        }
      }
    }
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int xv = xw + V * lane + v;
      const int slot = V * lane + v;
      const int b = phys_flux<D, 1>(S_[v], G_[v], gm1);
      bad |= ((slot >= 1) & (slot <= W - 2) & (xv < SX) & row_in) ? b : 0;
    }
    // ---- publish (U*, F_y) of row `warp` (reader: warp+1)
    if (warp <= NW - 2 && it >= 2) mbar_wait(&xyFree[p * NW + warp], (u - 1) & 1);
    {
      T* xr = xy + (p * NW + warp) * 2 * C * W + V * lane;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        VT sv, gv;
        if constexpr (V == 1) {
          sv = S_[0][c];
          gv = G_[0][c];
        } else {
          sv.x = S_[0][c];
          sv.y = S_[1][c];
          gv.x = G_[0][c];
          gv.y = G_[1][c];
        }
        *reinterpret_cast<VT*>(xr + c * W) = sv;
        *reinterpret_cast<VT*>(xr + (C + c) * W) = gv;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&xyReady[p * NW + warp]);
    // ---- y-face between rows warp-1 and warp (reader of the face: warp-1)
    T Py[V][C];
    if (warp >= 1) {
      mbar_wait(&xyReady[p * NW + warp - 1], u & 1);
      const T* pr = xy + (p * NW + warp - 1) * 2 * C * W + V * lane;
      T Sp[V][C], Gp[V][C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const VT sv = *reinterpret_cast<const VT*>(pr + c * W);
        const VT gv = *reinterpret_cast<const VT*>(pr + (C + c) * W);
        if constexpr (V == 1) {
          Sp[0][c] = sv;
          Gp[0][c] = gv;
        } else {
          Sp[0][c] = sv.x;
          Sp[1][c] = sv.y;
          Gp[0][c] = gv.x;
          Gp[1][c] = gv.y;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&xyFree[p * NW + warp - 1]);
#pragma unroll
      for (int v = 0; v < V; ++v) force_face<D, 1>(Sp[v], Gp[v], S_[v], G_[v], Py[v], qy, nqy, gm1);
      if (warp >= 2 && it >= 2) mbar_wait(&fyFree[p * (NW - 1) + warp - 1], (u - 1) & 1);
      T* fw = fy + (p * (NW - 1) + warp - 1) * C * W + V * lane;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        VT pv;
        if constexpr (V == 1) {
          pv = Py[0][c];
        } else {
          pv.x = Py[0][c];
          pv.y = Py[1][c];
        }
        *reinterpret_cast<VT*>(fw + c * W) = pv;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&fyReady[p * (NW - 1) + warp - 1]);
    }
    // ---- update rows 1..NW-2 with the face from warp+1
    if (warp >= 1 && warp <= NW - 2) {
      mbar_wait(&fyReady[p * (NW - 1) + warp], u & 1);
      const T* fu = fy + (p * (NW - 1) + warp) * C * W + V * lane;
      T o[V][C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const VT pv = *reinterpret_cast<const VT*>(fu + c * W);
        if constexpr (V == 1) {
          o[0][c] = S_[0][c] - (pv - Py[0][c]);
        } else {
          o[0][c] = S_[0][c] - (pv.x - Py[0][c]);
          o[1][c] = S_[1][c] - (pv.y - Py[1][c]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&fyFree[p * (NW - 1) + warp]);
      if (yr < SY) {
        T* dst = a.out + g.row(yr, 0) * g.rstride + g.xo + xw + V * lane;
        bool ok[V];
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const int slot = V * lane + v;
          ok[v] = (slot >= 1) & (slot <= W - 2) & (xw + slot < SX);
        }
        if constexpr (V == 2) {
          if (ok[0] & ok[1]) {
#pragma unroll
            for (int c = 0; c < C; ++c) {
              VT w;
              w.x = o[0][c];
              w.y = o[1][c];
              *reinterpret_cast<VT*>(dst + c * g.cstride) = w;
            }
          } else {
#pragma unroll
            for (int v = 0; v < V; ++v)
              if (ok[v])
#pragma unroll
                for (int c = 0; c < C; ++c) dst[c * g.cstride + v] = o[v][c];
          }
        } else {
          if (ok[0])
#pragma unroll
            for (int c = 0; c < C; ++c) dst[c * g.cstride] = o[0][c];
        }
        const bool yface = (yr < g.pad) | (yr >= SY - g.pad);
#pragma unroll
        for (int v = 0; v < V; ++v) {
          if (ok[v]) {
            nan = max(nan, max(naninf(o[v][0]), naninf(o[v][C - 1])));
            const int xv = xw + V * lane + v;
            if (yface | (xv < g.pad) | (xv >= SX - g.pad)) images<D, 0>(a, xv, yr, 0, o[v]);
          }
        }
      }
    }
  }
  if (__any_sync(kFull, bad < 0 || nan >= kExpMask<T>) && lane == 0) atomicOr(a.flag, 1u);
}

template <typename T, int V, int NW, int MB>
static void launch_pp2d(const KArgs<T>& a, const void* tmap, cudaStream_t s) {
  constexpr int W = 32 * V;
  using SM = SmemPP<T, V, NW>;
  const int nwin = (int)((a.g.S[0] + (W - 2) - 1) / (W - 2));
  const int nyb = (int)((a.g.S[1] + (NW - 2) - 1) / (NW - 2));
  const int ntiles = nwin * nyb;
  static int per_sm = 0;
  if (!per_sm) {
    cudaFuncSetAttribute(k_step2d_pp<T, V, NW, MB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)SM::bytes());
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_step2d_pp<T, V, NW, MB>,
                                                  32 * (NW + 1), SM::bytes());
    if (per_sm < 1) per_sm = 1;
  }
  int nsm = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  int grid = per_sm * nsm;
  if (grid > ntiles) grid = ntiles;
  k_step2d_pp<T, V, NW, MB><<<grid, 32 * (NW + 1), SM::bytes(), s>>>(
      a, *reinterpret_cast<const CUtensorMap*>(tmap), nwin, ntiles);
}

// 2-D fused variants (RPL_VARIANT): 0/34 persistent TMA V=1 NW=8, 3 CTAs/SM
// (default, fastest measured: 29.2 us at 1024^2 fp64), 32 same at 2 CTAs/SM,
// 30 V=1 NW=16, 31 V=2 NW=8, 33 V=2 NW=16, 35/36 other occupancies;
// 40-43 column-march (correct, slower: 39-48 us);
// 10/11/14 non-persistent tiles;
// 2/3/4 per-warp march.  Box of the TMA variants:
int tmap2d_box(const Geom& g, int variant, int* box_w, int* box_rows) {
  const int al = 16 / g.elem;  // see SmemPT::AL
  switch (variant) {
    case 30: *box_w = 32 + al; *box_rows = 16; return 1;
    case 31: *box_w = 64 + al; *box_rows = 8; return 1;
    case 32: case 34: case 35: *box_w = 32 + al; *box_rows = 8; return 1;
    case 36: *box_w = 64 + al; *box_rows = 8; return 1;
    case 0: case 37: case 39: *box_w = 32 + al; *box_rows = 12; return 1;
    case 38: *box_w = 32 + al; *box_rows = 10; return 1;
    case 44: *box_w = 32 + al; *box_rows = 24; return 1;
    case 80: case 83: *box_w = 32 + al; *box_rows = 8; return 1;
    case 90: case 91: case 92: case 93: case 94: case 95:
      *box_w = 32 + al; *box_rows = 1; return 1;
    case 81: *box_w = 32 + al; *box_rows = 16; return 1;
    case 82: *box_w = 32 + al; *box_rows = 12; return 1;
    case 84: *box_w = 32 + al; *box_rows = 10; return 1;
    case 46: *box_w = 32 + al; *box_rows = 14; return 1;
    case 47: *box_w = 32 + al; *box_rows = 20; return 1;
    case 40: case 41: *box_w = 32 + al; *box_rows = 8; return 1;
    case 42: *box_w = 64 + al; *box_rows = 8; return 1;
    case 43: *box_w = 32 + al; *box_rows = 16; return 1;
    case 60: case 61: *box_w = 32 + al; *box_rows = 8; return 1;
    case 62: *box_w = 32 + al; *box_rows = 16; return 1;
    case 63: *box_w = 64 + al; *box_rows = 8; return 1;
    case 33: *box_w = 64 + al; *box_rows = 16; return 1;
    default: return 0;
  }
}

// ---------------------------------------------------------------------------
// Ghost fill of partition `part` from the current buffers of all partitions
// (inverse of the image map: per dim, a ghost index maps to its source by the
// boundary kind, interior indices of other partitions map to themselves).
// ---------------------------------------------------------------------------
template <typename T, int D, int L>
__global__ void __launch_bounds__(256) k_fill(const Geom g, int part, T* const* bufs) {
  int pc[3];
  g.part_coords(part, pc);
  const int64_t n = g.P[0] * g.P[1] * g.P[2];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l[3] = {i % g.P[0] - g.off[0], (i / g.P[0]) % g.P[1] - g.off[1],
                          i / (g.P[0] * g.P[1]) - g.off[2]};
    bool interior = true;
#pragma unroll
    for (int d = 0; d < D; ++d) interior &= (l[d] >= 0) & (l[d] < g.S[d]);
    if (interior) continue;
    int64_t s[3] = {0, 0, 0};
    int sp[3] = {0, 0, 0};
    bool flip[3] = {false, false, false};
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int64_t N = g.N[d];
      const int64_t q = (int64_t)pc[d] * g.S[d] + l[d];
      int64_t src = q;
      if (q < 0 || q >= N) {
        const int k = q < 0 ? g.bc_lo[d] : g.bc_hi[d];
        if (k == 0) {
          src = q < 0 ? 0 : N - 1;
        } else if (k == 1) {
          src = ((q % N) + N) % N;
        } else {
          src = q < 0 ? -1 - q : 2 * N - 1 - q;
          flip[d] = true;
        }
      }
      sp[d] = (int)(src / g.S[d]);
      s[d] = src - (int64_t)sp[d] * g.S[d];
    }
    const T* sb = bufs[g.part_index(sp[0], sp[1], sp[2])];
    if (sb == nullptr) continue;  // other rank: filled by the halo exchange
    T v[D + 2];
    load_cell<D, L>(g, sb, s[0], s[1], s[2], v);
#pragma unroll
    for (int d = 0; d < D; ++d)
      if (flip[d]) v[1 + d] = -v[1 + d];
    store_cell<D, L>(g, bufs[part], l[0], l[1], l[2], v);
  }
}

// ---------------------------------------------------------------------------
// max over interior cells of |u| + c, c = sqrt(gamma p / rho), evaluated in fp64
// for both storage types.  Non-negative doubles order like their bit patterns,
// so the block maxima meet in one 64-bit atomicMax.  A NaN/negative state sets
// the domain flag.
// ---------------------------------------------------------------------------
template <typename T, int D, int L>
__global__ void __launch_bounds__(256) k_maxws(const Geom g, const T* __restrict__ in,
                                               double gamma, unsigned long long* smax,
                                               unsigned* flag) {
  double m = 0.0;
  bool bad = false;
  const int64_t n = g.cells();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = i % g.S[0], y = (i / g.S[0]) % g.S[1], z = i / (g.S[0] * g.S[1]);
    T v[D + 2];
    load_cell<D, L>(g, in, x, y, z, v);
    const double rho = (double)v[0];
    double usq = 0.0, msq = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const double u = (double)v[1 + k] / rho;
      usq += u * u;
      msq += (double)v[1 + k] * (double)v[1 + k];
    }
    const double p = (gamma - 1.0) * ((double)v[D + 1] - 0.5 * msq / rho);
    const double w = sqrt(usq) + sqrt(gamma * p / rho);
    if (!(rho > 0.0) || !(p > 0.0) || !(w < 1e300)) bad = true;
    else m = fmax(m, w);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(kFull, m, o));
  __shared__ double sm[8];
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, sm[w]);
    atomicMax(smax, (unsigned long long)__double_as_longlong(m));
  }
  if (bad) atomicOr(flag, 1u);
}

// ------------------------------------------------------------------ launchers
static int grid_for(int64_t n, int block) {
  int64_t b = (n + block - 1) / block;
  const int64_t cap = 148 * 16;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

template <typename T, int D, int L>
static void sweep_dispatch_d(const KArgs<T>& a, int d, cudaStream_t s) {
  const int grid = grid_for(a.g.cells(), 256);
  if (a.order == 2) {
    if (d == 0) k_sweep2<T, D, 0, L><<<grid, 256, 0, s>>>(a);
    if constexpr (D > 1)
      if (d == 1) k_sweep2<T, D, 1, L><<<grid, 256, 0, s>>>(a);
    if constexpr (D > 2)
      if (d == 2) k_sweep2<T, D, 2, L><<<grid, 256, 0, s>>>(a);
    return;
  }
  if (d == 0) k_sweep<T, D, 0, L><<<grid, 256, 0, s>>>(a);
  if constexpr (D > 1)
    if (d == 1) k_sweep<T, D, 1, L><<<grid, 256, 0, s>>>(a);
  if constexpr (D > 2)
    if (d == 2) k_sweep<T, D, 2, L><<<grid, 256, 0, s>>>(a);
}

template <typename T>
void launch_sweep(const KArgs<T>& a, int d, cudaStream_t s) {
  const int D = a.g.D, L = a.g.layout;
  if (D == 1) L == 0 ? sweep_dispatch_d<T, 1, 0>(a, d, s) : sweep_dispatch_d<T, 1, 1>(a, d, s);
  if (D == 2) L == 0 ? sweep_dispatch_d<T, 2, 0>(a, d, s) : sweep_dispatch_d<T, 2, 1>(a, d, s);
  if (D == 3) L == 0 ? sweep_dispatch_d<T, 3, 0>(a, d, s) : sweep_dispatch_d<T, 3, 1>(a, d, s);
}

int auto_rows_2d(const Geom& g) {
  // aim for ~16 resident warps per SM over 148 SMs, march at least 8 rows
  const int64_t target = 148 * 16;
  int64_t rows = (g.S[1] * g.nwin + target - 1) / target;
  if (rows < 8) rows = 8;
  if (rows > g.S[1]) rows = g.S[1];
  return (int)rows;
}

int auto_rows_3d(const Geom& g) {
  // z-planes per CTA: enough CTAs for ~6 waves of 148, at least 8 planes per march
  const int64_t ww = window3d(g);
  const int64_t tiles = ((g.S[0] + ww - 1) / ww) * ((g.S[1] + 13) / 14);  // (TY = 14 estimate)
  int64_t nzc = (148 * 6 + tiles - 1) / tiles;
  if (nzc < 1) nzc = 1;
  int64_t rows = (g.S[2] + nzc - 1) / nzc;
  if (rows < 8) rows = 8;
  if (rows > g.S[2]) rows = g.S[2];
  return (int)rows;
}

template <typename T>
void launch_step2d(const KArgs<T>& a, const void* tmap, cudaStream_t s) {
  if (a.order == 2) return launch_step2d_o2<T>(a, tmap, s);
  switch (a.variant) {
    case 30: return launch_pt2d<T, 1, 16>(a, tmap, s);
    case 31: return launch_pt2d<T, 2, 8>(a, tmap, s);
    case 32: return launch_pt2d<T, 1, 8>(a, tmap, s);
    case 33: return launch_pt2d<T, 2, 16>(a, tmap, s);
    case 34: return launch_pt2d<T, 1, 8, 3>(a, tmap, s);
    case 40: return launch_cm2d<T, 1, 8, 3>(a, tmap, s);
    case 60: return launch_pp2d<T, 1, 8, 3>(a, tmap, s);
    case 61: return launch_pp2d<T, 1, 8, 2>(a, tmap, s);
    case 62: return launch_pp2d<T, 1, 16, 1>(a, tmap, s);
    case 63: return launch_pp2d<T, 2, 8, 2>(a, tmap, s);
    case 41: return launch_cm2d<T, 1, 8, 2>(a, tmap, s);
    case 42: return launch_cm2d<T, 2, 8, 2>(a, tmap, s);
    case 43: return launch_cm2d<T, 1, 16, 1>(a, tmap, s);
    case 35: return launch_pt2d<T, 1, 8, 4>(a, tmap, s);
    case 36: return launch_pt2d<T, 2, 8, 2>(a, tmap, s);
    case 0: case 37: return launch_pt2d<T, 1, 12, 2>(a, tmap, s);  // default (DESIGN.md tuning)
    case 38: return launch_pt2d<T, 1, 10, 3>(a, tmap, s);
    case 39: return launch_pt2d<T, 1, 12, 3>(a, tmap, s);
    case 44: return launch_pt2d<T, 1, 24, 1>(a, tmap, s);
    case 90: return launch_wm2d<T, 3, 8, 3>(a, tmap, s);
    case 91: return launch_wm2d<T, 4, 8, 3>(a, tmap, s);
    case 92: return launch_wm2d<T, 3, 8, 4>(a, tmap, s);
    case 93: return launch_wm2d<T, 6, 8, 3>(a, tmap, s);
    case 94: return launch_wm2d<T, 3, 8, 2>(a, tmap, s);
    case 95: return launch_wm2d<T, 4, 16, 1>(a, tmap, s);
    case 80: return launch_lr2d<T, 8, 4>(a, tmap, s);
    case 81: return launch_lr2d<T, 16, 2>(a, tmap, s);
    case 82: return launch_lr2d<T, 12, 2>(a, tmap, s);
    case 83: return launch_lr2d<T, 8, 3>(a, tmap, s);
    case 84: return launch_lr2d<T, 10, 3>(a, tmap, s);
    case 46: return launch_pt2d<T, 1, 14, 2>(a, tmap, s);
    case 47: return launch_pt2d<T, 1, 20, 1>(a, tmap, s);
    default: break;
  }
  KArgs<T> am = a;
  if (am.rows <= 0) am.rows = auto_rows_2d(a.g);
  const int nchunk = (int)((a.g.S[1] + am.rows - 1) / am.rows);
  const int ntask = a.g.nwin * nchunk;
  const int wpb = 4;
  const int grid = (ntask + wpb - 1) / wpb;
  const int sm = wpb * Ring2<T>::WB;
  // occupancy variant (min resident blocks of 128 threads per SM): register cap
  // 128 / 168 / 255; default chosen by measurement
  const int v = a.variant;
  if (v == 10) return launch_tile2d<T, 1, 16>(a, s);
  if (v == 11) return launch_tile2d<T, 1, 8>(a, s);
  if (v == 14) return launch_tile2d<T, 2, 8>(a, s);
  if (v == 4) k_step2d<T, 4><<<grid, 32 * wpb, sm, s>>>(am, a.g.nwin, ntask);
  else if (v == 2) k_step2d<T, 2><<<grid, 32 * wpb, sm, s>>>(am, a.g.nwin, ntask);
  else k_step2d<T, 3><<<grid, 32 * wpb, sm, s>>>(am, a.g.nwin, ntask);
}

template <typename T>
void launch_fill(const Geom& g, int part, T* const* bufs, cudaStream_t s) {
  const int grid = grid_for(g.P[0] * g.P[1] * g.P[2], 256);
  const int D = g.D, L = g.layout;
#define RPL_FILL(DD, LL) k_fill<T, DD, LL><<<grid, 256, 0, s>>>(g, part, bufs)
  if (D == 1) { if (L == 0) RPL_FILL(1, 0); else RPL_FILL(1, 1); }
  if (D == 2) { if (L == 0) RPL_FILL(2, 0); else RPL_FILL(2, 1); }
  if (D == 3) { if (L == 0) RPL_FILL(3, 0); else RPL_FILL(3, 1); }
#undef RPL_FILL
}

template <typename T>
void launch_maxws(const Geom& g, const T* in, double gamma, unsigned long long* smax,
                  unsigned* flag, cudaStream_t s) {
  const int grid = grid_for(g.cells(), 256);
  const int D = g.D, L = g.layout;
#define RPL_MWS(DD, LL) k_maxws<T, DD, LL><<<grid, 256, 0, s>>>(g, in, gamma, smax, flag)
  if (D == 1) { if (L == 0) RPL_MWS(1, 0); else RPL_MWS(1, 1); }
  if (D == 2) { if (L == 0) RPL_MWS(2, 0); else RPL_MWS(2, 1); }
  if (D == 3) { if (L == 0) RPL_MWS(3, 0); else RPL_MWS(3, 1); }
#undef RPL_MWS
}

template void launch_sweep<float>(const KArgs<float>&, int, cudaStream_t);
template void launch_sweep<double>(const KArgs<double>&, int, cudaStream_t);
template void launch_step2d<float>(const KArgs<float>&, const void*, cudaStream_t);
template void launch_step2d<double>(const KArgs<double>&, const void*, cudaStream_t);
template void launch_fill<float>(const Geom&, int, float* const*, cudaStream_t);
template void launch_fill<double>(const Geom&, int, double* const*, cudaStream_t);
template void launch_maxws<float>(const Geom&, const float*, double, unsigned long long*,
                                  unsigned*, cudaStream_t);
template void launch_maxws<double>(const Geom&, const double*, double, unsigned long long*,
                                   unsigned*, cudaStream_t);

}  // namespace rpl

namespace rpl {

// ---------------------------------------------------------------------------
// Flux difference (sec. 7.3): the paper's
// single-GPU FV benchmark (Table 4).  For every interior cell
//   R = sum_d (F_{i+1/2,d} - F_{i-1/2,d}),   F = Toro's FORCE flux at step dt,
// "performed for all four faces of each cell": thread per cell,
// both faces of every direction evaluated by the cell (the paper's algorithm,
// not the shared-face scheme of the step kernels).  Reads the current state
// (ghosts filled), writes R to the scratch buffer.
// ---------------------------------------------------------------------------
template <typename T, int D, int L>
__global__ void __launch_bounds__(256) k_fluxdiff(const __grid_constant__ KArgs<T> a) {
  constexpr int C = D + 2;
  const Geom& g = a.g;
  const int64_t n = g.cells();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = i % g.S[0];
    const int64_t y = (i / g.S[0]) % g.S[1];
    const int64_t z = i / (g.S[0] * g.S[1]);
    T U0[C], R[C];
    load_cell<D, L>(g, a.in, x, y, z, U0);
#pragma unroll
    for (int c = 0; c < C; ++c) R[c] = T(0);
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int64_t dx = d == 0, dy = d == 1, dz = d == 2;
      T Um[C], Up[C], Fm[C], F0[C], Fp[C], PL[C], PR[C];
      load_cell<D, L>(g, a.in, x - dx, y - dy, z - dz, Um);
      load_cell<D, L>(g, a.in, x + dx, y + dy, z + dz, Up);
      const T inv_lam = T(0.25) / a.q[d];  // 1/lam: Phi = lam F_FORCE
      if (d == 0) {
        phys_flux<D, 0>(Um, Fm, a.gm1);
        phys_flux<D, 0>(U0, F0, a.gm1);
        phys_flux<D, 0>(Up, Fp, a.gm1);
        force_face<D, 0>(Um, Fm, U0, F0, PL, a.q[0], a.nq2[0], a.gm1);
        force_face<D, 0>(U0, F0, Up, Fp, PR, a.q[0], a.nq2[0], a.gm1);
      } else if (d == 1) {
        if constexpr (D > 1) {
          phys_flux<D, 1>(Um, Fm, a.gm1);
          phys_flux<D, 1>(U0, F0, a.gm1);
          phys_flux<D, 1>(Up, Fp, a.gm1);
          force_face<D, 1>(Um, Fm, U0, F0, PL, a.q[1], a.nq2[1], a.gm1);
          force_face<D, 1>(U0, F0, Up, Fp, PR, a.q[1], a.nq2[1], a.gm1);
        }
      } else {
        if constexpr (D > 2) {
          phys_flux<D, 2>(Um, Fm, a.gm1);
          phys_flux<D, 2>(U0, F0, a.gm1);
          phys_flux<D, 2>(Up, Fp, a.gm1);
          force_face<D, 2>(Um, Fm, U0, F0, PL, a.q[2], a.nq2[2], a.gm1);
          force_face<D, 2>(U0, F0, Up, Fp, PR, a.q[2], a.nq2[2], a.gm1);
        }
      }
#pragma unroll
      for (int c = 0; c < C; ++c) R[c] = fma(PR[c] - PL[c], inv_lam, R[c]);
    }
    store_cell<D, L>(g, a.out, x, y, z, R);
  }
}

// ---------------------------------------------------------------------------
// f2, tiled 2-D SoA form: every face computed once.  Persistent CTAs of NW
// warps stream [NW rows][C][32+AL] boxes (TMA, 2-stage ring); warp j owns row
// y0 - 1 + j.  Per row: F_x, F_y of every cell; x-face l+1/2 via shuffles (the
// lane's right face, left face from the neighbour lane); (U, F_y) published,
// y-face between rows j-1 and j computed once and published; rows 1..NW-2 sum
// R = (dPhi_x) / lam_x + (dPhi_y) / lam_y with exactly k_fluxdiff's operations,
// so both kernels agree bitwise.  One read of U, one write of R per cell.
// ---------------------------------------------------------------------------
template <typename T, int NW>
struct SmemFD {
  static constexpr int W = 32, C = 4;
  static constexpr int AL = 16 / (int)sizeof(T);
  static constexpr int WB = W + AL;
  static constexpr int STAGE = NW * C * WB;
  static constexpr int UF = NW * 2 * C * W;
  static constexpr int FY = NW * C * W;
  static constexpr size_t bytes() { return (size_t)(2 * STAGE + UF + FY) * sizeof(T) + 64; }
};

template <typename T, int NW, int MB>
__global__ void __launch_bounds__(32 * NW, MB)
    k_fluxdiff_pt(const __grid_constant__ KArgs<T> a, const __grid_constant__ CUtensorMap tmap,
                  int nwin, int ntiles) {
  constexpr int D = 2, C = 4, W = 32;
  using SM = SmemFD<T, NW>;
  extern __shared__ __align__(1024) unsigned char smem[];
  T* stage = reinterpret_cast<T*>(smem);
  T* uf = stage + 2 * SM::STAGE;
  T* fyb = uf + SM::UF;
  uint64_t* bar = reinterpret_cast<uint64_t*>(fyb + SM::FY);
  const Geom& g = a.g;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int SX = (int)g.S[0], SY = (int)g.S[1];
  const int G = gridDim.x;
  const T gm1 = a.gm1;
  const T ilx = T(0.25) / a.q[0], ily = T(0.25) / a.q[1];
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
  }
  __syncthreads();
  auto issue = [&](int i) {
    const int tile = blockIdx.x + i * G;
    if (tile >= ntiles) return;
    const int s = i & 1;
    const int w = tile % nwin, yb = tile / nwin;
    mbar_arrive_expect_tx(&bar[s], SM::STAGE * (unsigned)sizeof(T));
    const int x0 = (int)g.xo + w * (W - 2) - 1;
    tma_load_box(stage + s * SM::STAGE, &tmap, &bar[s], x0 - x0 % SM::AL, 0,
                 (int)g.off[1] + yb * (NW - 2) - 1, 0);
  };
  if (threadIdx.x == 0) {
    issue(0);
    issue(1);
  }
  const int Gq = G / nwin, Gr = G - (G / nwin) * nwin;
  int win = (int)blockIdx.x % nwin, yb = (int)blockIdx.x / nwin;
  const int nyb = ntiles / nwin;
  for (int i = 0;; ++i) {
    if (yb >= nyb) break;
    const int xw = win * (W - 2) - 1;
    const int yr = yb * (NW - 2) - 1 + warp;
    const int s = i & 1;
    mbar_wait(&bar[s], (i >> 1) & 1);
    T U[C], Fx[C], Fy[C], Rx[C];
    {
      const int sh = ((int)g.xo + xw) % SM::AL;
      const T* st = stage + s * SM::STAGE + warp * C * SM::WB + sh + lane;
#pragma unroll
      for (int c = 0; c < C; ++c) U[c] = st[c * SM::WB];
    }
    phys_flux<D, 0>(U, Fx, gm1);
    phys_flux<D, 1>(U, Fy, gm1);
    {
      T Un[C], Fn[C], Pnx[C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        Un[c] = __shfl_down_sync(kFull, U[c], 1);
        Fn[c] = __shfl_down_sync(kFull, Fx[c], 1);
      }
      force_face<D, 0>(U, Fx, Un, Fn, Pnx, a.q[0], a.nq2[0], gm1);
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const T Ppv = __shfl_up_sync(kFull, Pnx[c], 1);
        Rx[c] = fma(Pnx[c] - Ppv, ilx, T(0));
      }
    }
    {
      T* w = uf + warp * 2 * C * W + lane;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        w[c * W] = U[c];
        w[(C + c) * W] = Fy[c];
      }
    }
    __syncthreads();  // (A) stage consumed, (U, F_y) published
    if (threadIdx.x == 0) {
      fence_proxy_async();
      issue(i + 2);
    }
    T Py[C];
    if (warp >= 1) {
      T Up[C], Fp[C];
      const T* r = uf + (warp - 1) * 2 * C * W + lane;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        Up[c] = r[c * W];
        Fp[c] = r[(C + c) * W];
      }
      force_face<D, 1>(Up, Fp, U, Fy, Py, a.q[1], a.nq2[1], gm1);
      T* fw = fyb + warp * C * W + lane;
#pragma unroll
      for (int c = 0; c < C; ++c) fw[c * W] = Py[c];
    }
    __syncthreads();  // (B) y-faces published
    if (warp >= 1 && warp <= NW - 2 && yr < SY && lane >= 1 && lane <= 30 && xw + lane < SX) {
      const T* fu = fyb + (warp + 1) * C * W + lane;
      T* dst = a.out + ((int64_t)((int)g.off[1] + yr) * g.rstride + (int)g.xo + xw + lane);
      const int64_t cs = g.cstride;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        *dst = fma(fu[c * W] - Py[c], ily, Rx[c]);
        dst += cs;
      }
    }
    win += Gr;
    yb += Gq;
    if (win >= nwin) {
      win -= nwin;
      ++yb;
    }
  }
}

template <typename T, int NW, int MB>
static void launch_fd_pt(const KArgs<T>& a, const void* tmap, cudaStream_t s) {
  constexpr int W = 32;
  using SM = SmemFD<T, NW>;
  const int nwin = (int)((a.g.S[0] + (W - 2) - 1) / (W - 2));
  const int nyb = (int)((a.g.S[1] + (NW - 2) - 1) / (NW - 2));
  const int ntiles = nwin * nyb;
  static int per_sm = 0;
  if (!per_sm) {
    cudaFuncSetAttribute(k_fluxdiff_pt<T, NW, MB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)SM::bytes());
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fluxdiff_pt<T, NW, MB>, 32 * NW,
                                                  SM::bytes());
    if (per_sm < 1) per_sm = 1;
  }
  int nsm = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  int grid = per_sm * nsm;
  if (grid > ntiles) grid = ntiles;
  k_fluxdiff_pt<T, NW, MB><<<grid, 32 * NW, SM::bytes(), s>>>(
      a, *reinterpret_cast<const CUtensorMap*>(tmap), nwin, ntiles);
}

int fd_tile_rows(int elem) { return 16; }

template <typename T>
void launch_fluxdiff_tiled(const KArgs<T>& a, const void* tmap, cudaStream_t s) {
  if (sizeof(T) == 4) return launch_fd_pt<T, 16, 2>(a, tmap, s);
  return launch_fd_pt<T, 16, 2>(a, tmap, s);
}
template void launch_fluxdiff_tiled<float>(const KArgs<float>&, const void*, cudaStream_t);
template void launch_fluxdiff_tiled<double>(const KArgs<double>&, const void*, cudaStream_t);

template <typename T>
void launch_fluxdiff(const KArgs<T>& a, cudaStream_t s) {
  int64_t b = (a.g.cells() + 255) / 256;
  if (b > 148 * 32) b = 148 * 32;
  const int grid = (int)(b < 1 ? 1 : b);
  const int D = a.g.D, L = a.g.layout;
#define RPL_FD(DD, LL) k_fluxdiff<T, DD, LL><<<grid, 256, 0, s>>>(a)
  if (D == 1) { if (L == 0) RPL_FD(1, 0); else RPL_FD(1, 1); }
  if (D == 2) { if (L == 0) RPL_FD(2, 0); else RPL_FD(2, 1); }
  if (D == 3) { if (L == 0) RPL_FD(3, 0); else RPL_FD(3, 1); }
#undef RPL_FD
}

template void launch_fluxdiff<float>(const KArgs<float>&, cudaStream_t);
template void launch_fluxdiff<double>(const KArgs<double>&, cudaStream_t);

}  // namespace rpl
