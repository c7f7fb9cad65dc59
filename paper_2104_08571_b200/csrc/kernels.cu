// kernels.cu -- sm_100a kernels of the split FORCE step.
//
//   k_sweep     (K-A)  one sweep along d, one thread per cell: the paper's
//                      update_state_x / update_state_y node (Listing 8).
//   k_sweep2           the same with order-2 (MUSCL-Hancock) reconstruction (f3).
//   k_step2d_ra (K-B)  all sweeps of a 2-D step in one HBM pass, TMA tiles,
//                      adjacent row pairs per warp.
//   k_step2d_o2        the same with order-2 reconstruction (f3).
//   k_fill             set_boundary + halo for every ghost of a partition.
//   k_maxws            max |u| + c over the interior (Listing 8 set_wavespeeds +
//                      then_reduce(Max)).
//   k_fluxdiff[_ra]    the sec. 7.3 flux difference (Table 4; f2): per cell / tiled.
// (Slower 2-D designs measured in rounds 1 and 2 -- one row per warp, per-warp row
// march, column march, point-to-point hand-offs, low-register, warp march,
// software-pipelined -- are described in DESIGN.md's tuning log; their code is in
// git history.)
// All step kernels write the ghost images of the cells they produce (scheme.cuh),
// so no separate boundary or halo kernel runs between steps on one rank.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "async.cuh"
#include "launch.cuh"
#include "kernels.hpp"
#include "packed.cuh"
#include "scheme.cuh"

namespace rpl {

constexpr unsigned kFull = 0xffffffffu;

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
    T Um[C], U0[C], Up[C], Am[C], Bm[C], A0[C], B0[C], Ap[C], Bp[C];
    load_cell<D, L>(g, a.in, x - dm[0], y - dm[1], z - dm[2], Um);
    load_cell<D, L>(g, a.in, x, y, z, U0);
    load_cell<D, L>(g, a.in, x + dm[0], y + dm[1], z + dm[2], Up);
    cell_ab<D, d>(Um, Am, Bm, k.lam[d], a.gm1);
    bad |= dom_word(U0[0], cell_ab<D, d>(U0, A0, B0, k.lam[d], a.gm1));
    cell_ab<D, d>(Up, Ap, Bp, k.lam[d], a.gm1);
    T PL[C], PR[C], o[C];
    face_psi<D, d>(Am, B0, PL, k.lam[d], a.gm1);
    face_psi<D, d>(A0, Bp, PR, k.lam[d], a.gm1);
#pragma unroll
    for (int c = 0; c < C; ++c) o[c] = psi_update(U0[c], PL[c], PR[c]);
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
    // FORCE between the evolved values (Ubar^R_i, Ubar^L_{i+1}) through their half-states
    // (scheme.cuh hancock_ab / face_psi, reading A1)
    T BL[3][C], AR[3][C];
#pragma unroll
    for (int j = 0; j < 3; ++j)
      bad |= hancock_ab<D, d>(U[j], U[j + 1], U[j + 2], k.h2[d], k.lam[d], a.gm1, BL[j], AR[j]);
    T PL[C], PR[C], o[C];
    face_psi<D, d>(AR[0], BL[1], PL, k.lam[d], a.gm1);
    face_psi<D, d>(AR[1], BL[2], PR, k.lam[d], a.gm1);
#pragma unroll
    for (int c = 0; c < C; ++c) o[c] = psi_update(U[2][c], PL[c], PR[c]);
    nan = max(nan, max(naninf(o[0]), naninf(o[C - 1])));
    store_cell<D, L>(g, a.out, x, y, z, o);
    if (ws) wmax = fmax(wmax, wavespeed<D>(o, a.gm1, gam));
    if (near_face<D>(g, x, y, z)) images<D, L>(a, x, y, z, o);
  }
  if (bad < 0 || nan >= kExpMask<T>) atomicOr(a.flag, 1u);
  if (ws) publish_max(a, wmax);
}

constexpr int kRows2 = 24;  // 2-D order-1 tile rows (box), 22 outputs

// TMA tile load (cp.async.bulk.tensor.4d, mbarrier completion) used by the
// persistent 2-D kernels: box [rows][C comps][32+AL slots] of a SoA buffer.
__device__ __forceinline__ void tma_load_box(void* dst, const CUtensorMap* map, uint64_t* bar,
                                             int x, int c, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(c), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
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
//       values; the half-state A = Ubar^R + lam F_y(Ubar^R) published;
//   Y2  rows 2..NW-2: y-face Psi between rows j-1 and j (face_psi with this row's
//       B = Ubar^L - lam F_y(Ubar^L)), published;
//   upd rows 2..NW-3: U^{n+1} = U* - 1/4 (Psi_{j+1/2} - Psi_{j-1/2}), store + images.
// ---------------------------------------------------------------------------
template <typename T, int NW, int C_ = 4>
struct SmemO2 {
  static constexpr int W = 32, C = C_;
  static constexpr int AL = 16 / (int)sizeof(T);
  static constexpr int WB = W + AL;
  static constexpr int STAGE = NW * C * WB;
  static constexpr int SX = NW * C * W;
  static constexpr int BR = NW * C * W;
  static constexpr int FY = NW * C * W;
  static constexpr size_t bytes() { return (size_t)(2 * STAGE + SX + BR + FY) * sizeof(T) + 64; }
};

// D = 3: the x- and y-sweeps of every z-plane (tiles over (window, row block,
// plane)); the z-sweep of the step follows as a separate pass (k_sweep2).
template <typename T, int D, int NW, int MB>
__global__ void __launch_bounds__(32 * NW, MB)
    k_step2d_o2(const __grid_constant__ KArgs<T> a, const __grid_constant__ CUtensorMap tmap,
                int nwin, int nyb, int ntiles) {
  constexpr int C = D + 2, W = 32;
  using SM = SmemO2<T, NW, C>;
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
  const bool ws = a.cf.dev != nullptr && a.cf.last;
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
    const int w = tile % nwin, r = tile / nwin, yb = r % nyb, zp = r / nyb;
    mbar_arrive_expect_tx(&bar[s], SM::STAGE * (unsigned)sizeof(T));
    const int x0 = (int)g.xo + w * (W - 4) - 2;
    tma_load_box(stage + s * SM::STAGE, &tmap, &bar[s], x0 - x0 % SM::AL, 0,
                 (int)g.off[1] + yb * (NW - 4) - 2, (int)g.off[2] + zp);
  };
  if (threadIdx.x == 0) {
    issue(0);
    issue(1);
  }
  int bad = 0;  // sign bit: domain error or NaN/Inf output (one accumulator, see k_step2d_ra)
  const bool lane_in = (lane >= 1) & (lane <= 30);   // has both x-neighbours
  const bool lane_out = (lane >= 2) & (lane <= 29);  // U* valid
  const int SZ = (int)g.S[2];
  for (int i = 0, t = (int)blockIdx.x; t < ntiles; ++i, t += G) {
    const int win = t % nwin, yq = t / nwin;  // yq = z * nyb + yb
    const int yb = D == 2 ? yq : yq % nyb;
    const int zp = D == 2 ? 0 : yq / nyb;
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
      T Pnx[C];
      {
        T A[C], B[C], Bn[C];
        const int b = hancock_ab<D, 0>(Um, U, Up, kc.h2[0], kc.lam[0], gm1, B, A);
        bad |= (lane_in & (xv >= -1) & (xv <= SX) & row_in) ? b : 0;
#pragma unroll
        for (int c = 0; c < C; ++c) Bn[c] = __shfl_down_sync(kFull, B[c], 1);
        face_psi<D, 0>(A, Bn, Pnx, kc.lam[0], gm1);
      }
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const T Ppv = __shfl_up_sync(kFull, Pnx[c], 1);
        S_[c] = psi_update(U[c], Ppv, Pnx[c]);
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
    T By[C];  // B_y of this row's evolved lower value
    if (warp >= 1 && warp <= NW - 2) {
      T Sm[C], Sp[C], Ay[C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        Sm[c] = sx[(warp - 1) * C * W + c * W + lane];
        Sp[c] = sx[(warp + 1) * C * W + c * W + lane];
      }
      const int b = hancock_ab<D, 1>(Sm, S_, Sp, kc.h2[1], kc.lam[1], gm1, By, Ay);
      bad |= (lane_out & (xv < SX) & (yr >= -1) & (yr <= SY)) ? b : 0;
      T* w = br + warp * C * W + lane;  // A_y of the evolved upper value, for warp + 1
#pragma unroll
      for (int c = 0; c < C; ++c) w[c * W] = Ay[c];
    }
    __syncthreads();  // (B) Ubar^R_y published
    // ---- Y2: face between rows warp-1 and warp
    T Py[C];
    if (warp >= 2 && warp <= NW - 2) {
      T pA[C];
      const T* r = br + (warp - 1) * C * W + lane;
#pragma unroll
      for (int c = 0; c < C; ++c) pA[c] = r[c * W];
      face_psi<D, 1>(pA, By, Py, kc.lam[1], gm1);
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
      for (int c = 0; c < C; ++c) o[c] = psi_update(S_[c], Py[c], fu[c * W]);
      T* dst = a.out + (g.row(yr, zp) * g.rstride + (int)g.xo + xv);
      const int64_t cs = g.cstride;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        *dst = o[c];
        dst += cs;
      }
      bad |= (kExpMask<T> - 1) - max(naninf(o[0]), naninf(o[C - 1]));
      if (ws) wmax = fmax(wmax, wavespeed<D>(o, gm1, gam));
      const bool zf = D == 3 && ((zp < g.pad) | (zp >= SZ - g.pad));
      if ((yr < g.pad) | (yr >= SY - g.pad) | (xv < g.pad) | (xv >= SX - g.pad) | zf)
        images<D, 0>(a, xv, yr, zp, o);
    }
  }
  if (__any_sync(kFull, bad < 0) && lane == 0) atomicOr(a.flag, 1u);
  if (ws) publish_max(a, wmax);
}

template <typename T, int NW, int MB, int D = 2>
static void launch_o2(const KArgs<T>& a, const void* tmap, cudaStream_t s) {
  constexpr int W = 32;
  using SM = SmemO2<T, NW, D + 2>;
  const int nwin = (int)((a.g.S[0] + (W - 4) - 1) / (W - 4));
  const int nyb = (int)((a.g.S[1] + (NW - 4) - 1) / (NW - 4));
  const int ntiles = nwin * nyb * (D == 3 ? (int)a.g.S[2] : 1);
  static int cache[kMaxDevices] = {0};
  const int per_sm = resident_ctas(k_step2d_o2<T, D, NW, MB>, 32 * NW, SM::bytes(), cache);
  const int nsm = sm_count();
  int grid = per_sm * nsm;
  if (grid > ntiles) grid = ntiles;
  k_step2d_o2<T, D, NW, MB><<<grid, 32 * NW, SM::bytes(), s>>>(
      a, *reinterpret_cast<const CUtensorMap*>(tmap), nwin, nyb, ntiles);
}


// Order-2 2-D tile: 24 warps (20 output rows) at one CTA per SM (DESIGN.md tuning log:
// 16 warps 72.4 us, the row-pair form 68.4 us vs 66.4 us at 1024^2).
constexpr int kRowsO2 = 24;

int tmap2d_box_o2(const Geom& g, int variant, int* box_w, int* box_rows) {
  (void)variant;
  *box_w = 32 + 16 / g.elem;
  *box_rows = kRowsO2;
  return 1;
}

template <typename T>
static void launch_step2d_o2(const KArgs<T>& a, const void* tmap, cudaStream_t s) {
  launch_o2<T, kRowsO2, 1>(a, tmap, s);
}

// ---------------------------------------------------------------------------
// Order 2, 3-D: the z-sweep as a march (SoA).  A thread owns one (x, y) column
// and a chunk of ZC planes; it carries U(z), U(z+1), the evolved upper boundary
// value of plane z and the face below plane z in registers, so every evolved
// value and every z-face is computed once (k_sweep2 evaluates each three times).
// Coalesced: a warp's threads hold consecutive x.  Same operations per cell and
// face as k_sweep2 along z: bitwise identical.  128 registers (16 warps/SM, a
// few spilled bytes) beat 168 (12 warps/SM) and 96 (heavy spills): 256^3 fp64
// order-2 step 1890 -> 1779 us; the L1 prefetch one plane ahead 1947 -> 1890 us.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(128, 4) k_zmarch2(const __grid_constant__ KArgs<T> a, int zc) {
  constexpr int D = 3, C = 5;
  const Geom& g = a.g;
  const int SX = (int)g.S[0], SY = (int)g.S[1], SZ = (int)g.S[2];
  Coef<T> k;
  if (!step_coef(a, k)) return;
  const bool ws = a.cf.dev != nullptr && a.cf.last;
  const T gam = (T)a.cf.gamma;
  const T lam = k.lam[2], h2 = k.h2[2], gm1 = a.gm1;
  T wmax = T(0);
  int bad = 0, nan = 0;
  const int64_t col = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (col < (int64_t)SX * SY) {
    const int x = (int)(col % SX), y = (int)(col / SX);
    const int z0 = blockIdx.y * zc, z1 = min(z0 + zc, SZ);
    T U0[C], U1[C], Um[C], AR[C], Pp[C];  // AR: half-state A of plane z's evolved upper value
    {
      T Umm[C], B[C], Ac[C], unused[C];
      load_cell<D, 0>(g, a.in, x, y, z0 - 2, Umm);
      load_cell<D, 0>(g, a.in, x, y, z0 - 1, Um);
      load_cell<D, 0>(g, a.in, x, y, z0, U0);
      load_cell<D, 0>(g, a.in, x, y, z0 + 1, U1);
      bad |= hancock_ab<D, 2>(Umm, Um, U0, h2, lam, gm1, unused, Ac);  // plane z0 - 1
      bad |= hancock_ab<D, 2>(Um, U0, U1, h2, lam, gm1, B, AR);        // plane z0
      face_psi<D, 2>(Ac, B, Pp, lam, gm1);                             // face z0 - 1/2
    }
    for (int z = z0; z < z1; ++z) {
      T U2[C], B[C], nA[C], P[C], o[C];
      // L1 prefetch of the plane the next iteration loads (no registers held
      // across the iteration; hides the HBM latency behind this plane's work)
      const int dist = a.variant == 76 ? 4 : 3;  // RPL_VARIANT 75: no prefetch
      if (a.variant != 75 && z + dist <= z1 + 1) {
        const T* pf = a.in + g.at(0, x, y, z + dist);
#pragma unroll
        for (int c = 0; c < C; ++c)
          asm volatile("prefetch.global.L1 [%0];" ::"l"(pf + c * g.cstride));
      }
      load_cell<D, 0>(g, a.in, x, y, z + 2, U2);
      bad |= hancock_ab<D, 2>(U0, U1, U2, h2, lam, gm1, B, nA);  // plane z + 1
      face_psi<D, 2>(AR, B, P, lam, gm1);                        // face z + 1/2
#pragma unroll
      for (int c = 0; c < C; ++c) o[c] = psi_update(U0[c], Pp[c], P[c]);
      nan = max(nan, max(naninf(o[0]), naninf(o[C - 1])));
      store_cell<D, 0>(g, a.out, x, y, z, o);
      if (ws) wmax = fmax(wmax, wavespeed<D>(o, gm1, gam));
      if (near_face<D>(g, x, y, z)) images<D, 0>(a, x, y, z, o);
#pragma unroll
      for (int c = 0; c < C; ++c) {
        Pp[c] = P[c];
        AR[c] = nA[c];
        U0[c] = U1[c];
        U1[c] = U2[c];
      }
    }
  }
  if (bad < 0 || nan >= kExpMask<T>) atomicOr(a.flag, 1u);
  if (ws) publish_max(a, wmax);
}

template <typename T>
void launch_zmarch2(const KArgs<T>& a, cudaStream_t s) {
  const int64_t cols = a.g.S[0] * a.g.S[1];
  const int bx = (int)((cols + 127) / 128);
  // z-chunks: about 8 waves of resident blocks (short tail), at least 16 planes each
  static int cache[kMaxDevices] = {0};
  const int slots = resident_ctas(k_zmarch2<T>, 128, 0, cache) * sm_count();
  int nzc = (int)((8LL * slots + bx - 1) / bx);
  const int SZ = (int)a.g.S[2];
  if (nzc > SZ / 16) nzc = SZ / 16;
  if (nzc < 1) nzc = 1;
  const int zc = (SZ + nzc - 1) / nzc;
  nzc = (SZ + zc - 1) / zc;
  k_zmarch2<T><<<dim3(bx, nzc), 128, 0, s>>>(a, zc);
}
template void launch_zmarch2<float>(const KArgs<float>&, cudaStream_t);
template void launch_zmarch2<double>(const KArgs<double>&, cudaStream_t);

// order 2, 3-D: x/y sweeps of every plane in one pass (box {32+AL, C, 16, 1})
template <typename T>
void launch_xy3d_o2(const KArgs<T>& a, const void* tmap, cudaStream_t s) {
  launch_o2<T, 16, 1, 3>(a, tmap, s);
}
template void launch_xy3d_o2<float>(const KArgs<float>&, const void*, cudaStream_t);
template void launch_xy3d_o2<double>(const KArgs<double>&, const void*, cudaStream_t);

// 2-D order-1 tile rows: 24 (22 outputs, 12 warps x 2 CTAs/SM) unless one wave of those
// CTAs covers less than one band of tiles (more x-windows than resident CTAs), where
// 16-row tiles (8 warps x 3 CTAs/SM) are faster: 9600x6000 812 vs 935 us, while
// 6400x4000 355 vs 360 us and 1024^2 are unchanged (profiles/r2/variants_2d_ab.txt).
// A 3-stage ring was slower at every size (9600x6000: 1105 / 966 us).  RPL_VARIANT 3
// forces 16 rows, any other nonzero variant 24.
int rows2d(const Geom& g, int variant) {
  if (variant == 3) return 16;
  if (variant != 0) return kRows2;
  const int nwin = (int)((g.S[0] + 29) / 30);
  return nwin > 2 * sm_count() ? 16 : kRows2;
}

int tmap2d_box(const Geom& g, int variant, int* box_w, int* box_rows) {
  *box_w = 32 + 16 / g.elem;  // 16-byte-aligned TMA box start (AL extra elements)
  *box_rows = rows2d(g, variant);
  return 1;
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


int auto_rows_3d(const Geom& g) {
  // z-planes per CTA march (each chunk recomputes 2 planes).  fp64 (k_step3d_sp, one
  // CTA per SM): 5 full-length chunks and a last one a third as long, whose short CTAs
  // fill the final wave -- round 2, profiles/r2/rows_sweep*.txt: 512^3 96 planes
  // 3.78 ms vs 64 planes 3.90 ms, 86 and 103 planes 3.90 ms (after the half-state
  // FORCE: 96 planes 3.34 ms, 80 3.36, 112 3.39, 64 3.45).  fp32 (k_step3d_rb, two CTAs
  // per SM): 20-24 planes -- after the half-state FORCE, profiles/r2/rows_sweep4.txt:
  // 384^3 22 planes 870 us vs 26: 881, 39: 890, 64: 943; 256^3 20 planes 324 us vs
  // 16: 330, 26: 329.
  int64_t rows;
  if (g.elem == 8) {
    rows = (3 * g.S[2] + 15) / 16;
  } else {
    rows = g.S[2] / 18;
    if (rows < 20) rows = 20;
    if (rows > 24) rows = 24;
  }
  if (rows < 16) rows = 16;
  if (rows > g.S[2]) rows = g.S[2];
  return (int)rows;
}


// ---------------------------------------------------------------------------
// K-B (2-D), adjacent row pairs: warp w owns tile rows 2w and 2w+1 (P = pd: two
// scalar doubles; P = pk: packed fp32), so the y-face between them is evaluated
// in registers together with the face below row 2w, and only row 2w+1's half-state
// A_y (scheme.cuh cell_ab) and that lower face go through shared memory.  Same tile walk, TMA ring and
// per-cell / per-face operations as the split kernel k_sweep: bitwise equal.
// ---------------------------------------------------------------------------
template <typename P, int NW, int MB, int NS>
__global__ void __launch_bounds__(32 * NW, MB)
    k_step2d_ra(const __grid_constant__ KArgs<typename PairElem<P>::T> a,
                const __grid_constant__ CUtensorMap tmap, int nwin, int ntiles) {
  using T = typename PairElem<P>::T;
  constexpr int D = 2, C = 4, W = 32, R = 2 * NW;
  constexpr int AL = 16 / (int)sizeof(T), WB = W + AL, STAGE = R * C * WB;
  extern __shared__ __align__(1024) unsigned char smem[];
  T* stage = reinterpret_cast<T*>(smem);
  T* xy = stage + NS * STAGE;          // A_y(U*) of row 2w+1, per warp
  T* fy = xy + NW * C * W;             // face below row 2w, per warp
  uint64_t* bar = reinterpret_cast<uint64_t*>(fy + NW * C * W);
  const Geom& g = a.g;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j0 = 2 * warp, j1 = 2 * warp + 1;
  const int wdn = max(warp - 1, 0), wup = min(warp + 1, NW - 1);
  const int SX = (int)g.S[0], SY = (int)g.S[1];
  const int G = gridDim.x;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NS; ++k) mbar_init(&bar[k], 1);
    fence_barrier_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  Coef<T> kc;
  if (!step_coef(a, kc)) return;
  const bool ws = a.cf.dev != nullptr;
  const T gam = (T)a.cf.gamma;
  T wmax = T(0);
  const P gm1(a.gm1), lx(kc.lam[0]), ly(kc.lam[1]);
  __syncthreads();
  const int* tl = a.tiles;  // tile list (shell-first halo overlap) or nullptr: every tile
  auto issue = [&](int i) {
    const int idx = blockIdx.x + i * G;
    if (idx >= ntiles) return;
    const int tile = tl ? tl[idx] : idx;
    const int s = i % NS;
    const int w = tile % nwin, yb = tile / nwin;
    mbar_arrive_expect_tx(&bar[s], STAGE * (unsigned)sizeof(T));
    const int x0 = (int)g.xo + w * (W - 2) - 1;
    tma_load_box(stage + s * STAGE, &tmap, &bar[s], x0 - x0 % AL, 0,
                 (int)g.off[1] + yb * (R - 2) - 1, 0);
  };
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NS; ++k) issue(k);
  }
  // one domain accumulator (sign bit: rho <= 0 or p <= 0 in a flux evaluation, or a
  // NaN/Inf output) and a stateless tile index keep the loop at 80 registers
  int bad = 0;
  const unsigned bar_a0 = smem_u32(&bar[0]);
  int idx = (int)blockIdx.x;
  const int64_t cs = g.cstride;
  for (int i = 0; idx < ntiles; ++i, idx += G) {
    const int tile = tl ? tl[idx] : idx;
    const int win = tile % nwin, yb = tile / nwin;
    const int xw = win * (W - 2) - 1;
    const int yr0 = yb * (R - 2) - 1 + j0, yr1 = yr0 + 1;
    const int xv = xw + lane;
    const bool in_x = (xv >= -1) & (xv <= SX);
    const bool out_x = (lane >= 1) & (lane <= W - 2) & (xv < SX);
    const int s = NS == 2 ? (i & 1) : i % NS;
    mbar_wait_u32(bar_a0 + 8 * s, (i / NS) & 1);
    // ---- X (both rows)
    P S_[C], Ay[C], By[C];
    {
      // U^n of the two rows is read from the stage twice (for A, B and again for the
      // update) instead of being held across the x-face evaluation: 80 registers
      const int sh = ((int)g.xo + xw) % AL;
      const T* r0 = stage + s * STAGE + j0 * C * WB + sh + lane;
      const T* r1 = r0 + C * WB;
      P A[C], Bn[C], Pnx[C];
      {
        P U[C], B[C];
#pragma unroll
        for (int c = 0; c < C; ++c) U[c] = P(r0[c * WB], r1[c * WB]);
        const PkDom b = dom_word(U[0], cell_ab<D, 0>(U, A, B, lx, gm1));
        bad |= ((in_x & (yr0 <= SY)) ? b.a : 0) | ((in_x & (yr1 <= SY)) ? b.b : 0);
#pragma unroll
        for (int c = 0; c < C; ++c) Bn[c] = shfl_down1(B[c]);
      }
      face_psi<D, 0>(A, Bn, Pnx, lx, gm1);
#pragma unroll
      for (int c = 0; c < C; ++c)
        S_[c] = psi_update(P(r0[c * WB], r1[c * WB]), shfl_up1(Pnx[c]), Pnx[c]);
    }
    {
      const PkDom b = dom_word(S_[0], cell_ab<D, 1>(S_, Ay, By, ly, gm1));
      bad |= ((out_x & (yr0 <= SY)) ? b.a : 0) | ((out_x & (yr1 <= SY)) ? b.b : 0);
    }
    {
      T* x1 = xy + warp * C * W + lane;
#pragma unroll
      for (int c = 0; c < C; ++c) x1[c * W] = Ay[c].y;
    }
    P Py[C];
    __syncthreads();  // (A) stage s consumed; row 2w+1 published
    if (threadIdx.x == 0) {
      fence_proxy_async();
      issue(i + NS);
    }
    // ---- Y faces (2w-1 | 2w) and (2w | 2w+1), one pair evaluation
    {
      const T* pdn = xy + wdn * C * W + lane;
      P AL_[C];
#pragma unroll
      for (int c = 0; c < C; ++c) AL_[c] = P(pdn[c * W], Ay[c].x);
      face_psi<D, 1>(AL_, By, Py, ly, gm1);
      T* f0 = fy + warp * C * W + lane;
#pragma unroll
      for (int c = 0; c < C; ++c) f0[c * W] = Py[c].x;
    }
    __syncthreads();  // (B) faces below each pair published
    // ---- update + store
    {
      const T* fu = fy + wup * C * W + lane;  // face below row 2w+2
      P o[C];
#pragma unroll
      for (int c = 0; c < C; ++c) o[c] = psi_update(S_[c], Py[c], P(Py[c].y, fu[c * W]));
      const bool st0 = out_x & (j0 >= 1) & (yr0 < SY);
      const bool st1 = out_x & (j1 <= R - 2) & (yr1 < SY);
      const bool xface = (xv < g.pad) | (xv >= SX - g.pad);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const bool st = h ? st1 : st0;
        if (!st) continue;
        const int yr = h ? yr1 : yr0;
        T v[C];
#pragma unroll
        for (int c = 0; c < C; ++c) v[c] = h ? o[c].y : o[c].x;
        T* dst = a.out + ((int64_t)((int)g.off[1] + yr) * g.rstride + (int)g.xo + xv);
#pragma unroll
        for (int c = 0; c < C; ++c) dst[c * cs] = v[c];
        bad |= (kExpMask<T> - 1) - max(naninf(v[0]), naninf(v[C - 1]));
        if (ws) wmax = fmax(wmax, wavespeed<D>(v, a.gm1, gam));
        if (xface | (yr < g.pad) | (yr >= SY - g.pad)) images<D, 0>(a, xv, yr, 0, v);
      }
    }
  }
  if (__any_sync(kFull, bad < 0) && lane == 0) atomicOr(a.flag, 1u);
  if (ws) publish_max(a, wmax);
}

template <typename P, int NW, int MB, int NS>
static void launch_ra2d(const KArgs<typename PairElem<P>::T>& a, const void* tmap,
                        cudaStream_t s) {
  using T = typename PairElem<P>::T;
  constexpr int W = 32, R = 2 * NW, C = 4, AL = 16 / (int)sizeof(T);
  const size_t bytes = (size_t)(NS * R * C * (W + AL) + NW * 2 * C * W) * sizeof(T) + 64;
  const int nwin = (int)((a.g.S[0] + (W - 2) - 1) / (W - 2));
  const int nyb = (int)((a.g.S[1] + (R - 2) - 1) / (R - 2));
  const int ntiles = a.tiles ? a.ntiles : nwin * nyb;
  if (ntiles <= 0) return;
  if constexpr (sizeof(T) == 4) pk_set_negzero(s);
  static int cache[kMaxDevices] = {0};
  const int per_sm = resident_ctas(k_step2d_ra<P, NW, MB, NS>, 32 * NW, bytes, cache);
  int grid = per_sm * sm_count();
  if (grid > ntiles) grid = ntiles;
  launch_pdl(k_step2d_ra<P, NW, MB, NS>, grid, 32 * NW, bytes, s, a,
             *reinterpret_cast<const CUtensorMap*>(tmap), nwin, ntiles);
}

// 2-D order-1 kernel: adjacent row pairs (k_step2d_ra), 24-row tiles (22 outputs) of
// 12 warps, 2 CTAs/SM, 80 registers: round 2, profiles/r2/variants_2d_tiles.txt --
// 6400x4000 402 -> 384 us, 9600x6000 884 -> 847 us, 1024^2 27.0 / 27.1 us against the
// round-1 16-row tiles of 8 warps x 3 CTAs (a 3-stage ring: slower); 14 warps x 2
// (72 registers) 398 / 1007 us, 10 warps x 2 418 / 919 us, 20 warps x 1 413 / 949 us
// (profiles/r2/variants_2d_tiles2.txt).
template <typename T>
void launch_step2d(const KArgs<T>& a, const void* tmap, cudaStream_t s) {
  if (a.order == 2) return launch_step2d_o2<T>(a, tmap, s);
  using P = typename std::conditional<sizeof(T) == 8, pd, pk>::type;
  if (rows2d(a.g, a.variant) == 16) return launch_ra2d<P, 8, 3, 2>(a, tmap, s);
  launch_ra2d<P, kRows2 / 2, 2, 2>(a, tmap, s);
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
      T Um[C], Up[C], Am[C], Bm[C], A0[C], B0[C], Ap[C], Bp[C], PL[C], PR[C];
      load_cell<D, L>(g, a.in, x - dx, y - dy, z - dz, Um);
      load_cell<D, L>(g, a.in, x + dx, y + dy, z + dz, Up);
      const T lam = a.lam[d];
      const T inv4l = T(0.25) / lam;  // 1/(4 lam): Psi = 4 lam F_FORCE
      if (d == 0) {
        cell_ab<D, 0>(Um, Am, Bm, lam, a.gm1);
        cell_ab<D, 0>(U0, A0, B0, lam, a.gm1);
        cell_ab<D, 0>(Up, Ap, Bp, lam, a.gm1);
        face_psi<D, 0>(Am, B0, PL, lam, a.gm1);
        face_psi<D, 0>(A0, Bp, PR, lam, a.gm1);
      } else if (d == 1) {
        if constexpr (D > 1) {
          cell_ab<D, 1>(Um, Am, Bm, lam, a.gm1);
          cell_ab<D, 1>(U0, A0, B0, lam, a.gm1);
          cell_ab<D, 1>(Up, Ap, Bp, lam, a.gm1);
          face_psi<D, 1>(Am, B0, PL, lam, a.gm1);
          face_psi<D, 1>(A0, Bp, PR, lam, a.gm1);
        }
      } else {
        if constexpr (D > 2) {
          cell_ab<D, 2>(Um, Am, Bm, lam, a.gm1);
          cell_ab<D, 2>(U0, A0, B0, lam, a.gm1);
          cell_ab<D, 2>(Up, Ap, Bp, lam, a.gm1);
          face_psi<D, 2>(Am, B0, PL, lam, a.gm1);
          face_psi<D, 2>(A0, Bp, PR, lam, a.gm1);
        }
      }
#pragma unroll
      for (int c = 0; c < C; ++c) R[c] = fma(PR[c] - PL[c], inv4l, R[c]);
    }
    store_cell<D, L>(g, a.out, x, y, z, R);
  }
}

// ---------------------------------------------------------------------------
// f2, tiled 2-D SoA form: every face computed once.  Persistent CTAs of NW
// warps stream [NW rows][C][32+AL] boxes (TMA, 2-stage ring); warp j owns row
// y0 - 1 + j.  Per row: the half-states A, B (scheme.cuh cell_ab) of every cell in x
// and y; x-face l+1/2 via shuffles (the lane's right face from its A and the
// neighbour's B, left face from the neighbour lane); A_y published, y-face between
// rows j-1 and j computed once and published; rows 1..NW-2 sum
// R = (dPsi_x) / (4 lam_x) + (dPsi_y) / (4 lam_y) with exactly k_fluxdiff's
// operations, so both kernels agree bitwise.  One read of U, one write of R per cell.
// ---------------------------------------------------------------------------
template <typename T, int NW>
struct SmemFD {
  static constexpr int W = 32, C = 4;
  static constexpr int AL = 16 / (int)sizeof(T);
  static constexpr int WB = W + AL;
  static constexpr int STAGE = NW * C * WB;
  static constexpr int UF = NW * C * W;
  static constexpr int FY = NW * C * W;
  static constexpr size_t bytes() { return (size_t)(2 * STAGE + UF + FY) * sizeof(T) + 64; }
};

template <int NW, int MB, typename P = pk>
__global__ void __launch_bounds__(32 * NW, MB)
    k_fluxdiff_ra(const __grid_constant__ KArgs<typename PairElem<P>::T> a,
                  const __grid_constant__ CUtensorMap tmap, int nwin, int ntiles) {
  using T = typename PairElem<P>::T;
  constexpr int D = 2, C = 4, W = 32, R = 2 * NW;
  using SM = SmemFD<T, R>;  // stage geometry of the 2 NW-row box
  extern __shared__ __align__(1024) unsigned char smem[];
  T* stage = reinterpret_cast<T*>(smem);
  T* uf = stage + 2 * SM::STAGE;
  T* fyb = uf + NW * C * W;
  uint64_t* bar = reinterpret_cast<uint64_t*>(fyb + NW * C * W);
  const Geom& g = a.g;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j0 = 2 * warp, j1 = 2 * warp + 1;
  const int wdn = max(warp - 1, 0), wup = min(warp + 1, NW - 1);
  const int SX = (int)g.S[0], SY = (int)g.S[1];
  const int G = gridDim.x;
  const P gm1(a.gm1);
  const P lx(a.lam[0]), ly(a.lam[1]);
  const P ilx(T(0.25) / a.lam[0]), ily(T(0.25) / a.lam[1]);
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
                 (int)g.off[1] + yb * (R - 2) - 1, 0);
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
    const int yr0 = yb * (R - 2) - 1 + j0, yr1 = yr0 + 1;
    const int s = i & 1;
    mbar_wait(&bar[s], (i >> 1) & 1);
    P U[C], Ay[C], By[C], Rx[C];
    {
      const int sh = ((int)g.xo + xw) % SM::AL;
      const T* s0 = stage + s * SM::STAGE + j0 * C * SM::WB + sh + lane;
      const T* s1 = s0 + C * SM::WB;
#pragma unroll
      for (int c = 0; c < C; ++c) U[c] = P(s0[c * SM::WB], s1[c * SM::WB]);
    }
    {
      P Ax[C], Bx[C], Bn[C], Pnx[C];
      cell_ab<D, 0>(U, Ax, Bx, lx, gm1);
#pragma unroll
      for (int c = 0; c < C; ++c) Bn[c] = shfl_down1(Bx[c]);
      face_psi<D, 0>(Ax, Bn, Pnx, lx, gm1);
#pragma unroll
      for (int c = 0; c < C; ++c) Rx[c] = fma(Pnx[c] - shfl_up1(Pnx[c]), ilx, P(T(0)));
    }
    cell_ab<D, 1>(U, Ay, By, ly, gm1);
    {
      T* w1 = uf + warp * C * W + lane;  // row 2w+1 for warp w+1
#pragma unroll
      for (int c = 0; c < C; ++c) w1[c * W] = Ay[c].y;
    }
    __syncthreads();  // (A)
    if (threadIdx.x == 0) {
      fence_proxy_async();
      issue(i + 2);
    }
    P Py[C];
    {
      const T* pdn = uf + wdn * C * W + lane;
      P AL_[C];
#pragma unroll
      for (int c = 0; c < C; ++c) AL_[c] = P(pdn[c * W], Ay[c].x);
      face_psi<D, 1>(AL_, By, Py, ly, gm1);
      T* f0 = fyb + warp * C * W + lane;  // face below row 2w, for warp w-1
#pragma unroll
      for (int c = 0; c < C; ++c) f0[c * W] = Py[c].x;
    }
    __syncthreads();  // (B)
    {
      const bool xok = lane >= 1 && lane <= 30 && xw + lane < SX;
      const bool ok0 = xok && j0 >= 1 && yr0 < SY;
      const bool ok1 = xok && j1 <= R - 2 && yr1 < SY;
      const T* fu = fyb + wup * C * W + lane;  // face below row 2w+2
      P o[C];
#pragma unroll
      for (int c = 0; c < C; ++c)
        o[c] = fma(P(Py[c].y, fu[c * W]) - P(Py[c].x, Py[c].y), ily, Rx[c]);
      const int64_t cs = g.cstride;
      if (ok0) {
        T* dst = a.out + ((int64_t)((int)g.off[1] + yr0) * g.rstride + (int)g.xo + xw + lane);
#pragma unroll
        for (int c = 0; c < C; ++c) dst[c * cs] = o[c].x;
      }
      if (ok1) {
        T* dst = a.out + ((int64_t)((int)g.off[1] + yr1) * g.rstride + (int)g.xo + xw + lane);
#pragma unroll
        for (int c = 0; c < C; ++c) dst[c * cs] = o[c].y;
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

template <int NW, int MB, typename P = pk>
static void launch_fd_ra(const KArgs<typename PairElem<P>::T>& a, const void* tmap,
                         cudaStream_t s) {
  using T = typename PairElem<P>::T;
  constexpr int W = 32, R = 2 * NW, C = 4;
  using SM = SmemFD<T, R>;
  const size_t bytes = (size_t)(2 * SM::STAGE + NW * 2 * C * W) * sizeof(T) + 64;
  const int nwin = (int)((a.g.S[0] + (W - 2) - 1) / (W - 2));
  const int nyb = (int)((a.g.S[1] + (R - 2) - 1) / (R - 2));
  const int ntiles = nwin * nyb;
  if constexpr (sizeof(T) == 4) pk_set_negzero(s);
  static int cache[kMaxDevices] = {0};
  const int per_sm = resident_ctas(k_fluxdiff_ra<NW, MB, P>, 32 * NW, bytes, cache);
  const int nsm = sm_count();
  int grid = per_sm * nsm;
  if (grid > ntiles) grid = ntiles;
  k_fluxdiff_ra<NW, MB, P><<<grid, 32 * NW, bytes, s>>>(
      a, *reinterpret_cast<const CUtensorMap*>(tmap), nwin, ntiles);
}

// fp32: 24-row tiles (12 warps x 2 CTAs/SM) -- round 2, profiles/r2/variants_fd_tiles2.txt:
// 32768^2 13.0-13.7 -> 8.3 ms, 16384^2 2.12 -> 1.97 ms, 8192^2 505 -> 497 us against the
// 16-row tiles of 8 warps x 4 CTAs (RPL_VARIANT 4: 8 warps x 3 CTAs, 5: the old tiles).
// fp64: 16-row tiles x 2 CTAs (RPL_VARIANT 3: 24-row tiles x 1 CTA)
int fd_tile_rows(int elem, int variant) {
  if (variant == 6) return 32;
  if (elem == 4) return (variant == 4 || variant == 5) ? 16 : 24;
  return variant == 3 ? 24 : 16;
}

template <typename T>
void launch_fluxdiff_tiled(const KArgs<T>& a, const void* tmap, cudaStream_t s) {
  // adjacent row pairs: fp32 packed (FFMA2) 24-row tiles of 12 warps x 2 CTAs/SM, fp64
  // double pairs 16-row tiles x 2 CTAs/SM (round 1: the one-row-per-warp and
  // rows-w,w+8 forms were slower -- profiles/r1/fd_*.txt; tile shapes: fd_tile_rows)
  if constexpr (sizeof(T) == 4) {
    if (a.variant == 4) return launch_fd_ra<8, 3>(a, tmap, s);
    if (a.variant == 5) return launch_fd_ra<8, 4>(a, tmap, s);
    if (a.variant == 6) return launch_fd_ra<16, 2>(a, tmap, s);
    return launch_fd_ra<12, 2>(a, tmap, s);
  } else {
    if (a.variant == 3) return launch_fd_ra<12, 1, pd>(a, tmap, s);
    if (a.variant == 6) return launch_fd_ra<16, 1, pd>(a, tmap, s);
    return launch_fd_ra<8, 2, pd>(a, tmap, s);
  }
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
