// kernels3d.cu -- K-B (3-D): the x-, y- and z-sweeps of one step fused into one
// HBM pass, TMA-staged.
//
// CTA tile: one x-window of 32 slots (lane l <-> x = 30 w - 1 + l; lanes 0 and 31
// are the x-halo), 16 tile rows in y (8 warps, warp w owns the adjacent rows 2w and
// 2w+1 as a pair: packed FFMA2 lanes `pk` in fp32, two scalar doubles `pd` in
// fp64; rows 0 and 15 are the y-halo, 14 output rows), and a chunk of z-planes the
// CTA marches through (2.5-D streaming).  Per z-plane:
//   TMA   one elected thread streams the plane tile [16 rows][C comps][32+AL] into
//         an NS-stage shared-memory ring (cp.async.bulk.tensor.4d, mbarrier
//         completion), NS planes ahead of the compute;
//   X     every warp x-sweeps its two rows in registers (half-states A, B of every
//         cell, scheme.cuh cell_ab; one warp shuffle of B shares each x-face, which
//         is computed once by face_psi), forms the y half-states (A_y, B_y) of the
//         result and publishes row 2w+1's A_y in shared memory;
//   Y     warp w computes the y-faces (2w-1|2w) and (2w|2w+1) in one pair
//         evaluation (the second in registers) and publishes the first;
//   Z     every warp keeps a z-march state per cell in registers (U** of the
//         previous plane, its A_z and the previous z-face Psi), computes the
//         z-face, updates and stores plane z-1 (+ ghost images on partition faces).
// Two __syncthreads per plane order the shared-memory hand-offs.  HBM traffic per
// cell-step is one read of U^n (plus the tile halo, mostly L2 hits) and one write
// of U^{n+1}; the halo rows/planes are recomputed, not re-stored.
// k_step3d_rb runs the phases in this order; k_step3d_sp overlaps the X phase of
// plane k+1 with the Z phase of plane k (software pipelining, fp64 default).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <limits.h>
#include <stdlib.h>

#include <type_traits>

#include "async.cuh"
#include "launch.cuh"
#include "kernels.hpp"
#include "packed.cuh"
#include "scheme.cuh"

namespace rpl {

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int x, int c, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(c), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

template <int D, int L, typename T>
__device__ __noinline__ void images3_nl(const KArgs<T>* a, int64_t x, int64_t y, int64_t z, T v0,
                                        T v1, T v2, T v3, T v4) {
  const T v[5] = {v0, v1, v2, v3, v4};
  write_images<D, L>(a->g, a->outs, a->lo, x, y, z, v);
}

// ------------------------------------------------------------------------
// k_step3d_rb: the round-1 row-pair tile walk (adjacent row pairs, TMA ring, two CTA
// barriers per plane) with the per-plane bookkeeping taken off the issue path
// (round-1 ncu: 61 % of that kernel's issued instructions were not arithmetic,
// and IMAD moves compete with FFMA2 for the FMA pipe):
//  * domain check: per row of the pair one running minimum of hi(rho),
//    hi(p) over the states the sweeps read -- U^n (x-flux), U* (y-flux), U** (z-flux)
//    -- and one running maximum of the outputs' |bits| (NaN/Inf), unmasked in the
//    loop (one VIMNMX3 per state); the lane's loop-invariant output mask is applied
//    once after the march.  Checking exactly the tile's output cells covers every
//    interior cell once (the ghost and halo cells other tiles' lanes hold are copies
//    of interior cells, checked by their owners);
//  * ghost images behind a CTA-uniform test (tile within pad of a partition face in
//    x or y, or a boundary plane); stores predicated;
//  * NS-stage TMA ring (loads issued NS planes ahead).
// Per cell and face the operations are scheme.cuh's, in the same order: bitwise
// equal to the split kernel k_sweep.
// ------------------------------------------------------------------------
template <int NW, typename T, int NS>
struct SmemRB {
  static constexpr int W = 32, R = 2 * NW, C = 5;
  static constexpr int AL = 16 / (int)sizeof(T);
  static constexpr int WB = W + AL;
  static constexpr int STAGE = R * C * WB;
  static constexpr int XY = NW * C * W;      // A_y(U*) of row 2w+1, per warp
  static constexpr int FY = NW * C * W;      // face below row 2w, per warp
  static constexpr size_t bytes() { return (size_t)(NS * STAGE + XY + FY) * sizeof(T) + 8 * NS; }
};

template <typename P>
struct ZPlane {
  P us[5];  // U** of the previous plane
  P az[5];  // A_z(U**) = U** + lam_z F_z(U**) of the previous plane (scheme.cuh cell_ab)
  P ph[5];  // z-face Psi below the previous plane
};

template <int NW, int MB, int L, typename P, int NS>
__global__ void __launch_bounds__(32 * NW, MB)
    k_step3d_rb(const __grid_constant__ KArgs<typename PairElem<P>::T> a,
                const __grid_constant__ CUtensorMap tmap, int nwin, int nyb) {
  using T = typename PairElem<P>::T;
  constexpr int D = 3, C = 5, W = 32, R = 2 * NW, TY = R - 2;
  using SM = SmemRB<NW, T, NS>;
  extern __shared__ __align__(1024) unsigned char smem[];
  T* stage = reinterpret_cast<T*>(smem);
  T* xy = stage + NS * SM::STAGE;
  T* fyb = xy + SM::XY;
  uint64_t* bar = reinterpret_cast<uint64_t*>(fyb + SM::FY);
  const Geom& g = a.g;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int t = a.tiles ? a.tiles[blockIdx.x] : (int)blockIdx.x;
  const int win = t % nwin;
  t /= nwin;
  const int yb = t % nyb;
  const int zc = t / nyb;
  const int xw = win * (W - 2) - 1;
  const int y0 = yb * TY;
  const int z0 = zc * a.rows;
  const int z1 = min(z0 + a.rows, (int)g.S[2]);
  const int SX = (int)g.S[0], SY = (int)g.S[1], SZ = (int)g.S[2], pad = g.pad;
  const int j0 = 2 * warp, j1 = 2 * warp + 1;
  const int yr0 = y0 - 1 + j0, yr1 = y0 - 1 + j1;
  const int xs = xw + lane;
  // CTA-uniform: some output cell of the tile lies within pad of an x or y partition face
  const bool edge_xy = (xw + 1 < pad) | (xw + W - 2 >= SX - pad) | (y0 < pad) |
                       (y0 + TY - 1 >= SY - pad);
  Coef<T> kc;
  if (!step_coef(a, kc)) return;
  const bool ws = a.cf.dev != nullptr;

  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < NS; ++s) mbar_init(&bar[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  const int sh = (int)(g.xo + xw) % SM::AL;
  const int tx = (int)(g.xo + xw) - sh, ty = (int)(g.off[1] + y0 - 1);
  const int nplanes = z1 - (z0 - 1) + 1;
  auto issue = [&](int kz) {
    if (kz >= nplanes) return;
    const int s = kz % NS;
    mbar_arrive_expect_tx(&bar[s], SM::STAGE * (unsigned)sizeof(T));
    tma_load_4d(stage + s * SM::STAGE, &tmap, &bar[s], L == 0 ? tx : tx * C, 0, ty,
                (int)(g.off[2] + z0 - 1 + kz));
  };
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < NS; ++s) issue(s);
  }

  // domain minima (U^n, U*, U**) and output NaN/Inf maxima, per row of the pair
  int dm0 = INT_MAX, dm1 = INT_MAX, nn0 = 0, nn1 = 0;
  T wmax = T(0);
  const P gm1(a.gm1);
  const P lx(kc.lam[0]), ly(kc.lam[1]), lz(kc.lam[2]);
  const int64_t plane = g.rstride * g.P[1], cs = g.cstride;
  T* dst0 = a.out + g.row(yr0, z0 - 1) * g.rstride + (g.xo + xs) * g.xstride;
  T* dst1 = dst0 + g.rstride;
  const int wdn = max(warp - 1, 0), wup = min(warp + 1, NW - 1);
  // stage reads of this lane's two rows
  constexpr int cst = L == 0 ? SM::WB : 1;
  const int xoff = (L == 0 ? sh + lane : (sh + lane) * C) + j0 * C * SM::WB;
  // per-lane output masks (loop-invariant)
  const bool out_x = (lane >= 1) & (lane <= W - 2) & (xs < SX);
  const bool st0 = out_x & (j0 >= 1) & (yr0 < SY);
  const bool st1 = out_x & (j1 <= TY) & (yr1 < SY);

  auto body = [&](const int kz, const ZPlane<P>& zp, ZPlane<P>& zn) {
    const int s = kz % NS;
    mbar_wait(&bar[s], (kz / NS) & 1);
    P U[C], S_[C], Ay[C], By[C];
    {
      const T* r0 = stage + s * SM::STAGE + xoff;
      const T* r1 = r0 + C * SM::WB;
#pragma unroll
      for (int c = 0; c < C; ++c) U[c] = P(r0[c * cst], r1[c * cst]);
    }
    {
      P A[C], B[C], Bn[C], Pnx[C];
      dom_min(dm0, dm1, U[0], cell_ab<D, 0>(U, A, B, lx, gm1));
#pragma unroll
      for (int c = 0; c < C; ++c) Bn[c] = shfl_down1(B[c]);
      face_psi<D, 0>(A, Bn, Pnx, lx, gm1);
#pragma unroll
      for (int c = 0; c < C; ++c) S_[c] = psi_update(U[c], shfl_up1(Pnx[c]), Pnx[c]);
    }
    dom_min(dm0, dm1, S_[0], cell_ab<D, 1>(S_, Ay, By, ly, gm1));
    {
      T* x1 = xy + warp * C * W + lane;  // row 2w+1 for warp w+1
#pragma unroll
      for (int c = 0; c < C; ++c) x1[c * W] = Ay[c].y;
    }
    P Py[C];
    __syncthreads();  // (A) stage s consumed, rows 2w+1 published
    if (threadIdx.x == 0) {
      fence_proxy_async();
      issue(kz + NS);
    }
    // Y: faces (2w-1 | 2w) and (2w | 2w+1) in one pair evaluation
    {
      const T* pdn = xy + wdn * C * W + lane;
      P AL_[C];
#pragma unroll
      for (int c = 0; c < C; ++c) AL_[c] = P(pdn[c * W], Ay[c].x);
      face_psi<D, 1>(AL_, By, Py, ly, gm1);
      T* f0 = fyb + warp * C * W + lane;  // face below row 2w, for warp w-1
#pragma unroll
      for (int c = 0; c < C; ++c) f0[c * W] = Py[c].x;
    }
    __syncthreads();  // (B) faces published
    {
      const T* fu = fyb + wup * C * W + lane;  // face below row 2w+2 (warp w+1)
#pragma unroll
      for (int c = 0; c < C; ++c) zn.us[c] = psi_update(S_[c], Py[c], P(Py[c].y, fu[c * W]));
      P Bz[C];
      dom_min(dm0, dm1, zn.us[0], cell_ab<D, 2>(zn.us, zn.az, Bz, lz, gm1));
      if (kz >= 1) {
        face_psi<D, 2>(zp.az, Bz, zn.ph, lz, gm1);
        if (kz >= 2) {
          // update and store plane z - 1
          P o[C];
#pragma unroll
          for (int c = 0; c < C; ++c) o[c] = psi_update(zp.us[c], zp.ph[c], zn.ph[c]);
          dst0 += plane;
          dst1 += plane;
          nn0 = max(nn0, max(naninf(o[0].x), naninf(o[C - 1].x)));
          nn1 = max(nn1, max(naninf(o[0].y), naninf(o[C - 1].y)));
          if (st0) {
#pragma unroll
            for (int c = 0; c < C; ++c) dst0[c * cs] = o[c].x;
          }
          if (st1) {
#pragma unroll
            for (int c = 0; c < C; ++c) dst1[c * cs] = o[c].y;
          }
          if (ws) {
            T v0[C], v1[C];
#pragma unroll
            for (int c = 0; c < C; ++c) {
              v0[c] = o[c].x;
              v1[c] = o[c].y;
            }
            const T gam = (T)a.cf.gamma;
            if (st0) wmax = fmax(wmax, wavespeed<D>(v0, a.gm1, gam));
            if (st1) wmax = fmax(wmax, wavespeed<D>(v1, a.gm1, gam));
          }
          const int zo = z0 - 2 + kz;  // the stored plane
          const bool zf = (zo < pad) | (zo >= SZ - pad);
          if (edge_xy | zf) {
            const bool xface = (xs < pad) | (xs >= SX - pad);
            const bool yf0 = (yr0 < pad) | (yr0 >= SY - pad);
            const bool yf1 = (yr1 < pad) | (yr1 >= SY - pad);
            if (st0 & (xface | yf0 | zf)) {
              T v[C];
#pragma unroll
              for (int c = 0; c < C; ++c) v[c] = o[c].x;
              if (g.img_fast)
                images_single<D>(g, a.out, xs, yr0, zo, v);
              else
                images3_nl<D, L, T>(&a, xs, yr0, zo, v[0], v[1], v[2], v[3], v[4]);
            }
            if (st1 & (xface | yf1 | zf)) {
              T v[C];
#pragma unroll
              for (int c = 0; c < C; ++c) v[c] = o[c].y;
              if (g.img_fast)
                images_single<D>(g, a.out, xs, yr1, zo, v);
              else
                images3_nl<D, L, T>(&a, xs, yr1, zo, v[0], v[1], v[2], v[3], v[4]);
            }
          }
        }
      }
    }
  };

  ZPlane<P> za, zb;
  int kz = 0;
#pragma unroll 1
  for (; kz < nplanes; ++kz) {
    body(kz, za, zb);
    za = zb;
  }

  // the output masks, applied once
  const bool bad = (st0 & ((dm0 <= 0) | (nn0 >= kExpMask<T>))) |
                   (st1 & ((dm1 <= 0) | (nn1 >= kExpMask<T>)));
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(a.flag, 1u);
  if (ws) publish_max(a, wmax);
}

// ------------------------------------------------------------------------
// k_step3d_sp: k_step3d_rb software-pipelined across planes.  After barrier (B) of
// plane k a warp waits for stage k+1 and then runs, in one basic block, the
// x-sweep of plane k+1 and the y-update + z-march of plane k -- two independent
// instruction streams the scheduler interleaves (ncu on k_step3d_rb: the z-march
// region stalled on fixed-latency dependencies while the FMA pipe idled).  Row
// 2w+1 of plane k+1 is published after (B) of plane k, when every warp is done
// reading plane k's rows.  Stores are predicated (no branch splits the block);
// ghost images and the device-CFL wavespeed follow it behind uniform branches.
// Same per-cell operations as k_step3d_rb (bitwise equal).
// ------------------------------------------------------------------------
template <int NW, int MB, int L, typename P, int NS>
__global__ void __launch_bounds__(32 * NW, MB)
    k_step3d_sp(const __grid_constant__ KArgs<typename PairElem<P>::T> a,
                const __grid_constant__ CUtensorMap tmap, int nwin, int nyb) {
  using T = typename PairElem<P>::T;
  constexpr int D = 3, C = 5, W = 32, R = 2 * NW, TY = R - 2;
  using SM = SmemRB<NW, T, NS>;
  extern __shared__ __align__(1024) unsigned char smem[];
  T* stage = reinterpret_cast<T*>(smem);
  T* xy = stage + NS * SM::STAGE;
  T* fyb = xy + SM::XY;
  uint64_t* bar = reinterpret_cast<uint64_t*>(fyb + SM::FY);
  const Geom& g = a.g;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int t = a.tiles ? a.tiles[blockIdx.x] : (int)blockIdx.x;
  const int win = t % nwin;
  t /= nwin;
  const int yb = t % nyb;
  const int zc = t / nyb;
  const int xw = win * (W - 2) - 1;
  const int y0 = yb * TY;
  const int z0 = zc * a.rows;
  const int z1 = min(z0 + a.rows, (int)g.S[2]);
  const int SX = (int)g.S[0], SY = (int)g.S[1], SZ = (int)g.S[2], pad = g.pad;
  const int j0 = 2 * warp, j1 = 2 * warp + 1;
  const int yr0 = y0 - 1 + j0, yr1 = y0 - 1 + j1;
  const int xs = xw + lane;
  const bool edge_xy = (xw + 1 < pad) | (xw + W - 2 >= SX - pad) | (y0 < pad) |
                       (y0 + TY - 1 >= SY - pad);
  Coef<T> kc;
  if (!step_coef(a, kc)) return;
  const bool ws = a.cf.dev != nullptr;

  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < NS; ++s) mbar_init(&bar[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  const int sh = (int)(g.xo + xw) % SM::AL;
  const int tx = (int)(g.xo + xw) - sh, ty = (int)(g.off[1] + y0 - 1);
  const int nplanes = z1 - (z0 - 1) + 1;  // >= 3
  auto issue = [&](int kz) {
    if (kz >= nplanes) return;
    const int s = kz % NS;
    mbar_arrive_expect_tx(&bar[s], SM::STAGE * (unsigned)sizeof(T));
    tma_load_4d(stage + s * SM::STAGE, &tmap, &bar[s], L == 0 ? tx : tx * C, 0, ty,
                (int)(g.off[2] + z0 - 1 + kz));
  };
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < NS; ++s) issue(s);
  }

  int dm0 = INT_MAX, dm1 = INT_MAX, nn0 = 0, nn1 = 0;
  T wmax = T(0);
  const P gm1(a.gm1);
  const P lx(kc.lam[0]), ly(kc.lam[1]), lz(kc.lam[2]);
  const int64_t plane = g.rstride * g.P[1], cs = g.cstride;
  T* dst0 = a.out + g.row(yr0, z0 - 1) * g.rstride + (g.xo + xs) * g.xstride;
  T* dst1 = dst0 + g.rstride;
  const int wdn = max(warp - 1, 0), wup = min(warp + 1, NW - 1);
  constexpr int cst = L == 0 ? SM::WB : 1;
  const int xoff = (L == 0 ? sh + lane : (sh + lane) * C) + j0 * C * SM::WB;
  const bool out_x = (lane >= 1) & (lane <= W - 2) & (xs < SX);
  const bool st0 = out_x & (j0 >= 1) & (yr0 < SY);
  const bool st1 = out_x & (j1 <= TY) & (yr1 < SY);
  T* const x1 = xy + warp * C * W + lane;   // row 2w+1 for warp w+1
  const T* const pdn = xy + wdn * C * W + lane;
  T* const f0 = fyb + warp * C * W + lane;      // face below row 2w, for warp w-1
  const T* const fu = fyb + wup * C * W + lane;  // face below row 2w+2 (warp w+1)

  // X: stage of plane kz -> U* and its y half-states (A_y, B_y) of rows 2w, 2w+1
  auto xphase = [&](const int kz, P* S_, P* Ay, P* By) {
    const int s = kz % NS;
    mbar_wait(&bar[s], (kz / NS) & 1);
    P U[C], A[C], B[C];
    const T* r0 = stage + s * SM::STAGE + xoff;
    const T* r1 = r0 + C * SM::WB;
#pragma unroll
    for (int c = 0; c < C; ++c) U[c] = P(r0[c * cst], r1[c * cst]);
    dom_min(dm0, dm1, U[0], cell_ab<D, 0>(U, A, B, lx, gm1));
    P Bn[C], Pnx[C];
#pragma unroll
    for (int c = 0; c < C; ++c) Bn[c] = shfl_down1(B[c]);
    face_psi<D, 0>(A, Bn, Pnx, lx, gm1);
#pragma unroll
    for (int c = 0; c < C; ++c) S_[c] = psi_update(U[c], shfl_up1(Pnx[c]), Pnx[c]);
    dom_min(dm0, dm1, S_[0], cell_ab<D, 1>(S_, Ay, By, ly, gm1));
  };
  auto publish = [&](const P* Ay) {
#pragma unroll
    for (int c = 0; c < C; ++c) x1[c * W] = Ay[c].y;
  };
  // A, TMA refill, Y faces, B
  auto yphase = [&](const int kz, const P* Ay, const P* By, P* Py) {
    __syncthreads();  // (A) stage kz consumed, rows 2w+1 of plane kz published
    if (threadIdx.x == 0) {
      fence_proxy_async();
      issue(kz + NS);
    }
    P AL_[C];
#pragma unroll
    for (int c = 0; c < C; ++c) AL_[c] = P(pdn[c * W], Ay[c].x);
    face_psi<D, 1>(AL_, By, Py, ly, gm1);
#pragma unroll
    for (int c = 0; c < C; ++c) f0[c * W] = Py[c].x;
    __syncthreads();  // (B) faces published; every warp is done reading plane kz's rows
  };
  // y-update + z-march of plane kz: output o of plane kz-1 (kz >= 2), predicated stores
  // (M: 0 = first plane of the march, 1 = second, 2 = steady state -- compile-time, so
  // the steady-state block has no branch)
  auto zphase = [&](auto M, const P* S_, const P* Py, const ZPlane<P>& zp, ZPlane<P>& zn, P* o) {
#pragma unroll
    for (int c = 0; c < C; ++c) zn.us[c] = psi_update(S_[c], Py[c], P(Py[c].y, fu[c * W]));
    P Bz[C];
    dom_min(dm0, dm1, zn.us[0], cell_ab<D, 2>(zn.us, zn.az, Bz, lz, gm1));
    constexpr int m = decltype(M)::value;
    if constexpr (m >= 1) {
      face_psi<D, 2>(zp.az, Bz, zn.ph, lz, gm1);
      if constexpr (m >= 2) {
#pragma unroll
        for (int c = 0; c < C; ++c) o[c] = psi_update(zp.us[c], zp.ph[c], zn.ph[c]);
        dst0 += plane;
        dst1 += plane;
#pragma unroll
        for (int c = 0; c < C; ++c) {
          if (st0) dst0[c * cs] = o[c].x;
          if (st1) dst1[c * cs] = o[c].y;
        }
        nn0 = max(nn0, max(naninf(o[0].x), naninf(o[C - 1].x)));
        nn1 = max(nn1, max(naninf(o[0].y), naninf(o[C - 1].y)));
      }
    }
  };
  // ghost images and wavespeed of the stored plane (uniform branches)
  auto tail = [&](auto M, const int kz, const P* o) {
    constexpr int m = decltype(M)::value;
    if constexpr (m < 2) return;
    if (ws) {
      T v0[C], v1[C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        v0[c] = o[c].x;
        v1[c] = o[c].y;
      }
      const T gam = (T)a.cf.gamma;
      if (st0) wmax = fmax(wmax, wavespeed<D>(v0, a.gm1, gam));
      if (st1) wmax = fmax(wmax, wavespeed<D>(v1, a.gm1, gam));
    }
    const int zo = z0 - 2 + kz;
    const bool zf = (zo < pad) | (zo >= SZ - pad);
    if (edge_xy | zf) {
      const bool xface = (xs < pad) | (xs >= SX - pad);
      const bool yf0 = (yr0 < pad) | (yr0 >= SY - pad);
      const bool yf1 = (yr1 < pad) | (yr1 >= SY - pad);
      if (st0 & (xface | yf0 | zf)) {
        T v[C];
#pragma unroll
        for (int c = 0; c < C; ++c) v[c] = o[c].x;
        if (g.img_fast)
          images_single<D>(g, a.out, xs, yr0, zo, v);
        else
          images3_nl<D, L, T>(&a, xs, yr0, zo, v[0], v[1], v[2], v[3], v[4]);
      }
      if (st1 & (xface | yf1 | zf)) {
        T v[C];
#pragma unroll
        for (int c = 0; c < C; ++c) v[c] = o[c].y;
        if (g.img_fast)
          images_single<D>(g, a.out, xs, yr1, zo, v);
        else
          images3_nl<D, L, T>(&a, xs, yr1, zo, v[0], v[1], v[2], v[3], v[4]);
      }
    }
  };
  // one plane with the next plane's x-sweep overlapped: (Sa, Aa, Ba) -> (Sb, Ab, Bb)
  auto full = [&](auto M, const int kz, const P* Sa, const P* Aa, const P* Ba, P* Sb, P* Ab,
                  P* Bb, const ZPlane<P>& zp, ZPlane<P>& zn) {
    P Py[C], o[C];
    yphase(kz, Aa, Ba, Py);
    xphase(kz + 1, Sb, Ab, Bb);
    zphase(M, Sa, Py, zp, zn, o);
    publish(Ab);
    tail(M, kz, o);
  };
  auto last = [&](const int kz, const P* Sa, const P* Aa, const P* Ba, const ZPlane<P>& zp,
                  ZPlane<P>& zn) {
    P Py[C], o[C];
    yphase(kz, Aa, Ba, Py);
    zphase(std::integral_constant<int, 2>(), Sa, Py, zp, zn, o);
    tail(std::integral_constant<int, 2>(), kz, o);
  };
  using M0 = std::integral_constant<int, 0>;
  using M1 = std::integral_constant<int, 1>;
  using M2 = std::integral_constant<int, 2>;

  P SA[C], AA[C], BA[C], SB[C], AB[C], BB[C];
  ZPlane<P> za, zb;
  xphase(0, SA, AA, BA);
  publish(AA);
  full(M0(), 0, SA, AA, BA, SB, AB, BB, za, zb);  // nplanes >= 3
  full(M1(), 1, SB, AB, BB, SA, AA, BA, zb, za);
  int kz = 2;
  for (; kz + 2 < nplanes; kz += 2) {
    full(M2(), kz, SA, AA, BA, SB, AB, BB, za, zb);
    full(M2(), kz + 1, SB, AB, BB, SA, AA, BA, zb, za);
  }
  if (kz + 1 < nplanes) {
    full(M2(), kz, SA, AA, BA, SB, AB, BB, za, zb);
    last(kz + 1, SB, AB, BB, zb, za);
  } else {
    last(kz, SA, AA, BA, za, zb);
  }

  const bool bad = (st0 & ((dm0 <= 0) | (nn0 >= kExpMask<T>))) |
                   (st1 & ((dm1 <= 0) | (nn1 >= kExpMask<T>)));
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(a.flag, 1u);
  if (ws) publish_max(a, wmax);
}

// ------------------------------------------------------------------ host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// L2 sector promotion of the TMA loads (RPL_L2PROMO: 0 none, 1 64B, 2 128B, 3 256B;
// default 2 -- the SoA box rows are only 136-272 bytes long)
static CUtensorMapL2promotion l2_promotion() {
  int v = 2;
  if (const char* e = getenv("RPL_L2PROMO")) v = atoi(e);
  switch (v) {
    case 0: return CU_TENSOR_MAP_L2_PROMOTION_NONE;
    case 1: return CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
    case 3: return CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    default: return CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
  }
}

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// Tile geometry of every 3-D step kernel: 32-slot x-windows (30 outputs), 8 warps
// x 2 adjacent rows = 16-row boxes (14 output rows), z-chunks of a.rows planes.
constexpr int kRows3 = 16;
template <int NW, int MB, int L, typename P, int NS>
static int launch3_rb(const KArgs<typename PairElem<P>::T>& a, const void* tmap,
                      cudaStream_t s) {
  using T = typename PairElem<P>::T;
  constexpr int W = 32, TY = 2 * NW - 2;
  const Geom& g = a.g;
  const int nwin = (int)((g.S[0] + (W - 2) - 1) / (W - 2));
  const int nyb = (int)((g.S[1] + TY - 1) / TY);
  const int nzc = (int)((g.S[2] + a.rows - 1) / a.rows);
  const int grid = a.tiles ? a.ntiles : nwin * nyb * nzc;
  if (grid <= 0) return 0;
  const size_t sm = SmemRB<NW, T, NS>::bytes();
  if constexpr (sizeof(T) == 4) pk_set_negzero(s);
  static int cache[kMaxDevices] = {0};
  resident_ctas(k_step3d_rb<NW, MB, L, P, NS>, 32 * NW, sm, cache);
  k_step3d_rb<NW, MB, L, P, NS><<<grid, 32 * NW, sm, s>>>(
      a, *reinterpret_cast<const CUtensorMap*>(tmap), nwin, nyb);
  return 0;
}

template <int NW, int MB, int L, typename P, int NS>
static int launch3_sp(const KArgs<typename PairElem<P>::T>& a, const void* tmap,
                      cudaStream_t s) {
  using T = typename PairElem<P>::T;
  constexpr int W = 32, TY = 2 * NW - 2;
  const Geom& g = a.g;
  const int nwin = (int)((g.S[0] + (W - 2) - 1) / (W - 2));
  const int nyb = (int)((g.S[1] + TY - 1) / TY);
  const int nzc = (int)((g.S[2] + a.rows - 1) / a.rows);
  const int grid = a.tiles ? a.ntiles : nwin * nyb * nzc;
  if (grid <= 0) return 0;
  const size_t sm = SmemRB<NW, T, NS>::bytes();
  if constexpr (sizeof(T) == 4) pk_set_negzero(s);
  static int cache[kMaxDevices] = {0};
  resident_ctas(k_step3d_sp<NW, MB, L, P, NS>, 32 * NW, sm, cache);
  k_step3d_sp<NW, MB, L, P, NS><<<grid, 32 * NW, sm, s>>>(
      a, *reinterpret_cast<const CUtensorMap*>(tmap), nwin, nyb);
  return 0;
}

int make_tmap(const Geom& g, const void* buf, void* map_out, int box_w, int box_rows) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return -1;
  const cuuint64_t dims[4] = {(cuuint64_t)g.pitch, (cuuint64_t)g.C, (cuuint64_t)g.P[1],
                              (cuuint64_t)g.P[2]};
  const cuuint64_t strides[3] = {(cuuint64_t)(g.pitch * g.elem), (cuuint64_t)(g.rstride * g.elem),
                                 (cuuint64_t)(g.rstride * g.P[1] * g.elem)};
  const cuuint32_t box[4] = {(cuuint32_t)box_w, (cuuint32_t)g.C, (cuuint32_t)box_rows, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(reinterpret_cast<CUtensorMap*>(map_out),
                   g.elem == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                   4, const_cast<void*>(buf), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   l2_promotion(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -2;
}


// Default (variant 0; round 2, profiles/r2/): fp64 k_step3d_sp (software-pipelined
// planes, 8 warps, 1 CTA/SM, 246 registers, 3-stage ring): 512^3 4.34 -> 3.90 ms vs the
// round-1 row-pair kernel; fp32 k_step3d_rb (8 warps, 2 CTAs/SM, 120 registers,
// 3-stage ring): 384^3 1.06 -> 0.99 ms.  Variant 1 swaps the two forms (fp64 rb:
// 4.43 ms; fp32 sp needs 186 registers, 1 CTA/SM: 1.25 ms) -- kept as the measured
// alternative; the split kernel (RPL_KERNEL_SPLIT) is the fallback.
template <typename T>
int launch_step3d(const KArgs<T>& a, const void* tmap, cudaStream_t s) {
  const bool aos = a.g.layout == 1;
  if constexpr (sizeof(T) == 8) {
    if (a.variant == 1)
      return aos ? launch3_rb<8, 1, 1, pd, 3>(a, tmap, s) : launch3_rb<8, 1, 0, pd, 3>(a, tmap, s);
    return aos ? launch3_sp<8, 1, 1, pd, 3>(a, tmap, s) : launch3_sp<8, 1, 0, pd, 3>(a, tmap, s);
  } else {
    if (a.variant == 1)
      return aos ? launch3_sp<8, 1, 1, pk, 3>(a, tmap, s) : launch3_sp<8, 1, 0, pk, 3>(a, tmap, s);
    return aos ? launch3_rb<8, 2, 1, pk, 3>(a, tmap, s) : launch3_rb<8, 2, 0, pk, 3>(a, tmap, s);
  }
}

const char* step3d_kernel_name(int elem, int variant) {
  if (elem == 8) return variant == 1 ? "k_step3d_rb<pd>" : "k_step3d_sp<pd>";
  return variant == 1 ? "k_step3d_sp<pk>" : "k_step3d_rb<pk>";
}

// AoS: the (x, component) pair is one contiguous dimension of pitch*C elements
int make_tmap_aos(const Geom& g, const void* buf, void* map_out, int box_cells, int box_rows) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return -1;
  const cuuint64_t dims[4] = {(cuuint64_t)(g.pitch * g.C), 1, (cuuint64_t)g.P[1],
                              (cuuint64_t)g.P[2]};
  const cuuint64_t strides[3] = {(cuuint64_t)(g.rstride * g.elem), (cuuint64_t)(g.rstride * g.elem),
                                 (cuuint64_t)(g.rstride * g.P[1] * g.elem)};
  const cuuint32_t box[4] = {(cuuint32_t)(box_cells * g.C), 1, (cuuint32_t)box_rows, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(reinterpret_cast<CUtensorMap*>(map_out),
                   g.elem == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                   4, const_cast<void*>(buf), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   l2_promotion(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -2;
}

int make_tmap3d(const Geom& g, const void* buf, void* map_out, int variant) {
  (void)variant;
  if (g.layout == 1) return make_tmap_aos(g, buf, map_out, 32 + 16 / g.elem, kRows3);
  return make_tmap(g, buf, map_out, 32 + 16 / g.elem, kRows3);  // + SmemRB::AL
}
template int launch_step3d<float>(const KArgs<float>&, const void*, cudaStream_t);
template int launch_step3d<double>(const KArgs<double>&, const void*, cudaStream_t);

}  // namespace rpl
