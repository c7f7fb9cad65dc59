// kernels3d.cu -- K-B (3-D): the x-, y- and z-sweeps of one step fused into one
// HBM pass, TMA-staged.
//
// CTA tile: one x-window of W = 32V slots (lane l owns slots V l .. V l+V-1;
// slot s <-> x = (W-2) w - 1 + s, slots 0 and W-1 are the x-halo), TY output rows
// in y, and a chunk of z-planes that the CTA marches through (2.5-D streaming).
// Warp j (0 <= j < TY+2) owns tile row y = y0 - 1 + j; warps 0 and TY+1 are the
// y-halo rows.  Per z-plane:
//   TMA   one elected thread streams whole plane tiles [TY+2 rows][C comps][W]
//         into a 2-stage shared-memory ring (cp.async.bulk.tensor.4d, mbarrier
//         completion), two planes ahead of the compute;
//   X     every warp x-sweeps its row in registers (warp shuffles share faces),
//         evaluates F_y of the result and publishes (U*, F_y) in shared memory;
//   Y     warp j >= 1 computes the y-face between rows j-1 and j once and
//         publishes it; warps 1..TY then update U** = U* - (Phi_{j+1/2} - Phi_{j-1/2});
//   Z     warps 1..TY keep a z-march state per cell in registers (U** of the
//         previous plane, its F_z and the previous z-face), compute the z-face,
//         update and store plane z-1 (+ ghost images on partition faces).
// Two __syncthreads per plane order the shared-memory hand-offs.  HBM traffic per
// cell-step is one read of U^n (plus the tile halo, mostly L2 hits) and one write
// of U^{n+1}; the halo rows/planes are recomputed, not re-stored.
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

template <typename T, int V>
struct ZState {
  T us[V][5];  // U** of the previous plane
  T fz[V][5];  // F_z(U**) of the previous plane
  T ph[V][5];  // previous z-face
};

template <int TY, int V, typename T>
struct Smem3 {
  static constexpr int W = 32 * V, R = TY + 2, C = 5, NS = 2;
  // TMA boxes start 16-byte aligned in x: AL extra elements, read at `shift`
  static constexpr int AL = 16 / (int)sizeof(T);
  static constexpr int WB = W + AL;
  static constexpr int STAGE = R * C * WB;          // elements per ring stage
  static constexpr int XY = R * 2 * C * W;          // (U*, F_y) per tile row
  static constexpr int FY = (R - 1) * C * W;        // y-faces
  static constexpr size_t bytes() { return (size_t)(NS * STAGE + XY + FY) * sizeof(T) + 64; }
};

template <typename T, int V, int TY, int MB, int L>
__global__ void __launch_bounds__(32 * (TY + 2), MB)
    k_step3d(const __grid_constant__ KArgs<T> a, const __grid_constant__ CUtensorMap tmap,
             int nwin, int nyb) {
  constexpr int D = 3, C = 5, W = 32 * V;
  using SM = Smem3<TY, V, T>;
  extern __shared__ __align__(1024) unsigned char smem[];
  T* stage = reinterpret_cast<T*>(smem);
  T* xy = stage + SM::NS * SM::STAGE;
  T* fyb = xy + SM::XY;
  uint64_t* bar = reinterpret_cast<uint64_t*>(fyb + SM::FY);
  const Geom& g = a.g;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int t = blockIdx.x;
  const int win = t % nwin;
  t /= nwin;
  const int yb = t % nyb;
  const int zc = t / nyb;
  const int xw = win * (W - 2) - 1;                 // x of slot 0
  const int y0 = yb * TY;
  const int z0 = zc * a.rows;
  const int z1 = min(z0 + a.rows, (int)g.S[2]);
  const int yr = y0 - 1 + warp;                     // this warp's row
  const int SX = (int)g.S[0], SY = (int)g.S[1], SZ = (int)g.S[2];
  // per-lane slot validity
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
  const bool row_in = yr <= SY;                      // row holds valid (interior/ghost) data
  const bool row_out = (warp >= 1) & (warp <= TY) & (yr < SY);
  const bool yface = (yr < g.pad) | (yr >= SY - g.pad);
  const T gm1 = a.gm1;
  Coef<T> kc;
  if (!step_coef(a, kc)) return;
  const bool ws = a.cf.dev != nullptr;
  const T gam = (T)a.cf.gamma;
  T wmax = T(0);

  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < SM::NS; ++s) mbar_init(&bar[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  const int sh = (int)(g.xo + xw) % SM::AL;
  const int tx = (int)(g.xo + xw) - sh, ty = (int)(g.off[1] + y0 - 1);
  const int nplanes = z1 - (z0 - 1) + 1;  // planes z0-1 .. z1
  auto issue = [&](int kz) {
    if (kz >= nplanes) return;
    const int s = kz % SM::NS;
    mbar_arrive_expect_tx(&bar[s], SM::STAGE * (unsigned)sizeof(T));
    tma_load_4d(stage + s * SM::STAGE, &tmap, &bar[s], L == 0 ? tx : tx * C, 0, ty,
                (int)(g.off[2] + z0 - 1 + kz));
  };
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < SM::NS; ++s) issue(s);
  }

  ZState<T, V> zs;
  int bad = 0, nan = 0;
  const T qx = kc.q[0], nqx = kc.nq2[0], qy = kc.q[1], nqy = kc.nq2[1], qz = kc.q[2], nqz = kc.nq2[2];
  const int64_t plane = g.rstride * g.P[1], cs = g.cstride, xst = g.xstride;
  // this lane's first output of plane z0 - 1 (advanced by one plane per store)
  T* dst = a.out + g.row(yr, z0 - 1) * g.rstride + (g.xo + xw + V * lane) * xst;

  for (int kz = 0; kz < nplanes; ++kz) {
    const int z = z0 - 1 + kz;
    const int s = kz % SM::NS;
    mbar_wait(&bar[s], (kz / SM::NS) & 1);
    // ---------------- X: this warp's row
    T U[V][C], F[V][C], S_[V][C], G[V][C];
    // stage row layout: SoA box [C][WB] (x fastest), AoS box [WB][C] (component fastest)
    const T* st = stage + s * SM::STAGE + warp * C * SM::WB +
                  (L == 0 ? sh + V * lane : (sh + V * lane) * C);
#pragma unroll
    for (int c = 0; c < C; ++c)
#pragma unroll
      for (int v = 0; v < V; ++v) U[v][c] = L == 0 ? st[c * SM::WB + v] : st[v * C + c];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int b = phys_flux<D, 0>(U[v], F[v], gm1);
      bad |= (in_ok[v] & row_in) ? b : 0;
    }
    {
      // faces: inside the lane (V == 2) and towards the next lane
      T Pin[C], Pnx[C], Un[C], Fn[C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        Un[c] = __shfl_down_sync(0xffffffffu, U[0][c], 1);
        Fn[c] = __shfl_down_sync(0xffffffffu, F[0][c], 1);
      }
      force_face<D, 0>(U[V - 1], F[V - 1], Un, Fn, Pnx, qx, nqx, gm1);
      if (V == 2) force_face<D, 0>(U[0], F[0], U[V - 1], F[V - 1], Pin, qx, nqx, gm1);
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const T Ppv = __shfl_up_sync(0xffffffffu, Pnx[c], 1);
        if (V == 2) {
          S_[0][c] = U[0][c] - (Pin[c] - Ppv);
          S_[V - 1][c] = U[V - 1][c] - (Pnx[c] - Pin[c]);
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
    T* xr = xy + warp * 2 * C * W + V * lane;
#pragma unroll
    for (int c = 0; c < C; ++c)
#pragma unroll
      for (int v = 0; v < V; ++v) {
        xr[c * W + v] = S_[v][c];
        xr[(C + c) * W + v] = G[v][c];
      }
    __syncthreads();  // (A): stage s consumed, (U*, F_y) published
    if (threadIdx.x == 0) {
      fence_proxy_async();
      issue(kz + SM::NS);
    }
    // ---------------- Y: face between rows warp-1 and warp
    T Py[V][C];
    if (warp >= 1) {
      const T* pr = xy + (warp - 1) * 2 * C * W + V * lane;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        T Sp[C], Gp[C];
#pragma unroll
        for (int c = 0; c < C; ++c) {
          Sp[c] = pr[c * W + v];
          Gp[c] = pr[(C + c) * W + v];
        }
        force_face<D, 1>(Sp, Gp, S_[v], G[v], Py[v], qy, nqy, gm1);
      }
      T* fw = fyb + (warp - 1) * C * W + V * lane;
#pragma unroll
      for (int c = 0; c < C; ++c)
#pragma unroll
        for (int v = 0; v < V; ++v) fw[c * W + v] = Py[v][c];
    }
    __syncthreads();  // (B): y-faces published
    // ---------------- Y update + Z march (rows 1..TY)
    if (warp >= 1 && warp <= TY) {
      const T* fu = fyb + warp * C * W + V * lane;  // face between warp and warp+1
      T Us[V][C], Gz[V][C];
#pragma unroll
      for (int v = 0; v < V; ++v) {
#pragma unroll
        for (int c = 0; c < C; ++c) Us[v][c] = S_[v][c] - (fu[c * W + v] - Py[v][c]);
        const int b = phys_flux<D, 2>(Us[v], Gz[v], gm1);
        bad |= (out_ok[v] & row_out) ? b : 0;
      }
      if (kz >= 1) {
        T Pz[V][C];
#pragma unroll
        for (int v = 0; v < V; ++v)
          force_face<D, 2>(zs.us[v], zs.fz[v], Us[v], Gz[v], Pz[v], qz, nqz, gm1);
        if (kz >= 2) {
          // update and store plane z-1
          T o[V][C];
#pragma unroll
          for (int v = 0; v < V; ++v)
#pragma unroll
            for (int c = 0; c < C; ++c) o[v][c] = zs.us[v][c] - (Pz[v][c] - zs.ph[v][c]);
          dst += plane;  // plane z - 1
#pragma unroll
          for (int v = 0; v < V; ++v) {
            if (out_ok[v] & row_out) {
              nan = max(nan, max(naninf(o[v][0]), naninf(o[v][C - 1])));
              if (ws) wmax = fmax(wmax, wavespeed<D>(o[v], gm1, gam));
              T* p = dst + v * xst;
#pragma unroll
              for (int c = 0; c < C; ++c) {
                *p = o[v][c];
                p += cs;
              }
              const bool zf = (z - 1 < g.pad) | (z - 1 >= SZ - g.pad);
              if (xface[v] | yface | zf) {
                if (g.img_fast)
                  images_single<D>(g, a.out, xs[v], yr, z - 1, o[v]);
                else
                  images3_nl<D, L, T>(&a, xs[v], yr, z - 1, o[v][0], o[v][1], o[v][2], o[v][3],
                                      o[v][4]);
              }
            }
          }
        }
#pragma unroll
        for (int v = 0; v < V; ++v)
#pragma unroll
          for (int c = 0; c < C; ++c) zs.ph[v][c] = Pz[v][c];
      }
#pragma unroll
      for (int v = 0; v < V; ++v)
#pragma unroll
        for (int c = 0; c < C; ++c) {
          zs.us[v][c] = Us[v][c];
          zs.fz[v][c] = Gz[v][c];
        }
    }
  }
  if (__any_sync(0xffffffffu, bad < 0 || nan >= kExpMask<T>) && lane == 0) atomicOr(a.flag, 1u);
  if (ws) publish_max(a, wmax);
}


// ------------------------------------------------------------------------
// fp32, SoA: the same fused x-y-z pass with two tile rows per lane, packed
// (packed.cuh: FFMA2/FADD2 do both rows' arithmetic in one instruction).
// Warp w owns tile rows j0 = w and j1 = w + NW (R = 2 NW rows, TY = R - 2
// outputs, rows 0 and R-1 are the y-halo).  Every per-cell operation is the
// scalar kernel's, so the result is bitwise that of k_step3d / k_sweep.
// ------------------------------------------------------------------------
template <int NW>
struct SmemRP {
  static constexpr int W = 32, R = 2 * NW, C = 5, NS = 2;
  static constexpr int AL = 4;                      // 16-byte TMA alignment in floats
  static constexpr int WB = W + AL;
  static constexpr int STAGE = R * C * WB;          // floats per ring stage
  static constexpr int XY = R * 2 * C * W;          // (U*, F_y) per tile row
  static constexpr int FY = (R - 1) * C * W;        // y-faces
  static constexpr size_t bytes() { return (size_t)(NS * STAGE + XY + FY) * 4 + 64; }
};

template <int NW, int MB, int L>
__global__ void __launch_bounds__(32 * NW, MB)
    k_step3d_rp(const __grid_constant__ KArgs<float> a, const __grid_constant__ CUtensorMap tmap,
                int nwin, int nyb) {
  constexpr int D = 3, C = 5, W = 32, R = 2 * NW, TY = R - 2;
  using SM = SmemRP<NW>;
  extern __shared__ __align__(1024) unsigned char smem[];
  float* stage = reinterpret_cast<float*>(smem);
  float* xy = stage + SM::NS * SM::STAGE;
  float* fyb = xy + SM::XY;
  uint64_t* bar = reinterpret_cast<uint64_t*>(fyb + SM::FY);
  const Geom& g = a.g;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int t = blockIdx.x;
  const int win = t % nwin;
  t /= nwin;
  const int yb = t % nyb;
  const int zc = t / nyb;
  const int xw = win * (W - 2) - 1;  // x of slot 0
  const int y0 = yb * TY;
  const int z0 = zc * a.rows;
  const int z1 = min(z0 + a.rows, (int)g.S[2]);
  const int SX = (int)g.S[0], SY = (int)g.S[1], SZ = (int)g.S[2];
  const int j0 = warp, j1 = warp + NW;           // tile rows of the two halves
  const int yr0 = y0 - 1 + j0, yr1 = y0 - 1 + j1;
  const int xs = xw + lane;
  const bool out_x = (lane >= 1) & (lane <= W - 2) & (xs < SX);
  const bool in_x = (xs >= -1) & (xs <= SX);
  const bool xface = (xs < g.pad) | (xs >= SX - g.pad);
  const bool in0 = in_x & (yr0 <= SY), in1 = in_x & (yr1 <= SY);
  const bool ok0 = out_x & (yr0 <= SY), ok1 = out_x & (yr1 <= SY);
  const bool st0 = out_x & (j0 >= 1) & (yr0 < SY);                // stores: rows 1..TY
  const bool st1 = out_x & (j1 <= TY) & (yr1 < SY);
  const bool yface0 = (yr0 < g.pad) | (yr0 >= SY - g.pad);
  const bool yface1 = (yr1 < g.pad) | (yr1 >= SY - g.pad);
  Coef<float> kc;
  if (!step_coef(a, kc)) return;
  const bool ws = a.cf.dev != nullptr;
  const float gam = (float)a.cf.gamma;
  float wmax = 0.0f;

  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < SM::NS; ++s) mbar_init(&bar[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  const int sh = (int)(g.xo + xw) % SM::AL;
  const int tx = (int)(g.xo + xw) - sh, ty = (int)(g.off[1] + y0 - 1);
  const int nplanes = z1 - (z0 - 1) + 1;  // planes z0-1 .. z1
  auto issue = [&](int kz) {
    if (kz >= nplanes) return;
    const int s = kz % SM::NS;
    mbar_arrive_expect_tx(&bar[s], SM::STAGE * 4u);
    tma_load_4d(stage + s * SM::STAGE, &tmap, &bar[s], L == 0 ? tx : tx * C, 0, ty,
                (int)(g.off[2] + z0 - 1 + kz));
  };
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < SM::NS; ++s) issue(s);
  }

  pk zus[C], zfz[C], zph[C];  // z-march state: U** and F_z of the previous plane, last z-face
  int bad = 0, nan = 0;
  const pk gm1(a.gm1);
  const pk qx(kc.q[0]), nqx(kc.nq2[0]), qy(kc.q[1]), nqy(kc.nq2[1]), qz(kc.q[2]), nqz(kc.nq2[2]);
  const int64_t plane = g.rstride * g.P[1], cs = g.cstride;
  float* dst0 = a.out + g.row(yr0, z0 - 1) * g.rstride + (g.xo + xs) * g.xstride;
  float* dst1 = a.out + g.row(yr1, z0 - 1) * g.rstride + (g.xo + xs) * g.xstride;
  // y-face rows: below row j (face j-1 | j) and above (face j | j+1), clamped into range
  const int fb0 = max(j0 - 1, 0), fa1 = min(j1, R - 2);

  for (int kz = 0; kz < nplanes; ++kz) {
    const int z = z0 - 1 + kz;
    const int s = kz % SM::NS;
    mbar_wait(&bar[s], (kz / SM::NS) & 1);
    // ---------------- X: rows j0 and j1
    pk U[C], F[C], S_[C], G[C];
    {
      // stage row layout: SoA box [C][WB] (x fastest), AoS box [WB][C] (component fastest)
      constexpr int cst = L == 0 ? SM::WB : 1;
      const int xo = L == 0 ? sh + lane : (sh + lane) * C;
      const float* r0 = stage + s * SM::STAGE + j0 * C * SM::WB + xo;
      const float* r1 = stage + s * SM::STAGE + j1 * C * SM::WB + xo;
#pragma unroll
      for (int c = 0; c < C; ++c) U[c] = pk(r0[c * cst], r1[c * cst]);
    }
    {
      const PkDom b = phys_flux<D, 0>(U, F, gm1);
      bad |= (in0 ? b.a : 0) | (in1 ? b.b : 0);
    }
    {
      pk Un[C], Fn[C], Pnx[C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        Un[c] = shfl_down1(U[c]);
        Fn[c] = shfl_down1(F[c]);
      }
      force_face<D, 0>(U, F, Un, Fn, Pnx, qx, nqx, gm1);
#pragma unroll
      for (int c = 0; c < C; ++c) S_[c] = U[c] - (Pnx[c] - shfl_up1(Pnx[c]));
    }
    {
      const PkDom b = phys_flux<D, 1>(S_, G, gm1);
      bad |= (ok0 ? b.a : 0) | (ok1 ? b.b : 0);
    }
    {
      float* x0 = xy + j0 * 2 * C * W + lane;
      float* x1 = xy + j1 * 2 * C * W + lane;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        x0[c * W] = S_[c].x;
        x0[(C + c) * W] = G[c].x;
        x1[c * W] = S_[c].y;
        x1[(C + c) * W] = G[c].y;
      }
    }
    __syncthreads();  // (A): stage s consumed, (U*, F_y) published
    if (threadIdx.x == 0) {
      fence_proxy_async();
      issue(kz + SM::NS);
    }
    // ---------------- Y: faces (j0-1 | j0) and (j1-1 | j1)
    pk Py[C];
    {
      const float* p0 = xy + fb0 * 2 * C * W + lane;
      const float* p1 = xy + (j1 - 1) * 2 * C * W + lane;
      pk Sp[C], Gp[C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        Sp[c] = pk(p0[c * W], p1[c * W]);
        Gp[c] = pk(p0[(C + c) * W], p1[(C + c) * W]);
      }
      force_face<D, 1>(Sp, Gp, S_, G, Py, qy, nqy, gm1);
      float* f0 = fyb + fb0 * C * W + lane;
      float* f1 = fyb + (j1 - 1) * C * W + lane;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        if (j0 >= 1) f0[c * W] = Py[c].x;
        f1[c * W] = Py[c].y;
      }
    }
    __syncthreads();  // (B): y-faces published
    // ---------------- Y update + Z march (row halves with outputs)
    {
      const float* u0 = fyb + j0 * C * W + lane;   // face (j0 | j0+1); j0 <= R-2 always
      const float* u1 = fyb + fa1 * C * W + lane;  // face (j1 | j1+1)
      pk Us[C], Gz[C];
#pragma unroll
      for (int c = 0; c < C; ++c) Us[c] = S_[c] - (pk(u0[c * W], u1[c * W]) - Py[c]);
      {
        const PkDom b = phys_flux<D, 2>(Us, Gz, gm1);
        bad |= (st0 ? b.a : 0) | (st1 ? b.b : 0);
      }
      if (kz >= 1) {
        pk Pz[C];
        force_face<D, 2>(zus, zfz, Us, Gz, Pz, qz, nqz, gm1);
        if (kz >= 2) {
          // update and store plane z-1
          pk o[C];
#pragma unroll
          for (int c = 0; c < C; ++c) o[c] = zus[c] - (Pz[c] - zph[c]);
          dst0 += plane;
          dst1 += plane;
          const bool zf = (z - 1 < g.pad) | (z - 1 >= SZ - g.pad);
          if (st0) {
            float v[C];
#pragma unroll
            for (int c = 0; c < C; ++c) v[c] = o[c].x;
            nan = max(nan, max(naninf(v[0]), naninf(v[C - 1])));
            if (ws) wmax = fmaxf(wmax, wavespeed<D>(v, a.gm1, gam));
#pragma unroll
            for (int c = 0; c < C; ++c) dst0[c * cs] = v[c];
            if (xface | yface0 | zf) {
              if (g.img_fast)
                images_single<D>(g, a.out, xs, yr0, z - 1, v);
              else
                images3_nl<D, L, float>(&a, xs, yr0, z - 1, v[0], v[1], v[2], v[3], v[4]);
            }
          }
          if (st1) {
            float v[C];
#pragma unroll
            for (int c = 0; c < C; ++c) v[c] = o[c].y;
            nan = max(nan, max(naninf(v[0]), naninf(v[C - 1])));
            if (ws) wmax = fmaxf(wmax, wavespeed<D>(v, a.gm1, gam));
#pragma unroll
            for (int c = 0; c < C; ++c) dst1[c * cs] = v[c];
            if (xface | yface1 | zf) {
              if (g.img_fast)
                images_single<D>(g, a.out, xs, yr1, z - 1, v);
              else
                images3_nl<D, L, float>(&a, xs, yr1, z - 1, v[0], v[1], v[2], v[3], v[4]);
            }
          }
        }
#pragma unroll
        for (int c = 0; c < C; ++c) zph[c] = Pz[c];
      }
#pragma unroll
      for (int c = 0; c < C; ++c) {
        zus[c] = Us[c];
        zfz[c] = Gz[c];
      }
    }
  }
  if (__any_sync(0xffffffffu, bad < 0 || nan >= kExpMask<float>) && lane == 0) atomicOr(a.flag, 1u);
  if (ws) publish_max(a, wmax);
}


// ------------------------------------------------------------------------
// fp32, adjacent row pairs (the fp32 default): warp w owns tile rows 2w and 2w+1, so the
// y-face between them is computed in registers, packed with the face below row
// 2w (one force_face for both); only row 2w+1's (U*, F_y) and the face below row
// 2w go through shared memory (half the hand-off traffic of k_step3d_rp).  Same
// per-cell and per-face operations: bitwise equal to k_step3d / k_sweep.
// ------------------------------------------------------------------------
template <int NW, typename T = float>
struct SmemRA {
  static constexpr int W = 32, R = 2 * NW, C = 5, NS = 2;
  static constexpr int AL = 16 / (int)sizeof(T);
  static constexpr int WB = W + AL;
  static constexpr int STAGE = R * C * WB;
  static constexpr int XY = NW * 2 * C * W;  // (U*, F_y) of row 2w+1, per warp
  static constexpr int FY = NW * C * W;      // face below row 2w, per warp
  static constexpr size_t bytes() { return (size_t)(NS * STAGE + XY + FY) * sizeof(T) + 64; }
};

// P = pk (fp32, packed FFMA2) or pd (fp64, a plain pair of scalar lanes)
template <int NW, int MB, int L, typename P = pk>
__global__ void __launch_bounds__(32 * NW, MB)
    k_step3d_ra(const __grid_constant__ KArgs<typename PairElem<P>::T> a,
                const __grid_constant__ CUtensorMap tmap, int nwin, int nyb) {
  using T = typename PairElem<P>::T;
  constexpr int D = 3, C = 5, W = 32, R = 2 * NW, TY = R - 2;
  using SM = SmemRA<NW, T>;
  extern __shared__ __align__(1024) unsigned char smem[];
  T* stage = reinterpret_cast<T*>(smem);
  T* xy = stage + SM::NS * SM::STAGE;
  T* fyb = xy + SM::XY;
  uint64_t* bar = reinterpret_cast<uint64_t*>(fyb + SM::FY);
  const Geom& g = a.g;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int t = blockIdx.x;
  const int win = t % nwin;
  t /= nwin;
  const int yb = t % nyb;
  const int zc = t / nyb;
  const int xw = win * (W - 2) - 1;
  const int y0 = yb * TY;
  const int z0 = zc * a.rows;
  const int z1 = min(z0 + a.rows, (int)g.S[2]);
  const int SX = (int)g.S[0], SY = (int)g.S[1], SZ = (int)g.S[2];
  const int j0 = 2 * warp, j1 = 2 * warp + 1;
  const int yr0 = y0 - 1 + j0, yr1 = y0 - 1 + j1;
  const int xs = xw + lane;
  const bool out_x = (lane >= 1) & (lane <= W - 2) & (xs < SX);
  const bool in_x = (xs >= -1) & (xs <= SX);
  const bool xface = (xs < g.pad) | (xs >= SX - g.pad);
  const bool in0 = in_x & (yr0 <= SY), in1 = in_x & (yr1 <= SY);
  const bool ok0 = out_x & (yr0 <= SY), ok1 = out_x & (yr1 <= SY);
  const bool st0 = out_x & (j0 >= 1) & (yr0 < SY);
  const bool st1 = out_x & (j1 <= TY) & (yr1 < SY);
  const bool yface0 = (yr0 < g.pad) | (yr0 >= SY - g.pad);
  const bool yface1 = (yr1 < g.pad) | (yr1 >= SY - g.pad);
  Coef<T> kc;
  if (!step_coef(a, kc)) return;
  const bool ws = a.cf.dev != nullptr;
  const T gam = (T)a.cf.gamma;
  T wmax = T(0);

  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < SM::NS; ++s) mbar_init(&bar[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  const int sh = (int)(g.xo + xw) % SM::AL;
  const int tx = (int)(g.xo + xw) - sh, ty = (int)(g.off[1] + y0 - 1);
  const int nplanes = z1 - (z0 - 1) + 1;
  auto issue = [&](int kz) {
    if (kz >= nplanes) return;
    const int s = kz % SM::NS;
    mbar_arrive_expect_tx(&bar[s], SM::STAGE * (unsigned)sizeof(T));
    tma_load_4d(stage + s * SM::STAGE, &tmap, &bar[s], L == 0 ? tx : tx * C, 0, ty,
                (int)(g.off[2] + z0 - 1 + kz));
  };
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < SM::NS; ++s) issue(s);
  }

  P zus[C], zfz[C], zph[C];
  int bad = 0, nan = 0;
  const P gm1(a.gm1);
  const P qx(kc.q[0]), nqx(kc.nq2[0]), qy(kc.q[1]), nqy(kc.nq2[1]), qz(kc.q[2]), nqz(kc.nq2[2]);
  const int64_t plane = g.rstride * g.P[1], cs = g.cstride;
  T* dst0 = a.out + g.row(yr0, z0 - 1) * g.rstride + (g.xo + xs) * g.xstride;
  T* dst1 = a.out + g.row(yr1, z0 - 1) * g.rstride + (g.xo + xs) * g.xstride;
  // row 2w-1 lives in warp w-1's slot (warp 0: its own slot, value unused)
  const int wdn = max(warp - 1, 0), wup = min(warp + 1, NW - 1);

  for (int kz = 0; kz < nplanes; ++kz) {
    const int z = z0 - 1 + kz;
    const int s = kz % SM::NS;
    mbar_wait(&bar[s], (kz / SM::NS) & 1);
    P U[C], F[C], S_[C], G[C];
    {
      constexpr int cst = L == 0 ? SM::WB : 1;
      const int xo = L == 0 ? sh + lane : (sh + lane) * C;
      const T* r0 = stage + s * SM::STAGE + j0 * C * SM::WB + xo;
      const T* r1 = stage + s * SM::STAGE + j1 * C * SM::WB + xo;
#pragma unroll
      for (int c = 0; c < C; ++c) U[c] = P(r0[c * cst], r1[c * cst]);
    }
    {
      const PkDom b = phys_flux<D, 0>(U, F, gm1);
      bad |= (in0 ? b.a : 0) | (in1 ? b.b : 0);
    }
    {
      P Un[C], Fn[C], Pnx[C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        Un[c] = shfl_down1(U[c]);
        Fn[c] = shfl_down1(F[c]);
      }
      force_face<D, 0>(U, F, Un, Fn, Pnx, qx, nqx, gm1);
#pragma unroll
      for (int c = 0; c < C; ++c) S_[c] = U[c] - (Pnx[c] - shfl_up1(Pnx[c]));
    }
    {
      const PkDom b = phys_flux<D, 1>(S_, G, gm1);
      bad |= (ok0 ? b.a : 0) | (ok1 ? b.b : 0);
    }
    {
      T* x1 = xy + warp * 2 * C * W + lane;  // row 2w+1 for warp w+1
#pragma unroll
      for (int c = 0; c < C; ++c) {
        x1[c * W] = S_[c].y;
        x1[(C + c) * W] = G[c].y;
      }
    }
    __syncthreads();  // (A)
    if (threadIdx.x == 0) {
      fence_proxy_async();
      issue(kz + SM::NS);
    }
    // ---------------- Y: faces (2w-1 | 2w) and (2w | 2w+1) in one packed evaluation
    P Py[C];
    {
      const T* pdn = xy + wdn * 2 * C * W + lane;
      P SL[C], GL[C], SR[C], GR[C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        SL[c] = P(pdn[c * W], S_[c].x);
        GL[c] = P(pdn[(C + c) * W], G[c].x);
        SR[c] = P(S_[c].x, S_[c].y);
        GR[c] = P(G[c].x, G[c].y);
      }
      force_face<D, 1>(SL, GL, SR, GR, Py, qy, nqy, gm1);
      T* f0 = fyb + warp * C * W + lane;  // face below row 2w, for warp w-1
#pragma unroll
      for (int c = 0; c < C; ++c) f0[c * W] = Py[c].x;
    }
    __syncthreads();  // (B)
    {
      const T* fu = fyb + wup * C * W + lane;  // face below row 2w+2 (warp w+1)
      P Us[C], Gz[C];
#pragma unroll
      for (int c = 0; c < C; ++c)
        Us[c] = S_[c] - (P(Py[c].y, fu[c * W]) - P(Py[c].x, Py[c].y));
      {
        const PkDom b = phys_flux<D, 2>(Us, Gz, gm1);
        bad |= (st0 ? b.a : 0) | (st1 ? b.b : 0);
      }
      if (kz >= 1) {
        P Pz[C];
        force_face<D, 2>(zus, zfz, Us, Gz, Pz, qz, nqz, gm1);
        if (kz >= 2) {
          P o[C];
#pragma unroll
          for (int c = 0; c < C; ++c) o[c] = zus[c] - (Pz[c] - zph[c]);
          dst0 += plane;
          dst1 += plane;
          const bool zf = (z - 1 < g.pad) | (z - 1 >= SZ - g.pad);
          if (st0) {
            T v[C];
#pragma unroll
            for (int c = 0; c < C; ++c) v[c] = o[c].x;
            nan = max(nan, max(naninf(v[0]), naninf(v[C - 1])));
            if (ws) wmax = fmax(wmax, wavespeed<D>(v, a.gm1, gam));
#pragma unroll
            for (int c = 0; c < C; ++c) dst0[c * cs] = v[c];
            if (xface | yface0 | zf) {
              if (g.img_fast)
                images_single<D>(g, a.out, xs, yr0, z - 1, v);
              else
                images3_nl<D, L, T>(&a, xs, yr0, z - 1, v[0], v[1], v[2], v[3], v[4]);
            }
          }
          if (st1) {
            T v[C];
#pragma unroll
            for (int c = 0; c < C; ++c) v[c] = o[c].y;
            nan = max(nan, max(naninf(v[0]), naninf(v[C - 1])));
            if (ws) wmax = fmax(wmax, wavespeed<D>(v, a.gm1, gam));
#pragma unroll
            for (int c = 0; c < C; ++c) dst1[c * cs] = v[c];
            if (xface | yface1 | zf) {
              if (g.img_fast)
                images_single<D>(g, a.out, xs, yr1, z - 1, v);
              else
                images3_nl<D, L, T>(&a, xs, yr1, z - 1, v[0], v[1], v[2], v[3], v[4]);
            }
          }
        }
#pragma unroll
        for (int c = 0; c < C; ++c) zph[c] = Pz[c];
      }
#pragma unroll
      for (int c = 0; c < C; ++c) {
        zus[c] = Us[c];
        zfz[c] = Gz[c];
      }
    }
  }
  if (__any_sync(0xffffffffu, bad < 0 || nan >= kExpMask<T>) && lane == 0) atomicOr(a.flag, 1u);
  if (ws) publish_max(a, wmax);
}

// ------------------------------------------------------------------------
// k_step3d_rb: the k_step3d_ra tile walk (adjacent row pairs, TMA ring, two CTA
// barriers per plane) with the per-plane bookkeeping taken off the issue path
// (round-2 ncu: 61 % of k_step3d_ra's issued instructions were not arithmetic,
// and IMAD moves compete with FFMA2 for the FMA pipe):
//  * domain check: per row of the pair one running minimum of hi(rho),
//    hi(p) over the states the sweeps read -- U^n (x-flux), U* (y-flux), U** (z-flux)
//    -- and one running maximum of the outputs' |bits| (NaN/Inf), unmasked in the
//    loop (one VIMNMX3 per state); the lane's loop-invariant output mask is applied
//    once after the march.  Checking exactly the tile's output cells covers every
//    interior cell once (the ghost and halo cells other tiles' lanes hold are copies
//    of interior cells, checked by their owners);
//  * the z-march state (U**, F_z of the previous plane, the last z-face) ping-pongs
//    between two register sets (plane loop unrolled by two): nothing is copied;
//  * ghost images behind a CTA-uniform test (tile within pad of a partition face in
//    x or y, or a boundary plane); stores predicated;
//  * NS-stage TMA ring (loads issued NS planes ahead).
// Per cell and face the operations are scheme.cuh's, in the same order: bitwise
// equal to k_step3d_ra / k_step3d / k_sweep.
// ------------------------------------------------------------------------
template <int NW, typename T, int NS>
struct SmemRB {
  static constexpr int W = 32, R = 2 * NW, C = 5;
  static constexpr int AL = 16 / (int)sizeof(T);
  static constexpr int WB = W + AL;
  static constexpr int STAGE = R * C * WB;
  static constexpr int XY = NW * 2 * C * W;  // (U*, F_y) of row 2w+1, per warp
  static constexpr int FY = NW * C * W;      // face below row 2w, per warp
  static constexpr size_t bytes() { return (size_t)(NS * STAGE + XY + FY) * sizeof(T) + 8 * NS; }
};

template <typename P>
struct ZPlane {
  P us[5];  // U** of the previous plane
  P fz[5];  // F_z(U**) of the previous plane
  P ph[5];  // z-face below the previous plane
};

template <int NW, int MB, int L, typename P, int NS, bool UZ>
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
  int t = blockIdx.x;
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
  const P qx(kc.q[0]), nqx(kc.nq2[0]), qy(kc.q[1]), nqy(kc.nq2[1]), qz(kc.q[2]), nqz(kc.nq2[2]);
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
    P U[C], F[C], S_[C], G[C];
    {
      const T* r0 = stage + s * SM::STAGE + xoff;
      const T* r1 = r0 + C * SM::WB;
#pragma unroll
      for (int c = 0; c < C; ++c) U[c] = P(r0[c * cst], r1[c * cst]);
    }
    dom_min(dm0, dm1, U[0], flux_p<D, 0>(U, F, gm1));
    {
      P Un[C], Fn[C], Pnx[C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        Un[c] = shfl_down1(U[c]);
        Fn[c] = shfl_down1(F[c]);
      }
      force_face<D, 0>(U, F, Un, Fn, Pnx, qx, nqx, gm1);
#pragma unroll
      for (int c = 0; c < C; ++c) S_[c] = U[c] - (Pnx[c] - shfl_up1(Pnx[c]));
    }
    dom_min(dm0, dm1, S_[0], flux_p<D, 1>(S_, G, gm1));
    {
      T* x1 = xy + warp * 2 * C * W + lane;  // row 2w+1 for warp w+1
#pragma unroll
      for (int c = 0; c < C; ++c) {
        x1[c * W] = S_[c].y;
        x1[(C + c) * W] = G[c].y;
      }
    }
    __syncthreads();  // (A) stage s consumed, rows 2w+1 published
    if (threadIdx.x == 0) {
      fence_proxy_async();
      issue(kz + NS);
    }
    // Y: faces (2w-1 | 2w) and (2w | 2w+1) in one pair evaluation
    P Py[C];
    {
      const T* pdn = xy + wdn * 2 * C * W + lane;
      P SL[C], GL[C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        SL[c] = P(pdn[c * W], S_[c].x);
        GL[c] = P(pdn[(C + c) * W], G[c].x);
      }
      force_face<D, 1>(SL, GL, S_, G, Py, qy, nqy, gm1);
      T* f0 = fyb + warp * C * W + lane;  // face below row 2w, for warp w-1
#pragma unroll
      for (int c = 0; c < C; ++c) f0[c * W] = Py[c].x;
    }
    __syncthreads();  // (B) faces published
    {
      const T* fu = fyb + wup * C * W + lane;  // face below row 2w+2 (warp w+1)
#pragma unroll
      for (int c = 0; c < C; ++c) zn.us[c] = S_[c] - (P(Py[c].y, fu[c * W]) - Py[c]);
      dom_min(dm0, dm1, zn.us[0], flux_p<D, 2>(zn.us, zn.fz, gm1));
      if (kz >= 1) {
        force_face<D, 2>(zp.us, zp.fz, zn.us, zn.fz, zn.ph, qz, nqz, gm1);
        if (kz >= 2) {
          // update and store plane z - 1
          P o[C];
#pragma unroll
          for (int c = 0; c < C; ++c) o[c] = zp.us[c] - (zn.ph[c] - zp.ph[c]);
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
  if constexpr (UZ) {
    for (; kz + 2 <= nplanes; kz += 2) {
      body(kz, za, zb);
      body(kz + 1, zb, za);
    }
    if (kz < nplanes) body(kz, za, zb);
  } else {
#pragma unroll 1
    for (; kz < nplanes; ++kz) {
      body(kz, za, zb);
      za = zb;
    }
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
__device__ __forceinline__ void st_if(float* p, float v, bool ok) {
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q st.global.f32 [%0], %1;\n}" ::"l"(p),
               "f"(v), "r"((int)ok)
               : "memory");
}
__device__ __forceinline__ void st_if(double* p, double v, bool ok) {
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q st.global.f64 [%0], %1;\n}" ::"l"(p),
               "d"(v), "r"((int)ok)
               : "memory");
}

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
  int t = blockIdx.x;
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
  const P qx(kc.q[0]), nqx(kc.nq2[0]), qy(kc.q[1]), nqy(kc.nq2[1]), qz(kc.q[2]), nqz(kc.nq2[2]);
  const int64_t plane = g.rstride * g.P[1], cs = g.cstride;
  T* dst0 = a.out + g.row(yr0, z0 - 1) * g.rstride + (g.xo + xs) * g.xstride;
  T* dst1 = dst0 + g.rstride;
  const int wdn = max(warp - 1, 0), wup = min(warp + 1, NW - 1);
  constexpr int cst = L == 0 ? SM::WB : 1;
  const int xoff = (L == 0 ? sh + lane : (sh + lane) * C) + j0 * C * SM::WB;
  const bool out_x = (lane >= 1) & (lane <= W - 2) & (xs < SX);
  const bool st0 = out_x & (j0 >= 1) & (yr0 < SY);
  const bool st1 = out_x & (j1 <= TY) & (yr1 < SY);
  T* const x1 = xy + warp * 2 * C * W + lane;   // row 2w+1 for warp w+1
  const T* const pdn = xy + wdn * 2 * C * W + lane;
  T* const f0 = fyb + warp * C * W + lane;      // face below row 2w, for warp w-1
  const T* const fu = fyb + wup * C * W + lane;  // face below row 2w+2 (warp w+1)

  // X: stage of plane kz -> (U*, F_y(U*)) of rows 2w, 2w+1
  auto xphase = [&](const int kz, P* S_, P* G) {
    const int s = kz % NS;
    mbar_wait(&bar[s], (kz / NS) & 1);
    P U[C], F[C];
    const T* r0 = stage + s * SM::STAGE + xoff;
    const T* r1 = r0 + C * SM::WB;
#pragma unroll
    for (int c = 0; c < C; ++c) U[c] = P(r0[c * cst], r1[c * cst]);
    dom_min(dm0, dm1, U[0], flux_p<D, 0>(U, F, gm1));
    P Un[C], Fn[C], Pnx[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
      Un[c] = shfl_down1(U[c]);
      Fn[c] = shfl_down1(F[c]);
    }
    force_face<D, 0>(U, F, Un, Fn, Pnx, qx, nqx, gm1);
#pragma unroll
    for (int c = 0; c < C; ++c) S_[c] = U[c] - (Pnx[c] - shfl_up1(Pnx[c]));
    dom_min(dm0, dm1, S_[0], flux_p<D, 1>(S_, G, gm1));
  };
  auto publish = [&](const P* S_, const P* G) {
#pragma unroll
    for (int c = 0; c < C; ++c) {
      x1[c * W] = S_[c].y;
      x1[(C + c) * W] = G[c].y;
    }
  };
  // A, TMA refill, Y faces, B
  auto yphase = [&](const int kz, const P* S_, const P* G, P* Py) {
    __syncthreads();  // (A) stage kz consumed, rows 2w+1 of plane kz published
    if (threadIdx.x == 0) {
      fence_proxy_async();
      issue(kz + NS);
    }
    P SL[C], GL[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
      SL[c] = P(pdn[c * W], S_[c].x);
      GL[c] = P(pdn[(C + c) * W], G[c].x);
    }
    force_face<D, 1>(SL, GL, S_, G, Py, qy, nqy, gm1);
#pragma unroll
    for (int c = 0; c < C; ++c) f0[c * W] = Py[c].x;
    __syncthreads();  // (B) faces published; every warp is done reading plane kz's rows
  };
  // y-update + z-march of plane kz: output o of plane kz-1 (kz >= 2), predicated stores
  // (M: 0 = first plane of the march, 1 = second, 2 = steady state -- compile-time, so
  // the steady-state block has no branch)
  auto zphase = [&](auto M, const P* S_, const P* Py, const ZPlane<P>& zp, ZPlane<P>& zn, P* o) {
#pragma unroll
    for (int c = 0; c < C; ++c) zn.us[c] = S_[c] - (P(Py[c].y, fu[c * W]) - Py[c]);
    dom_min(dm0, dm1, zn.us[0], flux_p<D, 2>(zn.us, zn.fz, gm1));
    constexpr int m = decltype(M)::value;
    if constexpr (m >= 1) {
      force_face<D, 2>(zp.us, zp.fz, zn.us, zn.fz, zn.ph, qz, nqz, gm1);
      if constexpr (m >= 2) {
#pragma unroll
        for (int c = 0; c < C; ++c) o[c] = zp.us[c] - (zn.ph[c] - zp.ph[c]);
        dst0 += plane;
        dst1 += plane;
#pragma unroll
        for (int c = 0; c < C; ++c) {
          st_if(dst0 + c * cs, o[c].x, st0);
          st_if(dst1 + c * cs, o[c].y, st1);
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
  // one plane with the next plane's x-sweep overlapped: (Sa, Ga) -> (Sb, Gb)
  auto full = [&](auto M, const int kz, const P* Sa, const P* Ga, P* Sb, P* Gb,
                  const ZPlane<P>& zp, ZPlane<P>& zn) {
    P Py[C], o[C];
    yphase(kz, Sa, Ga, Py);
    xphase(kz + 1, Sb, Gb);
    zphase(M, Sa, Py, zp, zn, o);
    publish(Sb, Gb);
    tail(M, kz, o);
  };
  auto last = [&](const int kz, const P* Sa, const P* Ga, const ZPlane<P>& zp, ZPlane<P>& zn) {
    P Py[C], o[C];
    yphase(kz, Sa, Ga, Py);
    zphase(std::integral_constant<int, 2>(), Sa, Py, zp, zn, o);
    tail(std::integral_constant<int, 2>(), kz, o);
  };
  using M0 = std::integral_constant<int, 0>;
  using M1 = std::integral_constant<int, 1>;
  using M2 = std::integral_constant<int, 2>;

  P SA[C], GA[C], SB[C], GB[C];
  ZPlane<P> za, zb;
  xphase(0, SA, GA);
  publish(SA, GA);
  full(M0(), 0, SA, GA, SB, GB, za, zb);  // nplanes >= 3
  full(M1(), 1, SB, GB, SA, GA, zb, za);
  int kz = 2;
  for (; kz + 2 < nplanes; kz += 2) {
    full(M2(), kz, SA, GA, SB, GB, za, zb);
    full(M2(), kz + 1, SB, GB, SA, GA, zb, za);
  }
  if (kz + 1 < nplanes) {
    full(M2(), kz, SA, GA, SB, GB, za, zb);
    last(kz + 1, SB, GB, zb, za);
  } else {
    last(kz, SA, GA, za, zb);
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

// Tile geometry.  fp64: k_step3d with 32-slot windows (V = 1) and 14-row tiles.
// fp32 runs a packed kernel unless a scalar variant is asked for (20: k_step3d
// V = 1; 21: V = 2, 64-slot windows, measured slower: 1.93 vs 1.35 ms at 384^3;
// 50-52: scalar tile shapes): by default k_step3d_ra (adjacent row pairs, 8 warps
// / 14 output rows, two CTAs per SM: 384^3 1047 us); 78: k_step3d_rp (rows w,
// w+8: 1111 us); 70: k_step3d_rp with 16 warps / 30 rows, one CTA per SM (slower
// still, SoA only).  AoS (configs[4] layout comparison) runs the 8-warp forms.
static bool use_rp(const Geom& g, int variant) {
  return g.elem == 4 && (variant == 0 || variant == 80 || variant == 78 ||
                         (variant == 70 && g.layout == 0));
}
static int rp_warps(int variant) { return variant == 70 ? 16 : 8; }

// tile rows of a 3-D launch (variants 50: 30 rows, 51: 22 rows; default 14;
// fp32 packed: 2 NW - 2 output rows, the box holds 2 NW rows incl. the y-halo)
static int ty3(const Geom& g, int variant) {
  if (use_rp(g, variant)) return 2 * rp_warps(variant) - 2;
  if (variant == 98) return 22;
  if (variant == 99) return 30;
  return variant == 50 ? 30 : (variant == 51 ? 22 : 14);
}

// x-window width of a 3-D launch (variant 21: fp32 with V = 2)
static int win3(const Geom& g, int variant) {
  return (g.elem == 4 && variant == 21) ? 64 : 32;
}

template <int NW, int MB, int L, typename P = pk>
static int launch3_ra(const KArgs<typename PairElem<P>::T>& a, const void* tmap,
                      cudaStream_t s) {
  using T = typename PairElem<P>::T;
  constexpr int W = 32, TY = 2 * NW - 2;
  const Geom& g = a.g;
  const int nwin = (int)((g.S[0] + (W - 2) - 1) / (W - 2));
  const int nyb = (int)((g.S[1] + TY - 1) / TY);
  const int nzc = (int)((g.S[2] + a.rows - 1) / a.rows);
  const size_t sm = SmemRA<NW, T>::bytes();
  if constexpr (sizeof(T) == 4) pk_set_negzero(s);
  static int cache[kMaxDevices] = {0};
  resident_ctas(k_step3d_ra<NW, MB, L, P>, 32 * NW, sm, cache);
  k_step3d_ra<NW, MB, L, P><<<nwin * nyb * nzc, 32 * NW, sm, s>>>(
      a, *reinterpret_cast<const CUtensorMap*>(tmap), nwin, nyb);
  return 0;
}

template <int NW, int MB, int L, typename P, int NS, bool UZ = false>
static int launch3_rb(const KArgs<typename PairElem<P>::T>& a, const void* tmap,
                      cudaStream_t s) {
  using T = typename PairElem<P>::T;
  constexpr int W = 32, TY = 2 * NW - 2;
  const Geom& g = a.g;
  const int nwin = (int)((g.S[0] + (W - 2) - 1) / (W - 2));
  const int nyb = (int)((g.S[1] + TY - 1) / TY);
  const int nzc = (int)((g.S[2] + a.rows - 1) / a.rows);
  const size_t sm = SmemRB<NW, T, NS>::bytes();
  if constexpr (sizeof(T) == 4) pk_set_negzero(s);
  static int cache[kMaxDevices] = {0};
  resident_ctas(k_step3d_rb<NW, MB, L, P, NS, UZ>, 32 * NW, sm, cache);
  k_step3d_rb<NW, MB, L, P, NS, UZ><<<nwin * nyb * nzc, 32 * NW, sm, s>>>(
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
  const size_t sm = SmemRB<NW, T, NS>::bytes();
  if constexpr (sizeof(T) == 4) pk_set_negzero(s);
  static int cache[kMaxDevices] = {0};
  resident_ctas(k_step3d_sp<NW, MB, L, P, NS>, 32 * NW, sm, cache);
  k_step3d_sp<NW, MB, L, P, NS><<<nwin * nyb * nzc, 32 * NW, sm, s>>>(
      a, *reinterpret_cast<const CUtensorMap*>(tmap), nwin, nyb);
  return 0;
}

template <int NW, int MB, int L>
static int launch3_rp(const KArgs<float>& a, const void* tmap, cudaStream_t s) {
  constexpr int W = 32, TY = 2 * NW - 2;
  const Geom& g = a.g;
  const int nwin = (int)((g.S[0] + (W - 2) - 1) / (W - 2));
  const int nyb = (int)((g.S[1] + TY - 1) / TY);
  const int nzc = (int)((g.S[2] + a.rows - 1) / a.rows);
  const size_t sm = SmemRP<NW>::bytes();
  pk_set_negzero(s);
  static int cache[kMaxDevices] = {0};
  resident_ctas(k_step3d_rp<NW, MB, L>, 32 * NW, sm, cache);  // sets the smem attribute
  k_step3d_rp<NW, MB, L><<<nwin * nyb * nzc, 32 * NW, sm, s>>>(
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

int window3d(const Geom& g) { return 30; }

template <typename T, int V, int TY, int MB = 1, int L = 0>
static int launch3(const KArgs<T>& a, const void* tmap, cudaStream_t s) {
  constexpr int W = 32 * V;
  const Geom& g = a.g;
  const int nwin = (int)((g.S[0] + (W - 2) - 1) / (W - 2));
  const int nyb = (int)((g.S[1] + TY - 1) / TY);
  const int nzc = (int)((g.S[2] + a.rows - 1) / a.rows);
  const size_t sm = Smem3<TY, V, T>::bytes();
  static int cache[kMaxDevices] = {0};
  resident_ctas(k_step3d<T, V, TY, MB, L>, 32 * (TY + 2), sm, cache);  // sets the smem attribute
  k_step3d<T, V, TY, MB, L><<<nwin * nyb * nzc, 32 * (TY + 2), sm, s>>>(
      a, *reinterpret_cast<const CUtensorMap*>(tmap), nwin, nyb);
  return 0;
}

template <typename T>
int launch_step3d(const KArgs<T>& a, const void* tmap, cudaStream_t s) {
  if (a.variant == 0) {
    // defaults (round 2, profiles/r2/): fp64 k_step3d_sp (software-pipelined planes,
    // 8 warps, 1 CTA/SM, 3-stage ring): 512^3 4.34 -> 3.90 ms; fp32 k_step3d_rb
    // (8 warps, 2 CTAs/SM, 3-stage ring): 384^3 1.06 -> 0.99 ms
    const bool aos = a.g.layout == 1;
    if constexpr (sizeof(T) == 8)
      return aos ? launch3_sp<8, 1, 1, pd, 3>(a, tmap, s) : launch3_sp<8, 1, 0, pd, 3>(a, tmap, s);
    else
      return aos ? launch3_rb<8, 2, 1, pk, 3>(a, tmap, s) : launch3_rb<8, 2, 0, pk, 3>(a, tmap, s);
  }
  if (a.variant == 99) {
    using P = typename std::conditional<sizeof(T) == 8, pd, pk>::type;
    return a.g.layout == 1 ? launch3_rb<16, 1, 1, P, 3>(a, tmap, s) : launch3_rb<16, 1, 0, P, 3>(a, tmap, s);
  }
  if (a.variant == 98) {
    using P = typename std::conditional<sizeof(T) == 8, pd, pk>::type;
    return a.g.layout == 1 ? launch3_sp<12, 1, 1, P, 3>(a, tmap, s) : launch3_sp<12, 1, 0, P, 3>(a, tmap, s);
  }
  if (a.variant >= 95 && a.variant <= 97) {
    using P = typename std::conditional<sizeof(T) == 8, pd, pk>::type;
    constexpr int MB = sizeof(T) == 8 ? 1 : 2;
    const bool aos = a.g.layout == 1;
    switch (a.variant) {
      case 96: return aos ? launch3_sp<8, MB, 1, P, 3>(a, tmap, s) : launch3_sp<8, MB, 0, P, 3>(a, tmap, s);
      case 97: return aos ? launch3_sp<8, 1, 1, P, 3>(a, tmap, s) : launch3_sp<8, 1, 0, P, 3>(a, tmap, s);
      default: return aos ? launch3_sp<8, MB, 1, P, 2>(a, tmap, s) : launch3_sp<8, MB, 0, P, 2>(a, tmap, s);
    }
  }
  if (a.variant >= 90 && a.variant <= 94) {
    using P = typename std::conditional<sizeof(T) == 8, pd, pk>::type;
    constexpr int MB = sizeof(T) == 8 ? 1 : 2;
    const bool aos = a.g.layout == 1;
    switch (a.variant) {
      case 91: return aos ? launch3_rb<8, MB, 1, P, 3>(a, tmap, s) : launch3_rb<8, MB, 0, P, 3>(a, tmap, s);
      case 92: return aos ? launch3_rb<8, MB, 1, P, 4>(a, tmap, s) : launch3_rb<8, MB, 0, P, 4>(a, tmap, s);
      case 93: return aos ? launch3_rb<8, MB, 1, P, 2, true>(a, tmap, s) : launch3_rb<8, MB, 0, P, 2, true>(a, tmap, s);
      case 94: return aos ? launch3_rb<8, MB, 1, P, 4, true>(a, tmap, s) : launch3_rb<8, MB, 0, P, 4, true>(a, tmap, s);
      default: return aos ? launch3_rb<8, MB, 1, P, 2>(a, tmap, s) : launch3_rb<8, MB, 0, P, 2>(a, tmap, s);
    }
  }
  if constexpr (sizeof(T) == 4) {
    // packed row pairs (default) -- must match use_rp() / the TMA box
    if (use_rp(a.g, a.variant)) {
      // default: adjacent row pairs (k_step3d_ra); 78: rows w, w+8 (k_step3d_rp); 70: the
      // same with 16 warps / 30 rows
      if (a.variant == 70) return launch3_rp<16, 1, 0>(a, tmap, s);
      if (a.variant == 78)
        return a.g.layout == 1 ? launch3_rp<8, 2, 1>(a, tmap, s) : launch3_rp<8, 2, 0>(a, tmap, s);
      return a.g.layout == 1 ? launch3_ra<8, 2, 1>(a, tmap, s) : launch3_ra<8, 2, 0>(a, tmap, s);
    }
  }
  if constexpr (sizeof(T) == 8) {
    // 80: the round-1 fp64 default, adjacent row pairs of doubles (k_step3d_ra<pd>, 8
    // warps, 216 registers, 1 CTA/SM): 512^3 4340 us
    if (a.variant == 80)
      return a.g.layout == 1 ? launch3_ra<8, 1, 1, pd>(a, tmap, s) : launch3_ra<8, 1, 0, pd>(a, tmap, s);
  }
  if (a.g.layout == 1) return launch3<T, 1, 14, 1, 1>(a, tmap, s);  // AoS (configs[4])
  if constexpr (sizeof(T) == 4) {
    // V = 2 (two cells per lane) only for fp32 -- must match win3() / the TMA box
    if (a.variant == 21) return launch3<T, 2, 14>(a, tmap, s);
  }
  switch (a.variant) {
    case 50: return launch3<T, 1, 30>(a, tmap, s);
    case 51: return launch3<T, 1, 22>(a, tmap, s);
    case 52: return launch3<T, 1, 14, 2>(a, tmap, s);
    case 56: return launch3<T, 1, 14>(a, tmap, s);  // fp64: the one-row-per-warp kernel
    default: return launch3<T, 1, 14>(a, tmap, s);
  }
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
  if (g.layout == 1) return make_tmap_aos(g, buf, map_out, 32 + 16 / g.elem, ty3(g, variant) + 2);
  return make_tmap(g, buf, map_out, win3(g, variant) + 16 / g.elem,  // + Smem3::AL
                   ty3(g, variant) + 2);
}
template int launch_step3d<float>(const KArgs<float>&, const void*, cudaStream_t);
template int launch_step3d<double>(const KArgs<double>&, const void*, cudaStream_t);

}  // namespace rpl
