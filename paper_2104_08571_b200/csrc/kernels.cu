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
#include <cuda_runtime.h>
#include <stdint.h>

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
  for (int c = 0; c < D + 2; ++c) {
    const int64_t i = L == 0 ? c * g.comp_stride + g.row(y, z) * g.pitch + g.xo + x
                             : (g.row(y, z) * g.pitch + g.xo + x) * (D + 2) + c;
    v[c] = buf[i];
  }
}

template <int D, int L, typename T>
__device__ __noinline__ void write_images_noinline(const KArgs<T> a, int64_t x, int64_t y,
                                                   int64_t z, const T* v) {
  write_images<D, L>(a, x, y, z, v);
}

// ---------------------------------------------------------------------------
// K-A: one sweep along d.  Thread per interior cell; both faces of the cell are
// evaluated (the simple, unfused baseline: 3 flux evaluations + 2 faces).
// ---------------------------------------------------------------------------
template <typename T, int D, int d, int L>
__global__ void __launch_bounds__(256) k_sweep(const KArgs<T> a) {
  constexpr int C = D + 2;
  const Geom& g = a.g;
  const int64_t n = g.cells();
  bool ok = true;
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
    ok &= phys_flux<D, d>(U0, F0, a.gm1);
    phys_flux<D, d>(Up, Fp, a.gm1);
    T PL[C], PR[C], o[C];
    force_face<D, d>(Um, Fm, U0, F0, PL, a.q[d], a.nq2[d], a.gm1);
    force_face<D, d>(U0, F0, Up, Fp, PR, a.q[d], a.nq2[d], a.gm1);
#pragma unroll
    for (int c = 0; c < C; ++c) o[c] = U0[c] - (PR[c] - PL[c]);
    store_cell<D, L>(g, a.out, x, y, z, o);
    if (near_face<D>(g, x, y, z)) write_images_noinline<D, L>(a, x, y, z, o);
  }
  if (!ok) atomicOr(a.flag, 1u);
}

// ---------------------------------------------------------------------------
// K-B (2-D): x-sweep and y-sweep of one step fused into a single pass.
//
// A warp owns a 64-slot window of one row (lane l holds slots 2l, 2l+1 as one
// 128-bit (fp64) / 64-bit (fp32) vector; slot s <-> x = 62 w - 1 + s) and marches
// down a chunk of `rows` rows.  For each row: vector-load U, x-sweep in
// registers (face values shared across lanes with warp shuffles; slots 0 and 63
// are the window's halo), then the y-face between this row and the previous
// one from the march state (previous U*, F_y(U*), previous y-face), update and
// store the previous row.  HBM traffic per cell: one read of U^n, one write of
// U^{n+1}; the x-halo (2 of 64 slots) and the chunk's 2 halo rows are
// recomputed, not re-stored.  Vector loads are 2-element aligned because the
// layout puts x = -1 on an even element offset (geometry.hpp).
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(128) k_step2d(const KArgs<T> a, int nwin, int ntask) {
  constexpr int D = 2, C = 4;
  using V = typename Vec2<T>::type;
  const Geom& g = a.g;
  const int lane = threadIdx.x & 31;
  const int wid = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (wid >= ntask) return;
  const int win = wid % nwin;
  const int chunk = wid / nwin;
  const int64_t xa = (int64_t)win * kWinOut - 1 + 2 * lane;
  const int64_t y0 = (int64_t)chunk * a.rows;
  const int64_t y1 = min(y0 + (int64_t)a.rows, g.S[1]);
  const int64_t cs = g.comp_stride, pitch = g.pitch;
  const T* __restrict__ base = a.in + g.xo + xa;
  T* __restrict__ obase = a.out + g.xo + xa;
  const bool ina = (xa >= -1) & (xa <= g.S[0]);
  const bool inb = (xa + 1 >= -1) & (xa + 1 <= g.S[0]);
  const bool va = (lane >= 1) & (xa < g.S[0]);
  const bool vb = (lane <= 30) & (xa + 1 < g.S[0]);
  const T gm1 = a.gm1, qx = a.q[0], nqx = a.nq2[0], qy = a.q[1], nqy = a.nq2[1];
  bool ok = true;

  T usA[C], fyA[C], phA[C], usB[C], fyB[C], phB[C];
  V nxt[C];
  {
    const T* p = base + g.row(y0 - 1, 0) * pitch;
#pragma unroll
    for (int c = 0; c < C; ++c) nxt[c] = *reinterpret_cast<const V*>(p + c * cs);
  }
  for (int64_t y = y0 - 1; y <= y1; ++y) {
    T Ua[C], Ub[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
      Ua[c] = nxt[c].x;
      Ub[c] = nxt[c].y;
    }
    if (y < y1) {
      const T* p = base + g.row(y + 1, 0) * pitch;
#pragma unroll
      for (int c = 0; c < C; ++c) nxt[c] = *reinterpret_cast<const V*>(p + c * cs);
    }
    // ---- x-sweep of row y
    T Fa[C], Fb[C], Pab[C], Pbn[C], Un[C], Fn[C];
    ok &= phys_flux<D, 0>(Ua, Fa, gm1) | !ina;
    ok &= phys_flux<D, 0>(Ub, Fb, gm1) | !inb;
    force_face<D, 0>(Ua, Fa, Ub, Fb, Pab, qx, nqx, gm1);
#pragma unroll
    for (int c = 0; c < C; ++c) {
      Un[c] = __shfl_down_sync(kFull, Ua[c], 1);
      Fn[c] = __shfl_down_sync(kFull, Fa[c], 1);
    }
    force_face<D, 0>(Ub, Fb, Un, Fn, Pbn, qx, nqx, gm1);
    T Sa[C], Sb[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const T Ppa = __shfl_up_sync(kFull, Pbn[c], 1);
      Sa[c] = Ua[c] - (Pab[c] - Ppa);
      Sb[c] = Ub[c] - (Pbn[c] - Pab[c]);
    }
    // ---- y-sweep: face (y-1/2), update row y-1
    T Ga[C], Gb[C];
    ok &= phys_flux<D, 1>(Sa, Ga, gm1) | !va;
    ok &= phys_flux<D, 1>(Sb, Gb, gm1) | !vb;
    if (y >= y0) {
      T Qa[C], Qb[C];
      force_face<D, 1>(usA, fyA, Sa, Ga, Qa, qy, nqy, gm1);
      force_face<D, 1>(usB, fyB, Sb, Gb, Qb, qy, nqy, gm1);
      if (y > y0) {
        T oa[C], ob[C];
#pragma unroll
        for (int c = 0; c < C; ++c) {
          oa[c] = usA[c] - (Qa[c] - phA[c]);
          ob[c] = usB[c] - (Qb[c] - phB[c]);
        }
        T* p = obase + g.row(y - 1, 0) * pitch;
        if (va & vb) {
#pragma unroll
          for (int c = 0; c < C; ++c) {
            V w;
            w.x = oa[c];
            w.y = ob[c];
            *reinterpret_cast<V*>(p + c * cs) = w;
          }
        } else {
          if (va) {
#pragma unroll
            for (int c = 0; c < C; ++c) p[c * cs] = oa[c];
          }
          if (vb) {
#pragma unroll
            for (int c = 0; c < C; ++c) p[c * cs + 1] = ob[c];
          }
        }
        if (va && near_face<D>(g, xa, y - 1, 0)) write_images_noinline<D, 0>(a, xa, y - 1, 0, oa);
        if (vb && near_face<D>(g, xa + 1, y - 1, 0))
          write_images_noinline<D, 0>(a, xa + 1, y - 1, 0, ob);
      }
#pragma unroll
      for (int c = 0; c < C; ++c) {
        phA[c] = Qa[c];
        phB[c] = Qb[c];
      }
    }
#pragma unroll
    for (int c = 0; c < C; ++c) {
      usA[c] = Sa[c];
      fyA[c] = Ga[c];
      usB[c] = Sb[c];
      fyB[c] = Gb[c];
    }
  }
  if (!__all_sync(kFull, ok) && lane == 0) atomicOr(a.flag, 1u);
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
  // aim for ~12 resident warps per SM over 148 SMs, march at least 8 rows
  const int64_t target = 148 * 12;
  int64_t rows = (g.S[1] * g.nwin + target - 1) / target;
  if (rows < 8) rows = 8;
  if (rows > g.S[1]) rows = g.S[1];
  return (int)rows;
}

template <typename T>
void launch_step2d(const KArgs<T>& a, cudaStream_t s) {
  const int nchunk = (int)((a.g.S[1] + a.rows - 1) / a.rows);
  const int ntask = a.g.nwin * nchunk;
  const int wpb = 4;
  k_step2d<T><<<(ntask + wpb - 1) / wpb, 32 * wpb, 0, s>>>(a, a.g.nwin, ntask);
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
template void launch_step2d<float>(const KArgs<float>&, cudaStream_t);
template void launch_step2d<double>(const KArgs<double>&, cudaStream_t);
template void launch_fill<float>(const Geom&, int, float* const*, cudaStream_t);
template void launch_fill<double>(const Geom&, int, double* const*, cudaStream_t);
template void launch_maxws<float>(const Geom&, const float*, double, unsigned long long*,
                                  unsigned*, cudaStream_t);
template void launch_maxws<double>(const Geom&, const double*, double, unsigned long long*,
                                   unsigned*, cudaStream_t);

}  // namespace rpl

namespace rpl {
int auto_rows_3d(const Geom& g) { return (int)(g.S[2] < 16 ? g.S[2] : 16); }
}  // namespace rpl
