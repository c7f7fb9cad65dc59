// packed.cuh -- two fp32 lanes of the scheme per instruction (sm_100a FFMA2 /
// FADD2 / FMUL2, PTX add|sub|mul|fma.rn.f32x2).
//
// `pk` holds one component of two cells (a register pair).  The scheme's
// templates in scheme.cuh (cell_ab, face_psi, psi_update) run unchanged on it, so a
// packed kernel performs, per lane, exactly the IEEE operations of the scalar
// fp32 kernels -- results are bitwise identical.
// Measured on the B200 (tools/dp_microbench.cu): FFMA2 delivers the same lane
// rate as FFMA (126 lane-FMA/clk/SM) from half the issue slots, which is what
// the issue-bound fp32 3-D step needs.
//
// One ptxas caveat: it contracts mul.rn.f32x2 + add/sub.rn.f32x2 into FFMA2
// even under --fmad=false (and folds fma(a, b, -0) back to a multiply first),
// which would break bit-identity with the scalar kernels.  Products are
// therefore issued as fma(a, b, z) with z = -0.0 read from constant memory that
// the host sets at run time (pk_set_negzero): the compiler cannot see the
// value, so the multiply stays a stand-alone FFMA2 and fma(a, b, -0) == a*b
// exactly (including the sign of zero).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "launch.cuh"
#include "scheme.cuh"

namespace rpl {

// (-0.0f, -0.0f) -- written by the host (pk_set_negzero) before any packed launch;
// one copy per translation unit (static), each set by its own launchers
static __constant__ unsigned long long c_pk_negzero;

// Host: write c_pk_negzero of this translation unit on the current device, once,
// ordered before the caller's launch on `stream` and completed before returning
// (a pageable cudaMemcpyToSymbol may return before its DMA lands, and the
// library's stream does not synchronise with the legacy stream).
static inline void pk_set_negzero(cudaStream_t stream) {
  static int done[kMaxDevices] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) dev = 0;
  if (done[dev]) return;
  static const unsigned long long nz = 0x8000000080000000ull;
  if (cudaMemcpyToSymbolAsync(c_pk_negzero, &nz, sizeof(nz), 0, cudaMemcpyHostToDevice,
                              stream) == cudaSuccess &&
      cudaStreamSynchronize(stream) == cudaSuccess)
    done[dev] = 1;
}

struct __align__(8) pk {
  float x, y;
  __device__ __forceinline__ pk() {}
  __device__ __forceinline__ pk(float a, float b) : x(a), y(b) {}
  template <typename S>
  __device__ __forceinline__ explicit pk(S s) : x((float)s), y((float)s) {}
};

__device__ __forceinline__ unsigned long long pbits(pk a) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a.x), "f"(a.y));
  return r;
}
__device__ __forceinline__ pk punpack(unsigned long long r) {
  pk a;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a.x), "=f"(a.y) : "l"(r));
  return a;
}

__device__ __forceinline__ pk operator+(pk a, pk b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pbits(a)), "l"(pbits(b)));
  return punpack(r);
}
__device__ __forceinline__ pk operator-(pk a, pk b) {
  unsigned long long r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pbits(a)), "l"(pbits(b)));
  return punpack(r);
}
__device__ __forceinline__ pk operator*(pk a, pk b) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pbits(a)), "l"(pbits(b)), "l"(c_pk_negzero));
  return punpack(r);
}
__device__ __forceinline__ pk operator-(pk a) { return pk(-a.x, -a.y); }
using ::fma;  // keep the scalar overloads visible next to the packed one
__device__ __forceinline__ pk fma(pk a, pk b, pk c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pbits(a)), "l"(pbits(b)), "l"(pbits(c)));
  return punpack(r);
}
// 1/x per lane: the scalar MUFU + Newton sequence of scheme.cuh, the Newton step as
// two FFMA2 (per lane the same IEEE fma(r, fma(-x, r, 1), r) as the scalar rcp)
__device__ __forceinline__ pk rcp(pk a) {
  float r0, r1;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r0) : "f"(a.x));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r1) : "f"(a.y));
  const pk r(r0, r1);
  return fma(r, fma(-a, r, pk(1.0f)), r);
}

// running domain minimum per lane (scheme.cuh dom_min)
__device__ __forceinline__ void dom_min(int& a0, int& a1, pk rho, pk p) {
  dom_min(a0, rho.x, p.x);
  dom_min(a1, rho.y, p.y);
}

// domain word per lane (scheme.cuh dom_word)
struct PkDom {
  int a, b;
  __device__ __forceinline__ PkDom& operator|=(PkDom o) {
    a |= o.a;
    b |= o.b;
    return *this;
  }
};
__device__ __forceinline__ PkDom dom_word(pk rho, pk p) {
  return PkDom{dom_word(rho.x, p.x), dom_word(rho.y, p.y)};
}

// fp64 counterpart: two cells' values of one component as a plain pair (no packed
// FP64 instructions exist); lets the row-pair kernels run in double precision with
// exactly the scalar operations (mul stays a DMUL under -fmad=false).
struct pd {
  double x, y;
  __device__ __forceinline__ pd() {}
  __device__ __forceinline__ pd(double a, double b) : x(a), y(b) {}
  template <typename S>
  __device__ __forceinline__ explicit pd(S s) : x((double)s), y((double)s) {}
};
__device__ __forceinline__ pd operator+(pd a, pd b) { return pd(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ pd operator-(pd a, pd b) { return pd(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ pd operator*(pd a, pd b) { return pd(a.x * b.x, a.y * b.y); }
__device__ __forceinline__ pd operator-(pd a) { return pd(-a.x, -a.y); }
__device__ __forceinline__ pd fma(pd a, pd b, pd c) {
  return pd(::fma(a.x, b.x, c.x), ::fma(a.y, b.y, c.y));
}
__device__ __forceinline__ pd rcp(pd a) { return pd(rcp(a.x), rcp(a.y)); }
__device__ __forceinline__ PkDom dom_word(pd rho, pd p) {
  return PkDom{dom_word(rho.x, p.x), dom_word(rho.y, p.y)};
}
__device__ __forceinline__ void dom_min(int& a0, int& a1, pd rho, pd p) {
  dom_min(a0, rho.x, p.x);
  dom_min(a1, rho.y, p.y);
}
__device__ __forceinline__ pd shfl_down1(pd v) {
  return pd(__shfl_down_sync(0xffffffffu, v.x, 1), __shfl_down_sync(0xffffffffu, v.y, 1));
}
__device__ __forceinline__ pd shfl_up1(pd v) {
  return pd(__shfl_up_sync(0xffffffffu, v.x, 1), __shfl_up_sync(0xffffffffu, v.y, 1));
}

// componentwise minmod of pairs (scheme.cuh minmod per lane)
__device__ __forceinline__ pd minmod(pd a, pd b) { return pd(minmod(a.x, b.x), minmod(a.y, b.y)); }
__device__ __forceinline__ pk minmod(pk a, pk b) { return pk(minmod(a.x, b.x), minmod(a.y, b.y)); }

// element type of a pair type
template <typename P> struct PairElem;
template <> struct PairElem<pk> { using T = float; };
template <> struct PairElem<pd> { using T = double; };

__device__ __forceinline__ pk shfl_down1(pk v) {
  return pk(__shfl_down_sync(0xffffffffu, v.x, 1), __shfl_down_sync(0xffffffffu, v.y, 1));
}
__device__ __forceinline__ pk shfl_up1(pk v) {
  return pk(__shfl_up_sync(0xffffffffu, v.x, 1), __shfl_up_sync(0xffffffffu, v.y, 1));
}

}  // namespace rpl
