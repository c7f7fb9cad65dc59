// geometry.hpp -- padded, partitioned N-D tensor geometry (host + device).
//
// A Ripple tensor (sec. 4.1, Listing 1) is a global N-D grid of
// cells split into parts[0] x parts[1] x parts[2] equal partitions (P:299-310,
// divisibility required), each with `pad` ghost layers on every
// face (uniform padding S:194).
//
// HBM layout of one partition buffer:
//   SoA ("strided"):  [Pz][Py][C][pitch]   -- every row holds C
//       component sub-rows, each contiguous in x (coalesced 128-bit vectors);
//       component c of row r sits c*pitch elements after component 0
//   AoS ("contiguous"):          [Pz][Py][pitch][C]
// element (c,x,y,z) at  row(y,z)*rstride + c*cstride + (xo+x)*xstride  with
//   SoA: rstride = C*pitch, cstride = pitch, xstride = 1
//   AoS: rstride = C*pitch, cstride = 1,     xstride = C
// Pd = S_d + 2 pad for used dims, 1 for unused dims (oz/oy = pad or 0).
// xo is chosen odd-aligned so that x = -1 starts a 2-element vector (the fused
// kernel's 64-slot warp windows start at x = 62k - 1) and `pitch` is a multiple
// of 128 bytes covering every window slot; row starts are 128-byte aligned.
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define RPL_HD __host__ __device__ __forceinline__
#else
#define RPL_HD inline
#endif

namespace rpl {

constexpr int kMaxParts = 64;   // partitions per tensor (all may live on one rank)
constexpr int kMaxPad = 4;
constexpr int kWinSlots = 64;   // fused kernels: cells per warp window (32 lanes x 2)
constexpr int kWinOut = 62;     // outputs per window (slots 1..62)

struct Geom {
  int D;              // 1..3
  int C;              // D + 2 components
  int pad;            // ghost width
  int elem;           // bytes per element (4 or 8)
  int layout;         // 0 SoA, 1 AoS
  int bc_lo[3], bc_hi[3];
  int parts[3];
  int nparts;
  int64_t N[3];       // global interior extents (unused dims: 1)
  int64_t S[3];       // partition interior extents
  int64_t P[3];       // padded extents (unused dims: 1)
  int64_t off[3];     // padded index of interior cell 0 (pad or 0)
  int64_t xo;         // row offset of x = 0 (== off[0] shifted for alignment)
  int64_t pitch;      // elements (SoA) or cells (AoS) per row
  int64_t rstride;    // elements between consecutive rows (both layouts: C*pitch)
  int64_t cstride;    // elements between components of one cell (SoA pitch, AoS 1)
  int64_t xstride;    // elements between consecutive x cells (SoA 1, AoS C)
  int64_t buf_elems;  // elements per partition buffer
  int nwin;           // fused: 62-cell windows per row
  int img_fast;       // 1: single partition, pad <= 2, used extents >= 2 pad (images_single)

  // padded row index of (y, z) (signed interior coordinates)
  RPL_HD int64_t row(int64_t y, int64_t z) const { return (z + off[2]) * P[1] + (y + off[1]); }
  // element index of component c of cell (x, y, z)
  RPL_HD int64_t at(int c, int64_t x, int64_t y, int64_t z) const {
    return row(y, z) * rstride + c * cstride + (xo + x) * xstride;
  }
  RPL_HD int64_t cells() const { return S[0] * S[1] * S[2]; }
  RPL_HD void part_coords(int p, int pc[3]) const {
    pc[0] = p % parts[0];
    pc[1] = (p / parts[0]) % parts[1];
    pc[2] = p / (parts[0] * parts[1]);
  }
  RPL_HD int part_index(int a, int b, int c) const { return (c * parts[1] + b) * parts[0] + a; }
};

// Build the geometry; returns 0 or a negative rpl_status code.
int make_geom(int D, const int64_t size[3], int pad, const int parts[3], int elem, int layout,
              const int bc_lo[3], const int bc_hi[3], Geom* g, const char** why);

}  // namespace rpl
