// plan.cpp -- geometry and halo plan (host only; no CUDA calls, usable on CPU boxes).
//
// The halo plan is the paper's padding-transfer graph (concurrent_padded_access
// inserts one transfer node per neighbouring partition: 2/8/26 copies per
// partition in 1/2/3-D, sec. 5.4.1, Fig. 7) merged with set_boundary
// (P:283-297): every ghost cell gets exactly one source interior cell, so one
// list of boxes describes both the physical boundary fill and the exchange.
#include <string.h>

#include <vector>

#include "../../include/ripple_fv.h"
#include "geometry.hpp"
#include "plan.hpp"

namespace rpl {

int make_geom(int D, const int64_t size[3], int pad, const int parts[3], int elem, int layout,
              const int bc_lo[3], const int bc_hi[3], Geom* g, const char** why) {
  *why = "";
  memset(g, 0, sizeof(Geom));
  if (D < 1 || D > 3) { *why = "ndim must be 1, 2 or 3"; return RPL_E_INVALID_ARG; }
  if (pad < 1) { *why = "pad must be >= 1 (stencil radius 1)"; return RPL_E_PAD_TOO_SMALL; }
  if (pad > kMaxPad) { *why = "pad must be <= 4"; return RPL_E_INVALID_ARG; }
  if (elem != 4 && elem != 8) { *why = "dtype"; return RPL_E_INVALID_ARG; }
  if (layout != 0 && layout != 1) { *why = "layout"; return RPL_E_INVALID_ARG; }
  g->D = D;
  g->C = D + 2;
  g->pad = pad;
  g->elem = elem;
  g->layout = layout;
  g->nparts = 1;
  for (int d = 0; d < 3; ++d) {
    const bool used = d < D;
    if (size[d] < 1 || parts[d] < 1) { *why = "size and parts must be >= 1"; return RPL_E_INVALID_ARG; }
    if (!used && (size[d] != 1 || parts[d] != 1)) {
      *why = "unused dims must have size 1 and parts 1";
      return RPL_E_INVALID_ARG;
    }
    if (size[d] % parts[d] != 0) {
      *why = "size not divisible by partition count (SPEC S:135, S:192)";
      return RPL_E_NOT_DIVISIBLE;
    }
    g->N[d] = size[d];
    g->parts[d] = parts[d];
    g->S[d] = size[d] / parts[d];
    g->nparts *= parts[d];
    if (used && g->S[d] < pad) { *why = "partition extent must be >= pad"; return RPL_E_INVALID_ARG; }
    g->bc_lo[d] = used ? bc_lo[d] : 0;
    g->bc_hi[d] = used ? bc_hi[d] : 0;
    if (used && (bc_lo[d] < 0 || bc_lo[d] > 2 || bc_hi[d] < 0 || bc_hi[d] > 2)) {
      *why = "unknown boundary kind";
      return RPL_E_INVALID_ARG;
    }
    if (used && ((bc_lo[d] == 1) != (bc_hi[d] == 1))) {
      *why = "periodic must be set on both faces of a dim";
      return RPL_E_INVALID_ARG;
    }
    g->P[d] = used ? g->S[d] + 2 * pad : 1;
    g->off[d] = used ? pad : 0;
  }
  if (g->nparts > kMaxParts) { *why = "too many partitions (max 64)"; return RPL_E_INVALID_ARG; }
  g->nwin = (int)((g->S[0] + kWinOut - 1) / kWinOut);
  g->img_fast = (g->nparts == 1 && pad <= 2) ? 1 : 0;
  for (int d = 0; d < D; ++d)
    if (g->N[d] < 2 * pad) g->img_fast = 0;
  // x = -1 must sit on an even element offset: xo odd, xo >= pad
  g->xo = (pad % 2 == 1) ? pad : pad + 1;
  int64_t need = g->xo + (int64_t)kWinOut * g->nwin + 1;
  if (g->xo + g->S[0] + pad > need) need = g->xo + g->S[0] + pad;
  const int64_t align = 128 / elem;
  g->pitch = (need + align - 1) / align * align;
  g->rstride = (int64_t)g->C * g->pitch;
  g->cstride = layout == 0 ? g->pitch : 1;
  g->xstride = layout == 0 ? 1 : g->C;
  g->buf_elems = g->rstride * g->P[1] * g->P[2];
  return 0;
}

namespace {
struct Seg {
  int64_t s0, s1, t0, t1;
  int mode;
};
}  // namespace

void build_plan(const Geom& g, std::vector<rpl_halo_edge>* out) {
  out->clear();
  const int D = g.D, p = g.pad;
  for (int A = 0; A < g.nparts; ++A) {
    int a[3];
    g.part_coords(A, a);
    std::vector<Seg> segs[3];
    for (int d = 0; d < 3; ++d) {
      if (d >= D) {
        segs[d].push_back({0, 1, 0, 1, RPL_MAP_TRANSLATE});
        continue;
      }
      const int64_t N = g.N[d], lo = a[d] * g.S[d], hi = lo + g.S[d];
      segs[d].push_back({lo, hi, lo, hi, RPL_MAP_TRANSLATE});
      if (a[d] == 0) {
        const int k = g.bc_lo[d];
        if (k == 0) segs[d].push_back({0, 1, -p, 0, RPL_MAP_BROADCAST});
        else if (k == 1) segs[d].push_back({0, p, N, N + p, RPL_MAP_TRANSLATE});
        else segs[d].push_back({0, p, -p, 0, RPL_MAP_REFLECT});
      }
      if (a[d] == g.parts[d] - 1) {
        const int k = g.bc_hi[d];
        if (k == 0) segs[d].push_back({N - 1, N, N, N + p, RPL_MAP_BROADCAST});
        else if (k == 1) segs[d].push_back({N - p, N, -p, 0, RPL_MAP_TRANSLATE});
        else segs[d].push_back({N - p, N, N, N + p, RPL_MAP_REFLECT});
      }
    }
    for (int B = 0; B < g.nparts; ++B) {
      int b[3];
      g.part_coords(B, b);
      for (size_t i0 = 0; i0 < segs[0].size(); ++i0)
        for (size_t i1 = 0; i1 < segs[1].size(); ++i1)
          for (size_t i2 = 0; i2 < segs[2].size(); ++i2) {
            const Seg* sg[3] = {&segs[0][i0], &segs[1][i1], &segs[2][i2]};
            // per dim: pieces of the dst range inside B's padded range
            int64_t pc0[3][3], pc1[3][3];
            bool pin[3][3];
            int np[3] = {0, 0, 0};
            bool empty = false;
            for (int d = 0; d < 3; ++d) {
              if (d >= D) {
                pc0[d][0] = 0; pc1[d][0] = 1; pin[d][0] = true; np[d] = 1;
                continue;
              }
              const int64_t blo = b[d] * g.S[d], bhi = blo + g.S[d];
              const int64_t u0 = sg[d]->t0 > blo - p ? sg[d]->t0 : blo - p;
              const int64_t u1 = sg[d]->t1 < bhi + p ? sg[d]->t1 : bhi + p;
              if (u0 >= u1) { empty = true; break; }
              const int64_t cut[4] = {u0, u0 > blo ? u0 : (u1 < blo ? u1 : blo),
                                      u1 < bhi ? u1 : (u0 > bhi ? u0 : bhi), u1};
              for (int k = 0; k < 3; ++k)
                if (cut[k] < cut[k + 1]) {
                  pc0[d][np[d]] = cut[k];
                  pc1[d][np[d]] = cut[k + 1];
                  pin[d][np[d]] = (k == 1);
                  ++np[d];
                }
            }
            if (empty) continue;
            for (int j0 = 0; j0 < np[0]; ++j0)
              for (int j1 = 0; j1 < np[1]; ++j1)
                for (int j2 = 0; j2 < np[2]; ++j2) {
                  const int jj[3] = {j0, j1, j2};
                  bool all_in = true;
                  for (int d = 0; d < D; ++d) all_in &= pin[d][jj[d]];
                  if (all_in) continue;
                  rpl_halo_edge e;
                  memset(&e, 0, sizeof(e));
                  e.src_part = A;
                  e.dst_part = B;
                  for (int d = 0; d < 3; ++d) {
                    const Seg& s = *sg[d];
                    const int64_t v0 = pc0[d][jj[d]], v1 = pc1[d][jj[d]];
                    e.dst_lo[d] = v0;
                    e.dst_hi[d] = v1;
                    e.mode[d] = s.mode;
                    if (s.mode == RPL_MAP_TRANSLATE) {
                      e.src_lo[d] = v0 - s.t0 + s.s0;
                      e.src_hi[d] = v1 - s.t0 + s.s0;
                    } else if (s.mode == RPL_MAP_REFLECT) {
                      e.src_lo[d] = s.s0 + (s.t1 - v1);
                      e.src_hi[d] = s.s0 + (s.t1 - v0);
                    } else {
                      e.src_lo[d] = s.s0;
                      e.src_hi[d] = s.s0 + 1;
                    }
                  }
                  out->push_back(e);
                }
          }
    }
  }
}

}  // namespace rpl
