// kernels.hpp -- host-side launch entry points of kernels.cu (no torch types).
#pragma once
#include <cuda_runtime.h>

#include "geometry.hpp"

namespace rpl {

template <typename T>
struct KArgs;

// Tile of the fused order-1 step kernels: 30 output cells in x (32-lane windows); in
// y 22 output rows in 2-D (12 warps x 2 rows, 24-row boxes) and 14 in 3-D (8 warps x
// 2 rows, 16-row boxes); in 3-D a chunk of `rows` planes.  Tile t = (tz * ny + ty) * nx
// + tx; tile lists (KArgs::tiles) use this numbering.
constexpr int kTileX = 30, kTileY2 = 22, kTileY3 = 14;

template <typename T>
void launch_sweep(const KArgs<T>& a, int d, cudaStream_t s);      // K-A, one launch
template <typename T>
void launch_step2d(const KArgs<T>& a, const void* tmap, cudaStream_t s);  // K-B 2-D, one launch
template <typename T>
int launch_step3d(const KArgs<T>& a, const void* tmap, cudaStream_t s);  // K-B 3-D, one launch
int make_tmap3d(const Geom& g, const void* buf, void* map_out, int variant);
// 4-D tensor map {pitch, C, P1, P2} of a SoA buffer with box {box_w, C, box_rows, 1}
int make_tmap(const Geom& g, const void* buf, void* map_out, int box_w, int box_rows);
int tmap2d_box(const Geom& g, int variant, int* box_w, int* box_rows);
int tmap2d_box_o2(const Geom& g, int variant, int* box_w, int* box_rows);  // order-2 kernel
template <typename T>  // order 2, 3-D SoA: x/y sweeps of all planes (box {32+AL, C, 16, 1})
void launch_xy3d_o2(const KArgs<T>& a, const void* tmap, cudaStream_t s);
template <typename T>  // order 2, 3-D SoA: the z-sweep as a per-column march
void launch_zmarch2(const KArgs<T>& a, cudaStream_t s);  // 0 if 2-D uses TMA  // 128-byte CUtensorMap
template <typename T>
void launch_fill(const Geom& g, int part, T* const* bufs, cudaStream_t s);
template <typename T>
void launch_maxws(const Geom& g, const T* in, double gamma, unsigned long long* smax,
                  unsigned* flag, cudaStream_t s);

template <typename T>
void launch_fluxdiff(const KArgs<T>& a, cudaStream_t s);  // sec. 7.3 flux difference (f2)
template <typename T>  // tiled 2-D SoA form (TMA box {32+AL, C, fd_tile_rows, 1})
void launch_fluxdiff_tiled(const KArgs<T>& a, const void* tmap, cudaStream_t s);
int fd_tile_rows(int elem, int variant);

int auto_rows_3d(const Geom& g);
const char* step3d_kernel_name(int elem, int variant);  // the 3-D step kernel launch_step3d picks

}  // namespace rpl
