// runtime.cu -- the rpl_* C ABI (include/ripple_fv.h): domain lifetime, state
// transfer, padding fill, the step pipeline, the wavespeed reduction and the
// NCCL halo exchange.  One process per GPU; all device work is enqueued on one
// stream (the caller's, e.g. torch's current stream) in the order of Listing 8
// (P:1340-1358); no host synchronisation inside rpl_advance on one rank.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges cost nothing without a tool attached

#include "../../include/ripple_fv.h"
#include "geometry.hpp"
#include "kernels.hpp"
#include "plan.hpp"
#include "scheme.cuh"

using namespace rpl;

// ------------------------------------------------------------------ errors
static thread_local std::string g_err;

static rpl_status fail(rpl_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

#define CU(call)                                                                        \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return fail(RPL_E_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                                  \
  } while (0)

extern "C" const char* rpl_last_error(void) { return g_err.c_str(); }

// ------------------------------------------------------------------ NCCL (dlopen)
// NVTX range for profilers (Nsight Systems / ncu --nvtx): library calls, steps,
// halo exchanges.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

// NCCL is resolved at run time from the libnccl.so.2 already loaded in the
// process (torch's), else from the loader path: the library has no link-time
// NCCL dependency and single-rank use never touches it.
namespace {
struct Nccl {
  bool tried = false, ok = false;
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclSend) Send = nullptr;
  decltype(&ncclRecv) Recv = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
  decltype(&ncclAllReduce) AllReduce = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
  decltype(&ncclCommInitRankConfig) CommInitRankConfig = nullptr;  // optional (maxCTAs)
  bool load() {
    if (tried) return ok;
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) {
      const char* env = getenv("RPL_NCCL_LIB");
      h = dlopen(env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    }
    if (!h) return false;
#define RPL_SYM(n) n = (decltype(n))dlsym(h, "nccl" #n)
    RPL_SYM(GetUniqueId);
    RPL_SYM(CommInitRank);
    RPL_SYM(CommDestroy);
    RPL_SYM(Send);
    RPL_SYM(Recv);
    RPL_SYM(GroupStart);
    RPL_SYM(GroupEnd);
    RPL_SYM(AllReduce);
    RPL_SYM(GetErrorString);
    RPL_SYM(CommInitRankConfig);
#undef RPL_SYM
    ok = GetUniqueId && CommInitRank && CommDestroy && Send && Recv && GroupStart && GroupEnd &&
         AllReduce && GetErrorString;
    return ok;
  }
} g_nccl;
}  // namespace

#define NC(call)                                                                           \
  do {                                                                                     \
    ncclResult_t r_ = (call);                                                              \
    if (r_ != ncclSuccess)                                                                 \
      return fail(RPL_E_NCCL, "%s failed: %s", #call, g_nccl.GetErrorString(r_));         \
  } while (0)

// ------------------------------------------------------------------ small kernels
namespace {

struct DevEdge {
  int64_t src_lo[3], src_hi[3], dst_lo[3], dst_hi[3];
  int mode[3];
  int src_part, dst_part;
  int64_t count;   // cells in the dst box
  int64_t offset;  // element offset of this edge's message in the peer buffer
};

// pack (dir 0): message[c][i] = source cell of dst-box cell i (flips applied)
// unpack (dir 1): ghost cell i of dst <- message[c][i]
template <typename T, int D, int L>
__global__ void k_edge(const Geom g, const DevEdge e, T* buf, T* msg, int dir) {
  const int64_t ex = e.dst_hi[0] - e.dst_lo[0], ey = e.dst_hi[1] - e.dst_lo[1];
  int pcs[3], pcd[3];
  g.part_coords(e.src_part, pcs);
  g.part_coords(e.dst_part, pcd);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < e.count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t[3] = {e.dst_lo[0] + i % ex, e.dst_lo[1] + (i / ex) % ey,
                          e.dst_lo[2] + i / (ex * ey)};
    T v[D + 2];
    if (dir == 0) {
      int64_t s[3];
      bool flip[3] = {false, false, false};
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const int64_t k = t[d] - e.dst_lo[d];
        s[d] = e.mode[d] == RPL_MAP_TRANSLATE ? e.src_lo[d] + k
               : e.mode[d] == RPL_MAP_REFLECT ? e.src_hi[d] - 1 - k
                                              : e.src_lo[d];
        flip[d] = e.mode[d] == RPL_MAP_REFLECT;
        s[d] -= (d < D) ? (int64_t)pcs[d] * g.S[d] : 0;
      }
#pragma unroll
      for (int c = 0; c < D + 2; ++c) {
        v[c] = buf[g.at(c, s[0], s[1], s[2])];
      }
#pragma unroll
      for (int d = 0; d < D; ++d)
        if (flip[d]) v[1 + d] = -v[1 + d];
#pragma unroll
      for (int c = 0; c < D + 2; ++c) msg[c * e.count + i] = v[c];
    } else {
      int64_t l[3];
#pragma unroll
      for (int d = 0; d < 3; ++d) l[d] = t[d] - ((d < D) ? (int64_t)pcd[d] * g.S[d] : 0);
#pragma unroll
      for (int c = 0; c < D + 2; ++c) v[c] = msg[c * e.count + i];
      store_cell<D, L>(g, buf, l[0], l[1], l[2], v);
    }
  }
}

// All edges of one exchange direction in one launch (blockIdx.y = edge): pack (dir
// 0) reads the source partition's buffer tab[e.src_part], unpack (dir 1) writes
// tab[e.dst_part]; e.offset is the edge's element offset in msg.  Same cell map,
// flips and message layout as k_edge.
template <typename T, int D, int L>
__global__ void k_edges(const Geom g, const DevEdge* __restrict__ edges, T* const* tab, T* msg,
                        int dir) {
  const DevEdge& e = edges[blockIdx.y];
  T* buf = tab[dir == 0 ? e.src_part : e.dst_part];
  T* m = msg + e.offset;
  const int64_t ex = e.dst_hi[0] - e.dst_lo[0], ey = e.dst_hi[1] - e.dst_lo[1];
  int pcs[3], pcd[3];
  g.part_coords(e.src_part, pcs);
  g.part_coords(e.dst_part, pcd);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < e.count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t[3] = {e.dst_lo[0] + i % ex, e.dst_lo[1] + (i / ex) % ey,
                          e.dst_lo[2] + i / (ex * ey)};
    T v[D + 2];
    if (dir == 0) {
      int64_t sc[3];
      bool flip[3] = {false, false, false};
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const int64_t k = t[d] - e.dst_lo[d];
        sc[d] = e.mode[d] == RPL_MAP_TRANSLATE ? e.src_lo[d] + k
                : e.mode[d] == RPL_MAP_REFLECT ? e.src_hi[d] - 1 - k
                                               : e.src_lo[d];
        flip[d] = e.mode[d] == RPL_MAP_REFLECT;
        sc[d] -= (d < D) ? (int64_t)pcs[d] * g.S[d] : 0;
      }
#pragma unroll
      for (int c = 0; c < D + 2; ++c) v[c] = buf[g.at(c, sc[0], sc[1], sc[2])];
#pragma unroll
      for (int d = 0; d < D; ++d)
        if (flip[d]) v[1 + d] = -v[1 + d];
#pragma unroll
      for (int c = 0; c < D + 2; ++c) m[c * e.count + i] = v[c];
    } else {
      int64_t l[3];
#pragma unroll
      for (int d = 0; d < 3; ++d) l[d] = t[d] - ((d < D) ? (int64_t)pcd[d] * g.S[d] : 0);
#pragma unroll
      for (int c = 0; c < D + 2; ++c) v[c] = m[c * e.count + i];
      store_cell<D, L>(g, buf, l[0], l[1], l[2], v);
    }
  }
}

template <typename T>
void launch_edges(const Geom& g, const DevEdge* edges, int nedges, int64_t max_count,
                  T* const* tab, T* msg, int dir, cudaStream_t s) {
  if (nedges <= 0) return;
  int gx = (int)((max_count + 255) / 256);
  const int cap = (148 * 8 + nedges - 1) / nedges;
  if (gx > cap) gx = cap;
  if (gx < 1) gx = 1;
  const dim3 grid(gx, nedges);
#define RPL_E(DD, LL) k_edges<T, DD, LL><<<grid, 256, 0, s>>>(g, edges, tab, msg, dir)
  if (g.D == 1) { if (g.layout == 0) RPL_E(1, 0); else RPL_E(1, 1); }
  if (g.D == 2) { if (g.layout == 0) RPL_E(2, 0); else RPL_E(2, 1); }
  if (g.D == 3) { if (g.layout == 0) RPL_E(3, 0); else RPL_E(3, 1); }
#undef RPL_E
}

// interior <-> dense SoA staging [C][S2][S1][S0] (AoS layout transfers)
template <typename T, int D>
__global__ void k_stage(const Geom g, T* buf, T* stage, int dir) {
  const int64_t n = g.cells();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = i % g.S[0], y = (i / g.S[0]) % g.S[1], z = i / (g.S[0] * g.S[1]);
#pragma unroll
    for (int c = 0; c < D + 2; ++c) {
      const int64_t j = g.at(c, x, y, z);
      if (dir == 0) buf[j] = stage[c * n + i];
      else stage[c * n + i] = buf[j];
    }
  }
}

template <typename T>
void launch_edge(const Geom& g, const DevEdge& e, T* buf, T* msg, int dir, cudaStream_t s) {
  int grid = (int)((e.count + 255) / 256);
  if (grid > 148 * 8) grid = 148 * 8;
  if (grid < 1) grid = 1;
#define RPL_E(DD, LL) k_edge<T, DD, LL><<<grid, 256, 0, s>>>(g, e, buf, msg, dir)
  if (g.D == 1) { if (g.layout == 0) RPL_E(1, 0); else RPL_E(1, 1); }
  if (g.D == 2) { if (g.layout == 0) RPL_E(2, 0); else RPL_E(2, 1); }
  if (g.D == 3) { if (g.layout == 0) RPL_E(3, 0); else RPL_E(3, 1); }
#undef RPL_E
}

template <typename T>
void launch_stage(const Geom& g, T* buf, T* stage, int dir, cudaStream_t s) {
  int grid = (int)((g.cells() + 255) / 256);
  if (grid > 148 * 8) grid = 148 * 8;
  if (g.D == 1) k_stage<T, 1><<<grid, 256, 0, s>>>(g, buf, stage, dir);
  if (g.D == 2) k_stage<T, 2><<<grid, 256, 0, s>>>(g, buf, stage, dir);
  if (g.D == 3) k_stage<T, 3><<<grid, 256, 0, s>>>(g, buf, stage, dir);
}

struct Peer {
  int rank;
  std::vector<DevEdge> edges;  // edges of this peer, in plan order
  int64_t elems = 0;           // message elements
  int64_t offset = 0;          // offset into the send/recv arena
};

}  // namespace

// ------------------------------------------------------------------ the domain
struct rpl_domain {
  rpl_config cfg;
  Geom g;
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  void* arena = nullptr;
  bool own_arena = false;
  std::vector<int> local;              // global partition indices on this rank
  void* buf[2][kMaxParts] = {{nullptr}};
  void** d_tab = nullptr;              // device [2][kMaxParts]
  int cur = 0;                         // buffer holding the current state
  bool ghosts_stale = true;
  unsigned* d_flag = nullptr;
  unsigned long long* d_smax = nullptr;
  unsigned* h_flag = nullptr;          // pinned
  unsigned long long* h_smax = nullptr;
  void* stage = nullptr;               // AoS set/get staging (lazy)
  size_t stage_bytes = 0;
  // multi-rank
  ncclComm_t comm = nullptr;
  std::vector<Peer> send_peers, recv_peers;
  void* d_send = nullptr;
  void* d_recv = nullptr;
  // message exchange (xmode 1: NCCL between ranks; 2: loopback between the local
  // partitions of one rank through the same pack -> transfer -> unpack path, device
  // copies instead of send/recv): flat edge lists with absolute message offsets
  int xmode = 0;
  bool loop_nccl = false;  // loopback through ncclSend/ncclRecv to self (one-rank comm)
  DevEdge* d_sedges = nullptr;
  DevEdge* d_redges = nullptr;
  int n_sedges = 0, n_redges = 0;
  int64_t max_scount = 0, max_rcount = 0, n_selems = 0, n_relems = 0;
  void** d_tab_self = nullptr;  // loopback: [2][kMaxParts] tables holding one partition each
  // shell-first overlap (fused order-1 kernels): per local partition the tiles whose
  // cells are halo sources (shell) then the rest (interior), in d_tiles
  int* d_tiles = nullptr;
  int tile_off[kMaxParts] = {0}, n_shell[kMaxParts] = {0}, n_inter[kMaxParts] = {0};
  cudaStream_t xstream = nullptr;  // side stream of the exchange (high priority)
  cudaEvent_t ev_shell = nullptr, ev_halo = nullptr;
  int rows = 0;
  int variant = 0;
  // 3-D fused kernel: one TMA descriptor per (buffer, local partition)
  struct alignas(64) TMap {
    unsigned char b[128];
  };
  TMap tmap[2][kMaxParts];
  bool tmaps_ok = false;
  TMap tmap_fd[2][kMaxParts];  // tiled flux-difference kernel (lazy)
  bool fd_tmaps = false;
  // P2P transport
  unsigned long long* ctl = nullptr;        // [0,64): step flags from each rank, then 4 sets of
                                            // [64] wavespeed slots (set 0: rpl_max_wavespeed,
                                            // sets 1-3: device CFL, rotated by step)
  int64_t base_off = 0;                     // arena -> 256-aligned buffer base
  bool p2p = false, p2p_attached = false;
  bool p2p_broken = false;                  // a peer missed an epoch (sticky, see check_flag)
  void* peer_arena[kMaxParts] = {nullptr};  // IPC mappings (to close)
  unsigned long long** d_peer_ctl = nullptr;  // device [nranks]: each rank's control block
  unsigned long long epoch = 0;
  unsigned nbr_mask = 0;                    // P2P halo neighbours (bit r = rank r)
  // fault hook (RPL_FAULT_HALO=1, tests only): after every exchange flip one mantissa
  // bit (relative 2^-20) of rho in one ghost cell next to the interior, per local
  // partition that another partition sources -- proves the bitwise partition / rank
  // tests can fail
  int64_t fault_off[kMaxParts];
  bool fault = false;
  // device-side CFL (rpl_advance_to)
  CflDev* d_cfl = nullptr;
  CflDev* h_cfl = nullptr;  // pinned
  // kernel timing (rpl_profile)
  std::vector<cudaEvent_t> ev;  // pairs
  size_t ev_used = 0;
  // halo timing (rpl_profile_halo): (interior done = step kernels done, halo ready =
  // exchange / P2P epoch sync done) pairs, one per exchange, multi-rank only
  std::vector<cudaEvent_t> evh;
  size_t evh_used = 0;
};

static int64_t round_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

// control block after the buffers: P2P step flags [64] and 4 x wavespeed slots [64]
constexpr int64_t kCtlBytes = 5 * kMaxParts * 8;

extern "C" void rpl_config_init(rpl_config* c) {
  memset(c, 0, sizeof(*c));
  c->ndim = 1;
  c->size[0] = c->size[1] = c->size[2] = 1;
  c->pad = 2;
  c->parts[0] = c->parts[1] = c->parts[2] = 1;
  c->dtype = RPL_F64;
  c->layout = RPL_SOA;
  c->kernel = RPL_KERNEL_FUSED;
  c->gamma = 1.4;
  c->dx[0] = c->dx[1] = c->dx[2] = 1.0;
  c->nranks = 1;
  c->order = 1;
}

static rpl_status geom_of(const rpl_config* c, Geom* g) {
  if (!c) return fail(RPL_E_INVALID_ARG, "null config");
  const int bl[3] = {c->bc_lo[0], c->bc_lo[1], c->bc_lo[2]};
  const int bh[3] = {c->bc_hi[0], c->bc_hi[1], c->bc_hi[2]};
  const int pa[3] = {c->parts[0], c->parts[1], c->parts[2]};
  const char* why = "";
  int st = make_geom(c->ndim, c->size, c->pad, pa, c->dtype == RPL_F64 ? 8 : 4, (int)c->layout,
                     bl, bh, g, &why);
  if (st) return fail((rpl_status)st, "%s", why);
  if (!(c->gamma > 1.0)) return fail(RPL_E_INVALID_ARG, "gamma must be > 1");
  for (int d = 0; d < c->ndim; ++d)
    if (!(c->dx[d] > 0.0)) return fail(RPL_E_INVALID_ARG, "dx must be > 0");
  if (c->dtype != RPL_F32 && c->dtype != RPL_F64) return fail(RPL_E_INVALID_ARG, "dtype");
  if (c->kernel != RPL_KERNEL_FUSED && c->kernel != RPL_KERNEL_SPLIT)
    return fail(RPL_E_INVALID_ARG, "kernel");
  if (c->nranks < 1) return fail(RPL_E_INVALID_ARG, "nranks must be >= 1");
  if (c->nranks > 1 && c->nranks != g->nparts)
    return fail(RPL_E_INVALID_ARG, "nranks must be 1 or prod(parts) (one partition per rank)");
  if (c->rank < 0 || c->rank >= c->nranks) return fail(RPL_E_INVALID_ARG, "rank out of range");
  if (c->transport != RPL_TRANSPORT_NCCL && c->transport != RPL_TRANSPORT_P2P &&
      c->transport != RPL_TRANSPORT_LOOPBACK && c->transport != RPL_TRANSPORT_LOOPBACK_NCCL)
    return fail(RPL_E_INVALID_ARG, "transport");
  if ((c->transport == RPL_TRANSPORT_LOOPBACK || c->transport == RPL_TRANSPORT_LOOPBACK_NCCL) &&
      c->nranks != 1)
    return fail(RPL_E_INVALID_ARG, "LOOPBACK transports are for one rank (local partitions)");
  if (c->nranks > 1 && c->transport == RPL_TRANSPORT_NCCL && !c->nccl_id)
    return fail(RPL_E_INVALID_ARG, "nccl_id required");
  if (c->nranks > 32 && c->transport == RPL_TRANSPORT_P2P)
    return fail(RPL_E_INVALID_ARG, "P2P transport supports at most 32 ranks");
  if (c->transport == RPL_TRANSPORT_P2P && c->nranks > 1 && c->arena)
    return fail(RPL_E_INVALID_ARG, "P2P transport needs a library-owned arena (CUDA IPC)");
  if (c->rows_per_chunk < 0) return fail(RPL_E_INVALID_ARG, "rows_per_chunk must be >= 0");
  if (c->order != 1 && c->order != 2) return fail(RPL_E_INVALID_ARG, "order must be 1 or 2");
  if (c->order == 2 && c->pad < 2)
    return fail(RPL_E_PAD_TOO_SMALL, "order 2 (MUSCL-Hancock) needs pad >= 2 (stencil radius 2)");
  return RPL_OK;
}

extern "C" rpl_status rpl_config_check(const rpl_config* c) {
  Geom g;
  return geom_of(c, &g);
}

// + 512 B tail: the fused kernels' 16-byte-aligned bulk row copies may read up to
// 16 B past the last row of a buffer (never used).
static int64_t part_bytes(const Geom& g) { return round_up(g.buf_elems * g.elem + 512, 256); }

extern "C" rpl_status rpl_arena_bytes(const rpl_config* c, size_t* out) {
  Geom g;
  rpl_status st = geom_of(c, &g);
  if (st) return st;
  const int nloc = c->nranks > 1 ? 1 : g.nparts;
  *out = (size_t)(2 * nloc * part_bytes(g) + kCtlBytes + 256);
  return RPL_OK;
}

extern "C" rpl_status rpl_halo_plan(const rpl_config* c, rpl_halo_edge* edges, int32_t max_edges,
                                    int32_t* n_edges) {
  Geom g;
  rpl_status st = geom_of(c, &g);
  if (st) return st;
  std::vector<rpl_halo_edge> v;
  build_plan(g, &v);
  if (n_edges) *n_edges = (int32_t)v.size();
  if (max_edges > 0) {
    if (!edges) return fail(RPL_E_INVALID_ARG, "null edges");
    const int n = (int)v.size() < max_edges ? (int)v.size() : max_edges;
    memcpy(edges, v.data(), sizeof(rpl_halo_edge) * n);
  }
  return RPL_OK;
}

extern "C" rpl_status rpl_nccl_unique_id(void* out128) {
  if (!out128) return fail(RPL_E_INVALID_ARG, "null out");
  if (!g_nccl.load()) return fail(RPL_E_NCCL, "libnccl.so.2 not found (set RPL_NCCL_LIB)");
  ncclUniqueId id;
  NC(g_nccl.GetUniqueId(&id));
  memcpy(out128, &id, sizeof(id));
  return RPL_OK;
}

static void free_events(rpl_domain* d) {
  for (auto e : d->ev) cudaEventDestroy(e);
  for (auto e : d->evh) cudaEventDestroy(e);
  d->ev.clear();
  d->evh.clear();
  d->ev_used = 0;
  d->evh_used = 0;
}

static void free_domain(rpl_domain* d) {
  if (!d) return;
  free_events(d);
  for (int r = 0; r < kMaxParts; ++r)
    if (d->peer_arena[r]) cudaIpcCloseMemHandle(d->peer_arena[r]);
  if (d->d_peer_ctl) cudaFree(d->d_peer_ctl);
  if (d->comm) g_nccl.CommDestroy(d->comm);
  if (d->own_arena && d->arena) cudaFree(d->arena);
  if (d->d_tab) cudaFree(d->d_tab);
  if (d->d_flag) cudaFree(d->d_flag);
  if (d->d_smax) cudaFree(d->d_smax);
  if (d->d_cfl) cudaFree(d->d_cfl);
  if (d->h_cfl) cudaFreeHost(d->h_cfl);
  if (d->h_flag) cudaFreeHost(d->h_flag);
  if (d->h_smax) cudaFreeHost(d->h_smax);
  if (d->stage) cudaFree(d->stage);
  if (d->d_send) cudaFree(d->d_send);
  if (d->d_recv) cudaFree(d->d_recv);
  if (d->d_sedges) cudaFree(d->d_sedges);
  if (d->d_redges && d->d_redges != d->d_sedges) cudaFree(d->d_redges);
  if (d->d_tab_self) cudaFree(d->d_tab_self);
  if (d->d_tiles) cudaFree(d->d_tiles);
  if (d->ev_shell) cudaEventDestroy(d->ev_shell);
  if (d->ev_halo) cudaEventDestroy(d->ev_halo);
  if (d->xstream) cudaStreamDestroy(d->xstream);
  if (d->own_stream && d->stream) cudaStreamDestroy(d->stream);
  delete d;
}


// Message exchange plan (xmode 1: NCCL, 2: loopback): one flat edge list per
// direction, edges grouped per peer (NCCL) in plan order, absolute element offsets
// into the send / recv arenas; and, for the fused order-1 kernels, each local
// partition's tiles split into shell (some cell is a halo source) and interior.
static rpl_status setup_exchange(rpl_domain* d) {
  const Geom& g = d->g;
  const rpl_config* c = &d->cfg;
  std::vector<rpl_halo_edge> plan;
  build_plan(g, &plan);
  auto dev_edge = [&](const rpl_halo_edge& e) {
    DevEdge de;
    memset(&de, 0, sizeof(de));
    for (int k = 0; k < 3; ++k) {
      de.src_lo[k] = e.src_lo[k];
      de.src_hi[k] = e.src_hi[k];
      de.dst_lo[k] = e.dst_lo[k];
      de.dst_hi[k] = e.dst_hi[k];
      de.mode[k] = e.mode[k];
    }
    de.src_part = e.src_part;
    de.dst_part = e.dst_part;
    de.count = (e.dst_hi[0] - e.dst_lo[0]) * (e.dst_hi[1] - e.dst_lo[1]) *
               (e.dst_hi[2] - e.dst_lo[2]);
    return de;
  };
  std::vector<DevEdge> se, re;
  if (d->xmode == 1) {
    const int me = c->rank;
    auto add = [&](std::vector<Peer>& peers, int peer, const rpl_halo_edge& e) {
      Peer* P = nullptr;
      for (auto& q : peers)
        if (q.rank == peer) P = &q;
      if (!P) {
        peers.push_back(Peer());
        P = &peers.back();
        P->rank = peer;
      }
      DevEdge de = dev_edge(e);
      de.offset = P->elems;
      P->elems += de.count * g.C;
      P->edges.push_back(de);
    };
    for (const auto& e : plan) {
      if (e.src_part == me && e.dst_part != me) add(d->send_peers, e.dst_part, e);
      if (e.dst_part == me && e.src_part != me) add(d->recv_peers, e.src_part, e);
    }
    int64_t ns = 0, nr = 0;
    for (auto& P : d->send_peers) {
      P.offset = ns;
      ns += P.elems;
      for (auto e : P.edges) { e.offset += P.offset; se.push_back(e); }
    }
    for (auto& P : d->recv_peers) {
      P.offset = nr;
      nr += P.elems;
      for (auto e : P.edges) { e.offset += P.offset; re.push_back(e); }
    }
    d->n_selems = ns;
    d->n_relems = nr;
  } else {
    int64_t off = 0;  // loopback: one message list, packed and unpacked in place order
    for (const auto& e : plan)
      if (e.src_part != e.dst_part) {
        DevEdge de = dev_edge(e);
        de.offset = off;
        off += de.count * g.C;
        se.push_back(de);
      }
    re = se;
    d->n_selems = d->n_relems = off;
    // step kernels write ghost images into their own partition only: the other
    // partitions' halos travel through the messages
    std::vector<void*> tabs(2 * (size_t)kMaxParts * kMaxParts, nullptr);
    for (int b = 0; b < 2; ++b)
      for (int p : d->local) tabs[((size_t)b * kMaxParts + p) * kMaxParts + p] = d->buf[b][p];
    CU(cudaMalloc(&d->d_tab_self, sizeof(void*) * tabs.size()));
    CU(cudaMemcpy(d->d_tab_self, tabs.data(), sizeof(void*) * tabs.size(),
                  cudaMemcpyHostToDevice));
  }
  for (const auto& e : se) d->max_scount = std::max(d->max_scount, e.count);
  for (const auto& e : re) d->max_rcount = std::max(d->max_rcount, e.count);
  d->n_sedges = (int)se.size();
  d->n_redges = (int)re.size();
  if (d->n_selems) CU(cudaMalloc(&d->d_send, d->n_selems * g.elem));
  if (d->n_relems) CU(cudaMalloc(&d->d_recv, d->n_relems * g.elem));
  if (!se.empty()) {
    CU(cudaMalloc(&d->d_sedges, sizeof(DevEdge) * se.size()));
    CU(cudaMemcpy(d->d_sedges, se.data(), sizeof(DevEdge) * se.size(), cudaMemcpyHostToDevice));
  }
  if (d->xmode == 2) {
    d->d_redges = d->d_sedges;
  } else if (!re.empty()) {
    CU(cudaMalloc(&d->d_redges, sizeof(DevEdge) * re.size()));
    CU(cudaMemcpy(d->d_redges, re.data(), sizeof(DevEdge) * re.size(), cudaMemcpyHostToDevice));
  }
  int lo_prio = 0, hi_prio = 0;
  CU(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
  CU(cudaStreamCreateWithPriority(&d->xstream, cudaStreamNonBlocking, hi_prio));
  CU(cudaEventCreateWithFlags(&d->ev_shell, cudaEventDisableTiming));
  CU(cudaEventCreateWithFlags(&d->ev_halo, cudaEventDisableTiming));
  // shell / interior tiles of the fused order-1 kernels (2-D SoA, 3-D)
  if (g.D >= 2 && c->order == 1 && (g.D == 3 || g.layout == 0)) {
    const int64_t wx = kTileX, wy = g.D == 3 ? kTileY3 : kTileY2, wz = g.D == 3 ? d->rows : 1;
    const int64_t nx = (g.S[0] + wx - 1) / wx, ny = (g.S[1] + wy - 1) / wy,
                  nz = g.D == 3 ? (g.S[2] + wz - 1) / wz : 1;
    std::vector<int> all;
    for (int p : d->local) {
      int pc[3];
      g.part_coords(p, pc);
      std::vector<char> shell((size_t)(nx * ny * nz), 0);
      for (const auto& e : se) {
        if (e.src_part != p) continue;
        int64_t lo[3], hi[3];  // local source box (all pad layers the plan sends)
        for (int k = 0; k < 3; ++k) {
          const int64_t o = k < g.D ? (int64_t)pc[k] * g.S[k] : 0;
          lo[k] = e.src_lo[k] - o;
          hi[k] = e.src_hi[k] - o;
        }
        for (int64_t tz = 0; tz < nz; ++tz)
          for (int64_t ty = 0; ty < ny; ++ty)
            for (int64_t tx = 0; tx < nx; ++tx) {
              const int64_t a0[3] = {tx * wx, ty * wy, tz * wz};
              const int64_t a1[3] = {a0[0] + wx, a0[1] + wy, g.D == 3 ? a0[2] + wz : 1};
              bool hit = true;
              for (int k = 0; k < 3; ++k) hit &= a0[k] < hi[k] && lo[k] < a1[k];
              if (hit) shell[(size_t)((tz * ny + ty) * nx + tx)] = 1;
            }
      }
      d->tile_off[p] = (int)all.size();
      for (int64_t t = 0; t < nx * ny * nz; ++t)
        if (shell[(size_t)t]) all.push_back((int)t);
      d->n_shell[p] = (int)all.size() - d->tile_off[p];
      for (int64_t t = 0; t < nx * ny * nz; ++t)
        if (!shell[(size_t)t]) all.push_back((int)t);
      d->n_inter[p] = (int)all.size() - d->tile_off[p] - d->n_shell[p];
    }
    CU(cudaMalloc(&d->d_tiles, sizeof(int) * std::max<size_t>(all.size(), 1)));
    if (!all.empty())
      CU(cudaMemcpy(d->d_tiles, all.data(), sizeof(int) * all.size(), cudaMemcpyHostToDevice));
  }
  return RPL_OK;
}

static rpl_status create_impl(const rpl_config* c, rpl_domain* d) {
  d->cfg = *c;
  rpl_status st = geom_of(c, &d->g);
  if (st) return st;
  const Geom& g = d->g;
  d->device = c->device;
  CU(cudaSetDevice(d->device));
  if (c->stream) {
    d->stream = (cudaStream_t)c->stream;
  } else {
    CU(cudaStreamCreateWithFlags(&d->stream, cudaStreamNonBlocking));
    d->own_stream = true;
  }
  if (c->nranks > 1) d->local.push_back(c->rank);
  else
    for (int p = 0; p < g.nparts; ++p) d->local.push_back(p);
  size_t bytes = 0;
  st = rpl_arena_bytes(c, &bytes);
  if (st) return st;
  if (c->arena) {
    d->arena = c->arena;
  } else {
    cudaError_t e = cudaMalloc(&d->arena, bytes);
    if (e != cudaSuccess) return fail(RPL_E_OOM, "cudaMalloc(%zu): %s", bytes, cudaGetErrorString(e));
    d->own_arena = true;
  }
  char* base = (char*)round_up((int64_t)(uintptr_t)d->arena, 256);
  const int64_t pb = part_bytes(g);
  for (size_t i = 0; i < d->local.size(); ++i)
    for (int b = 0; b < 2; ++b) d->buf[b][d->local[i]] = base + (2 * i + b) * pb;
  CU(cudaMemsetAsync(base, 0, 2 * d->local.size() * pb + kCtlBytes, d->stream));
  d->ctl = reinterpret_cast<unsigned long long*>(base + 2 * d->local.size() * pb);
  d->base_off = base - (char*)d->arena;
  CU(cudaMalloc(&d->d_tab, sizeof(void*) * 2 * kMaxParts));
  CU(cudaMemcpy(d->d_tab, d->buf, sizeof(void*) * 2 * kMaxParts, cudaMemcpyHostToDevice));
  CU(cudaMalloc(&d->d_flag, sizeof(unsigned)));
  CU(cudaMalloc(&d->d_smax, sizeof(unsigned long long)));
  CU(cudaMemsetAsync(d->d_flag, 0, sizeof(unsigned), d->stream));
  CU(cudaMallocHost(&d->h_flag, sizeof(unsigned)));
  CU(cudaMallocHost(&d->h_smax, sizeof(unsigned long long)));
  CU(cudaMalloc(&d->d_cfl, sizeof(CflDev)));
  CU(cudaMallocHost(&d->h_cfl, sizeof(CflDev)));
  if (const char* v = getenv("RPL_VARIANT")) d->variant = atoi(v);
  if (g.D == 3) {  // SoA and AoS
    d->tmaps_ok = true;
    for (int p : d->local)
      for (int b = 0; b < 2; ++b) {
        // order 2 (SoA): the x/y-plane kernel's box {32+AL, C, 16, 1}
        const int r = (c->order == 2 && g.layout == 0)
                          ? make_tmap(g, d->buf[b][p], d->tmap[b][p].b, 32 + 16 / g.elem, 16)
                          : make_tmap3d(g, d->buf[b][p], d->tmap[b][p].b, d->variant);
        if (r != 0) d->tmaps_ok = false;
      }
    if (!d->tmaps_ok && c->kernel == RPL_KERNEL_FUSED)
      return fail(RPL_E_CUDA, "cuTensorMapEncodeTiled failed for the 3-D fused kernel");
  }
  {
    int bw = 0, br = 0;
    const bool box = c->order == 2 ? tmap2d_box_o2(g, d->variant, &bw, &br)
                                   : tmap2d_box(g, d->variant, &bw, &br);
    if (g.D == 2 && g.layout == 0 && box) {  // every 2-D fused kernel is TMA-fed
      for (int p : d->local)
        for (int b = 0; b < 2; ++b)
          if (make_tmap(g, d->buf[b][p], d->tmap[b][p].b, bw, br) != 0)
            return fail(RPL_E_CUDA, "cuTensorMapEncodeTiled failed for the 2-D fused kernel");
    }
  }
  d->rows = c->rows_per_chunk;
  // 0 = each fused launcher picks its own chunking (2-D); 3-D z-chunk planes:
  if (d->rows <= 0 && g.D == 3) d->rows = auto_rows_3d(g);
  d->p2p = c->nranks > 1 && c->transport == RPL_TRANSPORT_P2P;
  if (d->p2p) {
    CU(cudaMalloc(&d->d_peer_ctl, sizeof(void*) * kMaxParts));
    // halo neighbours: ranks whose partitions source a ghost of ours or take one of
    // ours as a ghost source (one partition per rank; symmetric by construction, the
    // same global plan on every rank) -- the only ranks a halo epoch waits on
    std::vector<rpl_halo_edge> plan;
    build_plan(g, &plan);
    for (const auto& e : plan) {
      if (e.src_part == c->rank && e.dst_part != c->rank) d->nbr_mask |= 1u << e.dst_part;
      if (e.dst_part == c->rank && e.src_part != c->rank) d->nbr_mask |= 1u << e.src_part;
    }
  }
  for (int p = 0; p < kMaxParts; ++p) d->fault_off[p] = -1;
  if (const char* f = getenv("RPL_FAULT_HALO")) {
    if (f[0] == '1') {
      std::vector<rpl_halo_edge> plan;
      build_plan(g, &plan);
      for (const auto& e : plan) {
        const int p = e.dst_part;
        if (e.src_part == p || d->fault_off[p] >= 0 || !d->buf[0][p]) continue;
        int pc[3];
        g.part_coords(p, pc);
        // a face edge (one dim outside the partition): its ghost layer next to the
        // interior, mid-face in the other dims -- a cell the next step reads
        int64_t q[3];
        int outside = 0;
        for (int k = 0; k < 3; ++k) {
          const int64_t o = k < g.D ? (int64_t)pc[k] * g.S[k] : 0;
          const int64_t lo = e.dst_lo[k] - o, hi = e.dst_hi[k] - o;
          if (k < g.D && hi <= 0) {
            q[k] = -1;
            ++outside;
          } else if (k < g.D && lo >= g.S[k]) {
            q[k] = g.S[k];
            ++outside;
          } else {
            q[k] = (lo + hi - 1) / 2;
          }
        }
        if (outside != 1) continue;
        d->fault_off[p] = g.at(0, q[0], q[1], q[2]);  // rho of that ghost
        d->fault = true;
      }
    }
  }
  const bool loop = c->transport == RPL_TRANSPORT_LOOPBACK ||
                    c->transport == RPL_TRANSPORT_LOOPBACK_NCCL;
  d->xmode = (c->nranks > 1 && !d->p2p) ? 1 : (c->nranks == 1 && loop && g.nparts > 1) ? 2 : 0;
  d->loop_nccl = d->xmode == 2 && c->transport == RPL_TRANSPORT_LOOPBACK_NCCL;
  if (d->xmode == 1 || d->loop_nccl) {
    if (!g_nccl.load()) return fail(RPL_E_NCCL, "libnccl.so.2 not found (set RPL_NCCL_LIB)");
    ncclUniqueId id;
    if (d->loop_nccl) NC(g_nccl.GetUniqueId(&id));  // one-rank communicator of our own
    else memcpy(&id, c->nccl_id, sizeof(id));
    const int nr = d->loop_nccl ? 1 : c->nranks, me = d->loop_nccl ? 0 : c->rank;
    if (g_nccl.CommInitRankConfig) {
      // cap NCCL's CTAs: the interior step kernel keeps the SMs while halos move
      ncclConfig_t cc = NCCL_CONFIG_INITIALIZER;
      const char* m = getenv("RPL_NCCL_MAX_CTAS");
      cc.maxCTAs = m ? atoi(m) : 8;
      NC(g_nccl.CommInitRankConfig(&d->comm, nr, id, me, &cc));
    } else {
      NC(g_nccl.CommInitRank(&d->comm, nr, id, me));
    }
  }
  if (d->xmode) {
    rpl_status st = setup_exchange(d);
    if (st) return st;
  }
  CU(cudaStreamSynchronize(d->stream));
  return RPL_OK;
}

extern "C" rpl_status rpl_create(const rpl_config* c, rpl_domain** out) {
  if (!out) return fail(RPL_E_INVALID_ARG, "null out");
  *out = nullptr;
  rpl_domain* d = new rpl_domain();
  rpl_status st = create_impl(c, d);
  if (st != RPL_OK) {
    std::string keep = g_err;
    free_domain(d);
    g_err = keep;
    return st;
  }
  *out = d;
  return RPL_OK;
}

extern "C" void rpl_destroy(rpl_domain* d) {
  if (!d) return;
  cudaSetDevice(d->device);
  cudaStreamSynchronize(d->stream);
  free_domain(d);
}

extern "C" rpl_status rpl_local_box(const rpl_domain* d, int64_t lo[3], int64_t hi[3]) {
  if (!d || !lo || !hi) return fail(RPL_E_INVALID_ARG, "null argument");
  const Geom& g = d->g;
  if (d->cfg.nranks > 1) {
    int pc[3];
    g.part_coords(d->cfg.rank, pc);
    for (int k = 0; k < 3; ++k) {
      lo[k] = pc[k] * g.S[k];
      hi[k] = lo[k] + g.S[k];
    }
  } else {
    for (int k = 0; k < 3; ++k) {
      lo[k] = 0;
      hi[k] = g.N[k];
    }
  }
  return RPL_OK;
}

// host box <-> partition interior copies (dense SoA host [C][bz][by][bx])
static rpl_status xfer(rpl_domain* d, void* host, bool to_dev, int which = -1) {
  const Geom& g = d->g;
  int64_t lo[3], hi[3];
  rpl_local_box(d, lo, hi);
  const int64_t bx = hi[0] - lo[0], by = hi[1] - lo[1], bz = hi[2] - lo[2];
  const size_t el = g.elem;
  for (int p : d->local) {
    int pc[3];
    g.part_coords(p, pc);
    const int64_t o[3] = {pc[0] * g.S[0] - lo[0], pc[1] * g.S[1] - lo[1], pc[2] * g.S[2] - lo[2]};
    char* dev = (char*)d->buf[which < 0 ? d->cur : which][p];
    if (g.layout == 0) {
      for (int c = 0; c < g.C; ++c) {
        cudaMemcpy3DParms m;
        memset(&m, 0, sizeof(m));
        cudaPitchedPtr hp = make_cudaPitchedPtr((char*)host + (size_t)c * bx * by * bz * el,
                                                bx * el, bx * el, by);
        cudaPitchedPtr dp = make_cudaPitchedPtr(dev + (size_t)c * g.cstride * el, g.rstride * el,
                                                g.pitch * el, g.P[1]);
        const cudaPos hpos = make_cudaPos(o[0] * el, o[1], o[2]);
        const cudaPos dpos = make_cudaPos(g.xo * el, g.off[1], g.off[2]);
        if (to_dev) {
          m.srcPtr = hp; m.srcPos = hpos; m.dstPtr = dp; m.dstPos = dpos;
          m.kind = cudaMemcpyHostToDevice;
        } else {
          m.srcPtr = dp; m.srcPos = dpos; m.dstPtr = hp; m.dstPos = hpos;
          m.kind = cudaMemcpyDeviceToHost;
        }
        m.extent = make_cudaExtent(g.S[0] * el, g.S[1], g.S[2]);
        CU(cudaMemcpy3DAsync(&m, d->stream));
      }
    } else {
      const size_t need = (size_t)g.C * g.cells() * el;
      if (d->stage_bytes < need) {
        CU(cudaStreamSynchronize(d->stream));
        if (d->stage) cudaFree(d->stage);
        d->stage = nullptr;
        d->stage_bytes = 0;
        CU(cudaMalloc(&d->stage, need));
        d->stage_bytes = need;
      }
      for (int c = 0; c < g.C; ++c) {
        cudaMemcpy3DParms m;
        memset(&m, 0, sizeof(m));
        cudaPitchedPtr hp = make_cudaPitchedPtr((char*)host + (size_t)c * bx * by * bz * el,
                                                bx * el, bx * el, by);
        cudaPitchedPtr sp = make_cudaPitchedPtr((char*)d->stage + (size_t)c * g.cells() * el,
                                                g.S[0] * el, g.S[0] * el, g.S[1]);
        const cudaPos hpos = make_cudaPos(o[0] * el, o[1], o[2]);
        if (to_dev) {
          m.srcPtr = hp; m.srcPos = hpos; m.dstPtr = sp; m.kind = cudaMemcpyHostToDevice;
        } else {
          m.srcPtr = sp; m.dstPtr = hp; m.dstPos = hpos; m.kind = cudaMemcpyDeviceToHost;
        }
        m.extent = make_cudaExtent(g.S[0] * el, g.S[1], g.S[2]);
        if (to_dev) {
          CU(cudaMemcpy3DAsync(&m, d->stream));
        }
        if (!to_dev && c == 0) {
          if (el == 8) launch_stage<double>(g, (double*)dev, (double*)d->stage, 1, d->stream);
          else launch_stage<float>(g, (float*)dev, (float*)d->stage, 1, d->stream);
          CU(cudaGetLastError());
        }
        if (!to_dev) CU(cudaMemcpy3DAsync(&m, d->stream));
      }
      if (to_dev) {
        if (el == 8) launch_stage<double>(g, (double*)dev, (double*)d->stage, 0, d->stream);
        else launch_stage<float>(g, (float*)dev, (float*)d->stage, 0, d->stream);
        CU(cudaGetLastError());
      }
    }
  }
  return RPL_OK;
}

static rpl_status check_flag(rpl_domain* d) {
  CU(cudaMemcpyAsync(d->h_flag, d->d_flag, sizeof(unsigned), cudaMemcpyDeviceToHost, d->stream));
  CU(cudaStreamSynchronize(d->stream));
  if (*d->h_flag & 2u) d->p2p_broken = true;  // the epoch protocol cannot recover
  if (d->p2p_broken)
    return fail(RPL_E_CUDA, "P2P transport: a peer rank did not reach the step epoch within "
                            "RPL_P2P_TIMEOUT_S (default 120 s)");
  if (*d->h_flag)
    return fail(RPL_E_DOMAIN, "numerical-domain error: rho<=0, p<=0 or non-finite state (S:588)");
  return RPL_OK;
}

extern "C" rpl_status rpl_set_state(rpl_domain* d, const void* host) {
  NvtxRange nvtx_("rpl_set_state");
  if (!d || !host) return fail(RPL_E_INVALID_ARG, "null argument");
  CU(cudaSetDevice(d->device));
  rpl_status st = xfer(d, (void*)host, true);
  if (st) return st;
  // a new state clears the domain-error bit (bit 0); a P2P timeout (bit 1) is sticky
  // for the domain's lifetime (p2p_broken), so it is read before the flag is reset
  CU(cudaMemcpyAsync(d->h_flag, d->d_flag, sizeof(unsigned), cudaMemcpyDeviceToHost, d->stream));
  CU(cudaStreamSynchronize(d->stream));
  if (*d->h_flag & 2u) d->p2p_broken = true;
  CU(cudaMemsetAsync(d->d_flag, 0, sizeof(unsigned), d->stream));
  CU(cudaStreamSynchronize(d->stream));
  d->ghosts_stale = true;
  if (d->p2p_broken)
    return fail(RPL_E_CUDA, "P2P transport: an earlier step epoch timed out (RPL_P2P_TIMEOUT_S)");
  return RPL_OK;
}

extern "C" rpl_status rpl_get_state(rpl_domain* d, void* host) {
  NvtxRange nvtx_("rpl_get_state");
  if (!d || !host) return fail(RPL_E_INVALID_ARG, "null argument");
  CU(cudaSetDevice(d->device));
  rpl_status st = xfer(d, host, false);
  if (st) return st;
  CU(cudaStreamSynchronize(d->stream));
  return check_flag(d);
}

extern "C" rpl_status rpl_get_padded(rpl_domain* d, int32_t part, void* host) {
  if (!d || !host) return fail(RPL_E_INVALID_ARG, "null argument");
  const Geom& g = d->g;
  if (part < 0 || part >= g.nparts || !d->buf[d->cur][part])
    return fail(RPL_E_INVALID_ARG, "partition %d is not on this rank", part);
  CU(cudaSetDevice(d->device));
  std::vector<char> raw((size_t)g.buf_elems * g.elem);
  CU(cudaMemcpyAsync(raw.data(), d->buf[d->cur][part], raw.size(), cudaMemcpyDeviceToHost,
                     d->stream));
  CU(cudaStreamSynchronize(d->stream));
  const int64_t n = g.P[0] * g.P[1] * g.P[2];
  for (int64_t i = 0; i < n; ++i) {
    const int64_t x = i % g.P[0] - g.off[0], y = (i / g.P[0]) % g.P[1] - g.off[1],
                  z = i / (g.P[0] * g.P[1]) - g.off[2];
    for (int c = 0; c < g.C; ++c)
      memcpy((char*)host + ((size_t)c * n + i) * g.elem,
             raw.data() + (size_t)g.at(c, x, y, z) * g.elem, g.elem);
  }
  return RPL_OK;
}

// Halo messages of buffer b on stream st: pack every send edge (one kernel) ->
// grouped ncclSend/ncclRecv (xmode 1) or one device copy (loopback) -> unpack every
// receive edge (one kernel).
template <typename T>
static rpl_status exchange_t(rpl_domain* d, int b, cudaStream_t st) {
  const Geom& g = d->g;
  T* const* tab = (T* const*)(d->d_tab + b * kMaxParts);
  launch_edges<T>(g, d->d_sedges, d->n_sedges, d->max_scount, tab, (T*)d->d_send, 0, st);
  CU(cudaGetLastError());
  if (d->xmode == 1) {
    const ncclDataType_t ty = g.elem == 8 ? ncclFloat64 : ncclFloat32;
    NC(g_nccl.GroupStart());
    for (auto& P : d->send_peers)
      NC(g_nccl.Send((T*)d->d_send + P.offset, P.elems, ty, P.rank, d->comm, st));
    for (auto& P : d->recv_peers)
      NC(g_nccl.Recv((T*)d->d_recv + P.offset, P.elems, ty, P.rank, d->comm, st));
    NC(g_nccl.GroupEnd());
  } else if (d->loop_nccl && d->n_selems) {
    // the same grouped calls, to ourselves on the one-rank communicator
    const ncclDataType_t ty = g.elem == 8 ? ncclFloat64 : ncclFloat32;
    NC(g_nccl.GroupStart());
    NC(g_nccl.Send((T*)d->d_send, d->n_selems, ty, 0, d->comm, st));
    NC(g_nccl.Recv((T*)d->d_recv, d->n_relems, ty, 0, d->comm, st));
    NC(g_nccl.GroupEnd());
  } else if (d->n_selems) {
    CU(cudaMemcpyAsync(d->d_recv, d->d_send, d->n_selems * g.elem, cudaMemcpyDeviceToDevice, st));
  }
  launch_edges<T>(g, d->d_redges, d->n_redges, d->max_rcount, tab, (T*)d->d_recv, 1, st);
  CU(cudaGetLastError());
  return RPL_OK;
}

// P2P: one warp publishes "rank `me` finished epoch e" into the control block of
// every peer it synchronises with (system-scope release after a system fence, so
// the step kernel's peer stores are visible first) and waits until each of them
// published e (acquire).  Mode 0 (halo epoch after a step) involves only the halo
// neighbours (`peers`, from the halo plan): they are the only ranks whose stores
// land in our buffers and the only ones whose buffers we store into, so "all
// neighbours finished step n" is all step n+1 needs -- a rank may run ahead of a
// non-neighbour by its graph distance, never of a neighbour.  Mode 1 (wavespeed max)
// involves every rank: it also publishes the local wavespeed max *smax into slot
// `me` of the peers' slot set `set` and, after the wait, reduces its own set into
// *smax (exact: max).  Sets rotate with the step (device CFL, one mode-1 sync per
// step): a rank is at most one epoch ahead of any peer, so a set is never rewritten
// before it was read.
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Bounded wait: a peer that never reaches this epoch (crashed or hung process)
// sets bit 1 of the sticky flag after timeout_ns instead of spinning forever;
// the next synchronising call reports it (RPL_E_CUDA).
__global__ void k_p2p_sync(unsigned long long* const* ctl, int me, int nranks,
                           unsigned long long epoch, unsigned long long* smax, int set, int mode,
                           unsigned* flag, unsigned long long timeout_ns, unsigned peers) {
  const int r = threadIdx.x;
  unsigned long long* mine = ctl[me];
  const int so = kMaxParts * (1 + set);
  // mode 0 (halo epoch): the halo neighbours only; mode 1 (wavespeed max): every rank
  if (r < nranks && r != me && (mode == 1 || ((peers >> r) & 1u))) {
    unsigned long long* peer = ctl[r];
    if (mode == 1) {
      const unsigned long long v = *smax;
      asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(peer + so + me), "l"(v)
                   : "memory");
    }
    __threadfence_system();
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(peer + me), "l"(epoch) : "memory");
    unsigned long long got = 0;
    const unsigned long long t0 = globaltimer_ns();
    do {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(got) : "l"(mine + r) : "memory");
      if (got < epoch) {
        __nanosleep(64);
        if (globaltimer_ns() - t0 > timeout_ns) {
          atomicOr(flag, 2u);
          break;
        }
      }
    } while (got < epoch);
  }
  __syncwarp();
  if (mode == 1 && r == 0) {
    unsigned long long m = *smax;
    for (int q = 0; q < nranks; ++q)
      if (q != me) {
        unsigned long long v;
        asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(mine + so + q)
                     : "memory");
        m = v > m ? v : m;
      }
    *smax = m;
  }
}

static rpl_status p2p_sync(rpl_domain* d, int mode, unsigned long long* smax = nullptr,
                           int set = 0) {
  if (!d->p2p_attached) return fail(RPL_E_INVALID_ARG, "P2P transport: call rpl_p2p_attach first");
  if (d->p2p_broken)
    return fail(RPL_E_CUDA, "P2P transport: an earlier step epoch timed out (RPL_P2P_TIMEOUT_S)");
  ++d->epoch;
  static const unsigned long long timeout_ns = [] {
    const char* e = getenv("RPL_P2P_TIMEOUT_S");
    const double sec = e ? atof(e) : 120.0;
    return (unsigned long long)((sec > 0 ? sec : 120.0) * 1e9);
  }();
  k_p2p_sync<<<1, 32, 0, d->stream>>>(d->d_peer_ctl, d->cfg.rank, d->cfg.nranks, d->epoch,
                                      smax ? smax : d->d_smax, set, mode, d->d_flag, timeout_ns,
                                      d->nbr_mask);
  CU(cudaGetLastError());
  return RPL_OK;
}

// Combine the ranks' wavespeed slot (max) on the stream; no-op for one rank.
static rpl_status reduce_max(rpl_domain* d, unsigned long long* slot, int set) {
  if (d->cfg.nranks <= 1) return RPL_OK;
  if (d->p2p) return p2p_sync(d, 1, slot, set);
  NC(g_nccl.AllReduce(slot, slot, 1, ncclUint64, ncclMax, d->comm, d->stream));
  return RPL_OK;
}

// flip mantissa bit 20 from the top (relative change 2^-20 -- a 1-ulp flip can be
// absorbed by rounding where the flux does not depend on rho, e.g. at rest)
__global__ void k_fault_flip(unsigned char* p, int elem) {
  if (elem == 8) p[4] ^= 1u;   // bit 32 of the double
  else p[0] ^= 8u;             // bit 3 of the float
}

static void inject_fault(rpl_domain* d, int b) {
  for (int p : d->local)
    if (d->fault_off[p] >= 0)
      k_fault_flip<<<1, 1, 0, d->stream>>>((unsigned char*)d->buf[b][p] +
                                           d->fault_off[p] * d->g.elem, d->g.elem);
}

static rpl_status exchange(rpl_domain* d, int b) {
  NvtxRange nvtx_("halo exchange");
  if (d->p2p) return p2p_sync(d, 0);  // halos were stored by the step kernel itself
  if (!d->xmode) return RPL_OK;       // one partition, or partitions writing each other's ghosts
  return d->g.elem == 8 ? exchange_t<double>(d, b, d->stream) : exchange_t<float>(d, b, d->stream);
}

template <typename T>
static rpl_status fill_t(rpl_domain* d) {
  if (d->p2p) {  // peers' states must be set before k_fill reads their interiors
    rpl_status st = p2p_sync(d, 0);
    if (st) return st;
  }
  T* const* tab = (T* const*)(d->d_tab + d->cur * kMaxParts);
  for (int p : d->local) launch_fill<T>(d->g, p, tab, d->stream);
  CU(cudaGetLastError());
  // P2P / one rank (loopback included): k_fill read the sources' interiors directly
  if (d->p2p || d->cfg.nranks == 1) return RPL_OK;
  return exchange(d, d->cur);
}

extern "C" rpl_status rpl_fill_padding(rpl_domain* d) {
  NvtxRange nvtx_("rpl_fill_padding");
  if (!d) return fail(RPL_E_INVALID_ARG, "null domain");
  CU(cudaSetDevice(d->device));
  rpl_status st = d->g.elem == 8 ? fill_t<double>(d) : fill_t<float>(d);
  if (st) return st;
  d->ghosts_stale = false;
  return RPL_OK;
}

static bool use_fused(const rpl_domain* d) {
  if (d->cfg.order == 2)  // order 2: fused 2-D / fused x-y + z pass in 3-D (SoA); AoS splits
    return d->cfg.kernel == RPL_KERNEL_FUSED && d->g.layout == 0 &&
           (d->g.D == 2 || (d->g.D == 3 && d->tmaps_ok));
  return d->cfg.kernel == RPL_KERNEL_FUSED &&
         ((d->g.D == 2 && d->g.layout == 0) || (d->g.D == 3 && d->tmaps_ok));
}

// shell-first overlap of the message exchange (NCCL / loopback) with the interior
// tiles: fused order-1 kernels with tile lists, fixed dt (the device-CFL step
// combines the wavespeed after the whole step)
static bool overlapped(const rpl_domain* d) {
  return d->xmode && d->d_tiles && use_fused(d) && d->cfg.order == 1;
}

// kernel passes per step: fused = 1 (3-D order 2: x-y pass + z pass), split = D
static int passes(const rpl_domain* d) {
  if (!use_fused(d)) return d->g.D;
  return (d->g.D == 3 && d->cfg.order == 2) ? 2 : 1;
}

extern "C" rpl_status rpl_launches_per_step(const rpl_domain* d, int32_t* out) {
  if (!d || !out) return fail(RPL_E_INVALID_ARG, "null argument");
  int n = (int)d->local.size() * passes(d);
  if (d->xmode) {
    n += ((d->n_sedges > 0) + (d->n_redges > 0)) * passes(d);  // pack + unpack kernels
    if (overlapped(d))  // shell and interior launches of the step kernel
      for (int p : d->local) n += (d->n_shell[p] > 0 && d->n_inter[p] > 0) ? 1 : 0;
  }
  if (d->p2p) n += passes(d);  // one flag kernel per exchange
  *out = n;
  return RPL_OK;
}

// Enqueue nsteps steps.  cf == nullptr: fixed dt.  Otherwise device-side CFL
// steps cf->step .. cf->step + nsteps - 1 (dt derived on the device, see
// scheme.cuh step_coef); after each step the ranks' wavespeed slot is combined.
template <typename T>
static rpl_status advance_t(rpl_domain* d, double dt, int nsteps, const CflArgs* cf = nullptr) {
  const Geom& g = d->g;
  KArgs<T> a;
  memset(&a, 0, sizeof(a));
  a.g = g;
  for (int k = 0; k < 3; ++k) {
    const double lam = k < g.D ? dt / d->cfg.dx[k] : 0.0;
    a.lam[k] = (T)lam;
    a.h2[k] = (T)(0.5 * lam);
  }
  a.gm1 = (T)(d->cfg.gamma - 1.0);
  a.flag = d->d_flag;
  a.rows = d->rows;
  a.variant = d->variant;
  a.order = d->cfg.order;
  if (cf) a.cf = *cf;
  const bool fused = use_fused(d);
  const bool xyz = fused && g.D == 3 && d->cfg.order == 2;  // x-y pass, then z pass
  const bool ov = overlapped(d) && !cf;  // shell tiles -> side-stream exchange || interior
  const bool hx = d->cfg.nranks > 1 || d->xmode;  // this domain exchanges halos
  // one step-kernel launch for partition p (sweep sw; tiles: optional tile list)
  auto launch = [&](int p, int sw, int nb, const int* tiles, int ntiles) {
    a.part = p;
    g.part_coords(p, a.pc);
    for (int k = 0; k < 3; ++k) a.lo[k] = a.pc[k] * g.S[k];
    a.in = (const T*)d->buf[d->cur][p];
    a.out = (T*)d->buf[nb][p];
    a.outs = d->xmode == 2 ? (T* const*)(d->d_tab_self + ((size_t)nb * kMaxParts + p) * kMaxParts)
                           : (T* const*)(d->d_tab + nb * kMaxParts);
    a.tiles = tiles;
    a.ntiles = ntiles;
    const bool prof = d->ev_used + 2 <= d->ev.size();
    if (prof) cudaEventRecord(d->ev[d->ev_used], d->stream);
    if (xyz && sw == 0) launch_xy3d_o2<T>(a, d->tmap[d->cur][p].b, d->stream);
    else if (xyz) launch_zmarch2<T>(a, d->stream);
    else if (fused && g.D == 2) launch_step2d<T>(a, d->tmap[d->cur][p].b, d->stream);
    else if (fused) launch_step3d<T>(a, d->tmap[d->cur][p].b, d->stream);
    else launch_sweep<T>(a, sw, d->stream);
    if (prof) {
      cudaEventRecord(d->ev[d->ev_used + 1], d->stream);
      d->ev_used += 2;
    }
  };
  for (int s = 0; s < nsteps; ++s) {
    NvtxRange nvtx_step("step");
    const int nsweep = passes(d);
    if (cf) a.cf.step = cf->step + s;
    for (int sw = 0; sw < nsweep; ++sw) {
      const int nb = d->cur ^ 1;
      a.cf.last = sw == nsweep - 1;
      rpl_status st = RPL_OK;
      const bool hprof = hx && d->evh_used + 2 <= d->evh.size();
      if (ov) {
        // shell tiles first; the side stream packs, exchanges and unpacks their halo
        // cells while the interior tiles run; the next step waits for the halos only
        for (int p : d->local)
          if (d->n_shell[p]) launch(p, sw, nb, d->d_tiles + d->tile_off[p], d->n_shell[p]);
        CU(cudaGetLastError());
        CU(cudaEventRecord(d->ev_shell, d->stream));
        CU(cudaStreamWaitEvent(d->xstream, d->ev_shell, 0));
        {
          NvtxRange nvtx_x("halo exchange (side stream)");
          st = d->g.elem == 8 ? exchange_t<double>(d, nb, d->xstream)
                              : exchange_t<float>(d, nb, d->xstream);
        }
        if (st) return st;
        if (hprof) cudaEventRecord(d->evh[d->evh_used + 1], d->xstream);  // halo ready
        CU(cudaEventRecord(d->ev_halo, d->xstream));
        for (int p : d->local)
          if (d->n_inter[p])
            launch(p, sw, nb, d->d_tiles + d->tile_off[p] + d->n_shell[p], d->n_inter[p]);
        CU(cudaGetLastError());
        if (hprof) {
          cudaEventRecord(d->evh[d->evh_used], d->stream);  // interior done
          d->evh_used += 2;
        }
        CU(cudaStreamWaitEvent(d->stream, d->ev_halo, 0));
      } else {
        for (int p : d->local) launch(p, sw, nb, nullptr, 0);
        CU(cudaGetLastError());
        if (cf && a.cf.last && d->cfg.nranks > 1) {
          const int sn = (a.cf.step + 1) % 3;
          if (d->p2p) {
            st = p2p_sync(d, 1, &cf->dev->S[sn], 1 + sn);  // halo epoch + wavespeed in one sync
          } else {
            st = exchange(d, nb);
            if (!st) st = reduce_max(d, &cf->dev->S[sn], 0);
          }
        } else {
          if (hprof) cudaEventRecord(d->evh[d->evh_used], d->stream);
          st = exchange(d, nb);
          if (hprof) {
            cudaEventRecord(d->evh[d->evh_used + 1], d->stream);
            d->evh_used += 2;
          }
        }
      }
      if (st) return st;
      if (d->fault) inject_fault(d, nb);
      d->cur = nb;  // Listing 8 swap: the current state is the last-written buffer
    }
  }
  return RPL_OK;
}

extern "C" rpl_status rpl_advance(rpl_domain* d, double dt, int32_t nsteps) {
  NvtxRange nvtx_("rpl_advance");
  if (!d) return fail(RPL_E_INVALID_ARG, "null domain");
  if (!(dt > 0.0) || nsteps < 0) return fail(RPL_E_INVALID_ARG, "dt must be > 0, nsteps >= 0");
  CU(cudaSetDevice(d->device));
  if (d->ghosts_stale) {
    rpl_status st = rpl_fill_padding(d);
    if (st) return st;
  }
  return d->g.elem == 8 ? advance_t<double>(d, dt, nsteps) : advance_t<float>(d, dt, nsteps);
}

extern "C" rpl_status rpl_max_wavespeed(rpl_domain* d, double* out) {
  NvtxRange nvtx_("rpl_max_wavespeed");
  if (!d || !out) return fail(RPL_E_INVALID_ARG, "null argument");
  CU(cudaSetDevice(d->device));
  CU(cudaMemsetAsync(d->d_smax, 0, sizeof(unsigned long long), d->stream));
  for (int p : d->local) {
    if (d->g.elem == 8)
      launch_maxws<double>(d->g, (const double*)d->buf[d->cur][p], d->cfg.gamma, d->d_smax,
                           d->d_flag, d->stream);
    else
      launch_maxws<float>(d->g, (const float*)d->buf[d->cur][p], d->cfg.gamma, d->d_smax,
                          d->d_flag, d->stream);
  }
  CU(cudaGetLastError());
  {
    rpl_status st = reduce_max(d, d->d_smax, 0);
    if (st) return st;
  }
  CU(cudaMemcpyAsync(d->h_smax, d->d_smax, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                     d->stream));
  rpl_status st = check_flag(d);
  if (st) return st;
  unsigned long long bits = *d->h_smax;
  memcpy(out, &bits, sizeof(double));
  return RPL_OK;
}

extern "C" rpl_status rpl_advance_cfl(rpl_domain* d, double t_end, double cfl, int32_t n_reduced,
                                      double reduce, int32_t max_steps, int32_t* nsteps_out) {
  if (!d) return fail(RPL_E_INVALID_ARG, "null domain");
  if (!(cfl > 0.0) || !(t_end >= 0.0) || max_steps < 0)
    return fail(RPL_E_INVALID_ARG, "cfl > 0, t_end >= 0, max_steps >= 0 required");
  double dxmin = d->cfg.dx[0];
  for (int k = 1; k < d->g.D; ++k)
    if (d->cfg.dx[k] < dxmin) dxmin = d->cfg.dx[k];
  double t = 0.0;
  int n = 0;
  rpl_status st = RPL_OK;
  while (t < t_end && n < max_steps) {
    double S = 0.0;
    st = rpl_max_wavespeed(d, &S);
    if (st) break;
    if (!(S > 0.0)) { st = fail(RPL_E_DOMAIN, "max wavespeed is not positive"); break; }
    const double c = n < n_reduced ? cfl * reduce : cfl;
    double dt = c * dxmin / S;
    bool last = false;
    if (t + dt >= t_end) {
      dt = t_end - t;
      last = true;
    }
    st = rpl_advance(d, dt, 1);
    ++n;
    if (st) break;
    t = last ? t_end : t + dt;
  }
  if (nsteps_out) *nsteps_out = n;
  if (st) return st;
  return rpl_synchronize(d);
}

// Device-side CFL run.  Same loop as rpl_advance_cfl, but S, dt, t
// and n live on the device: the initial S comes from k_maxws, each step kernel
// folds max |u| + c of the state it produces into the next slot, the slot is
// combined across ranks on the stream, and every step kernel derives its dt
// from it.  The host enqueues chunks of steps (kernels past t_end exit at once)
// and reads (t, n) back once per chunk.
template <typename T>
static rpl_status advance_to_t(rpl_domain* d, const CflArgs& base, int max_steps, double* t_out,
                               int32_t* n_out) {
  CflDev init;
  memset(&init, 0, sizeof(init));
  CU(cudaMemcpyAsync(d->d_cfl, &init, sizeof(init), cudaMemcpyHostToDevice, d->stream));
  for (int p : d->local)
    launch_maxws<T>(d->g, (const T*)d->buf[d->cur][p], d->cfg.gamma, &d->d_cfl->S[0], d->d_flag,
                    d->stream);
  CU(cudaGetLastError());
  rpl_status st = reduce_max(d, &d->d_cfl->S[0], 1);
  if (st) return st;
  const int nsweep = passes(d);
  const int cur0 = d->cur;
  int launched = 0, chunk = 8;
  double t_prev = 0.0;
  int n_prev = 0;
  if (const char* v = getenv("RPL_CFL_CHUNK")) chunk = atoi(v) > 0 ? atoi(v) : chunk;
  int n = 0;
  double t = 0.0;
  while (launched < max_steps) {
    const int k = std::min(chunk, max_steps - launched);
    CflArgs cf = base;
    cf.step = launched;
    st = advance_t<T>(d, 0.0, k, &cf);
    if (st) return st;
    launched += k;
    CU(cudaMemcpyAsync(d->h_cfl, d->d_cfl, sizeof(CflDev), cudaMemcpyDeviceToHost, d->stream));
    st = check_flag(d);  // synchronises the stream
    n = d->h_cfl->n;
    t = d->h_cfl->t[n & 1];
    if (st || n < launched || !(t < base.t_end)) break;
    // next chunk: the steps the last chunk's average dt predicts, +1
    const double rate = (t - t_prev) / (double)(n - n_prev);
    int want = rate > 0.0 ? (int)std::min(4096.0, (base.t_end - t) / rate) + 2 : chunk;
    chunk = std::max(1, std::min(want, 4 * chunk));
    t_prev = t;
    n_prev = n;
  }
  // kernels past the end exited without writing: the state is in buffer cur0 ^ (n nsweep)
  d->cur = cur0 ^ ((n * nsweep) & 1);
  if (t_out) *t_out = t;
  if (n_out) *n_out = n;
  return st;
}

extern "C" rpl_status rpl_advance_to(rpl_domain* d, double t_end, double cfl, int32_t n_reduced,
                                     double reduce, int32_t max_steps, double* t_out,
                                     int32_t* nsteps_out) {
  if (!d) return fail(RPL_E_INVALID_ARG, "null domain");
  if (!(cfl > 0.0) || !(t_end >= 0.0) || max_steps < 0)
    return fail(RPL_E_INVALID_ARG, "cfl > 0, t_end >= 0, max_steps >= 0 required");
  CU(cudaSetDevice(d->device));
  if (d->ghosts_stale) {
    rpl_status st = rpl_fill_padding(d);
    if (st) return st;
  }
  CflArgs cf;
  memset(&cf, 0, sizeof(cf));
  cf.dev = d->d_cfl;
  cf.t_end = t_end;
  cf.cfl = cfl;
  cf.reduce = reduce;
  cf.n_reduced = n_reduced;
  cf.gamma = d->cfg.gamma;
  double dxmin = d->cfg.dx[0];
  for (int k = 1; k < d->g.D; ++k)
    if (d->cfg.dx[k] < dxmin) dxmin = d->cfg.dx[k];
  cf.dxmin = dxmin;
  for (int k = 0; k < 3; ++k) cf.dx[k] = k < d->g.D ? d->cfg.dx[k] : 0.0;
  if (t_out) *t_out = 0.0;
  if (nsteps_out) *nsteps_out = 0;
  if (max_steps == 0 || !(t_end > 0.0)) return RPL_OK;
  return d->g.elem == 8 ? advance_to_t<double>(d, cf, max_steps, t_out, nsteps_out)
                        : advance_to_t<float>(d, cf, max_steps, t_out, nsteps_out);
}

extern "C" rpl_status rpl_synchronize(rpl_domain* d) {
  if (!d) return fail(RPL_E_INVALID_ARG, "null domain");
  CU(cudaSetDevice(d->device));
  CU(cudaStreamSynchronize(d->stream));
  CU(cudaGetLastError());
  return check_flag(d);
}

extern "C" rpl_status rpl_profile(rpl_domain* d, int32_t max_launches) {
  if (!d || max_launches < 0) return fail(RPL_E_INVALID_ARG, "bad argument");
  CU(cudaSetDevice(d->device));
  CU(cudaStreamSynchronize(d->stream));
  free_events(d);
  for (int i = 0; i < 2 * max_launches; ++i) {
    cudaEvent_t e;
    CU(cudaEventCreate(&e));
    d->ev.push_back(e);
    if (d->cfg.nranks > 1 || d->xmode) {
      CU(cudaEventCreate(&e));
      d->evh.push_back(e);
    }
  }
  return RPL_OK;
}

extern "C" rpl_status rpl_profile_halo(rpl_domain* d, double* halo_ms, int64_t* exchanges) {
  if (!d || !halo_ms || !exchanges) return fail(RPL_E_INVALID_ARG, "null argument");
  CU(cudaSetDevice(d->device));
  CU(cudaStreamSynchronize(d->stream));
  double tot = 0.0;
  for (size_t i = 0; i + 1 < d->evh_used; i += 2) {
    float ms = 0.f;
    CU(cudaEventElapsedTime(&ms, d->evh[i], d->evh[i + 1]));
    tot += ms > 0.f ? ms : 0.f;  // overlapped: the halos may be ready before the interior
  }
  *halo_ms = tot;
  *exchanges = (int64_t)(d->evh_used / 2);
  d->evh_used = 0;
  return RPL_OK;
}

extern "C" rpl_status rpl_profile_read(rpl_domain* d, double* kernel_ms, int64_t* launches) {
  if (!d || !kernel_ms || !launches) return fail(RPL_E_INVALID_ARG, "null argument");
  CU(cudaSetDevice(d->device));
  CU(cudaStreamSynchronize(d->stream));
  double tot = 0.0;
  for (size_t i = 0; i + 1 < d->ev_used; i += 2) {
    float ms = 0.f;
    CU(cudaEventElapsedTime(&ms, d->ev[i], d->ev[i + 1]));
    tot += ms;
  }
  *kernel_ms = tot;
  *launches = (int64_t)(d->ev_used / 2);
  d->ev_used = 0;
  return RPL_OK;
}

namespace {
struct P2PBlob {
  cudaIpcMemHandle_t h;
  int64_t base_off;  // arena -> buffer base
  int64_t pb;        // bytes per buffer
  int64_t ctl_off;   // buffer base -> control block
  int32_t rank, device;
};
}  // namespace

extern "C" rpl_status rpl_p2p_export(rpl_domain* d, void* blob, size_t* blob_bytes) {
  if (!d || !blob_bytes) return fail(RPL_E_INVALID_ARG, "null argument");
  if (!d->p2p) return fail(RPL_E_INVALID_ARG, "domain was not created with RPL_TRANSPORT_P2P");
  if (!blob) {
    *blob_bytes = sizeof(P2PBlob);
    return RPL_OK;
  }
  if (*blob_bytes < sizeof(P2PBlob)) return fail(RPL_E_INVALID_ARG, "blob too small");
  CU(cudaSetDevice(d->device));
  P2PBlob b;
  memset(&b, 0, sizeof(b));
  CU(cudaIpcGetMemHandle(&b.h, d->arena));
  b.base_off = d->base_off;
  b.pb = part_bytes(d->g);
  b.ctl_off = 2 * b.pb;  // one local partition per rank
  b.rank = d->cfg.rank;
  b.device = d->device;
  memcpy(blob, &b, sizeof(b));
  *blob_bytes = sizeof(b);
  return RPL_OK;
}

extern "C" rpl_status rpl_p2p_attach(rpl_domain* d, const void* blobs, size_t blob_bytes) {
  if (!d || !blobs) return fail(RPL_E_INVALID_ARG, "null argument");
  if (!d->p2p) return fail(RPL_E_INVALID_ARG, "domain was not created with RPL_TRANSPORT_P2P");
  if (blob_bytes != sizeof(P2PBlob)) return fail(RPL_E_SHAPE_MISMATCH, "blob size mismatch");
  CU(cudaSetDevice(d->device));
  const int me = d->cfg.rank, n = d->cfg.nranks;
  unsigned long long* ctl[kMaxParts] = {nullptr};
  for (int r = 0; r < n; ++r) {
    P2PBlob b;
    memcpy(&b, (const char*)blobs + (size_t)r * blob_bytes, sizeof(b));
    if (b.rank != r) return fail(RPL_E_INVALID_ARG, "blobs must be in rank order");
    if (r == me) {
      ctl[r] = d->ctl;
      continue;
    }
    void* p = nullptr;
    if (b.device != d->device) {  // the step kernel stores into the peer's memory directly
      int can = 0;
      CU(cudaDeviceCanAccessPeer(&can, d->device, b.device));
      if (!can) return fail(RPL_E_UNSUPPORTED, "no peer access between the ranks' GPUs (use NCCL)");
    }
    if (!d->peer_arena[r]) {
      CU(cudaIpcOpenMemHandle(&p, b.h, cudaIpcMemLazyEnablePeerAccess));
      d->peer_arena[r] = p;
    }
    char* base = (char*)d->peer_arena[r] + b.base_off;
    d->buf[0][r] = base;
    d->buf[1][r] = base + b.pb;
    ctl[r] = reinterpret_cast<unsigned long long*>(base + b.ctl_off);
  }
  CU(cudaMemcpy(d->d_tab, d->buf, sizeof(void*) * 2 * kMaxParts, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(d->d_peer_ctl, ctl, sizeof(void*) * kMaxParts, cudaMemcpyHostToDevice));
  d->p2p_attached = true;
  return RPL_OK;
}

// ------------------------------------------------------------------ flux difference (f2)
template <typename T>
static rpl_status fluxdiff_t(rpl_domain* d, double dt) {
  const Geom& g = d->g;
  KArgs<T> a;
  memset(&a, 0, sizeof(a));
  a.g = g;
  for (int k = 0; k < 3; ++k) {
    const double lam = k < g.D ? dt / d->cfg.dx[k] : 1.0;
    a.lam[k] = (T)lam;
  }
  a.gm1 = (T)(d->cfg.gamma - 1.0);
  a.flag = d->d_flag;
  a.variant = d->variant;
  // fused config, 2-D SoA: tiled kernel (each face once); otherwise the plain one
  const bool tiled = d->cfg.kernel == RPL_KERNEL_FUSED && g.D == 2 && g.layout == 0;
  if (tiled && !d->fd_tmaps) {
    for (int p : d->local)
      for (int b = 0; b < 2; ++b)
        if (make_tmap(g, d->buf[b][p], d->tmap_fd[b][p].b, 32 + 16 / g.elem,
                      fd_tile_rows(g.elem, d->variant)) != 0)
          return fail(RPL_E_CUDA, "cuTensorMapEncodeTiled failed for the flux-difference kernel");
    d->fd_tmaps = true;
  }
  for (int p : d->local) {
    a.part = p;
    g.part_coords(p, a.pc);
    for (int k = 0; k < 3; ++k) a.lo[k] = a.pc[k] * g.S[k];
    a.in = (const T*)d->buf[d->cur][p];
    a.out = (T*)d->buf[d->cur ^ 1][p];
    if (tiled) launch_fluxdiff_tiled<T>(a, d->tmap_fd[d->cur][p].b, d->stream);
    else launch_fluxdiff<T>(a, d->stream);
  }
  CU(cudaGetLastError());
  return RPL_OK;
}

extern "C" rpl_status rpl_flux_difference(rpl_domain* d, double dt) {
  NvtxRange nvtx_("rpl_flux_difference");
  if (!d) return fail(RPL_E_INVALID_ARG, "null domain");
  if (!(dt > 0.0)) return fail(RPL_E_INVALID_ARG, "dt must be > 0");
  CU(cudaSetDevice(d->device));
  if (d->ghosts_stale) {
    rpl_status st = rpl_fill_padding(d);
    if (st) return st;
  }
  return d->g.elem == 8 ? fluxdiff_t<double>(d, dt) : fluxdiff_t<float>(d, dt);
}

extern "C" const char* rpl_kernel_name(const rpl_domain* d, int32_t op) {
  if (!d) return "";
  const Geom& g = d->g;
  if (op == 1) {  // rpl_flux_difference (fluxdiff_t: tiled only for fused 2-D SoA)
    if (d->cfg.kernel == RPL_KERNEL_FUSED && g.D == 2 && g.layout == 0)
      return g.elem == 8 ? "k_fluxdiff_ra<pd>" : "k_fluxdiff_ra<pk>";
    return "k_fluxdiff";
  }
  if (op != 0) return "";
  if (!use_fused(d)) return d->cfg.order == 2 ? "k_sweep2" : "k_sweep";
  if (d->cfg.order == 2) return g.D == 2 ? "k_step2d_o2" : "k_step2d_o2<3> (x-y) + k_zmarch2 (z)";
  if (g.D == 2) return g.elem == 8 ? "k_step2d_ra<pd>" : "k_step2d_ra<pk>";
  return step3d_kernel_name(g.elem, d->variant);
}

extern "C" rpl_status rpl_get_flux_difference(rpl_domain* d, void* host) {
  if (!d || !host) return fail(RPL_E_INVALID_ARG, "null argument");
  CU(cudaSetDevice(d->device));
  rpl_status st = xfer(d, host, false, d->cur ^ 1);
  if (st) return st;
  CU(cudaStreamSynchronize(d->stream));
  return RPL_OK;
}
