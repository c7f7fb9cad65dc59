/*
 * ripple_fv.h -- C ABI of the B200-native Ripple finite-volume step.
 *
 * The operations follow the paper's problem statement (BASELINE.json north_star,
 * SURVEY.md 8(b)): create an N-D tensor with sizes, padding width and partition
 * count (sec. 4.1, Listing 1); set the initial state;
 * fill the padding (sec. 5.4.1); advance by dt over n steps
 * (the Euler step of Listing 8); read back the state.
 *
 * The scheme: dimensionally split x->y->z sweeps (Listing 8), each a FORCE flux
 * (Toro, sec. 7.3) on every face normal to the sweep followed by the
 * conservative update U' = U - dt/dx (F_{i+1/2} - F_{i-1/2});
 * ideal gas p = (gamma-1)(E - |m|^2/(2 rho)).  Conserved variables,
 * component order [rho, m_x, (m_y), (m_z), E], C = ndim + 2 (reading S6).
 *
 * Conventions
 *  - Every call returns rpl_status; no exceptions cross the ABI.  A failing call
 *    stores a message retrievable with rpl_last_error() (thread-local).
 *  - Asynchronous device errors (the numerical-domain flag: rho<=0, p<=0 or
 *    non-finite state; CUDA and NCCL errors) are sticky and reported by
 *    the next synchronising call (rpl_synchronize, rpl_get_state,
 *    rpl_max_wavespeed).  On RPL_E_DOMAIN the state is left as computed.
 *  - Collective calls (marked "collective") must be made by every rank with
 *    identical arguments.
 *  - Host arrays are always caller-owned and copied.  Device memory is
 *    library-owned unless rpl_config.arena is given (caller-owned, e.g. a torch
 *    tensor of rpl_arena_bytes() bytes, kept alive until rpl_destroy).
 *  - Host state layout ("dense SoA"): [C][nz][ny][nx] of the dtype, x fastest,
 *    covering the rank's box (rpl_local_box), unused dims of size 1.
 */
#ifndef RIPPLE_FV_H
#define RIPPLE_FV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rpl_domain rpl_domain; /* opaque; caller owns the handle, frees with rpl_destroy */

typedef enum {
  RPL_OK = 0,
  RPL_E_INVALID_ARG = -1,
  RPL_E_NOT_DIVISIBLE = -2,  /* size[d] % parts[d] != 0 */
  RPL_E_PAD_TOO_SMALL = -3,  /* pad < stencil radius (1; 2 for order 2) */
  RPL_E_OOM = -4,
  RPL_E_CUDA = -5,
  RPL_E_NCCL = -6,
  RPL_E_DOMAIN = -7,         /* rho <= 0, p <= 0 or non-finite */
  RPL_E_SHAPE_MISMATCH = -8,
  RPL_E_UNSUPPORTED = -9
} rpl_status;

typedef enum { RPL_F32 = 0, RPL_F64 = 1 } rpl_dtype;

/* Storage of the conserved-state struct per cell (sec. 4.2, Fig. 1):
 * SoA = "strided" (one plane per component), AoS = "contiguous". */
typedef enum { RPL_SOA = 0, RPL_AOS = 1 } rpl_layout;

/* Physical boundary kinds (readings S10/S11):
 * transmissive = SPEC "Clamp" (ghost = nearest interior cell), periodic (wrap,
 * also across partitions; must be set on both sides of a dim), reflective
 * (mirror with the normal momentum negated). */
typedef enum { RPL_BC_TRANSMISSIVE = 0, RPL_BC_PERIODIC = 1, RPL_BC_REFLECTIVE = 2 } rpl_bc;

/* Step kernel: FUSED = all D sweeps of a step in one HBM pass;
 * SPLIT = one launch per sweep, the paper's structure (update_state_x/_y nodes of
 * Listing 8), kept as the parity baseline / ablation (K-A).  Both give bitwise
 * identical results.  ndim == 1 always runs SPLIT (one sweep). */
typedef enum { RPL_KERNEL_FUSED = 0, RPL_KERNEL_SPLIT = 1 } rpl_kernel;

/* Halo transport between ranks (nranks > 1), the padding transfers of
 * P:840-927 / P:1417-1419:
 *  NCCL: pack kernel -> grouped ncclSend/ncclRecv -> unpack kernel (needs nccl_id);
 *  P2P:  the step kernel stores every halo cell straight into the neighbour's
 *        buffer over NVLink peer memory (CUDA IPC mappings), then a one-warp
 *        flag kernel orders the step against the neighbours (system-scope
 *        release/acquire); no pack, no copy, no NCCL.  Needs rpl_p2p_export /
 *        rpl_p2p_attach after rpl_create and a library-owned arena.  The flag
 *        wait is bounded: a peer that does not arrive within RPL_P2P_TIMEOUT_S
 *        seconds (environment, default 120) makes the next synchronising call
 *        return RPL_E_CUDA instead of hanging. */
/* Halo transport.  NCCL (nranks > 1): the step kernel runs on the partition's shell
 * tiles (halo sources) first; a side stream packs the halo slabs (one kernel),
 * exchanges them with grouped ncclSend/ncclRecv and unpacks them while the interior
 * tiles run; the next step waits only for that (sec. 5.4.1).
 * P2P (nranks > 1): the step kernel stores halo cells straight into the neighbours'
 * buffers over NVLink (CUDA IPC, rpl_p2p_export/attach) and a one-warp kernel syncs
 * with the halo neighbours.  LOOPBACK (nranks == 1, prod(parts) > 1): the local
 * partitions exchange halos through the NCCL path's pack -> transfer -> unpack
 * kernels and side stream, with a device copy instead of send/recv (the single-GPU
 * test of that choreography); LOOPBACK_NCCL does the transfer with grouped
 * ncclSend/ncclRecv to itself over a one-rank communicator the library creates
 * (the NCCL calls of the multi-rank path, on one GPU).  Otherwise partitions of one
 * rank write each other's ghosts directly. */
typedef enum {
  RPL_TRANSPORT_NCCL = 0,
  RPL_TRANSPORT_P2P = 1,
  RPL_TRANSPORT_LOOPBACK = 2,
  RPL_TRANSPORT_LOOPBACK_NCCL = 3
} rpl_transport;

typedef struct {
  int32_t ndim;            /* 1, 2 or 3 */
  int64_t size[3];         /* global interior cells per dim, x fastest; unused dims 1 */
  int32_t pad;             /* uniform ghost width, 1 <= pad <= 4 */
  int32_t parts[3];        /* partitions per dim; size[d] % parts[d] == 0 and
                              size[d]/parts[d] >= pad; unused dims 1 */
  rpl_dtype dtype;
  rpl_layout layout;
  rpl_kernel kernel;
  double gamma;            /* ratio of specific heats, > 1 (default 1.4) */
  double dx[3];            /* cell widths, > 0 */
  rpl_bc bc_lo[3];         /* per dim, low face */
  rpl_bc bc_hi[3];         /* per dim, high face */
  int32_t nranks;          /* SPMD ranks (one process per GPU); 1, or prod(parts) */
  int32_t rank;            /* this rank; partition linear index (x fastest) when nranks > 1 */
  const void* nccl_id;     /* 128-byte ncclUniqueId from rpl_nccl_unique_id on rank 0,
                              broadcast by the caller; NULL iff nranks == 1 */
  int32_t device;          /* CUDA device ordinal */
  void* stream;            /* cudaStream_t to enqueue on (e.g. torch's); NULL -> library stream */
  void* arena;             /* optional caller-owned device memory of rpl_arena_bytes() bytes */
  int32_t rows_per_chunk;  /* fused kernels: rows (2-D) / planes (3-D) marched per warp task;
                              0 -> automatic */
  rpl_transport transport; /* nranks > 1: NCCL (default) or P2P; nranks == 1: LOOPBACK
                              (optional, multi-partition) */
  int32_t order;           /* reconstruction order (the paper's Listing 8 is
                              order 1, reading S7): 1 = piecewise constant (default);
                              2 = MUSCL-Hancock with minmod slopes + FORCE (Toro's SLIC,
                              DESIGN.md readings F3a-F3d), needs pad >= 2.  Order 2 runs
                              the fused kernel for 2-D SoA, the split kernel otherwise. */
} rpl_config;

/* Fill *cfg with defaults: ndim 1, size {1,1,1}, pad 2, parts {1,1,1}, F64, SOA,
 * FUSED, gamma 1.4, dx {1,1,1}, transmissive, nranks 1, device 0, order 1. */
void rpl_config_init(rpl_config* cfg);

/* Validate cfg without touching a GPU (host only). */
rpl_status rpl_config_check(const rpl_config* cfg);

/* Device bytes this rank needs (two padded buffers per local partition + 256 B
 * alignment slack).  Host only. */
rpl_status rpl_arena_bytes(const rpl_config* cfg, size_t* out);

/* 128-byte ncclUniqueId (rank 0; caller broadcasts it). */
rpl_status rpl_nccl_unique_id(void* out128);

/* Create the domain (collective when nranks > 1).  Allocates or adopts device
 * buffers, sets up NCCL when nranks > 1.  *out receives the handle. */
rpl_status rpl_create(const rpl_config* cfg, rpl_domain** out);

/* This rank's interior box [lo, hi) in global cell indices (all dims). */
rpl_status rpl_local_box(const rpl_domain* dom, int64_t lo[3], int64_t hi[3]);

/* Copy the rank's interior state from host (dense SoA, see Conventions) into the
 * current buffer; blocking.  Marks the padding stale (filled before the next step). */
rpl_status rpl_set_state(rpl_domain* dom, const void* host);

/* Copy the rank's interior state to host (dense SoA); synchronises the stream. */
rpl_status rpl_get_state(rpl_domain* dom, void* host);

/* Copy one local partition's full padded buffer (ghosts included) to host as
 * dense SoA [C][pz][py][px] (pz = nz+2 pad for 3-D, else 1, ...); for tests of
 * halo soundness.  part = global partition linear index. */
rpl_status rpl_get_padded(rpl_domain* dom, int32_t part, void* host);

/* Fill every ghost layer of every local partition (collective): physical BCs
 * per kind and neighbour halos, corners included; equivalent to sequential
 * per-dim fills over the full padded extent. */
rpl_status rpl_fill_padding(rpl_domain* dom);

/* Advance nsteps split FORCE steps with fixed dt (collective).  Enqueues on the
 * stream and returns without a host sync (unless nranks > 1 needs one). */
rpl_status rpl_advance(rpl_domain* dom, double dt, int32_t nsteps);

/* Global max over interior cells of |u| + c, c = sqrt(gamma p / rho) (
 * Listing 8 set_wavespeeds + then_reduce(Max)).  Collective
 * (allreduce MAX over ranks, exact); synchronises. */
rpl_status rpl_max_wavespeed(rpl_domain* dom, double* out);

/* CFL-driven advance to t_end (Listing 8's set_dt; reading S8):
 * each step dt = cfl_n * min_d dx_d / S with cfl_n = cfl*reduce for the first
 * n_reduced steps, the last step clipped to land on t_end.  Synchronises every step.
 * Writes the steps taken to *nsteps_out. */
rpl_status rpl_advance_cfl(rpl_domain* dom, double t_end, double cfl, int32_t n_reduced,
                           double reduce, int32_t max_steps, int32_t* nsteps_out);

/* Device-side CFL-adaptive advance (the same loop as rpl_advance_cfl,
 * Listing 8 set_wavespeeds -> reduce(Max) -> set_dt):
 * S, dt, t and the step count live in device memory.  The initial S is computed
 * once; afterwards every step kernel folds max |u| + c of the state it writes
 * into a per-step slot (per-warp max, ordered-bits atomicMax), the slot is
 * combined over ranks on the stream (P2P: inside the step's flag sync; NCCL: one
 * 8-byte allreduce MAX), and the next step kernel derives dt = cfl_n min dx / S
 * (clipped to t_end) itself.  The host only enqueues chunks of steps and reads
 * (t, n) back once per chunk; kernels launched past t_end exit immediately.
 * In-kernel |u| + c uses MUFU rsqrt/rcp + Newton (within a few ulp of
 * rpl_max_wavespeed's IEEE formula), so dt may differ from rpl_advance_cfl's
 * in the last bits (reading "device CFL").  Writes the time reached
 * (t_end unless max_steps ran out) and the steps taken; either pointer may be
 * NULL.  Collective; synchronises once per chunk.  Errors: RPL_E_INVALID_ARG
 * (cfl <= 0, t_end < 0, max_steps < 0, a 2-D RPL_VARIANT without the device
 * step), RPL_E_DOMAIN (rho <= 0, p <= 0, non-finite state or S <= 0). */
rpl_status rpl_advance_to(rpl_domain* dom, double t_end, double cfl, int32_t n_reduced,
                          double reduce, int32_t max_steps, double* t_out, int32_t* nsteps_out);

/* Wait for all enqueued work; report deferred RPL_E_DOMAIN / CUDA / NCCL errors. */
rpl_status rpl_synchronize(rpl_domain* dom);

/* Kernel launches enqueued per step by rpl_advance on this rank. */
rpl_status rpl_launches_per_step(const rpl_domain* dom, int32_t* out);

/* Kernel timing for roofline reports.  While enabled, rpl_advance records a CUDA
 * event pair on its stream around every step-kernel launch (fused step or split
 * sweep; not the halo pack/unpack).  rpl_profile_read synchronises, returns the
 * summed kernel milliseconds and launch count since the last read, and resets.
 * Enabling pre-allocates max_launches event pairs (0 disables). */
rpl_status rpl_profile(rpl_domain* dom, int32_t max_launches);
rpl_status rpl_profile_read(rpl_domain* dom, double* kernel_ms, int64_t* launches);

/* Name of the kernel that rpl_advance (op 0) or rpl_flux_difference (op 1) launches
 * for this domain's configuration (for roofline reports, e.g. "k_step3d_sp<pd>").
 * Static string, owned by the library; "" for a null domain or an unknown op. */
const char* rpl_kernel_name(const rpl_domain* dom, int32_t op);

/* Exposed halo time (event-timed: t(halo_ready) - t(interior_done)).
 * While rpl_profile is enabled on a multi-rank domain, rpl_advance also records an
 * event pair around every halo exchange: after the step kernels (interior done) and
 * after the exchange (NCCL pack/send/recv/unpack, or the P2P epoch sync that waits
 * for the neighbours' halo stores: halo ready).  Synchronises; returns the summed
 * milliseconds and exchange count since the last read, and resets.  Single-rank
 * domains have no exchange: 0 ms, 0 exchanges.  Errors: RPL_E_INVALID_ARG (null). */
rpl_status rpl_profile_halo(rpl_domain* dom, double* halo_ms, int64_t* exchanges);

/* Halo transfer plan (host only, no GPU).  Every ghost cell of every partition
 * has exactly one source interior cell (sequential per-dim fill semantics,
 * S:193); the plan lists, for every (source partition, destination partition)
 * pair, the boxes of ghost cells of dst_part whose sources lie in src_part.
 * Per dim d the ghost index t in [dst_lo[d], dst_hi[d]) maps to the source
 * index s in [src_lo[d], src_hi[d]) by mode[d]:
 *   RPL_MAP_TRANSLATE: s = t - dst_lo[d] + src_lo[d]   (neighbour halo, periodic wrap)
 *   RPL_MAP_REFLECT:   s = src_hi[d] - 1 - (t - dst_lo[d]); m_d is negated
 *   RPL_MAP_BROADCAST: s = src_lo[d] (src extent 1: transmissive/clamp layers)
 * Coordinates are global cell indices; ghosts of physical faces lie outside
 * [0, size).  Entries with src_part == dst_part are the physical boundary fill;
 * the others are the halo exchange (Fig. 7) -- when the two
 * partitions live on different ranks they are the NCCL messages.
 * With max_edges == 0 only *n_edges is written. */
enum { RPL_MAP_TRANSLATE = 0, RPL_MAP_REFLECT = 1, RPL_MAP_BROADCAST = 2 };
typedef struct {
  int32_t src_part, dst_part;
  int64_t src_lo[3], src_hi[3];
  int64_t dst_lo[3], dst_hi[3];
  int32_t mode[3];
} rpl_halo_edge;
rpl_status rpl_halo_plan(const rpl_config* cfg, rpl_halo_edge* edges, int32_t max_edges,
                         int32_t* n_edges);

/* Flux difference of the paper's single-GPU FV benchmark (sec. 7.3,
 * P:1264-1284, Table 4): for every interior cell of the current
 * state, R = sum_d (F_{i+1/2} - F_{i-1/2}) along each dim d, F = FORCE flux at
 * step dt.  kernel SPLIT (and 1-D/3-D/AoS): the paper's form, both faces of
 * every direction evaluated per cell ("all four faces of each cell");
 * kernel FUSED, 2-D SoA: a TMA-tiled kernel that evaluates every face once and
 * shares it between its two cells -- bitwise the same R.  Fills stale ghosts
 * first; writes R into the scratch buffer (the state is unchanged; the next
 * rpl_advance overwrites R).  Not a time integrator.  Enqueued, no
 * host sync. */
rpl_status rpl_flux_difference(rpl_domain* dom, double dt);

/* Copy R of the last rpl_flux_difference to host (dense SoA, like rpl_get_state). */
rpl_status rpl_get_flux_difference(rpl_domain* dom, void* host);

/* P2P transport, step 1 (after rpl_create): write this rank's CUDA IPC handle
 * blob (at most *blob_bytes bytes; *blob_bytes receives the size used, the same
 * on every rank).  With blob == NULL only the size is returned. */
rpl_status rpl_p2p_export(rpl_domain* dom, void* blob, size_t* blob_bytes);

/* P2P transport, step 2 (collective): `blobs` = the blobs of all ranks in rank
 * order (e.g. all_gather through the caller's process group), each blob_bytes
 * long.  Maps every peer's buffers; halos then travel inside the step kernels.
 * RPL_E_UNSUPPORTED when a peer's GPU is not peer-accessible from this one (the
 * caller then recreates the domain with the NCCL transport, as bench.py does). */
rpl_status rpl_p2p_attach(rpl_domain* dom, const void* blobs, size_t blob_bytes);

/* Free everything (collective). */
void rpl_destroy(rpl_domain* dom);

/* Thread-local message describing the last failing call ("" if none). */
const char* rpl_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
