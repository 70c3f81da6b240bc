/*
 * lbm.h — C ABI of the B200-native fused lattice Boltzmann stream–collide library.
 *
 * Computes the lattice Boltzmann time step of Bauer, Köstler, Rüde, "lbmpy: Automatic code
 * generation for efficient parallel lattice Boltzmann methods" (arXiv 2001.11806), cited as
 * P:<line> of PAPER.md; readings of the paper are named G<k> as in DESIGN.md.
 *
 *   - D3Q19 / D3Q27 stencils, direction order G10: index 0 = (0,0,0), then by |c|_1,
 *     then lexicographic on (cx, cy, cz) with -1 < 0 < 1.
 *   - Collision: SRT/BGK Eq. (1); TRT with Guo forcing split by moment
 *     parity (G4); weighted-orthogonal MRT Eq. (4) (G5/G6; D3Q19); cumulant
 *     (G7; D3Q27 and D3Q19); Smagorinsky SRT and KBC.
 *     Equilibrium Eq. (3), 2nd order, compressible (G1), or its incompressible and
 *     moment-matched variants (LBM_EQ_*).
 *   - Storage patterns: two-array stream-pull-collide and collide-stream-push, the
 *     single-array AA and EsoTwist patterns; collision-only kernel.
 *   - Boundaries from a uint8 flag field: 0 = fluid, 1 = no-slip bounce-back,
 *     2 = velocity bounce-back UBB (G8), compiled into the update or applied
 *     by a separate kernel from per-link index lists with per-link wall velocities.
 *   - Multi-GPU: z-slab decomposition, one ghost plane per side, for every pattern; the exchanged
 *     populations move by NCCL send/recv overlapped with the interior update, or (LBM_HALO_FUSED)
 *     are stored by the boundary-plane kernel straight into the neighbour's planes over NVLink
 *     (P:1056-1071). AA slabs: ghost fill after even steps, return of ghost writes after odd steps;
 *     push: return after every step; EsoTwist: lower-face fill and return after every step.
 *   - Bulk kernels: plain register gathers or TMA-staged persistent kernels (lbm_set_kernel_path).
 *
 * Layout (part of the ABI): populations are SoA  f[q][z][y][x], x fastest. Host-visible arrays
 * passed to this API always use the canonical layout of the *local* slab (no ghost planes):
 * cell index i = x + nx * (y + ny * z_local). Vector fields are SoA [3][cells].
 *
 * Ownership ("raw pointer, together with shape and stride information"):
 * the population arrays pdf[2], the device flag bytes and the halo staging buffer may be BORROWED
 * from the caller (lbm_config.pdf_dev / flags_dev / halo_dev, e.g. torch tensors; sizes from
 * lbm_buffer_sizes): the library then never allocates or frees them, and the caller keeps them
 * alive until lbm_destroy returns. Left NULL, the library allocates them itself. The fused halo
 * (LBM_HALO_FUSED) needs its population arrays in NCCL symmetric memory (ncclMemAlloc windows) and
 * therefore always owns them. The library always owns its scratch memory, the boundary lists, its
 * events, CUDA graphs and NCCL communicator. The caller may pass its own compute stream (e.g.
 * torch.cuda.current_stream().cuda_stream); the library then launches every kernel of lbm_step on
 * it. Output buffers are caller-allocated.
 *
 * Errors: every function returns an int status, 0 = LBM_OK, negative = error. No C++ exception
 * crosses the ABI. Asynchronous CUDA errors surface at the next lbm_step / lbm_sync.
 * lbm_last_error(h) returns a human-readable message for the last failure on a handle.
 * A handle is not thread-safe; several handles per process are allowed.
 */
#ifndef LBM_B200_H
#define LBM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------------------------ */
#define LBM_OK 0
#define LBM_EINVAL (-1)       /* invalid configuration or argument */
#define LBM_EUNSUPPORTED (-2) /* valid but not implemented combination */
#define LBM_ECUDA (-3)        /* CUDA runtime error */
#define LBM_ENCCL (-4)        /* NCCL error */
#define LBM_ENAN (-5)         /* NaN detected in the populations */
#define LBM_EOOM (-6)         /* device allocation failed */

/* ---- enums --------------------------------------------------------------------------------- */
#define LBM_D3Q19 19
#define LBM_D3Q27 27

#define LBM_SRT 0      /* rates = [omega]                                              */
#define LBM_TRT 1      /* rates = [omega_even, omega_odd]                              */
#define LBM_MRT 2      /* rates = [omega_shear, omega_bulk, omega_3, omega_4] (D3Q19), or one rate per
                          moment via lbm_config.n_row_rates / row_rates                  */
#define LBM_CUMULANT 3 /* rates = [omega_shear, omega_bulk, omega_3..omega_6]; missing = 1. D3Q27, and
                          D3Q19 (the cumulants of the 19 basis monomials, orders 2-4;
                          omega_5, omega_6 unused) */
#define LBM_IDENTITY 4 /* debug: no collision (pure data movement, bit-exact tests)    */
#define LBM_SMAGORINSKY 5 /* SRT with the local Smagorinsky omega (Eqs. 11-14):
                             rates = [omega_0, C_S]                                    */
#define LBM_KBC 6      /* entropic KBC (Eqs. 15-19), D3Q19 and D3Q27: rates = [omega_s];
                          s = shear moments, h = the other non-conserved moments        */
#define LBM_GEN_SRT 8   /* generated operators: derived in moment space and simplified
                           for minimal FLOPs by paper_2001_11806_b200/codegen into
                           csrc/generated/gen_collide.cuh. SRT rates = [omega], D3Q19/D3Q27 */
#define LBM_GEN_TRT 9   /* generated TRT, rates = [omega_e, omega_o], D3Q19/D3Q27 (no forcing)    */
#define LBM_GEN_MRT 10  /* generated weighted MRT, rates = [omega_shear, omega_bulk, omega_3,
                           omega_4 (all orders >= 4)] (missing = 1), D3Q19 and D3Q27           */
#define LBM_GEN_SMAGORINSKY 11 /* generated Smagorinsky SRT, rates = [omega_0, C_S], D3Q19/D3Q27.
                           LBM_GEN_SRT / LBM_GEN_TRT also take LBM_EQ_INCOMPRESSIBLE          */
#define LBM_KBC_EXACT 7 /* KBC with omega_h maximising the entropy of Eq. (17) exactly, per cell, by
                           Newton's method started from Eq. (19); rates =
                           [omega_s]. A step that would make a population <= 0 is halved; stops after a
                           full step |d omega_h| <= 1e-8 (fp64) / 1e-4 (fp32) (quadratic convergence:
                           remaining error ~1e-16 / 1e-8) or 30 / 8 steps. ALU-bound.             */

#define LBM_F64 0
#define LBM_F32 1

#define LBM_PULL 0 /* two arrays, fused stream-pull-collide: state P(n) = (C o S)^n P(0) */
#define LBM_AA 1   /* one array, AA pattern: state F(n) = (S o C)^n f0 (G11)            */
#define LBM_PUSH 3  /* two arrays, fused collide-stream-push: state F(n) as AA */
#define LBM_ESOTWIST 2 /* one array, EsoTwist as even/odd kernels: populations stored on
                          their links at x - c_q^+, slot q or qbar by parity; state F(n) as AA.
                          Flag boundaries; any slab decomposition and halo mode */

#define LBM_FLAG_FLUID 0
#define LBM_FLAG_NOSLIP 1
#define LBM_FLAG_UBB 2

#define LBM_HOST 0   /* pointer argument is host memory   */
#define LBM_DEVICE 1 /* pointer argument is device memory */
#define LBM_HOST_ASYNC 2 /* host memory (pinned for overlap), asynchronous: lbm_init_equilibrium and
                            lbm_get_macroscopic return once the work is enqueued; uploads and downloads run on
                            their own streams (double-buffered device staging, PCIe full duplex) overlapped with
                            the compute stream. Inputs must stay unchanged and outputs are valid only after
                            lbm_sync. Other calls ignore it (treated as LBM_HOST where accepted). */

/* Equilibrium of SRT/TRT/MRT:
 * COMPRESSIBLE   Eq. (3), 2nd order, rho0 = rho; u = j / rho (G1; default)
 * INCOMPRESSIBLE Eq. (3) with rho0 = 1 (He & Luo): u = j (Eq. 2), f_eq = w rho + w [3 c.u + ...];
 *                macroscopic readout then reports u = j +- F/2
 * MOMENT_MATCHED the raw moments of the basis monomials are those of the continuous Maxwellian
 *                Eq. (7)-(8) truncated at 2nd order in u: differs from Eq. (3) for D3Q19 in
 *                the three x^2 y^2-type moments (by rho u_k^2 / 6), identical for D3Q27 */
#define LBM_EQ_COMPRESSIBLE 0
#define LBM_EQ_INCOMPRESSIBLE 1
#define LBM_EQ_MOMENT_MATCHED 2

/* Boundary handling:
 * FLAGS: compiled into the update: the bulk kernel skips walls and near-wall fluid cells (one flag
 *        byte), an edge kernel updates the near-wall cells from an index list with the bounce-back /
 *        UBB substitution inline (default).
 * LINKS: index-list boundaries: the flag field only seeds one list entry per boundary link (wall cell
 *        b, direction q from b to the fluid cell b + c_q, per-link UBB term); the update kernels are
 *        flag-free and a separate boundary kernel writes, before each pull step (AA and push: after
 *        each step), the values the fluid cells stream from the wall cells. Per-link wall
 *        velocities: lbm_boundary_links / lbm_set_link_velocities. Wall cells are updated like fluid
 *        cells and hold meaningless values. Every pattern (EsoTwist: the fix moves the departing slot of
 *        the link's location L = b + c_q^- into its arriving slot, by parity) and any slab decomposition
 *        (the link kernel also fills the wall slots of ghost planes, after the exchange; with the fused
 *        halo a step's fix runs after the next LSA gate, and lbm_step ends with a closing gate).
 *        In-kernel links (pull and AA, halo modes other than fused; by default for fp64 except D3Q27 AA,
 *        where it measured at least as fast; LBM_LINKS_FUSED=1 / 0 in the environment forces it on / off):
 *        the update kernels read one flag byte per cell (wall cells are skipped) and each
 *        near-wall fluid cell stores, right after its collision, the wall slots of its links that the next
 *        stream reads — the link kernel's writes, same values, no separate launch and no re-read of the
 *        fluid slots; links whose wall cell lies in a ghost plane stay with the link kernel (after the
 *        exchange). Before the first step after init / set / load the full list runs once (priming). A
 *        call of lbm_set_link_velocities switches the handle to the separate link kernel for good.
 *        Results are identical to the separate-kernel form. */
/* LBM_BOUNDARY_INLINE: the flag field compiled into every cell's update ("compiled-in conditionals",
 *        P:1230-1238): the bulk kernels test the flags of all q neighbours of every cell, no separate
 *        boundary launch. Same results as LBM_BOUNDARY_FLAGS. Not with the fused halo (LBM_EUNSUPPORTED). */
#define LBM_BOUNDARY_FLAGS 0
#define LBM_BOUNDARY_LINKS 1
#define LBM_BOUNDARY_INLINE 2
/* With LBM_BOUNDARY_FLAGS, a flag field whose walls are exactly the faces of the non-periodic axes (each
 * face one type; a cell on several wall faces takes the first of -x, +x, -y, +y, -z, +z — e.g. the channel
 * and the lid-driven cavity, G9) runs face-aligned kernels for the pull and AA patterns of the plain-path
 * operators (SRT/TRT, cumulant): wall and near-wall cells are recognised from their coordinates, no
 * flag read and no separate boundary launch, same substitutions and results. LBM_FACES=0 in the
 * environment disables it. lbm_boundary_impl reports what a handle runs. */
#define LBM_IMPL_NONE 0   /* no flag field */
#define LBM_IMPL_SPLIT 1  /* bulk kernel + near-wall edge-list kernel */
#define LBM_IMPL_INLINE 2 /* every cell tests its neighbours' flags */
#define LBM_IMPL_LINKS 3  /* flag-free update + index-list link kernel */
#define LBM_IMPL_FACES 4  /* face-aligned walls from coordinates */
#define LBM_IMPL_LINKS_FUSED 5 /* index lists stored by the pull / AA update kernels (+ residual link kernel) */

#define LBM_HALO_ZEROCOPY 0 /* one NCCL message per crossing population plane */
#define LBM_HALO_PACKED 1   /* pack kernel + one message per face            */
#define LBM_HALO_FUSED 2    /* NCCL ranks (or nccl_self): the boundary-plane kernel stores the
                               exchanged populations straight into the neighbours' planes through
                               NCCL symmetric-window (LSA) pointers over NVLink (pull: their ghost
                               planes; AA/push/EsoTwist: the planes the exchange phases of
                               lbm_halo_schedule_phase target); an LSA barrier kernel orders the
                               steps. Arrays live in ncclMemAlloc memory. */

typedef struct lbm_config {
    int32_t stencil;   /* LBM_D3Q19 | LBM_D3Q27 */
    int32_t collision; /* LBM_SRT .. LBM_GEN_SMAGORINSKY */
    int32_t dtype;     /* LBM_F64 | LBM_F32: storage and arithmetic precision. Populations are
                          stored zero-centred, g_q = f_q - w_q (G12), in both precisions. */
    int32_t pattern;   /* LBM_PULL | LBM_AA | LBM_ESOTWIST | LBM_PUSH */
    int32_t n_rates;
    double rates[8];      /* see the collision enum; every rate must lie in (0, 2) */
    double force[3];      /* Guo body force per cell (SRT/TRT only); all zero = force-free kernel */
    int64_t global[3];    /* global lattice nx, ny, nz (cells) */
    int32_t periodic[3];  /* 1 = periodic axis; a non-periodic axis must carry wall cells on both faces */
    const uint8_t *flags; /* host, global nx*ny*nz, x fastest; NULL = all fluid */
    double ubb_velocity[3]; /* wall velocity of UBB cells; wall density rho_w = 1 (G8) */
    int32_t rank, nranks;   /* z-slab decomposition across processes (NCCL); nranks = 1: single GPU */
    const uint8_t *nccl_id; /* 128-byte ncclUniqueId from lbm_nccl_unique_id on rank 0; NULL if nranks = 1 */
    int32_t n_local_slabs;  /* >1: decompose this process's domain into slabs on one GPU, exchanged
                               with device copies (loopback; tests the multi-GPU path on one GPU) */
    int32_t device;         /* CUDA device ordinal */
    void *stream;           /* cudaStream_t for compute; NULL = library-created stream */
    int32_t halo_mode;      /* LBM_HALO_ZEROCOPY | LBM_HALO_PACKED | LBM_HALO_FUSED */
    int32_t use_graph;      /* small single-slab domains (launch-bound): 1 = replay a captured two-step
                               CUDA graph; 2 = one persistent cooperative kernel per lbm_step call with a
                               grid-wide barrier between steps (walls inline; pull and AA, compressible
                               equilibrium, flag boundaries; otherwise plain launches) */
    int32_t block_x;        /* threads per block along x (0 = default: the extent with the fewest idle lanes at
                             * the row end, or, for full x-rows whose nx leaves idle lanes in every extent, 256
                             * threads indexing the rows' contiguous cells linearly ("flat rows"; LBM_FLAT=0 in
                             * the environment keeps the 2-D blocks); > 0 forces the 2-D block extent */
    int32_t check_nan_every;/* >0: check for NaN every k steps inside lbm_step (LBM_ENAN) */
    int32_t nccl_self;      /* nranks == 1 only: keep ghost planes and exchange them through a
                               1-rank NCCL communicator (self send/recv) instead of wrapping z
                               locally — exercises and times the multi-GPU exchange path on 1 GPU */
    int32_t equilibrium;    /* LBM_EQ_*: what SRT/TRT/MRT relax to (and what lbm_init_equilibrium writes);
                               other operators require LBM_EQ_COMPRESSIBLE (LBM_EUNSUPPORTED) */
    int32_t boundary_mode;  /* LBM_BOUNDARY_FLAGS | LBM_BOUNDARY_LINKS | LBM_BOUNDARY_INLINE (see below) */
    int32_t n_row_rates;    /* 0, or 15 with LBM_MRT: one relaxation rate per non-conserved moment,
                               row_rates[k] for the rows of the weighted Gram-Schmidt basis in the paper's
                               order: x^2-y^2, xy, xz, y^2-z^2, yz (orthogonalised), bulk,
                               x^2y, x^2z, xy^2, xz^2, y^2z, yz^2, x^2y^2, x^2z^2, y^2z^2 (orthogonalised);
                               rates[] is then ignored (D3Q19, compressible equilibrium, not in the
                               low-level kernel ABI) */
    double row_rates[15];
    /* Borrowed device memory (NULL = allocated by the library). One slab per process only
       (n_local_slabs <= 1) and not with LBM_HALO_FUSED (LBM_EUNSUPPORTED); every pointer 16-byte aligned
       (LBM_EINVAL). Byte sizes from lbm_buffer_sizes. Contents on entry are ignored: lbm_create zeroes
       the arrays and writes the prepared flag bytes. */
    void *pdf_dev[2];       /* population arrays, layout of the low-level kernel ABI (SoA [q][zs][y][x] with
                               the ghost planes, zero-centred, dtype elements); pdf_dev[1] for PULL/PUSH only */
    uint8_t *flags_dev;     /* device flag bytes (one per storage cell, ghost planes included); with a flag field */
    void *halo_dev;         /* halo staging: 4 faces of n_cross * nx * ny dtype elements; decomposed runs only */
} lbm_config;

/* Byte sizes of the device buffers a configuration needs (for borrowed memory, lbm_config.pdf_dev /
 * flags_dev / halo_dev): out[0] = one population array, out[1] = the flag bytes (0 without a flag field),
 * out[2] = the halo staging buffer (0 without a decomposition). Host-only; validates cfg like lbm_create
 * (LBM_EINVAL / LBM_EUNSUPPORTED). */
int lbm_buffer_sizes(const lbm_config *cfg, int64_t out[3]);

typedef struct lbm_handle_s *lbm_handle;

/* Fill `cfg` with defaults (D3Q19 SRT fp64 pull, omega = 1.8, 32^3 periodic, 1 rank). */
void lbm_config_default(lbm_config *cfg);

/* Create a simulation. Validates cfg (LBM_EINVAL: bad enum, rate outside (0,2), nz % nranks != 0,
 * slabs thinner than 2 planes, non-periodic axis without walls on its faces, misaligned borrowed
 * buffers; LBM_EUNSUPPORTED: hand-written MRT other than D3Q19, force with operators other than SRT/TRT,
 * equilibrium variants with other operators, inline boundaries with the fused halo, borrowed buffers with
 * several local slabs or the fused halo), allocates (or borrows) device memory and, for nranks > 1 (or
 * nccl_self), creates the NCCL communicator (collective: every rank must call it). The state is zero until
 * an init call. */
int lbm_create(const lbm_config *cfg, lbm_handle *out);
int lbm_destroy(lbm_handle h);

/* Host-only: 1 if cfg's flag field is face-aligned (see LBM_IMPL_FACES; face_out = wall type of the faces
 * -x, +x, -y, +y, -z, +z, 0 = none), 0 if not (or no flag field), LBM_EINVAL / LBM_EUNSUPPORTED if cfg is
 * invalid. */
int lbm_detect_faces(const lbm_config *cfg, int8_t face_out[6]);
/* Boundary implementation the handle runs: LBM_IMPL_* (or LBM_EINVAL). */
int lbm_boundary_impl(lbm_handle h);

/* Local extent of this process: out[0] = z0 (global index of local plane 0), out[1] = nz_local,
 * out[2] = nx, out[3] = ny. */
int lbm_local_extent(lbm_handle h, int64_t out[4]);

/* Initialise the populations to the equilibrium of (rho, u) per local cell: Eq. (3) for
 * SRT/TRT/MRT/IDENTITY, the product equilibrium (G2) for the cumulant. rho: [cells], u: [3][cells]
 * (fp64), in host or device memory per `where`. Resets the step counter to 0. */
int lbm_init_equilibrium(lbm_handle h, const double *rho, const double *u, int32_t where);

/* Same, with rho = 1 + U(-rho_amp, rho_amp), u_i = U(-u_amp, u_amp) from the counter-based
 * generator keyed by the GLOBAL cell index (G13), so every decomposition gives the same state.
 * profile = 1 adds profile_amp * sin(2 pi z / nz_global) to u_x (shear wave, config 2). */
int lbm_init_random(lbm_handle h, uint64_t seed, double rho_amp, double u_amp, int32_t profile,
                    double profile_amp);

/* Advance n time steps (pull: n stream-pull-collide updates; AA: alternating even/odd). */
int lbm_step(lbm_handle h, int64_t n);
/* Block until all work of the handle finished; returns any pending asynchronous error (CUDA: LBM_ECUDA;
 * NCCL communicator errors from ncclCommGetAsyncError: LBM_ENCCL — also checked at every lbm_step). */
int lbm_sync(lbm_handle h);
int64_t lbm_steps_done(lbm_handle h);

/* Density and velocity of every local cell (fp64). Pull state (post-collision): u = (j - F/2)/rho;
 * AA state (pre-collision): u = (j + F/2)/rho (G11). Wall cells report their stored values. */
int lbm_get_macroscopic(lbm_handle h, double *rho, double *u, int32_t where);

/* Canonical populations f_q (fp64, [q][cells]) of the local slab: f = g + w_q. For AA after an
 * odd number of steps the reversed-slot layout is gathered back (F(n)_q(y) = a[y - c_q](qbar)).
 * raw = 1 returns/accepts the stored values g (no +w_q, no AA gather; bit-exact data movement). */
int lbm_get_populations(lbm_handle h, double *out, int32_t where, int32_t raw);
int lbm_set_populations(lbm_handle h, const double *in, int32_t where, int32_t raw);

/* Canonical populations (fp64) of n local cells given by their local linear indices
 * i = x + nx * (y + ny * z_local) (host array `cells`); out[q * n + k] (host). For sampled
 * full-size parity checks without copying the whole lattice. */
int lbm_get_populations_at(lbm_handle h, const int64_t *cells, int64_t n, double *out);

/* Halo reference: the crossing populations of local plane z (c_qz == dir, dir = +1 or -1) of the
 * current state in canonical order (q ascending over {q : c_qz = dir}, then y, then x), raw stored
 * values, fp64. `out` holds n_cross * nx * ny values (n_cross = 5 for D3Q19, 9 for D3Q27). */
int lbm_pack_face(lbm_handle h, int64_t z, int32_t dir, double *out, int32_t where);

/* Timing support: record CUDA events around every kernel of the next lbm_step call on the
 * launching stream; lbm_kernel_time_ms returns the summed kernel time of that call. */
int lbm_kernel_time_ms(lbm_handle h, double *ms, int64_t *launches);
/* Number of kernel launches issued by this handle since creation (all kernels). */
int64_t lbm_launch_count(lbm_handle h);

/* Phase timeline of the last timed step of a decomposed run (timing switched on with
 * lbm_kernel_time_ms(h, NULL, NULL)): out = {boundary begin, boundary end, exchange begin, exchange end,
 * interior begin, interior end} in ms relative to the boundary begin, from CUDA events recorded on the
 * stream each phase runs on (the exchange on the comm stream with NCCL send/recv, so an exchange interval
 * inside the interior interval is the measured overlap; the fused halo reports its LSA gate as the
 * exchange). LBM_EINVAL if no decomposed step was timed. The same phases carry NVTX ranges
 * ("lbm.boundary_planes", "lbm.exchange", "lbm.interior", "lbm.lsa_gate", "lbm.step") for nsys. */
int lbm_step_phases_ms(lbm_handle h, double out[6]);

/* Checkpoint / resume, bit-exact: the complete stored state of the handle is the array holding the current
 * state of every local slab, ghost planes included, in the storage layout (lbm_state_bytes bytes, slabs in
 * z order) plus the step count (which fixes the AA / EsoTwist parity). lbm_save_state copies it to `out`
 * (host or device per `where`) and returns the step count; lbm_load_state restores it into a handle of the
 * same configuration (any handle: a fresh one or the same), after which lbm_step continues exactly as
 * the saved run would have. Asynchronous CUDA/NCCL errors surface as usual. */
int64_t lbm_state_bytes(lbm_handle h);
int lbm_save_state(lbm_handle h, void *out, int32_t where, int64_t *steps_done);
int lbm_load_state(lbm_handle h, const void *in, int32_t where, int64_t steps_done);

/* NCCL bootstrap: 128-byte unique id (call on rank 0, broadcast with torch.distributed). */
int lbm_nccl_unique_id(uint8_t out[128]);

/* Host-only decomposition plan (no GPU): slab of `rank` in a z-decomposition of nz cells over
 * nranks ranks: out[0] = z0, out[1] = nz_local, out[2] = rank below (z - 1 side, periodic),
 * out[3] = rank above. Returns LBM_EINVAL if nz % nranks != 0 or nz / nranks < 2. */
int lbm_slab_plan(int64_t nz, int32_t nranks, int32_t rank, int64_t out[4]);
/* Crossing directions of a z face: writes the stencil indices q with c_qz == dir into q_out
 * (ascending) and returns their count (5 for D3Q19, 9 for D3Q27), or LBM_EINVAL. */
int lbm_crossing_directions(int32_t stencil, int32_t dir, int32_t *q_out);
/* Host-only zero-copy halo schedule of `rank` in a decomposition over nranks ranks with nz_local
 * interior planes: the point-to-point operations one step posts inside one NCCL group, in posting
 * order. Row k of `out` (4 int32 each): {kind (0 = send, 1 = recv), peer rank, q, storage plane}
 * where storage plane 0 is the lower ghost plane, 1..nz_local the interior, nz_local + 1 the upper
 * ghost plane; each message is the contiguous nx*ny run of population q in that plane. Returns the
 * number of operations (4 * n_cross) or LBM_EINVAL (also if cap is too small). */
int lbm_halo_schedule(int32_t stencil, int64_t nz_local, int32_t rank, int32_t nranks, int32_t *out, int32_t cap);
/* The same for every exchange phase (crossing slot set c_z(slot) = +-1 of one storage plane per face):
 * LBM_PHASE_PULL (after every pull step), LBM_PHASE_AA_FILL (after AA even steps), LBM_PHASE_AA_RETURN
 * (after AA odd steps; with walls the library unpacks it masked), LBM_PHASE_ESO_AFTER_EVEN /
 * LBM_PHASE_ESO_AFTER_ODD (EsoTwist: lower-ghost fill from the down neighbour's top plane and return
 * of the bottom plane's writes; masked with walls). lbm_halo_schedule == phase LBM_PHASE_PULL. */
#define LBM_PHASE_PULL 0
#define LBM_PHASE_AA_FILL 1
#define LBM_PHASE_AA_RETURN 2
#define LBM_PHASE_ESO_AFTER_EVEN 3
#define LBM_PHASE_ESO_AFTER_ODD 4
int lbm_halo_schedule_phase(int32_t stencil, int32_t phase, int64_t nz_local, int32_t rank, int32_t nranks, int32_t *out,
                            int32_t cap);
/* Direction table of a stencil in ABI order: c_out[3*q + d], w_out[q]. Returns Q or LBM_EINVAL. */
int lbm_stencil_table(int32_t stencil, int32_t *c_out, double *w_out);

/* ---- Low-level kernel ABI ("raw pointer, together with shape and stride
 * information ... relaxation rates or constant external forces become parameters") -------------
 * One launch of one fused kernel on caller-owned device memory, asynchronous on `stream`.
 * Layout: contiguous SoA, element (q, zs, y, x) at q*Sq + (zs*ny + y)*nx + x with
 * Sq = nx*ny*(nz + 2*ghost); zs = z + ghost; populations stored zero-centred (g = f - w_q) in the
 * dtype's precision. `flags` (device, one byte per storage cell, or NULL) must have been prepared
 * by lbm_prepare_flags. The kernel updates interior planes z in [z_begin, z_end). Returns LBM_OK
 * once the launch is enqueued; LBM_EINVAL / LBM_EUNSUPPORTED for bad arguments; LBM_ECUDA if the
 * launch failed. */
typedef struct lbm_kernel_args {
    int32_t stencil, collision, dtype;
    const void *src;      /* pull: read array; AA: unused */
    void *dst;            /* pull: write array; AA: the single array (read and written) */
    const uint8_t *flags; /* prepared flags or NULL (all fluid) */
    int64_t shape[3];     /* nx, ny, nz (interior planes) */
    int32_t ghost;        /* 0: z wraps within the array; 1: one ghost plane per z side */
    int64_t z_begin, z_end;
    double rates[8];      /* as lbm_config.rates (SRT: [omega]) */
    double force[3];
    double ubb_velocity[3];
    void *stream;         /* cudaStream_t */
    int32_t equilibrium;  /* LBM_EQ_* (SRT/TRT/MRT) */
} lbm_kernel_args;

/* Fused stream-pull-collide: dst = C(S(src)) on the fluid cells of planes [z_begin, z_end). */
int lbm_kernel_pull(const lbm_kernel_args *a);
/* AA even (odd = 0) or odd (odd = 1) step on dst in place (ghost must be 0). */
int lbm_kernel_aa(const lbm_kernel_args *a, int32_t odd);
/* Fused collide-stream-push: dst(x + c_q)(q) = C(src(x))_q on the fluid cells of [z_begin, z_end);
 * a population pushed toward a wall is bounced into dst(x)(qbar) (+ UBB term). */
int lbm_kernel_push(const lbm_kernel_args *a);
/* Collision only, in place on dst, fluid cells of [z_begin, z_end). */
int lbm_kernel_collide(const lbm_kernel_args *a);
/* Device flag bytes for the kernels: copies host flags (nx*ny*nplanes, values 0/1/2) and marks
 * fluid cells that have a non-fluid neighbour (bit 7). nplanes includes ghost planes. */
int lbm_prepare_flags(const uint8_t *host_flags, int64_t nx, int64_t ny, int64_t nplanes, int32_t ghost,
                      uint8_t *device_out, void *stream);

/* Index-list boundaries (boundary_mode == LBM_BOUNDARY_LINKS). lbm_boundary_links returns the number
 * of links n and, if the arrays are non-NULL (cap >= n, else LBM_EINVAL), per link i: cells[i] = global
 * linear index x + nx (y + ny z) of the wall cell, dirs[i] = q (the fluid cell is at cells[i] + c_q,
 * periodic wrap), types[i] = LBM_FLAG_NOSLIP | LBM_FLAG_UBB. Returns 0 in flag mode.
 * lbm_set_link_velocities sets the wall velocity of every link (host uw[3*i + d], n == link count);
 * UBB links then use 6 w_q rho_w c_q.u_w(i) (G8, rho_w = 1), no-slip links ignore it. Synchronises the
 * handle's stream. The initial velocities are cfg.ubb_velocity. */
int64_t lbm_boundary_links(lbm_handle h, int64_t *cells, int32_t *dirs, int32_t *types, int64_t cap);
int lbm_set_link_velocities(lbm_handle h, const double *uw, int64_t n);

/* Roofline probe "copy-q" (the analogue of the paper's copy-19 / update-19 bandwidth probes, Table III,
 * P:1083-1127): allocates two q x nx x ny x nz arrays of the dtype on `device`, copies every cell's q
 * populations from one to the other `reps` times (gathered from x - c_q with periodic wrap when
 * shifted != 0 — the pull access pattern — else aligned) and returns the achieved read + write
 * bandwidth in GB/s (CUDA events). Frees everything before returning. LBM_EOOM if the arrays do not fit. */
int lbm_probe_copy(int32_t stencil, int32_t dtype, int32_t shifted, int64_t nx, int64_t ny, int64_t nz, int32_t reps,
                   int32_t device, double *gbs_out);

/* Roofline probe "update-q" (the analogue of the paper's in-place update-19 probe, Table III):
 * one q x nx x ny x nz array of the dtype, the AA-pattern access streams without collision, in place:
 * mode 0 even (read f[x](q), write f[x](qbar)), 1 odd (read f[x - c_q](qbar), write f[x + c_q](q)),
 * 2 alternating even/odd. Returns read + write GB/s: the ceiling of the AA / EsoTwist update kernels. */
int lbm_probe_update(int32_t stencil, int32_t dtype, int32_t mode, int64_t nx, int64_t ny, int64_t nz, int32_t reps,
                     int32_t device, double *gbs_out);
/* ALU ceiling probe: TFLOP/s of independent FMA chains (DFMA for LBM_F64, FFMA for LBM_F32; 2 FLOP per
 * FMA; 8 x 256 threads per SM, no memory traffic) — the peak the FP64-ALU-bound operators (cumulant,
 * KBC, exact KBC) are reported against. */
int lbm_probe_fma(int32_t dtype, int32_t device, double *tflops_out);

/* ---- Kernel path of the bulk update kernels (process-wide; affects launches issued afterwards) ----
 * LBM_PATH_PLAIN : one thread per cell gathers its q populations straight into registers (ld.global.nc).
 * LBM_PATH_STAGED: persistent CTAs; a producer warp moves the source rows of each direction into a
 *                  shared-memory ring with 1-D bulk copies (cp.async.bulk, the TMA engine, mbarrier
 *                  completion) and consumer warps gather from shared memory. Needs nx * sizeof(real)
 *                  % 16 == 0 (and nx % 16 == 0 with walls); otherwise the plain kernel runs.
 * LBM_PATH_AUTO  : the measured per-operator choice. Default; the environment
 *                  variable LBM_KERNEL_PATH=auto|plain|staged sets the initial value.
 * Both paths compute the same update (same arithmetic in the same order). Returns LBM_EINVAL for an
 * unknown path. */
#define LBM_PATH_AUTO 0
#define LBM_PATH_PLAIN 1
#define LBM_PATH_STAGED 2
int lbm_set_kernel_path(int32_t path);
int32_t lbm_get_kernel_path(void);

const char *lbm_strerror(int status);
const char *lbm_last_error(lbm_handle h);
/* Library version string. */
const char *lbm_version(void);

#ifdef __cplusplus
}
#endif
#endif /* LBM_B200_H */
