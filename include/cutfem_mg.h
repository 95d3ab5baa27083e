/*
 * cutfem_mg.h — C ABI of the B200-native CutFEM vertex-patch multigrid path.
 *
 * Implements the data-parallel hot path of arxiv 2508.11608:
 * the multiplicative vertex-patch smoother with Cartesian (fast
 * diagonalisation) and cut (dense inverse) patches for the Nitsche +
 * ghost-penalty Poisson problem on an unfitted Cartesian mesh, inside a
 * V-cycle and preconditioned CG.  Paper citations are "P l.<line>" of
 * PAPER.md; readings R<n> are listed in DESIGN.md.
 *
 * Conventions for every call
 *  - All functions return 0 on success and a nonzero cutfem_status code on
 *    failure; cutfem_last_error() then returns a message (thread-local).
 *    No call aborts the process.  Invalid arguments are detected before any
 *    device work is queued.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *    stream).  Device work is queued on it asynchronously unless the call
 *    says otherwise.
 *  - Vectors are DEVICE pointers to fp64 "lattice vectors" of a level: NL rows
 *    (NL*NL rows in 3D, row c*NL + b) of LD doubles (cutfem_level_info),
 *    entry [b*LD + a] (3D: [(c*NL + b)*LD + a]) is lattice node
 *    (a, b) = x-index a, y-index b, at position
 *    x0 + (a div p + xi_{a mod p}) h (xi = Gauss-Lobatto nodes on [0,1]).
 *    Entries of nodes that carry no DoF (P l.121: no DoFs on exterior cells)
 *    and the padding columns a >= NL are ignored on input (they may hold any
 *    value, NaN included); output vectors (y of cutfem_apply_operator, x of
 *    cutfem_solve_cg_mg) are 0 there, vectors updated in place (x of
 *    cutfem_smooth / cutfem_vcycle / cutfem_colour_step) keep their non-DoF
 *    entries unchanged -- except on a fitted box (cutfem_params.domain = 1),
 *    where their entries on the box boundary are set to 0.
 *    Vectors are owned by the caller; the library never frees them.
 *  - The problem handle owns all device memory it allocates (mesh data,
 *    patch data, local inverses, workspaces); cutfem_destroy releases it.
 *  - A handle is not thread-safe; calls on one handle must be serialised.
 */
#ifndef CUTFEM_MG_H
#define CUTFEM_MG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct cutfem_problem_s* cutfem_problem;

enum cutfem_status {
  CUTFEM_OK = 0,
  CUTFEM_ERR_ARG = 1,      /* invalid argument (null pointer, bad level, ...) */
  CUTFEM_ERR_CUDA = 2,     /* a CUDA runtime call failed */
  CUTFEM_ERR_STATE = 3,    /* call out of order (e.g. smooth before build_patches) */
  CUTFEM_ERR_GEOMETRY = 4, /* the hierarchy violates Omega_l ⊆ Omega_{l-1} (P l.128-129), or a
                              level has no DoF (the domain misses the background box) */
  CUTFEM_ERR_SIZE = 5      /* a size limit was exceeded (coarse DoFs, patch size) */
};

/* Problem description (P l.43-121, l.217; BASELINE.json configs). */
typedef struct {
  double x0, y0;        /* lower-left corner of the square background box */
  double length;        /* side of the box */
  int n_coarse;         /* cells per side on level 0 (P l.217: 2) */
  int n_levels;         /* levels 0..n_levels-1, n_l = n_coarse 2^l cells per side */
  int degree;           /* p of Q_p, 1..4 (P l.79) */
  double cx, cy, r;     /* level set phi(x) = |x - c| - r, Omega = {phi < 0} (P l.217) */
  double gamma_D;       /* Nitsche penalty (P l.85); <= 0 selects 5 p (p+1) (R7) */
  double gamma_k[4];    /* ghost penalty gamma_1..gamma_p (P l.104-108); < 0 selects 0.1 (R5) */
  int sigma;            /* ghost scaling h^(2k+sigma) (R5; -1 = H^1 scaling) */
  int n_q;              /* Gauss points per direction on cut cells; 0 selects p+1 (R6) */
  int n_c;              /* sweeps over cut patches per smoothing step (P l.203; >= 1) */
  int symmetric;        /* 1: post-smoother = reverse colour order (R9, needed by CG) */
  int cut_mode;         /* cut-cell operator: 0 = element matrix of bulk + Nitsche terms precomputed
                           from the cut quadrature at setup, 1 = quadrature on the fly */
  int dim;              /* 2 (circle, default when 0) or 3 (sphere; degree 1..3) */
  double z0, cz;        /* 3D: box corner z and sphere centre z (the box is a cube of side length) */
  int domain;           /* 0: the circle / sphere level set above (unfitted, cut cells, Nitsche +
                           ghost penalty); 1: FITTED box -- Omega = the open background box itself,
                           homogeneous Dirichlet condition imposed strongly (no DoF on the box
                           boundary), every patch at an interior vertex is Cartesian (the paper's
                           "Square" baseline, P Table 1 / Fig. 2; BASELINE configs[4]); cx, cy, cz,
                           r are ignored */
} cutfem_params;

/* Per-level sizes and counts. */
typedef struct {
  int dim;              /* 2 or 3 */
  int n;                /* cells per side */
  int nl;               /* lattice nodes per side = n p + 1 */
  int ld;               /* row stride of lattice vectors (doubles), even, >= nl */
  int64_t n_dofs;       /* active DoFs n_l (P l.120) */
  int n_inside, n_cut;  /* cells of M_{l,Omega} \ M_{l,Gamma} and of M_{l,Gamma} (P l.69) */
  int n_ghost_faces;    /* |F_G| (P l.97-101) */
  int n_cart[8];        /* Cartesian patches per colour (R4); 4 colours in 2D, 8 in 3D */
  int n_cutp[8];        /* cut patches per colour */
  int64_t n_vol_qp, n_surf_qp; /* cut-cell quadrature points (R6) */
  double h;
  int64_t cut_step_bytes[8];   /* algorithmic bytes of one cut colour step per colour with the
                                  precomputed patch maps (descriptor, map, gathered x and b,
                                  written x per patch); 0 without maps */
  int64_t cut_method_bytes[8]; /* the method's bytes of one cut colour step per colour, whatever
                                  the implementation: per patch
                                  8 (m^2 [A_j^{-1}] + n_cut (p+1)^{2d} [cut-cell matrices]
                                  + 3 m + nnz [b_I, x_I read, x_I written, coupled x_E]) */
  int sweep_ctas[2];           /* 2D: CTAs of the one-launch cut sweep (forward, reverse) of
                                  cutfem_smooth on an unpartitioned level; 0 = not built (the
                                  sweep then runs one launch per colour step) */
  double sweep_redundancy[2];  /* map bytes the sweep's CTAs stream / map bytes of the 4 n_c
                                  colour steps (>= 1: patches recomputed near CTA boundaries) */
  int64_t sweep_map_bytes[2];  /* map bytes streamed by all CTAs of one sweep */
  int64_t host_span_doubles;   /* 2D: doubles of the DoF spans of the lattice rows (what
                                  cutfem_smooth_host moves per vector for pinned host memory) */
} cutfem_level_info;

/* ---- setup ------------------------------------------------------------ */

/* setup_mesh: builds the level hierarchy, classifies cells against the level
 * set (P l.69, reading R2), marks DoF nodes (P l.121), lists ghost faces
 * (P l.97-101) and generates cut-cell quadrature (P l.190, reading R6), all
 * on the device.  Blocks until done.  Returns CUTFEM_ERR_GEOMETRY if a fine
 * active cell has an inactive parent. */
int cutfem_setup_mesh(const cutfem_params* prm, void* stream, cutfem_problem* out);

/* build_patches: vertex patches at every vertex of an active cell (R3),
 * Cartesian/cut split (R4), colouring (I mod 2) + 2 (J mod 2) (P l.179),
 * interior DoF sets, local matrices A_{l,j} of the cut patches assembled
 * matrix-free and inverted (P l.193, R10), fast-diagonalisation data for the
 * Cartesian patches (P l.192), and the exact coarse inverse of A_0 (P l.124).
 * Blocks until done. */
int cutfem_build_patches(cutfem_problem pb, void* stream);

int cutfem_destroy(cutfem_problem pb);
const char* cutfem_last_error(void);
int cutfem_level_info_get(cutfem_problem pb, int level, cutfem_level_info* out);

/* ---- hot path ----------------------------------------------------------- */

/* y = A_l x, A_l = a_l + g_l (P eq. cutfem-ghost l.92-95), matrix-free:
 * sum factorisation on uncut cells, quadrature with Nitsche terms on cut
 * cells, ghost-penalty faces.  x and y must not alias. */
int cutfem_apply_operator(cutfem_problem pb, int level, const double* x, double* y, void* stream);

/* One smoothing step x <- S(x, b) of eq. (smoother-split) (P l.196-210):
 * Cartesian colours 0..3, then n_c sweeps over cut colours 0..3; reverse = 1
 * applies the steps in the opposite order (R9).  In place on x.  In 2D the
 * cut colour steps run as one cooperative launch (cutfem_level_info.sweep_ctas
 * CTAs, at most one per SM), bit-identical to one launch per colour step: a
 * concurrent kernel that holds SMs delays it until they free up.  Returns
 * CUTFEM_ERR_CUDA if the launch fails. */
int cutfem_smooth(cutfem_problem pb, int level, double* x, const double* b, int reverse, void* stream);

/* One colour step of the smoother (P l.179-181, R9): kind 0 = Cartesian,
 * 1 = cut patches; colour 0..3 (0..7 in 3D).  2D only: kind 2 runs the
 * whole Cartesian sweep and kind 3 the n_c cut sweeps of a smoothing step
 * (forward, or reversed if colour is odd) exactly as cutfem_smooth does.  x <- x + sum_j Q_j^T A_j^{-1} Q_j (b - A x)
 * with the residual taken before the step.  Used by the sampled full-size
 * parity tests. */
int cutfem_colour_step(cutfem_problem pb, int level, int kind, int colour, double* x, const double* b, void* stream);

/* x <- x + V(b - A_L x)-style V-cycle on the finest level with the current x
 * as initial guess (P l.124, one pre- and one post-smoothing step, l.217).
 * In place on x. */
int cutfem_vcycle(cutfem_problem pb, double* x, const double* b, void* stream);

/* CG on the finest level preconditioned by one V-cycle (zero initial guess),
 * x_0 = 0, stop when ||r_k||_2 <= tol ||b||_2 or after max_it iterations.
 * Writes the solution to x; iterations and final relative residual to the
 * host pointers (may be NULL).  Blocks (reads the residual norm each
 * iteration). */
int cutfem_solve_cg_mg(cutfem_problem pb, double* x, const double* b, double tol, int max_it,
                       int* iters, double* rel_res, void* stream);

/* Same as the calls above with HOST (pageable or pinned) lattice vectors:
 * host->device copy of the inputs, the device call, device->host copy of the
 * result, all on `stream`; blocks until the result is on the host.  For
 * pinned, device-mapped host memory (cudaHostAlloc, cudaHostRegister) on a 2D
 * level-set problem, cutfem_smooth_host moves only the DoF span of every
 * lattice row, read and written by kernels over PCIe
 * (cutfem_level_info.host_span_doubles per vector); otherwise whole vectors. */
int cutfem_smooth_host(cutfem_problem pb, int level, double* x_host, const double* b_host, int reverse,
                       void* stream);
int cutfem_solve_cg_mg_host(cutfem_problem pb, double* x_host, const double* b_host, double tol,
                            int max_it, int* iters, double* rel_res, void* stream);

/* Intergrid transfer (P l.126-137): x_fine += P x_coarse, and
 * b_coarse = P^T r_fine, between levels `level` (fine) and level-1. */
int cutfem_prolongate_add(cutfem_problem pb, int level, const double* x_coarse, double* x_fine, void* stream);
int cutfem_restrict(cutfem_problem pb, int level, const double* r_fine, double* b_coarse, void* stream);

/* ---- slab partition over ranks (north_star: "the background mesh is
 * partitioned into slabs across the GPUs ... halo exchange per colour sweep
 * and per residual, coarse-grid solve on one rank") --
 *
 * A communicator endpoint is one rank's view of a group.  cutfem_partition
 * attaches it to a built 2D problem, which takes ownership of it.  Rank r of W
 * then owns the cell rows [r s, (r+1) s), s = n/W, of every level whose slab
 * is a whole number of fused Cartesian tiles and thicker than the halo, from
 * the finest level down; the remaining coarse levels (incl. the exact coarse
 * solve) are computed redundantly by every rank after one all-reduce of the
 * restricted residual.  Vectors stay full-size lattice vectors on every rank;
 * only the rank's rows are meaningful:
 *  - cutfem_smooth / cutfem_vcycle: x and b valid on the rows [v0, v1)
 *    (owned rows + halo, cutfem_partition_info); x is valid there on return.
 *  - cutfem_apply_operator: x valid on [v0, v1); y valid on the owned rows.
 *  - cutfem_solve_cg_mg(_host): b valid on the owned rows; x valid on the
 *    owned rows on return; iteration counts and residuals identical on all ranks.
 * Every rank must make the same sequence of calls (the exchanges pair up).
 * cutfem_colour_step: only kinds 2 and 3 (with their halo exchanges) on
 * partitioned levels. */
typedef struct cutfem_comm_s* cutfem_comm;
#define CUTFEM_NCCL_ID_BYTES 128

/* `world` endpoints of an in-process group (ranks = host threads of this
 * process sharing one device; halo rows copied device-to-device).  The
 * single-GPU harness of the decomposition. */
int cutfem_comm_local_create(int world, cutfem_comm* out /* [world] */);
/* NCCL (libnccl.so.2, loaded at first use): rank 0 creates the unique id, the
 * caller broadcasts its CUTFEM_NCCL_ID_BYTES bytes, every rank then calls
 * cutfem_comm_nccl_create (collective, blocking) on its own device. */
int cutfem_comm_nccl_unique_id(unsigned char* id_out);
int cutfem_comm_nccl_create(const unsigned char* id, int rank, int world, cutfem_comm* out);
/* destroys an endpoint that was not attached to a problem */
int cutfem_comm_destroy(cutfem_comm comm);
/* On failure the endpoint stays with the caller; a partition that failed
 * half-way leaves the problem unusable (every later call returns
 * CUTFEM_ERR_STATE; destroy it). */
int cutfem_partition(cutfem_problem pb, cutfem_comm comm);
/* out[8] = {partitioned, r0, r1, v0, v1, rank, world, halo}: owned lattice
 * rows [r0, r1) and valid rows [v0, v1) = owned rows +- `halo` cells of
 * `level` (the whole lattice if the level is not partitioned).  halo = 4
 * cells, or 12 n_c cells on levels whose slabs are thick enough for the
 * wide-halo cut sweeps (one exchange per sweep instead of one per step) */
int cutfem_partition_info(cutfem_problem pb, int level, int* out);
/* The slab plan the partition uses for one level (host only, no device):
 * out[17] = {c0, c1, r0, r1, v0, v1, n_xfers, then 2 x (peer, send_off,
 * send_n, recv_off, recv_n)} -- owned cell rows [c0, c1), owned lattice rows
 * [r0, r1), valid rows [v0, v1) after an exchange of `halo_cells` cells, and
 * the row bands exchanged with the neighbours (offsets / counts in lattice
 * rows; peer = -1 for an unused slot).  ERR_ARG unless n_cells % world == 0
 * and n_cells / world >= halo_cells + 1. */
int cutfem_slab_plan(int n_cells, int degree, int world, int rank, int halo_cells, int64_t* out);
/* The planner of the one-launch cut sweep (host only, no device; exposed for
 * the CPU tests of its dependency cones).  Input: npatch cut patches of a 2D
 * level (n cells per side, degree p, lattice row stride ld), patch k with
 * vertex (ijc[3k], ijc[3k+1]), colour ijc[3k+2], interior lattice nodes
 * in_nodes[in_off[k] .. in_off[k+1]) and coupled exterior window nodes
 * ex_nodes[ex_off[k] .. ex_off[k+1]); S = 4 n_c colour steps, reverse = the
 * adjoint order; nsm = CTA limit, force_ng > 0 forces the count; (ca, cb) =
 * the level-set centre in lattice coordinates.  Output: the CTA count
 * (*ncta), per CTA g its owned nodes own_nodes[own_off[g] .. own_off[g+1])
 * and per (g, step s) the cone's patches task_patch[task_off[g S + s] ..
 * task_off[g S + s + 1]).  The caller sizes the arrays (own_off: nsm + 1,
 * task_off: nsm S + 1, own_nodes / task_patch: own_cap / task_cap entries);
 * ERR_SIZE if they are too small, ERR_ARG for bad arguments. */
int cutfem_sweep_plan(int n, int p, int ld, int S, int reverse, int nsm, int force_ng, int npatch, const int* ijc,
                      const int* in_off, const int* in_nodes, const int* ex_off, const int* ex_nodes, double ca,
                      double cb, int* ncta, int* own_off, int* own_nodes, int own_cap, int* task_off, int* task_patch,
                      int task_cap);
/* exchange the halo rows of a lattice vector of `level` with the neighbours */
int cutfem_halo_exchange(cutfem_problem pb, int level, double* v, void* stream);

/* ---- export (host copies, blocking; used by the parity tests) ---------- */

/* cell types [j*n + i]: 0 outside, 1 inside, 2 cut */
int cutfem_export_cell_types(cutfem_problem pb, int level, int8_t* host_out);
/* DoF mask of the lattice [b*nl + a] (1 = node carries a DoF) */
int cutfem_export_dof_mask(cutfem_problem pb, int level, uint8_t* host_out);
/* patch vertices of one (kind, colour) list, kind 0 = Cartesian, 1 = cut,
 * packed I + (n+1) J, in list order; returns the count in *count.  host_out
 * may be NULL to query the count. */
int cutfem_export_patches(cutfem_problem pb, int level, int kind, int colour, int32_t* host_out, int* count);
/* interior DoF sets of the cut patches in (colour, list) order: offsets
 * (n_cut_patches + 1) and lattice indices b*nl + a.  NULL pointers query the
 * sizes through *n_patches and *n_entries. */
int cutfem_export_cut_interior(cutfem_problem pb, int level, int64_t* host_offsets, int32_t* host_nodes,
                               int* n_patches, int64_t* n_entries);
/* number of kernels this library has launched since load (for the bench's
 * gpu_launches claim) */
int64_t cutfem_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* CUTFEM_MG_H */
