/*
 * alyab200.h — C ABI of libalyab200.so, the B200 (sm_100a) hot path of the
 * arXiv 2005.05899 (Alya) fractional-step explicit-RK FE Navier-Stokes step.
 *
 * The reference package (coexbal 0.1.0) is pure Python; its "operator API" is
 * the set of functions listed against each entry point below.  Every entry
 * point here replaces one of them (or one of the time-step pieces the paper
 * describes and the reference leaves out) and is what a ctypes
 * binding on the reference side would call.
 *
 * ABI rules
 *  - plain C types only; every array argument is a DEVICE pointer owned by
 *    the caller (PyTorch tensors in the Python package); no allocation inside
 *    the launch functions except where documented;
 *  - every function returns 0 on success or a negative AB_E* code; the
 *    message is available from ab_last_error() (thread-local);
 *  - `stream` is a cudaStream_t passed as void*; all work is asynchronous on
 *    it, nothing synchronises the host;
 *  - "accumulated" outputs are added into (fp64 atomics): the caller zeroes
 *    them (the fused node kernels below re-zero the buffers they consume).
 *
 * Layouts: node vectors are [n_nodes][4] f64 (x,y,z,pad /
 * u,v,w,pad) so one 256-bit load fetches a node; connectivity is int32
 * [n_elem][nnode] per category in the reference's VTK node order.
 */
#ifndef ALYAB200_H
#define ALYAB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AB_OK 0
#define AB_EINVAL (-1)
#define AB_ECUDA (-2)
#define AB_ENOMEM (-3)

/* Integration rules (kernel template parameter).  Names and values follow
 * reference assembly.py:89-117 (tet1, tet4, hex8) plus pyr5/pri6. */
#define AB_RULE_TET1 0
#define AB_RULE_TET4 1
#define AB_RULE_PYR5 2
#define AB_RULE_PRI6 3
#define AB_RULE_HEX8 4

typedef struct ab_category {
  int32_t rule;          /* AB_RULE_* */
  int32_t pad_;
  int64_t n_elem;
  const int32_t* conn;   /* [n_elem][nnode] */
} ab_category;

typedef struct ab_mesh {
  int64_t n_nodes;
  const double* coords;  /* [n_nodes][4] */
  double period[3];      /* box length of periodic axes, 0 = not periodic */
  int32_t n_cat;
  int32_t pad_;
  ab_category cat[5];
} ab_mesh;

typedef struct ab_phys {
  double rho;            /* density */
  double mu;             /* molecular viscosity */
  double c_vreman;       /* Vreman constant, 0 disables the SGS model */
} ab_phys;

/* Sliced-ELL matrix, slice height 32. */
typedef struct ab_sell {
  int64_t n_rows;
  int64_t n_slices;
  int64_t max_width;         /* widest slice; > 0 enables the TMA-staged SpMV */
  const int64_t* slice_ptr;  /* [n_slices+1], offsets in entries */
  const int32_t* cols;       /* [slice_ptr[n_slices]], lane-innermost; padding col = row */
  const double* vals;        /* same layout; padding 0 */
} ab_sell;

/* ---- housekeeping ------------------------------------------------------ */
int ab_version(void);
const char* ab_last_error(void);
/* Number of kernels this library launched since load (evidence counter). */
int64_t ab_launch_count(void);


/* ---- K1: packed mass matrix + lumped mass -------------------------------
 * Replaces build_packs' Jacobians + assemble_packs (reference
 * assembly.py:129-141, :178-244) and scatter_global(...).row_sums()
 * (assembly.py:306-333).  For category `cat`: Ae[e][i][j] =
 * sum_g |detJ|_g w_g N_i N_j (Gauss ascending), J[e][g] = |detJ|_g, and
 * ml[node] += sum_j Ae[e][i][j].  Each output pointer may be NULL.
 * `tile` = elements per CTA (the pack size of the reference, <= 1024). */
int ab_mass(const ab_mesh* mesh, int32_t cat, double* ae, double* jdet, double* ml,
            int32_t tile, void* stream);

/* Register node windows for the category whose connectivity pointer is
 * `conn` (windowed gather/scatter); blk_ptr == NULL clears
 * them.  Elements are taken in blocks of `block` (must be 128): block b's
 * unique nodes are wnode[blk_ptr[b] .. blk_ptr[b+1]); window node k
 * collects the element slots wslot[wptr[k] .. wptr[k+1]) (slot offset
 * a * block + local element); loc[e][a] is the window index of element e's node
 * a; desc[b] = {blk_ptr[b], blk_ptr[b+1], wptr[blk_ptr[b]],
 * wptr[blk_ptr[b+1]]} (int32 x 4, nullable); wmax = largest window.  Every
 * K2/K4/K6 launch on that connectivity then gathers node data through the
 * shared-memory window and issues one fp64 reduction per (block, node)
 * instead of per (element, node); with `desc` it runs the persistent
 * two-stage pipelined kernel (bulk-async metadata, cp.async node gathers).
 * Every window array must be readable 16 bytes past its end. */
int ab_set_windows(const int32_t* conn, int32_t block, const int64_t* blk_ptr, const int32_t* wnode,
                   const int32_t* wptr, const uint16_t* wslot, const uint16_t* loc, const int32_t* desc,
                   int32_t wmax);
/* The pipelined kernels (desc != NULL) also need, per 128-element block b,
 * the block's 128 * nnode element-node references sorted by window node:
 * wref[b * 128 * nnode + j] = slot offset | (window index << 16), the last
 * block padded with 0xffff0000.  Thread t of the block then reduces
 * references t*nnode .. t*nnode+nnode-1 (one fp64 reduction per window node
 * it touches). */
int ab_set_window_refs(const int32_t* conn, const uint32_t* wref);
/* Colour mode of the pipelined kernels (the north star's "mesh colouring"
 * scatter, chosen against fp64 atomics by measurement): the
 * category's blocks are processed colour by colour (corder: block ids grouped
 * by colour, cptr [ncol+1] offsets), no two blocks of a colour share a window
 * node, and every node sum is formed in a fixed order, so K2/K4/K6 results
 * are bitwise reproducible run to run (the reference's scatter_global sums in
 * a fixed order, assembly.py:317-326).  gbar: ncol device uint32 (one
 * barrier counter per colour).  ncol 0 / NULL corder restores the fp64-atomic
 * scatter. */
int ab_set_window_colours(const int32_t* conn, int32_t ncol, const int32_t* corder, const int64_t* cptr,
                          uint32_t* gbar);
/* Jones-Plassmann colouring of the window blocks (setup): blocks b, b' are
 * neighbours when they share a window node; nptr/nblk: node -> blocks CSR
 * (N+1 / n_window_entries); flags: 2 device int32 scratch.  Synchronises the
 * stream once per round; colour[b] in [0, 64). */
int ab_colour_blocks(int64_t n_blocks, const int64_t* blk_ptr, const int32_t* wnode, const int64_t* nptr,
                     const int32_t* nblk, int32_t* colour, int32_t* flags, void* stream);

/* ---- Partition file I/O (host; reference sfc.py:385-417 `part 1` body) ----
 * ab_format_partition: lines "i parts[i]\n" for i = first .. first+n-1 into
 * buf (capacity cap); returns bytes written or < 0.  ab_parse_partition:
 * parts[id] = subdomain for every "id subdomain" line of buf (the file after
 * its header line); every id in [0, n) exactly once (seen: n bytes scratch);
 * returns lines parsed or < 0 (malformed, out of range, duplicate).  Replace
 * the per-element Python loops of store_partition / load_partition. */
int64_t ab_format_partition(const int32_t* parts, int64_t first, int64_t n, char* buf, int64_t cap);
int64_t ab_parse_partition(const char* buf, int64_t len, int32_t* parts, int64_t n, uint8_t* seen);

/* Vreman filter width of category k: delta2[e] = V_e^(2/3) (device, E_k
 * doubles; geometry only, computed once).  ab_set_filter_width registers it
 * for the category with connectivity `conn` and n_elem elements (delta2 NULL
 * clears); K2 then reads it
 * instead of evaluating the cube root per element and stage (same values). */
int ab_filter_width(const ab_mesh* m, int32_t k, double* delta2, void* stream);
int ab_set_filter_width(const int32_t* conn, int64_t n_elem, const double* delta2);

/* ---- K2: momentum RHS (EMAC convection + viscous + Vreman) --------------
 * New entry point; rhs4 accumulated. */
/* Diagnostics: grid size and element-block count of the most recent
 * pipelined (persistent) element kernel launched by the calling thread. */
int ab_last_pipe_shape(int64_t* grid, int64_t* n_blocks);
int ab_momentum_rhs(const ab_mesh* mesh, const ab_phys* phys, const double* u4, double* rhs4,
                    void* stream);

/* ---- K8: boundary assembly of the equilibrium wall model ---------------
 * (Algorithm 1 line 4).  Wall faces as
 * node quadruples (-1 in slot 3 for triangles) plus the off-face nodes of
 * the owning element (-1 padded) that define the exchange point; rhs4
 * accumulates -rho u_tau^2 u_t/|u_t| A/n_face_nodes per face node, u_tau
 * from Reichardt's law. */
typedef struct ab_wall {
  int64_t n_faces;
  const int32_t* face;  /* [n_faces][4] */
  const int32_t* off;   /* [n_faces][4] */
  /* optional fixed-order accumulation (all NULL/0: fp64 reductions per face
   * node): the face tractions go to ftrac [n_faces][3], then each of the
   * n_nodes wall nodes node[i] adds the tractions of its faces
   * fref[ptr[i] .. ptr[i+1]) (ascending face ids) in that order, so K8's
   * result is bitwise reproducible. */
  int64_t n_nodes;
  const int32_t* node;  /* [n_nodes] wall node ids */
  const int64_t* ptr;   /* [n_nodes + 1] */
  const int32_t* fref;  /* faces of each wall node, ascending */
  double* ftrac;        /* [n_faces][3] scratch */
} ab_wall;
int ab_wall_traction(const ab_wall* w, const ab_phys* phys, const double* coords4, const double* u4, double* rhs4,
                     void* stream);

/* ---- K4: divergence  out[a] += scale * sum_e int N_a div(u) ------------- */
int ab_divergence(const ab_mesh* mesh, const double* u4, double scale, double* out, void* stream);

/* ---- K6: gradient  out4[a] += scale * sum_e int N_a grad(p) ------------- */
int ab_gradient(const ab_mesh* mesh, const double* p, double scale, double* out4, void* stream);

/* ---- Laplacian L_ab = int grad N_a . grad N_b ------------
 * Values accumulated into a CSR whose pattern (row_ptr, sorted cols) the
 * caller built from the connectivity. */
int ab_laplacian_csr(const ab_mesh* mesh, const int64_t* row_ptr, const int32_t* cols, double* vals,
                     void* stream);
/* Dirichlet rows/cols -> identity (fixed[i] != 0), pattern kept. */
int ab_csr_dirichlet(int64_t n_rows, const int64_t* row_ptr, const int32_t* cols, double* vals,
                     const uint8_t* fixed, void* stream);
/* CSR -> SELL-32 (slice_ptr prepared by the caller from per-slice widths). */
int ab_csr_to_sell(int64_t n_rows, const int64_t* row_ptr, const int32_t* cols, const double* vals,
                   const int64_t* slice_ptr, int32_t* sell_cols, double* sell_vals, double* diag,
                   void* stream);
/* y = A x */
int ab_sell_spmv(const ab_sell* a, const double* x, double* y, void* stream);

/* ---- K5: Jacobi-PCG kernels --------------------
 * Vectors x, r, z, p, q (and t for decomposed domains), dinv are [n].  The
 * SpMV is applied to z and A p is formed recursively: p = z + beta p_old,
 * q = A z + beta q_old (one 8-byte gather per non-zero).  `red` = 8 doubles
 * of reduction results, `sc` = 8 doubles of solver scalars, `part` =
 * partial-sum scratch (>= 2*(nb + ng) doubles, nb = ceil(n/256),
 * ng = ceil(nb/64)), `cnt` = 1 + ng zero-initialised uint32 counters
 * (two-level deterministic grid reduction, re-armed by the kernels).  `own`
 * (nullable) = per-row ownership weights for the dots of a decomposed domain.
 *   init:   r = fixed ? 0 : b; b = 0 (if b_zero); x = p = q = 0; z = dinv r;
 *           red[RZN] = r.z, red[RR] = r.r, sc[RZ] = 0
 *   set_bb: sc[BB] = red[RR]
 *   spmv:   with_dot: beta = sc[RZ] ? red[RZN]/sc[RZ] : 0; p = z + beta p;
 *           q = A z + beta q; red[PQ] = p.q; sc[RZ] = red[RZN]
 *           !with_dot (decomposed): t = (A z)_local only
 *   dot:    (after the interface sum of t) p = z + beta p; q = t + beta q;
 *           red[PQ] = p.q; sc[RZ] = red[RZN]
 *   update: alpha = red[PQ] ? sc[RZ]/red[PQ] : 0; x += alpha p; r -= alpha q;
 *           z = dinv r; red[RZN] = r.z; red[RR] = r.r                      */
#define AB_RED_RZN 0
#define AB_RED_RR 1
#define AB_RED_PQ 2
#define AB_RED_ITERS 3
#define AB_RED_RQ 6    /* tiled single-pass CG (ab_cg_tile_iter): r'.q */
#define AB_RED_QQ 7    /* tiled single-pass CG: q.q */
#define AB_RED_FAIL 5  /* sticky failure flag of the decomposed solvers (1.0 = a peer wait timed out) */
#define AB_SC_RZ 0
#define AB_SC_BB 1
int ab_cg_init(int64_t n, const double* b_in, double* b_zero, const uint8_t* fixed, const double* dinv,
               double* x, double* r, double* z, double* p, double* q, const double* own, double* red, double* sc,
               double* part, uint32_t* cnt, void* stream);
int ab_cg_set_bb(double* red, double* sc, void* stream);
/* Single domain on P A P^T: ab_cg_init + ab_cg_set_bb with the right-hand
 * side read in node order, r_i = b[perm[i]] (b[perm[i]] = 0 if zero_b);
 * fixed, dinv in row order.  ab_perm_scatter: out[perm[i]] = in[i] (x back
 * to node order). */
int ab_cg_init_perm(int64_t n, const int64_t* perm, double* b, int32_t zero_b, const uint8_t* fixed,
                    const double* dinv, double* x, double* r, double* z, double* p, double* q, double* red, double* sc,
                    double* part, uint32_t* cnt, void* stream);
int ab_perm_scatter(int64_t n, const int64_t* perm, const double* in, double* out, void* stream);
/* Symmetrically scaled single-domain form: Jacobi-PCG on A is plain CG on
 * A' = D^-1/2 A D^-1/2 (same iterates in exact arithmetic), with r' =
 * D^-1/2 r playing z's role, so per iteration neither z nor D^-1 moves (16
 * bytes per row less).  ab_sell_symscale: vals *= s_row s_col (s = d^-1/2,
 * row order, on a copy the caller owns); init: r'_i = s_i b[perm[i]];
 * the SpMV is ab_cg_spmv with z := r'; update: x' += alpha p,
 * r' -= alpha q, red[RZN] = r'.r', red[RR] = sum d r'^2 (d non-NULL, when a
 * tolerance is tested) or r'.r'; finish: out[j] = s_i x'_i, i = iperm[j]
 * (the inverse permutation: coalesced writes). */
int ab_sell_symscale(const ab_sell* a, const double* s, void* stream);
/* The scaled SpMV with A' stored WITHOUT its diagonal (every diagonal entry
 * of A' is 1): q = A' z + beta q as z + offdiag . z (ab_cg_spmv with_dot,
 * own = NULL, otherwise). */
int ab_cg_spmv_unit(const ab_sell* a, const double* z, double* p, double* q, double* red, double* sc, double* part,
                    uint32_t* cnt, void* stream);
int ab_cg_init_scaled(int64_t n, const int64_t* perm, double* b, int32_t zero_b, const uint8_t* fixed,
                      const double* s, const double* d, double* x, double* r, double* p, double* q, double* red,
                      double* sc, double* part, uint32_t* cnt, void* stream);
int ab_cg_update_scaled(int64_t n, const double* p, const double* q, double* x, double* r, const double* d,
                        double* red, const double* sc, double* part, uint32_t* cnt, void* stream);
int ab_cg_finish_scaled(int64_t n, const int64_t* iperm, const double* s, const double* x, double* out,
                        void* stream);
int ab_cg_spmv(const ab_sell* a, const double* z, double* p, double* q, double* t, int32_t with_dot,
               const double* own, double* red, double* sc, double* part, uint32_t* cnt, void* stream);
int ab_cg_dot(int64_t n, const double* z, const double* t, double* p, double* q, const double* own, double* red,
              double* sc, double* part, uint32_t* cnt, void* stream);
int ab_cg_update(int64_t n, const double* p, const double* q, const double* dinv, double* x, double* r, double* z,
                 const double* own, double* red, const double* sc, double* part, uint32_t* cnt, void* stream);

/* Launch shape of the resident CG (one cooperative CTA per SM, each owning a
 * contiguous, slice-aligned row range): returns 1 when the per-CTA rows fit
 * the shared-memory vectors (x, r, z, p, q), and reports rows_per_cta/n_cta. */
int ab_cg_resident_fits(int64_t n, int64_t* rows_per_cta, int32_t* n_cta);

/* CTA-local column map of a SELL matrix for the resident CG (DESIGN.md
 * §4.3): CTA b owns rows [b*rows_per_cta, (b+1)*rows_per_cta) (the launch
 * shape of ab_cg_resident_fits); its remote columns ("ghost rows") are
 * ghost[ghost_ptr[b] .. ghost_ptr[b+1]) ascending, and cols[k] (same layout
 * as ab_sell.cols) is the local index of entry k: c - row0 for an own row,
 * rows_per_cta + g for ghost g.  rows_per_cta + max_ghost <= 65536.
 * perm (nullable): the matrix is P L P^T, row i of the system is node
 * perm[i] (a compact, SFC-ordered numbering keeps the ghost sets small);
 * b_in, b_zero and x are then in node order, fixed and dinv in row order.
 * prefetch_depth: SELL slices per warp bulk-prefetched into L2 ahead of
 * use (also across the grid barriers, so the matrix stream of the next
 * iteration starts while the reductions complete). */
typedef struct ab_cg_local {
  int64_t rows_per_cta;
  int32_t n_cta;
  int32_t max_ghost;
  const uint16_t* cols;
  const int32_t* ghost_ptr;  /* [n_cta+1] */
  const int32_t* ghost;
  const int32_t* perm;       /* [n_rows] or NULL */
  int32_t prefetch_depth;
  int32_t variant;           /* must be 0 (the tensor-memory and single-reduction variants
                                measured slower and live in tools/lab/cg_rejected_variants.cu) */
  const unsigned char* packed;  /* reserved (NULL) */
  int32_t group;                /* reserved (0) */
  int32_t force_mode;        /* variant 0: 0 = best shared-memory plan; 1..4 = the plan of
                                ab_cg_resident_local_fits (testing: every plan is exercised) */
  /* the CTAs owning each CTA's ghost rows, nbr[nbr_ptr[b] .. nbr_ptr[b+1])
   * (informational; NULL allowed) */
  const int32_t* nbr_ptr;
  const int32_t* nbr;
} ab_cg_local;
/* Tiled ab_cg_spmv_unit: CTA b owns rows [b R, (b+1) R), R = m->rows_per_cta
 * (a multiple of 64, m->n_cta * R >= n_rows, R + max_ghost <= 65536); it
 * stages z of its rows and of its ghost rows (m->ghost[m->ghost_ptr[b] ..
 * m->ghost_ptr[b+1]), the remote columns) in shared memory and reads the
 * slices of `a` (values; same entry order) with the 16-bit tile-local
 * columns m->cols (own row: c - b R, ghost g: R + g).  p and q are bitwise
 * those of ab_cg_spmv_unit; red[PQ] sums per-tile partials (rounding-level
 * different).  m->perm, prefetch_depth, variant, force_mode,
 * nbr are ignored. */
int ab_cg_spmv_tile(const ab_sell* a, const ab_cg_local* m, const double* z, double* p, double* q, double* red,
                    double* sc, double* part, uint32_t* cnt, void* stream);
/* Tiled single-pass scaled CG: ONE kernel per iteration on the same tiles
 * (rows_per_cta = 1024, 2048 or 4096) and A' without its unit diagonal.
 * Vectors as 16-byte pairs: xp[i] = (x'_i, p_i), in place; rq[i] = (r'_i,
 * q_i), ping-pong between two buffers (iteration k reads rq_in, writes
 * rq_out; the next swaps them).  Iteration: alpha = red[RZN]/red[PQ] (0 if
 * PQ == 0), beta = (RZN - 2 alpha red[RQ] + alpha^2 red[QQ]) / RZN; per row
 * r' -= alpha q (own and ghost rows, staged in shared memory), x' += alpha
 * p, p = r' + beta p, q = A' r' + beta q; then red[RZN] = r'.r', red[RR] =
 * sum d r'^2 (d non-NULL) or r'.r', red[PQ] = p.q, red[RQ] = r'.q, red[QQ] =
 * q.q.  init: rq = (s_i b[perm[i]], 0), xp = 0, red[PQ] = red[RQ] =
 * red[QQ] = 0, sc[BB] = red[RR] (b zeroed if zero_b).  After K iterations x'
 * holds x'_{K-1}: finish with apply = 1 adds the last alpha p (= K
 * iterations of the two-kernel loop), apply = 0 returns x'_{K-1} (tolerance
 * met); out[j] = s_i x'_i, i = iperm[j].  part: >= 5 (nb + nb/64 + 1)
 * doubles, nb = ceil(n / 256). */
int ab_cg_tile_init(int64_t n, const int64_t* perm, double* b, int32_t zero_b, const uint8_t* fixed,
                    const double* s, const double* d, double* xp, double* rq, double* red, double* sc, double* part,
                    uint32_t* cnt, void* stream);
int ab_cg_tile_iter(const ab_sell* a, const ab_cg_local* m, const double* rq_in, double* rq_out, double* xp,
                    const double* d, double* red, double* part, uint32_t* cnt, void* stream);
int ab_cg_tile_finish(int64_t n, const int64_t* iperm, const double* s, const double* xp, const double* red,
                      int32_t apply, double* out, void* stream);
/* Diagnostics: buf (device, >= 8 * n_cta int64, or NULL to disable) receives
 * globaltimer stamps of the resident solver's phase boundaries in iteration
 * 10 (per CTA: loop top, ghosts gathered, phase A reduced, barrier A,
 * phase B reduced, barrier B). */
int ab_debug_timeline(int64_t* buf);
/* 0: does not fit; otherwise 1 + (x kept in shared memory) + 2 * (the CTA's
 * slice pointers and ghost ids copied to shared memory) */
int ab_cg_resident_local_fits(int64_t rows_per_cta, int32_t max_ghost);
/* Resident Jacobi-PCG: init + up to `maxit` iterations (stop when
 * ||r||/||b|| <= tol, tested on the device; tol = 0 runs exactly maxit) in
 * one cooperative kernel, one CTA per SM; each CTA keeps its rows' vectors
 * on chip (x in tensor memory, r, p, q, z in shared memory), fetches its
 * ghost z values once per iteration, and the SpMV reads z through the
 * 16-bit local columns.  Same iterates as the two-kernel form above.
 * Outputs: x, z (scratch); red[RZN], red[RR], red[ITERS]; sc[BB].  `part` >=
 * 8 * n_cta + 20 * ceil4(n_cta) doubles (grid-barrier counter at 5 * n_cta,
 * replicated partial tables from 8 * n_cta). */
int ab_cg_resident_local(const ab_sell* a, const ab_cg_local* m, const double* b_in, double* b_zero,
                         const uint8_t* fixed, const double* dinv, double* x, double* z, int32_t maxit, double tol,
                         double* red, double* sc, double* part, void* stream);

/* ---- discrete gradient operator B_ab = int N_a grad N_b ----------------
 * (DESIGN.md §4).  Assembled once into the Laplacian's CSR pattern (3
 * value planes), stored as SELL-32 with three lane-innermost value planes;
 * K4 and K6(+K7) become sparse products streaming it at HBM speed. */
typedef struct ab_sell3 {
  int64_t n_rows;
  int64_t n_slices;
  const int64_t* slice_ptr;
  const int32_t* cols;
  const double* vx;
  const double* vy;
  const double* vz;
} ab_sell3;
int ab_gradop_csr(const ab_mesh* mesh, const int64_t* row_ptr, const int32_t* cols, double* vx, double* vy,
                  double* vz, void* stream);
/* K4:  out[a] += scale * sum_b B_ab . u4[b]  (replaces ab_divergence) */
int ab_gradop_div(const ab_sell3* b, const double* u4, double scale, double* out, void* stream);
/* K6:  out4[a] += scale * sum_b B_ab p[b]  (replaces ab_gradient) */
int ab_gradop_grad(const ab_sell3* b, const double* p, double scale, double* out4, void* stream);
/* K6 + K7 in one pass: gd = B dp; uout = uin - k*minv*gd; p += dp; gp += gd
 * (single domain: no interface sum between K6 and K7).  uin may == uout. */
int ab_gradop_correct(const ab_sell3* b, const double* dp, double k, const double* uin, double* uout,
                      const double* minv, double* p, double* gp, void* stream);

/* ---- K5 across ranks: resident CG fused with its interface exchange ----
 * (DESIGN.md §5).  One cooperative kernel per rank solves the decomposed
 * system without leaving the GPU: after the local SpMV every CTA writes the
 * partial products of its interface rows straight into the neighbours'
 * receive arrays (peer memory over NVLink, or the same device for virtual
 * ranks), signals per-peer arrival counters, and adds what the neighbours
 * sent; both dot products are reduced across CTAs (grid barrier) and then
 * across ranks through {value, epoch} records written into every rank's
 * reduction slots.  Counters and epochs are monotone over the whole run
 * (evbase), so no buffer is ever reset while a peer may write to it.
 * One launch may host several ranks ("virtual ranks": CTA groups of one
 * cooperative grid on one GPU), which is how the protocol is tested on a
 * single GPU; across GPUs every rank launches its own group and the peer
 * pointers come from ab_ipc_* handles. */
#define AB_DD_MAX_PEERS 8
typedef struct ab_cg_dd_rank {
  int64_t n_rows, rows_per_cta;
  int32_t cta0, n_cta;                /* CTAs [cta0, cta0 + n_cta) of the launch */
  int32_t max_ghost, rank;
  int32_t n_ranks, pad0_;
  const int64_t* slice_ptr;           /* SELL-32 of the rank's P L P^T (SFC row order) */
  const uint16_t* cols;               /* CTA-local columns (ab_cg_local) */
  const double* vals;
  const int32_t* ghost_ptr;           /* [n_cta + 1] */
  const int32_t* ghost;
  const int32_t* perm;                /* row -> local node (b, x are in node order) */
  const double* dinv;                 /* row order; D of the assembled global operator */
  const uint8_t* fixed;               /* row order, nullable */
  const double* own;                  /* row order: 1 on the rank owning the node, else 0 */
  const double* b_in;
  double* b_zero;                     /* nullable */
  double* x_out;
  double* zg;                         /* [n_rows] scratch */
  double* red;                        /* RZN, RR, -, ITERS (-1: peer timeout) */
  double* sc;                         /* BB */
  double* part;                       /* >= 6 * n_cta */
  unsigned* bar;                      /* [2] zeroed before every solve: grid barrier, failure flag */
  /* interface: rows whose partial products are exchanged */
  const uint32_t* ifmask;             /* bit per row */
  const int32_t* send_ptr;            /* [n_rows + 1] per row into send_peer/send_off (interface rows only) */
  const int32_t* send_peer;           /* index into peer_* */
  const int32_t* send_off;            /* offset in that peer's recv array */
  const int32_t* rrow_ptr;            /* [n_cta + 1] per CTA into rrow */
  const int32_t* rrow;                /* interface rows, ascending */
  const int32_t* recv_ptr;            /* [n_if + 1] per interface row into recv_off */
  const int32_t* recv_off;            /* offsets into recv, ascending peer rank */
  double* recv;                       /* written by the peers */
  unsigned long long* cnt_in;         /* [n_ranks]: CTAs of rank q done sending (monotone) */
  double* red_in;                     /* [3][n_ranks][2][2]: {value, epoch} records per set, rank, value */
  unsigned long long* evbase;         /* [2]: halo events, reduction epochs completed before this solve */
  int32_t n_peers;
  int32_t recv_stride;                /* M: recv slot q * M + k holds rank q's k-th value */
  int32_t peer_rank[AB_DD_MAX_PEERS];
  int32_t peer_ncta[AB_DD_MAX_PEERS];
  double* peer_recv[AB_DD_MAX_PEERS];
  unsigned long long* peer_cnt[AB_DD_MAX_PEERS];  /* &peer.cnt_in[rank] */
  double* peer_red[AB_DD_MAX_PEERS];              /* &peer.red_in[0] */
} ab_cg_dd_rank;
/* Solve the ranks described by groups[0 .. n_groups) (device array) in one
 * cooperative launch of sum(n_cta) CTAs; x0 = 0, exactly maxit iterations
 * or until ||r||/||b|| <= tol (identical decision on every rank). */
int ab_cg_dd(const ab_cg_dd_rank* groups_dev, int32_t n_groups, int32_t n_cta_total, int32_t maxit, double tol,
             int64_t max_rows_per_cta, int32_t max_ghost, void* stream);
/* CUDA IPC: export the allocation holding dev_ptr (64-byte handle + the
 * pointer's offset in it) / map a peer's allocation (returns its base). */
int ab_ipc_get_handle(const void* dev_ptr, unsigned char* handle64, int64_t* offset);
int ab_ipc_open_handle(const unsigned char* handle64, void** dev_ptr);
int ab_ipc_close(void* dev_ptr);

/* ---- Peer-memory interface exchange and decomposed CG for large subdomains
 * (DESIGN.md §5).  One process (rank) per GPU; the buffers a rank's peers
 * write into (recv, cnt_in, rec) are mapped into every peer with CUDA IPC
 * (ab_ipc_*), or are plain device pointers when several ranks share one GPU
 * in one process ("virtual ranks", tests).  All progress state (exchange
 * counts, record epochs, iteration counter, scalars) lives in device memory,
 * so every entry point below is asynchronous on the caller's stream and a
 * whole multi-rank time step can be captured in one CUDA graph.  Waits
 * poll with acquire loads and never time out silently: after 10 s they set
 * the sticky failure word (state[AB_PS_FAIL] / scal[AB_D2_FAIL]) and return.
 *
 * Interface sum (element operators): node i of
 * this rank shared with ranks S_i gets  sum_{q in S_i + {rank}} f_q(i)  added
 * in ascending global rank order, so every copy of the node holds the same
 * bits on every rank.  Two launches: put (this rank's partials into the
 * sharers' receive slots + one release-add per CTA on their arrival
 * counters) and add (acquire-wait for the neighbours, rank-ordered sum).
 * The receive area is double-buffered by exchange parity, which is all a
 * neighbour can run ahead (its next put needs this rank's next put). */
#define AB_PEER_MAX 8
#define AB_PS_EV 0      /* exchanges completed (u64 words of `state`) */
#define AB_PS_TICK 1    /* arrival ticket of the add kernel */
#define AB_PS_FAIL 2    /* sticky failure flag */
typedef struct ab_peer_halo {
  int32_t rank, n_ranks;
  int32_t n_if;                       /* interface nodes of this rank */
  int32_t n_cta;                      /* CTAs of this rank's put kernel (a neighbour waits for that many) */
  int32_t max_shared;                 /* M: longest shared-node list of any rank pair (all ranks agree) */
  int32_t n_nbr;
  const int32_t* if_node;             /* [n_if] local node ids, ascending */
  const int32_t* if_ptr;              /* [n_if + 1] into if_rank / if_slot */
  const int32_t* if_rank;             /* sharing rank of each copy (ascending per node, this rank excluded) */
  const int32_t* if_slot;             /* index k of the node in the (this rank, that rank) shared list */
  double* recv;                       /* [2][n_ranks][M][3] written by the neighbours */
  unsigned long long* cnt_in;         /* [n_ranks] put-CTA arrivals from rank q (monotone) */
  unsigned long long* state;          /* [4] AB_PS_* */
  int32_t nbr_rank[AB_PEER_MAX];
  int32_t nbr_ncta[AB_PEER_MAX];      /* put CTAs of that neighbour */
  double* nbr_recv[AB_PEER_MAX];      /* the neighbour's recv (mapped) */
  unsigned long long* nbr_cnt[AB_PEER_MAX];  /* &neighbour.cnt_in[rank] (mapped) */
} ab_peer_halo;
/* field[node * stride + c], c < ncomp <= 3 */
int ab_peer_halo_put(const ab_peer_halo* h, const double* field, int32_t ncomp, int32_t stride, void* stream);
int ab_peer_halo_add(const ab_peer_halo* h, double* field, int32_t ncomp, int32_t stride, void* stream);
int ab_peer_halo_grid(int32_t n_if);  /* the put kernel's CTA count for n_if interface nodes */

/* Decomposed Jacobi-PCG for subdomains too large to stay on chip (two
 * kernels + one small interface kernel per iteration, PAPER.md:327-330,
 * :449-454).  The rank's P L P^T is numbered with its interface rows FIRST
 * ([0, n_if), SFC order) and the interior rows after (SFC order), so the
 * blocks holding interface rows run first in the SpMV and their partial
 * products travel to the sharers while the interior rows stream:
 *   spmv    beta from the ranks' {r.z, r.r} records; t = (A z) per row;
 *           interface rows: t -> tif and into every sharer's receive slot,
 *           one release-add per signalling block; interior rows: p = z +
 *           beta p, q = t + beta q, p.q partials (grid sum -> scal)
 *   iface   wait for the neighbours' blocks; interface rows: (A z)_i = the
 *           sharers' partials summed in global rank order; p, q, p.q; the
 *           rank's p.q total -> {value, epoch} record into every rank
 *   update  alpha from the ranks' p.q records; x += alpha p, r -= alpha q,
 *           z = D^-1 r; {r.z, r.r} record into every rank
 * Records: the value is stored first, then the epoch with release
 * semantics; a reader acquires the epoch, then loads the value.  Every rank
 * sums the P records in rank order, so alpha, beta and the stopping
 * decision are identical everywhere.  Convergence (tol > 0) is decided on
 * the device; once done, later launches of the solve return immediately. */
#define AB_D2_IT 0        /* iterations completed (doubles of `scal`) */
#define AB_D2_DONE 1
#define AB_D2_BB 2
#define AB_D2_RZ0 3       /* rz of even / odd iterations: 3, 4 */
#define AB_D2_BETA 5
#define AB_D2_PQI 6       /* interior p.q of this rank */
#define AB_D2_EPOCH 7     /* publishes so far (monotone over the run, equal on all ranks) */
#define AB_D2_EPA 8       /* epoch of the last p.q record */
#define AB_D2_EPB 9       /* epoch of the last {r.z, r.r} record */
#define AB_D2_HEV 10      /* SpMV exchanges completed */
#define AB_D2_RR 11
#define AB_D2_FAIL 12     /* sticky failure flag (1.0 = a peer wait timed out) */
#define AB_D2_TOL 13
#define AB_D2_INT 16      /* single pass: this rank's interior dots of the current iteration, 16..20 */
#define AB_D2_NSCAL 24
typedef struct ab_ddcg2_rank {
  int64_t n_rows, n_if;
  int32_t rank, n_ranks;
  int32_t n_peers;                    /* every other rank (the reductions) */
  int32_t recv_stride;                /* M: recv slot q * M + k holds rank q's k-th shared row */
  const int64_t* slice_ptr;           /* SELL-32 of P L P^T (interface rows first) */
  const int32_t* cols;
  const double* vals;
  const double* dinv;                 /* row order, D of the assembled global operator */
  const uint8_t* fixed;               /* row order, nullable */
  const double* own;                  /* row order: 1 on the lowest sharing rank, else 0 */
  const double* s;                    /* scaled != 0: D^-1/2 (row order); the values are those of
                                         D^-1/2 P L P^T D^-1/2 and r' takes z's role (ab_sell_symscale) */
  const int32_t* perm;                /* row -> local node */
  double *x, *r, *z, *p, *q;          /* row order (z unused when scaled) */
  double* tif;                        /* [n_if] this rank's (A z) at the interface rows */
  const int32_t* send_ptr;            /* [n_if + 1] into send_peer / send_off */
  const int32_t* send_peer;           /* index into peer_* */
  const int32_t* send_off;            /* slot in that peer's recv */
  const int32_t* recv_ptr;            /* [n_if + 1] into recv_rank / recv_off */
  const int32_t* recv_rank;           /* sharing rank (ascending; this rank excluded) */
  const int32_t* recv_off;            /* slot in this rank's recv */
  double* recv;                       /* written by the neighbours */
  unsigned long long* cnt_in;         /* [n_ranks] signalling-block arrivals from rank q (monotone) */
  double* rec;                        /* [2 sets][n_ranks][2 values][value, epoch] written by every rank */
  double* part;                       /* grid partials */
  uint32_t* cnt;                      /* grid-sum counters (zeroed once) */
  double* scal;                       /* [AB_D2_NSCAL] */
  int32_t nsig;                       /* blocks of this rank's SpMV holding interface rows */
  int32_t scaled;                     /* symmetrically scaled form (see s) */
  int32_t peer_rank[AB_PEER_MAX];
  int32_t peer_nsig[AB_PEER_MAX];     /* that peer's signalling blocks (0: not a neighbour) */
  double* peer_recv[AB_PEER_MAX];     /* mapped */
  unsigned long long* peer_cnt[AB_PEER_MAX];  /* &peer.cnt_in[rank] (mapped) */
  double* peer_rec[AB_PEER_MAX];      /* &peer.rec[0] (mapped) */
  /* optional tiled SpMV (tile_rows > 0; NULL/0: the plain SELL gather): the
   * rows in tiles of tile_rows (1024, 2048 or 4096), per tile its ghost rows
   * tghost[tghost_ptr[b] .. tghost_ptr[b+1]) and 16-bit tile-local columns
   * tcols in the entry order of `cols` (ab_cg_spmv_tile's map); nsig and the
   * peers' peer_nsig then count tiles: ceil(n_if / tile_rows) */
  const uint16_t* tcols;
  const int32_t* tghost_ptr;
  const int32_t* tghost;
  int32_t tile_rows;
  int32_t tmax_ghost;
  /* single pass (single_pass != 0; scaled form and a tile map required):
   * TWO launches per iteration, ab_ddcg2_tile_iter + ab_ddcg2_tile_iface,
   * with x', p as 16-byte pairs xp[n][2] and r', q as pairs in the ping-pong
   * buffers rq[0], rq[1] ([n][2] each; x, r, z, p, q unused).  init and
   * finish follow the mode. */
  double* xp;
  double* rq[2];
  int32_t single_pass;
  int32_t pad_sp_;
} ab_ddcg2_rank;
/* b (node order) -> r = b (fixed rows 0), z = D^-1 r, x = p = q = 0, and the
 * {r.z, r.r} record; b_zero (nullable) is zeroed.  tol is kept for the solve. */
int ab_ddcg2_init(const ab_ddcg2_rank* d, const double* b, double* b_zero, double tol, void* stream);
int ab_ddcg2_spmv(const ab_ddcg2_rank* d, void* stream);
int ab_ddcg2_iface(const ab_ddcg2_rank* d, void* stream);
int ab_ddcg2_update(const ab_ddcg2_rank* d, void* stream);
/* Single-pass iteration (d->single_pass): tile_iter forms r' -= alpha q
 * (own and ghost rows of each tile), x += alpha p, p = r' + beta p, q = A r'
 * + beta q and the dots of the interior rows, and sends the interface rows'
 * partial products; tile_iface waits for the neighbours' partials, forms the
 * interface rows' q in global rank order, adds their ownership-weighted dots
 * and publishes {r'.r', the ||r||^2 form, p.q, r'.q, q.q} to every rank
 * (record sets alternate per iteration); beta from the three-dot recurrence
 * of ab_cg_tile_iter.  The record array `rec` holds [2 sets][n_ranks][10]
 * doubles in both modes. */
int ab_ddcg2_tile_iter(const ab_ddcg2_rank* d, void* stream);
int ab_ddcg2_tile_iface(const ab_ddcg2_rank* d, void* stream);
/* x (row order) -> x_node[perm[i]] (single pass: x' + alpha p with alpha
 * from the last published records unless the solve converged, scaled by s) */
int ab_ddcg2_finish(const ab_ddcg2_rank* d, double* x_node, void* stream);
/* doubles of `part` / uint32 of `cnt` the kernels need for n_rows */
int64_t ab_ddcg2_part_size(int64_t n_rows);

/* ---- Session: the whole time step behind four calls ---------------------
 * (the plugin path it serves is the reference's bench
 * timer / balancing loop, cli.py:171-187, balance.py:241).
 *   ab_ctx_create(device)            context + setup stream on one GPU
 *   ab_mesh_upload(ctx, desc)        HOST arrays in; on the device: SFC element
 *                                    order, node windows, Vreman filter width,
 *                                    lumped mass, CSR pattern (sort/unique),
 *                                    Laplacian + Dirichlet, gradient operator,
 *                                    SELL-32, Hilbert row order of the pressure
 *                                    system (synchronous, setup only)
 *   ab_state_set / ab_state_get      u [n][3], p [n] from/to host or device
 *                                    memory (UVA), asynchronous on `stream`
 *   ab_step(ctx, dt, cg_iters, s)    one fractional step (Algorithm 1): 3 x
 *                                    (K2 + K8 + K3 + velocity BC), K4, Jacobi-PCG
 *                                    with cg_iters iterations on P L P^T, K6+K7;
 *                                    asynchronous, no host synchronisation
 *   ab_ctx_destroy(ctx)
 * One context per GPU, one stream at a time, not shared across threads.
 * Element node order and the bank-spread reference order of the Python setup
 * are not applied (results differ from FlowSolver's by rounding only). */
typedef struct ab_ctx ab_ctx;
typedef struct ab_mesh_desc {
  int64_t n_nodes;
  const double* coords;        /* [n_nodes][3], host */
  double period[3];            /* periodic box lengths, 0 = not periodic */
  int32_t n_cat, pad_;
  ab_category cat[5];          /* conn in HOST memory, reference VTK node order */
  const uint8_t* p_fixed;      /* [n_nodes] pressure Dirichlet nodes (nullable), host */
  const uint8_t* u_fixed;      /* [n_nodes] velocity Dirichlet bits: 1 x, 2 y, 4 z (nullable), host */
  const double* u_values;      /* [n_nodes][3] their values (nullable = 0), host */
  int64_t n_wall_faces;        /* wall-model faces (meshgen.wall_model_bcs), 0 = none */
  const int32_t* wall_face;    /* [n_wall_faces][4], host */
  const int32_t* wall_off;     /* [n_wall_faces][4], host */
  ab_phys phys;
} ab_mesh_desc;
typedef struct ab_ctx_info_t {
  int64_t n_nodes, nnz;
  int32_t n_cat, ready;
  int64_t n_elem[5];
  int64_t n_velocity_bc, n_wall_faces;
} ab_ctx_info_t;
int ab_ctx_create(int32_t device, ab_ctx** ctx);
int ab_ctx_destroy(ab_ctx* ctx);
int ab_mesh_upload(ab_ctx* ctx, const ab_mesh_desc* desc);
int ab_ctx_info(const ab_ctx* ctx, ab_ctx_info_t* info);
int ab_state_set(ab_ctx* ctx, const double* u, const double* p, void* stream);
int ab_state_get(ab_ctx* ctx, double* u, double* p, void* stream);
int ab_step(ab_ctx* ctx, double dt, int32_t cg_iters, void* stream);

/* ---- K3: fused RK stage update (one HBM pass) -------------
 *   uout = a*u0 + b*(uprev + k*minv*(rhs - gp));  rhs = 0 afterwards.     */
int ab_rk_stage(int64_t n, double a, double b, double k, const double* u0, const double* uprev,
                double* rhs, const double* gp, const double* minv, double* uout, void* stream);
/* ---- K7: velocity correction + pressure increment --
 *   uout = uin - k*minv*gd; p += dp; gp += gd; gd = 0.  (uin may == uout) */
int ab_correct(int64_t n, double k, const double* uin, double* uout, double* gd, const double* minv,
               double* p, const double* dp, double* gp, void* stream);
/* Dirichlet velocity values on a node list: u4[idx[i]][c] = vals[i][c] where mask bit c set. */
int ab_apply_velocity_bc(int64_t n_fixed, const int32_t* idx, const uint8_t* mask, const double* vals,
                         double* u4, void* stream);
/* minv = 1/ml */
int ab_reciprocal(int64_t n, const double* in, double* out, void* stream);

/* Ordered segmented sum out[s] = sum_{k in [seg_ptr[s], seg_ptr[s+1])} vals[k],
 * left to right: the global COO accumulation of scatter_global
 * (reference assembly.py:317-333) done bit-exactly on the device. */
int ab_segment_sum(int64_t n_seg, const int64_t* seg_ptr, const double* vals, double* out, void* stream);

/* ---- interface halo ------------------------
 * pack:   buf[i*ncomp + c] = field[idx[i]*stride + c]
 * unpack: field[idx[i]*stride + c] += buf[i*ncomp + c]                    */
int ab_halo_pack(int64_t n, const int32_t* idx, const double* field, int32_t stride, int32_t ncomp,
                 double* buf, void* stream);
int ab_halo_unpack_add(int64_t n, const int32_t* idx, const double* buf, int32_t stride, int32_t ncomp,
                       double* field, void* stream);

/* ---- decomposition (reference mesh.py:371-384, sfc.py:114-148, :184-192) -
 * centroid[e] = (sum_a x_a)/nnode in node order (matches numpy mean);
 * keys = Hilbert index of floor((c - lo)/span * 2^level) clipped.         */
int ab_centroids(const ab_mesh* mesh, int32_t cat, double* out, void* stream);
int ab_hilbert_keys(int64_t n, const double* centroids, const double* lo, const double* span,
                    int32_t level, int64_t* keys, void* stream);
int ab_hilbert_cells(int64_t n, const int64_t* cells, int32_t level, int64_t* keys, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* ALYAB200_H */
