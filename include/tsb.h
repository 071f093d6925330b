/*
 * tsb.h -- C ABI of the B200-native implicit-FEM solve path (libtsb.so).
 *
 * The reference (tetsim, /root/reference/pkg/src/tetsim) is pure Python +
 * NumPy and has no native interface; each entry point below replaces one
 * reference function on the hot path named by BASELINE.json's north_star and
 * is cited with the reference file:line it replaces.  The Python host layer
 * (paper_2306_05893_b200/) keeps the reference's API and calls these through
 * ctypes; INTEGRATION.md shows the binding a tetsim maintainer would add.
 *
 * Conventions
 *   - every pointer named d_* is a DEVICE pointer (cudaMalloc / torch CUDA
 *     storage); plain pointers are host memory;
 *   - indices are int32 (CSR row_ptr/col_ind, element connectivity), offsets
 *     into factor storage are int64;
 *   - every call is ordered on the caller's stream (`stream` is a
 *     cudaStream_t passed as void*, NULL = legacy default stream) and never
 *     synchronises unless documented (tsb_pcg_solve reads back one report);
 *   - return value: 0 = ok, otherwise a TSB_E_* code; the message is kept
 *     per thread and read with tsb_last_error().  Codes map to the reference
 *     exceptions (see paper_2306_05893_b200/_lib.py).
 *   - handles are opaque, bound to one stream at a time, not thread-safe.
 */
#ifndef TSB_H
#define TSB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TSB_ABI_VERSION 3

enum tsb_status {
    TSB_OK = 0,
    TSB_E_ASSEMBLY = 1,       /* assembly.AssemblyError        assembly.py:42-43   */
    TSB_E_STALE_MAPPING = 2,  /* assembly.StaleMappingError    assembly.py:46-47   */
    TSB_E_SOLVER = 3,         /* krylov.SolverError            krylov.py:34-35     */
    TSB_E_LIFECYCLE = 4,      /* ndprecond.LifecycleError      ndprecond.py:65-66  */
    TSB_E_CUDA = 5,           /* CUDA runtime failure (RuntimeError)               */
    TSB_E_MODEL = 6,          /* models.ModelError             models.py:37-38     */
    TSB_E_ARG = 7,            /* bad argument (ValueError)                         */
    TSB_E_PRECOND = 8         /* ndprecond.PrecondError        ndprecond.py:57-58  */
};

int tsb_abi_version(void);
/* Copies the calling thread's last error message into buf (NUL-terminated). */
int tsb_last_error(char *buf, size_t len);
/* Number of kernels libtsb launched in this process (for bench evidence). */
int64_t tsb_launch_count(void);
/* sizeof of the ABI structs (0 asm_plan, 1 asm_coeffs, 2 ldlt_block,
 * 3 ldlt_desc, 4 report, 5 ldlt_tile) so bindings can verify their layouts;
 * -1 = unknown. */
int64_t tsb_struct_size(int32_t which);

/* ------------------------------------------------------------------------
 * CSR SpMV  y = A x                        replaces krylov.spmv  krylov.py:73-96
 * Bit-identical to the reference: per row y_i = p_0 + pairwise(p_1..p_{L-1})
 * with p_k = a_k * x[col_k], i.e. np.add.reduceat's summation order
 * (krylov.py:63-70).
 * ---------------------------------------------------------------------- */
int tsb_spmv(int64_t nrows, const int32_t *d_row_ptr, const int32_t *d_col_ind,
             const double *d_values, const double *d_x, double *d_y, void *stream);

/* Diagonal of a CSR matrix        replaces CsrMatrix.diagonal  assembly.py:154-159 */
int tsb_csr_diagonal(int64_t nrows, int64_t ncols, const int32_t *d_row_ptr,
                     const int32_t *d_col_ind, const double *d_values, double *d_diag,
                     void *stream);

/* ------------------------------------------------------------------------
 * Triplet merge through a compression mapping
 *                       replaces assembly.compress / compress_parallel
 *                       assembly.py:322-376
 * values[s] = sum over kept triplets t with slot s, ascending t, of
 *             coeffs[t]*vals[t]   (coeffs may be NULL), starting from 0.0,
 * which is np.bincount's order (assembly.py:341); pinned diagonal slots := 1.0.
 * d_slot_ptr (nnz+1) / d_slot_trip: kept triplet ids grouped by slot.
 * ---------------------------------------------------------------------- */
int tsb_compress(int64_t nnz, const int64_t *d_slot_ptr, const int32_t *d_slot_trip,
                 const double *d_vals, const double *d_coeffs,
                 const int32_t *d_fixed_diag_slots, int64_t nfixed, double *d_values,
                 void *stream);

/* ------------------------------------------------------------------------
 * Fused corotational assembly         replaces
 *   BackwardEulerIntegrator.assemble_system  integrator.py:145-169
 *   corotational_forces_and_stiffness        models.py:200-238
 *   MatrixAssembler.finish / compress        assembly.py:407-419, 332-343
 * One element pass (F, polar R, rotated gradients, f_e = R Ke (R^T x - x0),
 * K v) followed by deterministic gathers into the fixed CSR pattern (slot
 * sums in ascending triplet order, mass triplets first) and into the nodal
 * vectors (ascending element order, np.bincount's order, models.py:192-193).
 * All arrays are SoA on the device and owned by the caller.
 * ---------------------------------------------------------------------- */
typedef struct tsb_asm_plan {
    int64_t n_nodes;            /* N                                         */
    int64_t n_elems;            /* m                                         */
    int64_t n_blocks;           /* CSR 3x3 node blocks with >=1 contribution  */
    int64_t nnz;                /* CSR nnz                                   */
    int64_t n_fixed_slots;      /* pinned diagonal slots                     */
    const int32_t *d_conn;      /* [4][m] element node ids                   */
    const double *d_grads;      /* [m][12] rest shape gradients (a*3+i)      */
    const double *d_vol;        /* [m] rest volumes                          */
    const double *d_mass_share; /* [m] rho*V/4 (integrator._mass_vals)       */
    const double *d_rest;       /* [3N] rest positions                       */
    const double *d_mass_diag;  /* [3N] lumped mass diagonal                 */
    const double *d_gravity;    /* [3N] gravity force M g                    */
    const uint8_t *d_fixed_dof; /* [3N] 1 = pinned                           */
    const int32_t *d_blk;       /* [nb][4] slot0, rowlen, list_begin, list_end */
    const int32_t *d_blk_list;  /* contributions e*16 + a*4 + b, sorted by (block, e) */
    const int32_t *d_node_ptr;  /* [N+1] incidence offsets                   */
    const int32_t *d_node_list; /* e*4 + a, ascending e per node             */
    const int32_t *d_fixed_slots; /* [n_fixed_slots]                         */
    double *d_work;             /* [48][m] scratch: [m][36] grads', f_e, K v_e; [m][12] F F^T, S (StVK) */
    int32_t *d_flags;           /* [4] device status words                   */
    const double *d_gab;        /* [m][10] rest-gradient products g_a.g_b (tsb_assembly_setup) */
    const int32_t *d_blk_mirror;/* [nb][2] or NULL: block k is (I, J), I <= J, and also writes the
                                   transposed block (J, I) at slot0 / rowlen d_blk_mirror[k]
                                   (slot0 -1: diagonal block); d_blk then lists only I <= J */
} tsb_asm_plan;

enum { TSB_LAW_COROTATIONAL = 0, TSB_LAW_LINEAR = 1, TSB_LAW_STVK = 2 };

typedef struct tsb_asm_coeffs {
    double lam, mu;             /* Lame constants (models.py:57-64)          */
    double h;                   /* dt                                        */
    double rayleigh_stiffness;  /* beta                                      */
    double rayleigh_mass;       /* alpha                                     */
    double cm, ck;              /* per-triplet coefficients (integrator.py:135-143) */
    int32_t law;                /* TSB_LAW_*: 0 corotational, 1 linear (R := I), 2 StVK */
    int32_t want_matrix;        /* 0: forces only (model.internal_forces)    */
} tsb_asm_coeffs;

/* x, v: [3N] positions/velocities; f_ext_state: [3N] state.f_ext.
 * Outputs: d_values [nnz], d_b, d_f_int, d_kv, d_f_ext [3N] (NULL allowed for
 * d_values when want_matrix == 0, and for d_b/d_f_ext).  d_flags[0] is set
 * to 1 when a position or deformation gradient is non-finite (ModelError);
 * the caller reads it back when it reads the solve report. */
/* Plan setup (once per plan): fills d_gab from d_grads. */
int tsb_assembly_setup(const tsb_asm_plan *plan, void *stream);

int tsb_assemble_corot(const tsb_asm_plan *plan, const tsb_asm_coeffs *coeffs,
                       const double *d_x, const double *d_v, const double *d_f_ext_state,
                       double *d_values, double *d_b, double *d_f_int, double *d_kv,
                       double *d_f_ext, void *stream);

/* Kinematic update of one implicit step   replaces integrator.py:192-208
 * d_flags[1] := 1 if an acceleration is non-finite (StepError); pinned DOFs
 * get accel 0 and keep v, x; v' = v + h a, x' = x + h v' (NumPy rounding). */
int tsb_advance(int64_t n_dof, const double *d_accel, const double *d_v, const double *d_x,
                const uint8_t *d_fixed_dof, double h, double *d_acc_out, double *d_v_out,
                double *d_x_out, int32_t *d_flags, void *stream);

/* Element stiffness blocks R Ke R^T as the reference emits them
 * (models.py:231, 196-197): d_kblocks [m][144], row-major per element.
 * Used only by the API-compatibility path that fills a TripletStream. */
int tsb_element_blocks(const tsb_asm_plan *plan, const tsb_asm_coeffs *coeffs,
                       const double *d_x, double *d_kblocks, void *stream);

/* ------------------------------------------------------------------------
 * Nested-dissection LDL^T preconditioner apply
 *   replaces solve_lower  ndprecond.py:647-671 (+ _forward_block 623-631)
 *            solve_upper  ndprecond.py:674-691 (+ _backward_block 634-644)
 *            apply        ndprecond.py:694-700, LdlFactors.apply 497-498
 * Factor values come from the host factorisation (ldlt_factor,
 * ndprecond.py:501-572) and are packed by the host into the layout below.
 * ---------------------------------------------------------------------- */
/* Block-inverse layout (built by the host from LdlFactors, _ldlt_pack.py).
 * For every dissection block b (permuted rows [start, start+m), ancestors
 * anc[0..na)) the host forms
 *     G_b = [ inv(L11) - I   (strict lower triangle, rows 1..m-1)      ]
 *           [ M = L21 inv(L11)  (na x m)                               ]
 * -- the reference's tile inverses (ndprecond.py:575-587) widened to the
 * whole diagonal block, with the coupling panel pre-multiplied by it:
 *   lower (solve_lower, ndprecond.py:647-671):  y_b = x_b + (Linv-I) x_b,
 *          contributions to the ancestors  c_b = M x_b  (column-major
 *          pre-accumulation of the paper, one GEMV per block, no in-block chain);
 *   upper (solve_upper, ndprecond.py:674-691):  z_b = w_b + G_b^T v,
 *          v = [w_b; -z_anc]  (row-major pull, one GEMV per block).
 * Each sweep's rows (lower: rows of G_b over v = x_b; upper: rows of G_b^T
 * over v = [w_b; -z_anc]) are grouped in tiles of 32 rows, one per lane:
 * tile i covers v-columns [tl, tl + 2 np) (tl even) and stores entry
 * (row row0 + k, column tl + 2p + h) at off + (p*32 + k)*2 + h (zeros
 * outside the row's range), so a warp reads 512 contiguous bytes per column
 * pair and every lane accumulates its own row.
 * Items (int4 {block, t0, t1, seg}): tiles [t0, t1) of one block, staged by
 * one TMA bulk copy (<= 48 KB) issued before the dependency wait, one warp
 * per tile; seg = s + 1: column segment s (48 KB) of one large tile, the 8
 * warps splitting its pairs; the tile's last segment to finish adds the
 * segments' partial sums in segment order (deterministic) and emits.
 * Lower: x_b = r_b - (contributions of its descendants), summed in a fixed
 * order either by each of the block's items (mode 1) or once by nfin
 * finaliser items {block, row0, row1, -1} dispatched before the block's
 * items (mode 2).  Upper: an item of b waits for
 * every item of b's parent (z_anc final). */
typedef struct tsb_ldlt_block {
    int32_t start, m, na, parent;   /* parent: block elimination-tree parent, -1 = root */
    int32_t target_l;               /* lower items of all children (x_b complete)  */
    int32_t n_u;                    /* upper items of this block (z_b complete)    */
    int32_t mode;                   /* lower input: 0 no contributions (leaf),
                                       1 every item sums the contributions itself,
                                       2 nfin finaliser items form x_b once        */
    int32_t ncb;                    /* contributions into the block's rows         */
    int32_t nfin;                   /* finaliser items (mode 2)                     */
    int32_t nu_parent;              /* n_u of the parent (0 at a root): the upper
                                       items' dependency target                    */
    int64_t anc_off;                /* offset of the block's anc rows in d_anc      */
    int64_t cb_off;                 /* first cbuf slot of the block's rows          */
} tsb_ldlt_block;

typedef struct tsb_ldlt_tile {
    int64_t off;                    /* offset of the tile in d_g / d_gt (doubles)  */
    int32_t tl;                     /* first v-column (even)                        */
    int32_t np;                     /* column pairs                                 */
    int32_t row0, nrows;            /* block rows [row0, row0 + nrows)              */
    int32_t nseg;                   /* 0: small tile; else 48 KB column segments   */
    int32_t part;                   /* first partial-sum slot (x 32 doubles)        */
} tsb_ldlt_tile;

typedef struct tsb_ldlt_desc {
    int64_t n;
    int64_t n_blocks;
    int64_t n_items_lower;
    int64_t n_items_upper;
    int32_t max_m;                /* largest block                                  */
    int32_t max_v;                /* largest m + na                                 */
    int32_t max_cb;               /* contribution staging (doubles, <= 4096)        */
    int32_t grid;                 /* persistent CTAs (0 = fill the GPU)             */
    const tsb_ldlt_block *d_blocks;
    const int32_t *d_items_lower; /* [n_items_lower][4], topological dispatch order */
    const int32_t *d_items_upper; /* [n_items_upper][4]                            */
    const tsb_ldlt_tile *d_tiles_lower;
    const tsb_ldlt_tile *d_tiles_upper;
    const double *d_g;            /* lower tiles                                    */
    const double *d_gt;           /* upper tiles                                    */
    const int32_t *d_anc;         /* permuted ancestor rows, per block             */
    const int32_t *d_cslot;       /* cbuf slot of (block, anc k)                    */
    const int64_t *d_cin_ptr;     /* [n+1]: row r's contributions are cbuf[cin_ptr[r]..cin_ptr[r+1]) */
    const double *d_d;            /* [n] D                                          */
    const int32_t *d_perm;        /* [n] perm[k] = original index at position k    */
    double *d_cbuf;               /* scratch: lower contributions                  */
    double *d_x;                  /* scratch [n]: contribution sums (mode 2) / z    */
    double *d_y;                  /* scratch [n]: lower result inside apply         */
    int32_t *d_cnt_l, *d_ready_l; /* [n_blocks] counters (zeroed; reset on exit)    */
    int32_t *d_done_u, *d_pad;    /* [n_blocks]                                     */
    double *d_part_lower;         /* scratch: segment partial sums (32 per slot)    */
    double *d_part_upper;
    int32_t *d_tcnt_lower;        /* [n_tiles_lower] segment counters (zeroed)      */
    int32_t *d_tcnt_upper;        /* [n_tiles_upper]                                */
    int64_t n_tiles_lower, n_tiles_upper;
    const int32_t *d_ext_rows;    /* rows outside the handle's blocks that receive  */
    int64_t n_ext;                /* contributions (block subsets of a shard)        */
    int32_t *d_ctl;               /* [4] tickets / exit counters (zeroed)          */
    int64_t *d_trace_lower;       /* optional [n_items_lower][8] item timeline     */
    int64_t *d_trace_upper;       /* optional [n_items_upper][8]                   */
    double *d_rin;                /* scratch [n]: apply's input gathered through perm once, so
                                     the lower sweep's items read it directly (NULL: gather per item) */
} tsb_ldlt_desc;

typedef struct tsb_ldlt *tsb_ldlt_t;

int tsb_ldlt_create(const tsb_ldlt_desc *desc, tsb_ldlt_t *out);
int tsb_ldlt_destroy(tsb_ldlt_t h);
/* y = L^{-1} r, both in permuted order                 (solve_lower) */
int tsb_ldlt_lower(tsb_ldlt_t h, const double *d_r, double *d_y, void *stream);
/* z = L^{-T} w, both in permuted order                 (solve_upper) */
int tsb_ldlt_upper(tsb_ldlt_t h, const double *d_w, double *d_z, void *stream);
/* z = P^T L^{-T} D^{-1} L^{-1} P r, original order     (apply)       */
int tsb_ldlt_apply(tsb_ldlt_t h, const double *d_r, double *d_z, void *stream);
/* Multi-RHS lower sweep (the compliance columns of build_compliance,
 * contact.py:109-125): y_j = L^{-1} r_j for nr
 * right-hand sides [nr][n] (permuted order) in one pass over the factor;
 * scratch cbuf [nr][ld_cb], x [nr][n], part [nr][ld_part]. */
int tsb_ldlt_lower_multi(tsb_ldlt_t h, int32_t nr, const double *d_r, double *d_y, double *d_cbuf, int64_t ld_cb,
                         double *d_x, double *d_part, int64_t ld_part, void *stream);
/* Block subsets (one rank's shard, paper_2306_05893_b200/shard.py), permuted order:
 * y = L^{-1} (r - ext) on the handle's blocks (d_ext may be NULL) */
int tsb_ldlt_lower_ext(tsb_ldlt_t h, const double *d_r, const double *d_ext, double *d_y, void *stream);
/* z = L^{-T} D^{-1} y on the handle's blocks; z of ancestor rows outside them
 * is read from d_z (solved before) */
int tsb_ldlt_upper_scaled(tsb_ldlt_t h, const double *d_y, double *d_z, void *stream);
/* after a lower sweep: d_out[row] = sum of the contributions to each external
 * row (d_ext_rows), fixed order */
int tsb_ldlt_external_sums(tsb_ldlt_t h, double *d_out, void *stream);

/* ------------------------------------------------------------------------
 * Device pattern build                 replaces build_pattern (assembly.py:
 *                                      235-312) for whole pinned nodes: the
 * same CSR (row_ptr, col_ind) and gather lists as _plan.topology_pattern.
 * Two calls: count (synchronises once, fills n_blocks / nnz), then fill
 * into caller-allocated outputs (synchronises once, fills n_contrib).
 * ---------------------------------------------------------------------- */
typedef struct tsb_pattern {
    int64_t n_nodes, n_elems;
    const int32_t *d_conn;        /* [4][m] element node ids                      */
    const uint8_t *d_pinned;      /* [N] 1 = pinned node                          */
    int64_t *d_tmp;               /* scratch [N]                                  */
    int64_t *d_sums;              /* scratch [max(N, n_blocks) / 1024 + 1]        */
    int64_t *d_node_ptr;          /* out [N + 1]                                  */
    int32_t *d_node_list;         /* out [4 m]: e*4 + a, ascending per node       */
    int32_t *d_cand;              /* scratch [16 m]: sorted neighbours per node   */
    int64_t *d_nbr;               /* out [N]: node blocks per node row            */
    int64_t *d_blk_ptr;           /* out [N + 1]                                  */
    int64_t *d_row_base;          /* out [N + 1]: first slot of row 3I            */
    int64_t n_blocks, nnz, n_contrib;  /* filled by the calls                    */
    int64_t *d_ccount;            /* scratch [n_blocks]                           */
    int64_t *d_cptr;              /* out [n_blocks + 1]                           */
    int32_t *d_row_ptr;           /* out [3N + 1]                                 */
    int32_t *d_col_ind;           /* out [nnz]                                    */
    int32_t *d_blk;               /* out [n_blocks][4]                            */
    int32_t *d_blk_list;          /* out [<= 16 m]                                */
} tsb_pattern;

int tsb_pattern_count(tsb_pattern *p, void *stream);
int tsb_pattern_fill(tsb_pattern *p, void *stream);

/* ------------------------------------------------------------------------
 * Plane contact stage                   replaces detect_plane_contacts,
 *                                       build_compliance,
 * projected_gauss_seidel, correct_motion (contact.py:89-195).  J is CSR over
 * the constraint rows (int64 indptr, int32 columns).  With LDL^T factors
 * W = Y^T D^-1 Y with Y = L^-1 P J^T (tsb_ldlt_lower per column) and
 * S lambda = P^T L^-T D^-1 (Y lambda) (one tsb_ldlt_upper_scaled).
 * ---------------------------------------------------------------------- */
/* nodes with z < plane_z in ascending order, their penetration, the count and
 * max(plane_z - z, 0); d_nodes / d_pen may be NULL (count + max only) */
int tsb_plane_contacts(int64_t n_nodes, const double *d_pos, double plane_z, int32_t *d_nodes, double *d_pen,
                       int64_t *d_count, double *d_maxpen, void *stream);
/* R[:, i] = J^T e_i (scattered through iperm when non-NULL), R n x m column-major */
int tsb_contact_rhs(int64_t m, const int64_t *d_indptr, const int32_t *d_cols, const double *d_coefs,
                    const int32_t *d_iperm, int64_t n, double *d_R, void *stream);
/* W = scale * Y^T diag(1/d) Y (d may be NULL: identity); d_part scratch of
 * tsb_gram_scratch(n, m) doubles */
int64_t tsb_gram_scratch(int64_t n, int64_t m);
int tsb_gram(int64_t n, int64_t m, const double *d_Y, const double *d_d, double scale, double *d_part, double *d_W,
             void *stream);
/* W = scale * (J S + (J S)^T) / 2 for solution columns S (n x m) */
int tsb_compliance_from_columns(int64_t m, int64_t n, const int64_t *d_indptr, const int32_t *d_cols,
                                const double *d_coefs, const double *d_S, double scale, double *d_W, void *stream);
/* lambda of W lambda = rhs, lambda >= 0 on unilateral rows; info: sweeps,
 * complementarity residual sum |lambda (W lambda - rhs)|, dropped rows */
int tsb_pgs(int64_t m, const double *d_W, const double *d_rhs, const uint8_t *d_unilateral, double tol,
            int32_t max_sweeps, double *d_lam, double *d_info, void *stream);
/* out = Y lambda (n x m column-major) */
int tsb_gemv_cols(int64_t n, int64_t m, const double *d_Y, const double *d_lam, double *d_out, void *stream);
/* acc = acc_free - delta (delta in permuted order when iperm is non-NULL) */
int tsb_contact_correct(int64_t n, const double *d_acc_free, const double *d_delta, const int32_t *d_iperm,
                        double *d_acc, void *stream);

/* ------------------------------------------------------------------------
 * Device LDL^T refactorisation        replaces ldlt_factor (numeric phase)
 *                                     ndprecond.py:501-572 (+ the host pack
 *                                     of the factor into the sweep layout)
 * Multifrontal over the dissection tree: per front F = [A_bb A_b,anc; A_anc,b 0]
 * + extend-added children updates, a tiled (64 x 64) partial Cholesky of its
 * m pivots gives C, LS = F21 C^-T and U = F22 - LS LS^T (sent to the parent);
 * a right triangular solve gives [C^-1; LS C^-1] and the pack writes
 * Linv = diag(C) C^-1 and M = LS C^-1 into the tiles of an existing
 * tsb_ldlt handle layout (d_g, d_gt) and d = diag(C)^2 into d_d.  The host
 * "program" (8 int64 per op, built once per pattern by
 * paper_2306_05893_b200/refactor.py) lists the launches in order.
 * ---------------------------------------------------------------------- */
typedef struct tsb_front {
    int64_t off;                  /* front F (nf x nf, column-major) in d_ws    */
    int64_t woff;                 /* C^-1 (m x m, column-major) in d_wb         */
    int64_t ioff;                 /* pivot-tile inverses (P x 2 x 64 x 64) in d_inv */
    int32_t m, na, nf, P, NT;     /* pivots, coupling rows, m + na, pivot tiles, tiles */
    int32_t start;                /* first permuted row                          */
} tsb_front;

typedef struct tsb_front_pair {   /* extend-add child -> parent                  */
    int32_t child, parent;
    int64_t tp_off;               /* child's na positions in the parent front    */
} tsb_front_pair;

enum {
    TSB_RF_SCATTER = 1,           /* a: entries                                  */
    TSB_RF_EXTEND = 2,            /* a, b: pair range; c: max child na           */
    TSB_RF_DIAG = 3,              /* a: k; b: list offset; c: fronts             */
    TSB_RF_PANEL = 4,             /* a: k; b: list offset; c: fronts; d: tasks   */
    TSB_RF_UPDATE = 5,            /* same                                        */
    TSB_RF_TSCALE = 6,            /* same (right solve, column tile k)           */
    TSB_RF_TUPDATE = 7,           /* same                                        */
    TSB_RF_PACK = 8,              /* pack tiles + d                              */
    TSB_RF_IDENT = 9,             /* C^-1 buffers := I                           */
    TSB_RF_RECORD = 10,           /* a: event id, recorded on the op's stream    */
    TSB_RF_WAIT = 11              /* a: event id, waited for by the op's stream  */
};
/* op[5] selects the stream: 0 the caller's, 1 a side stream of the handle
 * (the right solve of a finished tree height overlaps the next heights). */

typedef struct tsb_refactor_desc {
    int64_t n_fronts;
    int64_t n_prog;               /* ops                                          */
    const int64_t *h_prog;        /* HOST [n_prog][8]: op, a, b, c, d, 0, 0, 0    */
    const tsb_front *d_fronts;
    const int32_t *d_lists;       /* [.][4]: front, panel/scale prefix, update prefix, 0 */
    const int32_t *d_sc_src;      /* A entry (original CSR order) ...           */
    const int64_t *d_sc_dst;      /* ... -> d_ws offset (lower triangle only)   */
    const tsb_front_pair *d_pairs;
    const int32_t *d_tp;
    const tsb_ldlt_tile *d_tiles_lower;
    const tsb_ldlt_tile *d_tiles_upper;
    const int32_t *d_tile_blk_lower;  /* tile -> front (= handle block) */
    const int32_t *d_tile_blk_upper;
    int64_t n_tiles_lower, n_tiles_upper;
    double *d_ws;                 /* fronts                                       */
    double *d_wb;                 /* C^-1 blocks                                  */
    double *d_inv;                /* pivot-tile inverses                          */
    int64_t ws_size, wb_size;     /* doubles                                      */
    int32_t *d_ctl;               /* [1] first failing front + 1 (0 = ok)         */
} tsb_refactor_desc;

typedef struct tsb_refactor *tsb_refactor_t;

int tsb_refactor_create(const tsb_refactor_desc *desc, tsb_refactor_t *out);
int tsb_refactor_destroy(tsb_refactor_t h);
/* Factor the values of A (original CSR order) into d_g / d_gt / d_d of the
 * handle layout the program was planned for.  A non-positive pivot is
 * reported in d_ctl[0] (IndefiniteMatrixError), read by the caller. */
int tsb_refactor_run(tsb_refactor_t h, const double *d_values, double *d_g, double *d_gt, double *d_d,
                     void *stream);

/* ------------------------------------------------------------------------
 * Vector kernels of the sharded PCG (shard.py): weights w = 1 on owned rows
 * (top rows on rank 0 only); d_part scratch of 2 * 148 doubles.
 * ---------------------------------------------------------------------- */
int tsb_wdot(int64_t n, const double *d_w, const double *d_a, const double *d_b, double *d_part,
             double *d_out, void *stream);
/* alpha = d_sc[0] / d_sc[1]; x += alpha p; r -= alpha ap; d_out[0] = sum w r^2.
 * d_done (may be NULL): device stop flag -- when set, nothing is updated. */
int tsb_pcg_update(int64_t n, const double *d_w, double *d_x, const double *d_p, double *d_r,
                   const double *d_ap, const double *d_sc, double *d_part, double *d_out,
                   const int32_t *d_done, void *stream);
/* beta = d_sc[0] / d_sc[1]; p = z + beta p; d_sc[1] = d_sc[0] (skipped when *d_done) */
int tsb_pcg_direction(int64_t n, double *d_p, const double *d_z, double *d_sc, const int32_t *d_done,
                      void *stream);
/* Device-side stop test of the sharded loop (krylov.py:150-153): unless
 * *d_done, count the iteration (*d_it += 1), res = sqrt(*d_rr) / bnorm into
 * *d_res, and set *d_done when res <= tol or *d_it == max_it.  With it the
 * iterations can be replayed from a CUDA graph with no host read. */
int tsb_pcg_check(const double *d_rr, double bnorm, double tol, int64_t max_it, int32_t *d_done,
                  int64_t *d_it, double *d_res, void *stream);
int tsb_gather_rows(int64_t m, const int32_t *d_idx, const double *d_src, double *d_dst, void *stream);
/* All-reduce over peer memory (shard.PeerAllreduce, replaces the NCCL
 * all-reduce of the exchanges): x (rows d_idx[0..m), or the first m entries
 * when d_idx is NULL) := sum over ranks in rank order.  d_bufs[r], d_flags[r]:
 * rank r's exchange buffer (2 x half doubles) and epoch word as mapped in this
 * process (CUDA IPC).  `epoch` is ignored: each exchange takes one more than
 * the rank's own epoch word (device-side numbering, CUDA-graph replayable). */
int tsb_peer_allreduce(int64_t m, int32_t world, int32_t rank, double *const *d_bufs, int64_t *const *d_flags,
                       const int32_t *d_idx, double *d_x, int64_t epoch, int64_t half, void *stream);
/* tsb_ldlt_external_sums + peer all-reduce of d_out's rows d_idx[0..m) in one
 * kernel (the shard's forward-sweep exchange); d_ticket: one int32, zero. */
int tsb_ldlt_external_sums_peer(tsb_ldlt_t h, double *d_out, int64_t m, int32_t world, int32_t rank,
                                double *const *d_bufs, int64_t *const *d_flags, const int32_t *d_idx, int64_t epoch,
                                int64_t half, int32_t *d_ticket, void *stream);
/* Fused SpMV + peer all-reduce of the shared rows (one kernel: the last CTA
 * of the product runs the exchange).  d_ticket: one int32, initially zero. */
int tsb_spmv_peer(int64_t nrows, const int32_t *d_row_ptr, const int32_t *d_col_ind, const double *d_values,
                  const double *d_x, double *d_y, int64_t m, int32_t world, int32_t rank, double *const *d_bufs,
                  int64_t *const *d_flags, const int32_t *d_idx, int64_t epoch, int64_t half, int32_t *d_ticket,
                  void *stream);
int tsb_scatter_rows(int64_t m, const int32_t *d_idx, const double *d_src, double *d_dst, void *stream);

/* ------------------------------------------------------------------------
 * Device-resident preconditioned CG      replaces krylov.pcg / krylov.cg
 *                                        krylov.py:120-163
 * The iteration loop runs inside one CUDA graph with a conditional WHILE
 * node: alpha, beta and the convergence test live on the device, no host
 * round-trip per iteration; one report is read back per solve.
 * ---------------------------------------------------------------------- */
enum tsb_precond_kind {
    TSB_PRECOND_IDENTITY = 0,   /* IdentityPreconditioner  krylov.py:99-101  */
    TSB_PRECOND_JACOBI = 1,     /* jacobi_precond           krylov.py:104-117 */
    TSB_PRECOND_LDLT = 2        /* LdlFactors.apply         ndprecond.py:497  */
};

typedef struct tsb_report {     /* krylov.SolveReport  krylov.py:55-60       */
    int64_t iterations;
    double final_residual;
    int32_t converged;
    int32_t status;             /* 0 ok, 3 zero diagonal (SolverError)        */
    int64_t zero_diag_row;
} tsb_report;

typedef struct tsb_pcg *tsb_pcg_t;

int tsb_pcg_create(int64_t n, tsb_pcg_t *out);
int tsb_pcg_destroy(tsb_pcg_t h);
/* Solve A x = b.  d_x0 may be NULL (x0 = 0).  precond_kind selects the
 * preconditioner; ldlt is required for TSB_PRECOND_LDLT.  For Jacobi,
 * d_inv_diag (may be NULL) supplies 1/diag, otherwise the diagonal is
 * extracted from the matrix and inverted on the device.  d_x receives the
 * solution.  When `report` is non-NULL the call synchronises the stream
 * once and fills it; otherwise the report stays on the device
 * (tsb_pcg_report reads it later). */
int tsb_pcg_solve(tsb_pcg_t h, int64_t nrows, const int32_t *d_row_ptr,
                  const int32_t *d_col_ind, const double *d_values, const double *d_b,
                  const double *d_x0, double *d_x, int32_t precond_kind, tsb_ldlt_t ldlt,
                  const double *d_inv_diag, double tol, int64_t max_iterations,
                  tsb_report *report, void *stream);
int tsb_pcg_report(tsb_pcg_t h, tsb_report *report, void *stream);
/* Diagnostics of the last solve: CTA 0's device time (ns) in SpMV, barrier +
 * alpha, vector update, barrier + beta, preconditioner, whole loop. */
int tsb_pcg_phase_times(tsb_pcg_t h, int64_t *out6, void *stream);

/* ------------------------------------------------------------------------
 * Host setup (not on the per-iteration path): nested-dissection ordering
 *   replaces nested_dissection / _dissect / _greedy_cover / _pseudo_peripheral
 *   ndprecond.py:107-267  (same algorithm and tie-breaking, so the
 *   permutation and block tree are identical to the reference's)
 * Graph: CSR adjacency (sorted neighbour lists, no self loops).
 * Outputs (host, caller-allocated with capacity n for the per-block arrays
 * and n for children): perm[n], blocks in creation order.
 * ---------------------------------------------------------------------- */
int tsb_nested_dissection(int64_t n, const int64_t *indptr, const int64_t *indices,
                          int64_t leaf_threshold, int64_t *perm, int64_t *n_blocks,
                          int64_t *blk_start, int64_t *blk_stop, int64_t *blk_tree_start,
                          int32_t *blk_is_sep, int64_t *blk_child_ptr, int64_t *blk_child);

#ifdef __cplusplus
}
#endif
#endif /* TSB_H */
