/*
 * bddc_b200.h -- C-ABI of the B200 (sm_100a) adaptive-BDDC hot path.
 *
 * The reference (arXiv 2501.01676, package `adbddc`) is pure Python with
 * no FFI; its boundary for this path is the Python API.
 * Each entry point below replaces the LAPACK / SuperLU / numpy call sites
 * named in its comment (paths relative to /root/reference/pkg/src/adbddc).
 * The Python host package paper_2501_01676_b200 mirrors the reference's
 * functions on top of these calls; a ctypes binding is in
 * paper_2501_01676_b200/_lib.py and INTEGRATION.md shows how a maintainer
 * binds them from the reference side.
 *
 * Conventions
 *  - All pointers are DEVICE pointers (caller-owned, e.g. torch tensors);
 *    nothing allocates inside.  Work is ordered on `stream`.
 *  - Batched ("vbatched") dense matrices live in one buffer: matrix b starts
 *    at base + off[b], row-major, leading dimension ld[b] (or n[b]).
 *  - Return value: 0 = launched, < 0 = -cudaError_t of the launch.
 *    Numerical failures are written per batch member into the caller's
 *    device `status` array (0 = ok, see enum below); the host maps them to
 *    the reference's NumericalError messages.
 *  - Stateless and thread-safe apart from one-time kernel attribute setup.
 */
#ifndef BDDC_B200_H
#define BDDC_B200_H

#include <cuda_runtime.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
enum {
  BDDC_OK = 0,
  BDDC_NOT_POSITIVE_DEFINITE = 1, /* cho_factor failure (Bsym, deluxe sums, dual certificate) */
  BDDC_SINGULAR_PIVOT = 2,        /* zero / non-finite pivot (lu_factor on a singular block) */
  BDDC_NOT_PSD = 3,               /* pencil right-hand side not PSD (linalg.py:151-152) */
  /* per-glob kernels: 100 + sharer index  = glob Schur block singular
                       200 + status        = pencil failure                      */
};

/* ---- local.cu : substructuring -------------------------------------------- */

/* Symbolic plan, element part: local dof index (interior first, then the
 * glob-major interface block, 2^30 for Dirichlet nodes) of every corner of
 * the rank's elements (input order); sub_of holds global subdomain ids, nI is
 * indexed by local subdomain (global - s0).
 * replaces the pos/loc maps of build_subdomain_operator substructuring.py:98-101. */
int bddc_plan_loc4(const long long* conn, const long long* sub_of, long long n_elements, int s0,
                   const int* iloc_of_node, const int* glob_of_node, const int* pos_in_glob,
                   const int* sh_start, const int* sh_sub, const int* sh_boff,
                   const long long* nI, int* loc4, cudaStream_t stream);

/* Dense local matrix [I|B] x [I|B|f] from element blocks with Dirichlet lifting;
 * writes every entry of each nloc[b] x ld[b] matrix (no memset needed) in a fixed
 * summation order (no atomics: bitwise reproducible).  lists: workspace of
 * 4 * elem_start[nbatch] ints (per-row corner lists; 4 x n_elements < 2^31),
 * keys: 4 * elem_start[nbatch] long longs of scratch; max_nl = max nloc.
 * general = 0: compact row lists (<= 16 distinct columns
 * per row); a row with more sets *overflow (device int, zeroed by the caller)
 * and the call must be repeated with general = 1 (dense row buffers, any
 * mesh).  Both give bitwise identical matrices.
 * nint / ndeep (both null: none): interior and deep-interior counts of the
 * two-phase elimination; the compact path then leaves the two blocks nobody
 * reads unwritten (deep rows x interface columns, interface rows x deep
 * columns: structurally zero and skipped by the panel kernels, the
 * extraction and the recovery).
 * replaces substructuring.py:98-114 (COO->CSR assembly, load, lifting). */
int bddc_local_assemble(double* K, const long long* off, const int* ld, const int* nloc,
                        const long long* elem_start, const long long* elem_ids, const int* loc4,
                        const long long* conn, const double* Ke, const double* Fe,
                        const double* gdir, int nbatch, int max_nl, int* lists, long long* keys,
                        int* overflow, int general, const int* nint, const int* ndeep,
                        cudaStream_t stream);

/* Blocked Schur elimination without pivoting (panel 64 or 128 = two 64-wide
 * sub-panels combined so the DMMA trailing update runs with K = 128):
 * eliminates npiv[b] leading pivots; trailing block becomes the Schur complement.
 * The factors are those of 64-wide panels in either case ("rows below only"
 * LU form): pivot rows keep W_k = P_k A12^(k) (P_k the inverse 64 x 64 pivot
 * block) for back-substitution, the column panels below keep A21^(k).
 * col_hole0 / col_hole1 (per matrix, both null: none): the pivot rows have no
 * entries in columns [col_hole0[b], col_hole1[b]), so the panel steps skip
 * them (first phase of the two-phase subdomain elimination: the deep interior
 * pivots touch only the interior block and the load column; nrows = nI there).
 * replaces splu(A_II) + lu.solve + A_BI @ (...)  substructuring.py:120-127,
 *          lu_factor(coarse) solver.py:123 (with piv_out for the pivot check :124-132),
 *          cho_factor(sym(Sdd)) certificate solver.py:94 (require_positive = 1). */
int bddc_schur_eliminate(double* M, const long long* off, const int* ld, const int* npiv,
                         const int* nrows, const int* ncols, int nbatch, int max_npiv,
                         int max_rows, int max_cols, int panel, double* pinv_ws,
                         long long pinv_stride, long long pinv_step_stride, int* status,
                         int require_positive, double* piv_out, long long piv_stride,
                         const int* col_hole0, const int* col_hole1, cudaStream_t stream);

/* Same, recording CUDA events around every trailing-update launch; the summed
 * device time (ms) is written to the HOST pointer host_trailing_ms (bench roofline). */
int bddc_schur_eliminate_timed(double* M, const long long* off, const int* ld, const int* npiv,
                               const int* nrows, const int* ncols, int nbatch, int max_npiv,
                               int max_rows, int max_cols, int panel, double* pinv_ws,
                               long long pinv_stride, long long pinv_step_stride, int* status,
                               int require_positive, double* piv_out, long long piv_stride,
                               const int* col_hole0, const int* col_hole1, cudaStream_t stream,
                               double* host_trailing_ms);

/* Event log of the bddc_schur_eliminate trailing-update launches (bench
 * roofline measured over the timed region without synchronising inside it):
 * bddc_trailing_log(1) starts logging, bddc_trailing_collect() synchronises on
 * the logged events, writes the summed duration (ms, HOST pointer) and the
 * number of logged launches, and clears the log.  The log is per calling host
 * thread (thread_local), so concurrent threads do not interfere. */
int bddc_trailing_log(int enable);
int bddc_trailing_collect(double* total_ms, long long* launches);

/* Envelope LU without pivoting of the coarse matrix (one n x n matrix at
 * C + off[0], leading dimension ldv[0], nv[0] = n) in a bandwidth-reducing
 * order: panel k updates only rows/cols below host_lim[k/64] (host array).
 * Scalar pivots go to piv_out (for the singularity check solver.py:124-132).
 * replaces lu_factor(coarse) solver.py:123. */
int bddc_coarse_factor(double* C, const long long* off, const int* ldv, const int* nv, int n,
                       const int* host_lim, double* pinv, double* piv_out, int* status,
                       cudaStream_t stream);

/* Blocked in-place Gauss-Jordan inverse (no pivoting).  symmetric = 1 (exactly
 * symmetric input): only the lower half of each trailing update is computed and
 * mirrored, the result is exactly symmetric.
 * replaces cho_factor/cho_solve(Bsym, I) substructuring.py:64-75 (require_positive = 1)
 *          lu_factor(Sdd) + lu_solve solver.py:99, 105, 187, 195 (require_positive = 0). */
int bddc_gj_inverse(double* M, const long long* off, const int* ld, const int* n, int nbatch,
                    int max_n, double* pinv_ws, long long pinv_stride, int* status,
                    int require_positive, int symmetric, cudaStream_t stream);

/* Symmetric in-place Gauss-Jordan inverse in 128-wide panels (K = 128 DMMA
 * trailing updates, half the passes of the 64-panel variant).  Per panel the
 * 128 x 128 pivot block is copied to work (nbatch x 128 x 128; work_off[b] =
 * b * 16384, work_ld[b] = 128; work_n: nbatch ints of scratch, distinct from
 * work_ld) and inverted there by bddc_gj_inverse (pinv_ws: nbatch x 4096);
 * a pivot block of at most 64 pivots (the last panel of a matrix) is
 * inverted by one register Gauss-Jordan instead, whatever the other matrices
 * of the batch need (results do not depend on the batch).  Positive pivots
 * <=> positive definite (the cho_factor criterion).
 * replaces cho_factor/cho_solve(Bsym, I) substructuring.py:64-75. */
int bddc_gj_inverse128(double* M, const long long* off, const int* ld, const int* n, int nbatch,
                       int max_n, double* work, const long long* work_off, const int* work_ld,
                       int* work_n, double* pinv_ws, int* status, int require_positive,
                       cudaStream_t stream);

/* S, g, Bsym = (S + S^T)/2 from the eliminated local matrices.  s_norm2 (or
 * null): ||S_b||_F^2 per matrix, accumulated while S is written (fixed
 * reduction order) through norm_ws (48 * nbatch doubles of scratch).
 * replaces SubdomainOperator.__init__ substructuring.py:35-40. */
int bddc_extract_schur(const double* M, const long long* off, const int* ld, const int* nI,
                       const int* nB, const long long* soff, const long long* voff, double* S,
                       double* Bsym, double* g, int nbatch, double* s_norm2, double* norm_ws,
                       cudaStream_t stream);

int bddc_symmetrize(double* X, const long long* soff, const int* n, int nbatch,
                    cudaStream_t stream);

/* out[b] = ||X_b||_F^2 (square n[b] x n[b] at soff[b]; deterministic reduction).
 * Feeds the certified shortcut of the dual-block Cholesky certificate
 * (engine.DevicePreconditioner, reference solver.py:91-98). */
int bddc_frob2(const double* X, const long long* soff, const int* n, int nbatch, double* out,
               cudaStream_t stream);

/* out[b] = trace(X_b)^2: for symmetric positive definite X_b an upper bound of
 * ||X_b||_F^2 from the diagonal alone (used for ||Bsym^-1|| in the certificates
 * that replace cho_factor(sym(Sdd)) solver.py:94 and the per-block checks of
 * substructuring.py:166-170). */
int bddc_trace2(const double* X, const long long* soff, const int* n, int nbatch, double* out,
                cudaStream_t stream);

/* u_I = A_II^-1 (f_I - A_IB u_B) by block back-substitution over the stored
 * W rows.  ndeep (per matrix, null: 0): the leading pivots eliminated in a
 * separate first phase (bddc_schur_eliminate with a column hole); the panels
 * of the second phase start at ndeep[b].
 * replaces recover_interior solver.py:318-326. */
int bddc_recover_interior(const double* M, const long long* off, const int* ld, const int* nI,
                          const int* nB, const long long* voff, const int* iface_perm,
                          const long long* ioff, const long long* interior_nodes,
                          const double* u_hat, double* u, int nbatch, int max_nloc, int panel,
                          const int* ndeep, cudaStream_t stream);

/* ---- plan_host.cu : host side of the symbolic plan ------------------------ */

/* Glob tables of the symbolic plan, all HOST arrays (no device work): from the
 * glob sizes gsize[G], sharer counts nsh[G] and the flat sharer list
 * (glob-major, ascending per glob) to the slot tables sh_start[G+1],
 * slot_glob[ns], sh_doff[ns+1] (n_g^2 per slot), the per-subdomain glob lists
 * sub_globs / sub_glob_sh[ns] with sub_glob_start[N+1], the block offset of
 * every glob in its sharer's glob-major interface order (sub_glob_boff[ns] by
 * (subdomain, glob), sh_boff[ns] by slot), nB[N] and the start of each glob's
 * nodes in the flat glob-node list b_starts[ns].  Returns -2 for a sharer id
 * outside [0, N).  replaces the per-subdomain glob bookkeeping of
 * build_subdomain_operator substructuring.py:85-96. */
int bddc_plan_glob_tables(int G, int N, const int* gsize, const long long* nsh,
                          const long long* sharers, int* sh_start, int* slot_glob,
                          long long* sh_doff, int* sub_globs, int* sub_glob_sh,
                          int* sub_glob_start, int* sub_glob_boff, int* sh_boff, long long* nB,
                          long long* b_starts);

/* ---- elements.cu : SUPG element blocks ------------------------------------ */

/* Ke (m x 16) and Fe (m x 4) of the SUPG-stabilised P1 tetrahedra for
 * device-evaluable coefficients: velocity a(x) = A x + a0, constant reaction
 * and source, viscosity nu[e] = nu_tab[e % nu_period].  fields (host array,
 * 16 doubles): A (row-major 3x3), a0, c, f, c - div(a)/2 (or c), tau.
 * bad_element (device, initialised to ~0ull by the caller): smallest element
 * index with a non-positive volume.  replaces element_contributions /
 * p1_gradients / stabilization discretization.py:91-158. */
int bddc_supg_elements(const double* nodes, const long long* conn, long long m,
                       const double* nu_tab, long long nu_period, const double* fields,
                       double* Ke, double* Fe, unsigned long long* bad_element,
                       cudaStream_t stream);

/* ---- globs.cu : scaling and adaptive coarse space ------------------------- */

/* Deluxe scaling D_s = (sum_k B_k)^-1 B_s per glob; vertices 1/|n(V)|.
 * Globs glob_ids[0..n_globs) (NULL: 0..n_globs-1); reads the slot blocks BsC.
 * replaces deluxe_scaling / vertex_scaling / build_scaling scaling.py:10-57. */
int bddc_deluxe(const int* kind, const int* size, const int* sh_start, const int* sh_sub,
                const int* sh_boff, const long long* sh_doff, const double* BsC, double* D,
                double* ws, const long long* ws_off, int* status, const int* glob_ids, int n_globs,
                cudaStream_t stream);

/* Batched linalg.py kernels on arbitrary symmetric n[b] x n[b] inputs at off[b]
 * (one CTA per member; workspace ws + ws_off[b] of bddc_ws_linalg(n[b]) doubles):
 *   mode 0: out = pseudo_inverse(A) with cut rel_tol (linalg.py:23-50);
 *   mode 1: out = parallel_sum(A, B) (linalg.py:53-67);
 *   mode 2: sym_pencil_gevp(A, B) (linalg.py:116-214): vals / degen at voff[b]
 *           (n[b] each; +inf first, finite descending, degenerate last), out =
 *           eigenvectors (columns aligned with vals), status[b] = 3 when B is not
 *           positive semidefinite (the reference's ValueError).
 * replaces scipy.linalg.eigh-based pseudo_inverse / parallel_sum / sym_pencil_gevp. */
long long bddc_ws_linalg(long long n);
int bddc_linalg_batched(int mode, const double* A, const double* B, const long long* off,
                        const int* n, int nbatch, double rel_tol, double* out, double* vals,
                        const long long* voff, int* degen, int* status, double* ws,
                        const long long* ws_off, int max_n, cudaStream_t stream);

/* Batched change of basis: Q (n[b] x n[b], orthogonal) whose first rank[b]
 * rows span the rows (m[b] x n[b], row-major) at roff[b]; rank at the
 * s >= 1e-10 s_max cut (one-sided Jacobi SVD + Householder completion).
 * Workspace bddc_ws_row_space(m, n) doubles per member.
 * replaces build_change_of_basis adaptive.py:190-206 and the SVD of
 * reduce_edge_constraints adaptive.py:172-187. */
long long bddc_ws_row_space(long long m, long long n);
int bddc_row_space_batched(const double* rows, const long long* roff, const int* m, const int* n,
                           int nbatch, double* Q, const long long* qoff, int* rank, double* ws,
                           const long long* ws_off, int max_dim, cudaStream_t stream);

/* Face GEP + selection + change of basis.  mode = 1: certified fast path in a
 * compact arena (faces whose certificate fails get status 900 and must be
 * re-run with mode 0); mode = 0: general kernel, certified shortcuts allowed;
 * mode = -1: the reference algorithm verbatim (eigen-based pseudo-inverse,
 * general pencil solver).  detail (NULL or per glob at detail_off[g], n = n_g):
 * [pencil_left n^2 | pencil_right n^2 | eigenvectors n^2 | constraint rows
 * n_sel x n (n^2 slot) | degenerate flags n], the reference GevpReport fields
 * (adaptive.py:36-47); implies mode -1.
 * SC / sc_status: the per-slot glob Schur blocks of bddc_slot_schur, or NULL; with
 * SC = NULL the fast path (mode 1, n <= 64) bounds their norms by the Bsym
 * principal blocks and needs sub_ok (per subdomain: 1 when cond(Bsym) is
 * certified, ||S||_F ||Bsym^-1||_F < 1e11) in place of the per-block PD checks;
 * faces of uncertified subdomains get status 900.
 * replaces face_gevp adaptive.py:57-72, glob_schur_block substructuring.py:152-171,
 *          parallel_sum / pseudo_inverse / sym_pencil_gevp linalg.py:23-214,
 *          build_change_of_basis adaptive.py:190-206. */
int bddc_face_gevp(const int* kind, const int* size, const int* sh_start, const int* sh_sub,
                   const int* sh_boff, const long long* sh_doff, const double* BsC,
                   const double* BiC, const double* SC, const int* sc_status, const int* sub_ok,
                   const double* D, double theta, double* eig,
                   const long long* eig_off, int* n_sel, int* r, double* Q, const long long* q_off,
                   int* status, double* ws, const long long* ws_off, const int* face_ids,
                   int n_faces, int max_n, int mode, double* detail, const long long* detail_off,
                   cudaStream_t stream);

/* Prior blocks of the face-transformed Bsym^-1 per subdomain.
 * replaces adaptive.py:310-329 (Minv = Q Bsym^-1 Q^T on face rows/cols, prior_idx). */
int bddc_priors(const int* kind, const int* size, const int* nB, const long long* soff,
                const double* Binv, const int* sub_glob_start, const int* sub_globs,
                const int* sub_glob_boff, const int* r, const double* Q, const long long* q_off,
                const long long* pb_off, const int* nH, double* PB, double* XHH,
                const long long* xhh_off, int n_sub, cudaStream_t stream);

/* Prior-aware ("new") edge GEP + SVD reduction + change of basis.
 * general = 1: reference algorithm verbatim (no certified pencil shortcut);
 * detail as bddc_face_gevp with n = nC = (|n(E)| - 1) n_E (implies general).
 * replaces edge_block_with_priors substructuring.py:174-190, edge_gevp_new
 *          adaptive.py:94-156, reduce_edge_constraints adaptive.py:172-187. */
int bddc_edge_gevp_new(const int* kind, const int* size, const int* sh_start, const int* sh_sub,
                       const int* sh_boff, const long long* sh_doff, const double* BsC,
                       const double* BiC, const double* SC, const int* sc_status,
                       const double* D, const double* EX,
                       const long long* ex_off, const int* ex_h, double theta, double* eig,
                       const long long* eig_off, int* n_sel, int* r, double* Q,
                       const long long* q_off, int* status, double* ws, const long long* ws_off,
                       const int* edge_ids, int n_edges, int max_dim, int general,
                       double* detail, const long long* detail_off, cudaStream_t stream);

/* Coupled ("old") edge GEP; general / detail as bddc_edge_gevp_new (n = n_E).
 * replaces edge_gevp_old adaptive.py:75-91,
 *          parallel_sum_chain linalg.py:70-78. */
int bddc_edge_gevp_old(const int* kind, const int* size, const int* sh_start, const int* sh_sub,
                       const int* sh_boff, const long long* sh_doff, const double* BsC,
                       const double* BiC, const double* SC, const int* sc_status,
                       const double* D, double theta, double* eig,
                       const long long* eig_off, int* n_sel, int* r, double* Q,
                       const long long* q_off, int* status, double* ws, const long long* ws_off,
                       const int* edge_ids, int n_edges, int max_n, int general, double* detail,
                       const long long* detail_off, cudaStream_t stream);

/* Slot-compact glob blocks.  Every (glob, sharer) slot k whose sharer is a
 * subdomain of this rank (slot_sub[k] = its local index, -1 otherwise) gets
 * the n_g x n_g principal blocks of Bsym / Bsym^-1 at BsC / BiC + sh_doff[k]
 * (BsC or BiC may be NULL); sym = 1: the first source is S and BsC receives
 * the blocks of Bsym = sym(S).  The per-glob kernels read only these
 * buffers; on the sharded path the cross-rank slots move point to point
 * (dist.SlotExchange).
 * replaces the per-glob Bsym[g_idx][:, g_idx] slicing of build_scaling
 *          scaling.py:33-41 and glob_schur_block substructuring.py:152-171. */
int bddc_extract_slot_blocks(const int* slot_sub, const int* slot_glob, const int* size,
                             const int* sh_boff, const long long* sh_doff, const int* nB,
                             const long long* soff, const double* Bsym, const double* Binv,
                             double* BsC, double* BiC, int n_slots, int sym,
                             cudaStream_t stream);

/* Glob Schur blocks sym(((Bsym^-1)[g,g])^-1) of the listed slots with
 * n_g <= 64 (register Gauss-Jordan, one CTA per slot) into SC (sh_doff
 * layout); sc_status[slot] = 1 when the block is not positive definite.  The
 * face / edge kernels take SC (or NULL: computed in-kernel).
 * replaces glob_schur_block substructuring.py:152-171. */
int bddc_slot_schur(const int* slots, int n_slots, const int* slot_glob, const int* size,
                    const long long* sh_doff, const double* BiC, double* SC, int* sc_status,
                    cudaStream_t stream);

/* Per local (edge, sharer) slot: X = [[Binv_EE, PB_E^T], [PB_E, XHH]] at
 * EX + ex_off[k] ((ne+nH) x (ne+nH)), the input of the prior-aware edge Schur
 * complement.  replaces edge_block_with_priors substructuring.py:174-190. */
int bddc_edge_x_extract(const int* slot_sub, const int* slot_glob, const int* size,
                        const int* kind, const int* sh_boff, const int* nB, const long long* soff,
                        const double* Binv, const long long* pb_off, const int* nH,
                        const double* PB, const double* XHH, const long long* xhh_off, double* EX,
                        const long long* ex_off, int n_slots, cudaStream_t stream);

/* workspace sizes (doubles) of the per-glob kernels, for the host planner */
long long bddc_ws_face(long long n);
long long bddc_ws_face_fast(long long n);
long long bddc_ws_edge_new(long long ns, long long ne, long long wd, long long nhmax);

/* ---- precond.cu : preconditioner setup / apply, interface operator -------- */

/* Sbar = Q_i S_i Q_i^T (block diagonal Q_i per glob; DMMA block products).
 * QT: caller scratch the size of the Q buffer.  replaces solver.py:85-86. */
int bddc_pc_transform_schur(const int* nB, const long long* soff, const int* sub_glob_start,
                            int nbatch, const int* sub_globs, const int* sub_glob_boff,
                            const int* sub_glob_sh, const int* gsize, const double* Q,
                            const long long* q_off, double* QT, int n_globs, int n_items,
                            int max_nB, int max_ng, int max_globs, const double* S, double* tmp,
                            double* Sbar, cudaStream_t stream);

/* Householder form of the change of basis: per glob with r > 0 (not a vertex,
 * n_g > 1) Q_g <- H_r ... H_1 from the Householder QR of Q_g[:r]^T (same
 * primal span), reflector j stored as w_j (H_j = I - w_j w_j^T) in row j of
 * HV at q_off[g]; W: scratch of n_g * r_g doubles per glob at w_off[g].
 * max_ng: largest n_g.  Part of replacing the transforms of solver.py:70-90. */
int bddc_pc_glob_reflectors(const int* kind, const int* gsize, const int* r, double* Q,
                            const long long* q_off, double* HV, double* W, const long long* w_off,
                            int n_globs, int max_ng, cudaStream_t stream);

/* Sbar_i = Q_i S_i Q_i^T with Q_i = blockdiag of the reflector products of
 * bddc_pc_glob_reflectors (2 r n_g nB flops per glob block and side).
 * replaces the S-bar transform solver.py:86-90. */
int bddc_pc_transform_refl(const int* nB, const long long* soff, const int* sub_glob_start,
                           const int* sub_globs, const int* sub_glob_boff, const int* kind,
                           const int* gsize, const int* r, const double* HV,
                           const long long* q_off, const double* S, double* Sbar, int nbatch,
                           cudaStream_t stream);

/* TT_(g,s) = D_g^(s) Q_g^T blocks.  replaces Dbar solver.py:87-90. */
int bddc_pc_ttblocks(const int* slot_glob, const int* gsize, const double* Q,
                     const long long* q_off, const double* D, const long long* sh_doff,
                     double* TT, int n_slots, cudaStream_t stream);

/* Zin = Sbar with primal rows/cols -> identity; Csym = sym(Zin).  solver.py:84, 91-94. */
int bddc_pc_dual_embed(const int* nB, const long long* soff, const long long* voff,
                       const unsigned char* primal_mask, const double* Sbar, double* Zin,
                       double* Csym, int nbatch, cudaStream_t stream);




int bddc_pc_primal_rows_T(const int* nB, const long long* voff, const int* pos2k,
                          const int* sub_globs, const int* sub_glob_boff, const int* sub_glob_sh,
                          const int* gsize, const long long* sh_doff, const double* TT,
                          const int* pstart, const long long* poff, const double* In, double* Out,
                          int nbatch, cudaStream_t stream);

/* Copy the per-panel inverse pivot blocks P_k^-1 of a batched 64-panel
 * schur_eliminate (pinv + k * step_stride + b * pinv_stride, ld 64) into the
 * diagonal blocks, completing the in-place LU used by the dual solves. */
int bddc_lu_diag_pinv(double* LU, const long long* soff, const int* nB, int nbatch, int max_n,
                      const double* pinv, long long pinv_stride, long long step_stride,
                      cudaStream_t stream);

/* The coarse restriction alone: cvals = G x, x = u[perm] (G = null in
 * bddc_pc_local_solve then skips it there), so that the coarse solve can run
 * on another stream next to the local solves.
 * replaces the primal part of Rtil^T Dtil^T ... solver.py:180-186. */
int bddc_pc_primal_restrict(const int* nB, const long long* voff, const int* iface_perm,
                            const double* u, const int* pstart, const long long* poff,
                            const double* G, double* cvals, int nbatch, int max_nB,
                            cudaStream_t stream);

/* Local part of the preconditioner and the coarse restriction per subdomain:
 * x = u[perm]; cvals = G x (skipped when G is null); y = TT (Sdd^-1 (TT^T x
 * with primal entries zeroed)) through the dual-block LU (the reference's
 * lu_solve of Stil, solver.py:187-195).
 * replaces BddcPreconditioner.apply local solves solver.py:138-209. */
int bddc_pc_local_solve(const int* nB, const long long* soff, const long long* voff,
                        const int* iface_perm, const double* LU, const int* pos2k,
                        const int* sub_globs, const int* sub_glob_boff, const int* sub_glob_sh,
                        const int* gsize, const long long* sh_doff, const double* TT,
                        const unsigned char* primal_mask, const double* u, double* y,
                        const int* pstart, const long long* poff, const double* G, double* cvals,
                        int nbatch, int max_nB, cudaStream_t stream);

/* Householder-path fusion of the S-bar transform and the dual embedding:
 * Sbar = Q S Q^T (reflectors HV, r per glob), Z = embedded dual block
 * (identity on primal rows / columns), Srows[q] = Sbar[ppos_q, :] and
 * Scols[q] = Sbar[:, ppos_q] (n_p x nB at poff); pidx: per local B position its
 * primal index or -1.  Left reflectors: one CTA per listed glob block
 * (left_k[i] into sub_globs, subdomain left_sub[i]); right reflectors and the
 * outputs: one warp per row, applying only the subdomain's reflected globs
 * refl_k[refl_start[b] .. refl_start[b + 1]).  replaces solver.py:85-99. */
int bddc_pc_transform_embed(const int* nB, const long long* soff, const long long* voff,
                            const int* pos2k, const int* sub_globs, const int* sub_glob_boff,
                            const int* kind, const int* gsize, const int* r, const double* HV,
                            const long long* q_off, const int* refl_start, const int* refl_k,
                            const int* left_k, const int* left_sub, int n_left, const int* pidx,
                            const long long* poff, const double* S, double* Z, double* Srows,
                            double* Scols, int nbatch, int max_nB, cudaStream_t stream);

/* Srows / Scols (as above) from a full Sbar (dense-Q path). */
int bddc_pc_primal_extract(const int* nB, const long long* soff, const long long* voff,
                           const int* pidx, const long long* poff, const double* Sbar,
                           double* Srows, double* Scols, int nbatch, cudaStream_t stream);

/* Primal pieces through the dual LU: MP = e_P - Z Sbar[:, P], RP = e_P -
 * Z^T Sbar[P, :]^T, coarse blocks C_i = Sbar[P, :] MP (Srows / Scols: the
 * compact primal rows / columns).  replaces solver.py:100-110. */
int bddc_pc_primal_pieces_lu(const int* nB, const long long* soff, const long long* voff,
                             const unsigned char* primal_mask, const int* pstart, const int* ppos,
                             const long long* poff, const double* Srows, const double* Scols,
                             const double* LU, double* MP, double* RP, double* Cl,
                             const long long* coff, int nbatch, int max_nB, cudaStream_t stream);

/* coarse = sum_i P_i^T C_i P_i (dense n_c x n_c, every entry written, fixed
 * summation order: no atomics).  cstart (n_c + 1) / csrc: for each coarse dof
 * the positions in pgid of its (subdomain, local primal) sources, ascending.
 * replaces solver.py:106. */
int bddc_coarse_scatter(const int* pstart, const int* pgid, const double* Cl,
                        const long long* coff, const long long* cstart, const long long* csrc,
                        double* C, long long ldc, int n_c, int nbatch, cudaStream_t stream);

/* Dense transformed deluxe weights per subdomain in nodal B order:
 * Dbar_b[pos, pos] = Q_g TT_(g,b) (= Q_g D_g^(b) Q_g^T) for each slot; nodal maps a
 * glob-major local position (voff layout) to its nodal one; W: slot-layout scratch;
 * Dbar zeroed by the caller.  replaces the Dbar loop of solver.py:86-90. */
int bddc_pc_dbar(const int* slot_glob, const int* slot_sub, const int* gsize, const int* sh_boff,
                 const long long* sh_doff, const double* Q, const long long* q_off,
                 const double* TT, const int* nB, const long long* soff, const long long* voff,
                 const int* nodal, double* W, double* Dbar, int n_slots, cudaStream_t stream);

/* out_b = X_b^T (square n[b] x n[b] at soff[b]). */
int bddc_transpose_batched(const double* X, const long long* soff, const int* n, int nbatch,
                           double* out, cudaStream_t stream);

/* y_i = M_i u[perm_i] (+ c_i = G_i u[perm_i]).  replaces interface_operator solver.py:229-233
 * (M = S) and the local half of BddcPreconditioner.apply solver.py:201-209 (M = A). */
int bddc_local_gemv(const int* nB, const long long* soff, const long long* voff,
                    const int* iface_perm, const double* M, const double* u, double* y,
                    const int* pstart, const long long* poff, const double* G, double* cvals,
                    int nbatch, int max_nB, int row_chunks, cudaStream_t stream);

/* y_i += N_i u_P[gprimal_i].  replaces solver.py:193-198 + scale + inject_t. */
int bddc_prolong_primal(const int* nB, const long long* voff, const int* pstart, const int* pgid,
                        const long long* poff, const double* Nt, const double* uP, double* y,
                        int nbatch, cudaStream_t stream);

/* out[t] = sum of y over the CSR sources of t (deterministic subassembly).
 * replaces out[op.iface_index] += ... solver.py:231-232, 159-160. */
int bddc_gather_reduce(const long long* tstart, const long long* tsrc, const double* y,
                       double* out, long long n, cudaStream_t stream);

/* Coarse solve with the envelope-LU factors of bddc_coarse_factor, one
 * cooperative persistent launch (grid-wide barrier per 64-wide panel):
 * forward panel k updates rows [k+64, lim[k/64]), backward panel k updates
 * rows [first[k/64], k) (device int arrays).  b is overwritten; the solution
 * is returned in t.  replaces lu_solve(coarse_lu) solver.py:192. */
int bddc_coarse_solve(const double* A, long long ld, int n, const double* pinv,
                      long long pinv_step_stride, const int* lim, const int* first, double* b,
                      double* t, cudaStream_t stream);

/* Same solve as a dataflow over 128-row super-panels (one cooperative launch,
 * per-super-panel ready flags instead of grid-wide barriers): jmin[Q] / jmax[Q]
 * = first / last super-panel coupled to super-panel Q in L' / W; flags: 2 *
 * ceil(n / 128) ints, epoch: a value different from every earlier call's. */
int bddc_coarse_solve_flow(const double* A, long long ld, int n, const double* pinv,
                           long long pinv_step_stride, const int* jmin, const int* jmax, double* b,
                           double* t, int* flags, int epoch, cudaStream_t stream);

/* ---- coarse.cu : block-inverse coarse solve --------------------------------- */

/* Build the block-inverse solve operators from the factors of
 * bddc_coarse_factor (A, ld, pinv as left by it).  Rows are grouped in blocks
 * of B = bddc_coarse_block_rows() (1024); for block D (rows [B D, B D + h)):
 *   F_D = Linv_DD [L_(D, cl[D]:B D) | I_h]       h x ldF, at foff[D]
 *   G_D = Uinv_DD [P_D | W_(D, B D + h:cu[D])]    h x ldG, at goff[D]
 * ldF = (B D - cl[D]) + roundup2(h), ldG = roundup2(cu[D] - B D); cl[D]
 * (64-aligned) is the first column of L coupled to the block, cu[D] the end
 * of its U coupling (device arrays; engine.coarse_blockinv_layout).  max_ldf /
 * max_ldg: largest ldF / ldG.  Part of replacing lu_factor(coarse) solver.py:123. */
int bddc_coarse_blockinv(const double* A, long long ld, int n, const double* pinv,
                         long long pinv_step_stride, int nD, const int* cl, const int* cu,
                         const long long* foff, const long long* goff, int max_ldf, int max_ldg,
                         double* F, double* G, cudaStream_t stream);

/* Rows per block of the block-inverse coarse solve (the layout's block size). */
int bddc_coarse_block_rows(void);

/* x = C^-1 b with the operators of bddc_coarse_blockinv: 2 nD dependent
 * row-parallel GEMV steps in one cooperative launch (128 CTAs).  z: n doubles
 * of scratch (the forward result); counters: 2 nD ints zeroed once, epoch:
 * 1, 2, 3, ... on successive calls with the same counters (reset counters and
 * restart at 1 before epoch * 128 overflows).  replaces lu_solve(coarse_lu)
 * solver.py:192. */
int bddc_coarse_solve_blockinv(const double* F, const double* G, int n, int nD, const int* cl,
                               const int* cu, const long long* foff, const long long* goff,
                               const double* b, double* z, double* x, int* counters, int epoch,
                               cudaStream_t stream);

/* ---- krylov.cu : GMRES vector kernels (solver.py:286-310) ------------------ */

/* As bddc_multi_dot over the first n entries of rows of stride ldv (owned
 * entries of a rank-local vector on the sharded path). */
int bddc_multi_dot_ld(const double* V, long long ldv, long long n, int m, const double* w,
                      double* h, double* partial, int nblocks, int accumulate,
                      cudaStream_t stream);
int bddc_multi_dot(const double* V, long long n, int m, const double* w, double* h,
                   double* partial, int nblocks, int accumulate, cudaStream_t stream);
int bddc_multi_axpy(const double* V, long long n, int m, const double* coef, double alpha,
                    double* w, cudaStream_t stream);
int bddc_norm2(const double* w, long long n, double* out, double* partial, int nblocks,
               cudaStream_t stream);
/* One step of the GMRES least-squares recurrence by Givens rotations on the
 * device: column m-1 of the Hessenberg matrix is h1[0:m] + h2[0:m] (the two
 * Gram-Schmidt passes), subdiagonal h2[m]; updates R (column-major, ldr
 * rows), the rotations cs / sn and the rotated rhs g (g[0] = beta), writes
 * y = R^-1 g[0:m] and out = {|g[m]|, h2[m]}.  m <= 1023.
 * replaces scipy.linalg.lstsq(H, beta e1, gelsd) per step, solver.py:297-300. */
int bddc_gmres_givens(const double* h1, const double* h2, int m, int ldr, double* R, double* cs,
                      double* sn, double* g, double* y, double* out, cudaStream_t stream);

/* One whole GMRES step after w = M^-1 S_hat v_(m-1) in a single cooperative
 * launch (one rank): CGS2 against V[0:m] (h1, h2[0:m], h2[m] = ||w||), the
 * Givens recurrence of bddc_gmres_givens (R, cs, sn, g, y, out), the next
 * basis vector vnext = w / ||w|| and the true residual norm
 * tres[0] = ||rhs - U[0:m]^T y||.  V, U: m rows of stride ldv; partial:
 * (2 m + 2) * bddc_gmres_step_blocks() doubles of workspace.  Returns 1 (nothing
 * launched) when the vectors do not fit the resident chunks: the caller then
 * uses the separate kernels above.  Fixed-order reductions (reproducible).
 * replaces the inner loop of gmres_solve, solver.py:283-306. */
int bddc_gmres_step(const double* V, const double* U, long long ldv, long long n, int m,
                    const double* w, const double* rhs, double* h1, double* h2, int ldr, double* R,
                    double* cs, double* sn, double* g, double* y, double* out, double* tres,
                    double* vnext, double* partial, cudaStream_t stream);
int bddc_gmres_step_blocks(void);

/* x[i] = sqrt(x[i]), i < n (norms after a cross-rank sum of squares). */
int bddc_sqrt_inplace(double* x, int n, cudaStream_t stream);

/* Halo / slot-exchange packing for the sharded path: dst[i] = src[idx[i]];
 * unpacking: dst[idx[i]] = src[i] (add = 0) or dst[idx[i]] += src[i] (add = 1),
 * idx duplicate-free.  replaces the implicit sums over all subdomains in one
 * process of solver.py:229-242 when subdomains live on several GPUs. */
int bddc_gather_idx(const double* src, const long long* idx, long long n, double* dst,
                    cudaStream_t stream);
int bddc_scatter_idx(double* dst, const long long* idx, long long n, const double* src, int add,
                     cudaStream_t stream);

int bddc_scale_copy(const double* a, long long n, const double* den, double* out,
                    cudaStream_t stream);

/* ---- counters.cu : launch accounting (bench "gpu_launches") ---------------- */
long long bddc_launch_count(void);
int bddc_launch_count_reset(void);

#ifdef __cplusplus
}
#endif
#endif /* BDDC_B200_H */
