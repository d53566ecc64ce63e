/*
 * mg_internal.h -- host-side setup routines of libmgb200.so, exported with the
 * prefix mgi_ so the CPU test-suite can check them without a GPU (they make
 * no CUDA calls).  Not part of the solver API (include/mg.h).
 *
 * All routines: plain host pointers, caller-owned outputs sized as stated,
 * return 0 on success or a negative mg_status code (mg.h) on invalid input.
 */
#ifndef MGB200_MG_INTERNAL_H
#define MGB200_MG_INTERNAL_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Validate a BSR / CSR matrix: row_ptr[0] == 0, non-decreasing, row_ptr[n] ==
 * nnz; columns strictly increasing within a row and in [0, n_cols); values
 * (nnz * vpe) finite; if need_diag, every row i holds column diag_offset + i.
 * Returns 0, MG_ERR_STRUCTURE (-3) or MG_ERR_NONFINITE (-4). */
int mgi_validate_csr(int64_t n, int64_t n_cols, const int64_t *row_ptr, const int64_t *col,
                     const double *val, int64_t vpe, int need_diag, int64_t diag_offset);

/* Sliced-ELL layout ("SELL-32-sigma") used on the device for every sparse
 * operator: rows are sorted by length
 * (descending, stable) inside windows of `sigma` rows (sigma % 32 == 0),
 * then cut into slices of 32 rows (one warp, lane = row).  Slice s holds
 * len_s = max row length entries per lane; entry k of lane t sits at
 * e = slice_ptr[s] + 32*k + t.  Values of entry e (vpe doubles) are chunked
 * for coalesced 16-byte loads: element 2j, 2j+1 (j < vpe/2) at
 * (e - t)*vpe + 64*j + 2*t + {0,1}; the last element of odd vpe at
 * (e - t)*vpe + 64*(vpe/2) + t.  Padding entries have value 0 and repeat
 * the row's last real column (0 for empty rows and padding lanes), so every
 * stored column is in range, also for rectangular operators (P, R);
 * perm[s*32 + t] = row or -1.
 *
 * mgi_sell_size: *n_slices and *n_entries (= slice_ptr[n_slices]). */
int mgi_sell_size(int64_t n, const int64_t *row_ptr, int sigma, int64_t *n_slices,
                  int64_t *n_entries);

/* Fill the layout: slice_ptr[n_slices+1], perm[n_slices*32], col[n_entries],
 * val[n_entries*vpe] (val may be NULL for structure only). */
int mgi_sell_fill(int64_t n, const int64_t *row_ptr, const int64_t *col_in, const double *val_in,
                  int vpe, int sigma, int64_t *slice_ptr, int32_t *perm, int32_t *col,
                  double *val);

/* Same layout with fp32 values (mixed-precision V-cycle operators):
 * 4-float chunks -- element 4j+t (j < vpe/4) at (e - lane)*vpe + 128*j + 4*lane + t
 * -- then the vpe % 4 remaining elements as planes at (e - lane)*vpe + 128*(vpe/4)
 * + 32*k + lane.  Values are rounded to nearest fp32. */
int mgi_sell_fill_f32(int64_t n, const int64_t *row_ptr, const int64_t *col_in, const double *val_in,
                      int vpe, int sigma, int64_t *slice_ptr, int32_t *perm, int32_t *col,
                      float *val);

/* Transfer layout (P_l, R_l): SELL-C-sigma with C = 32 / bs rows per
 * slice, so a warp's lane (r, q) = (lane / bs, lane % bs) handles component q
 * of the slice's row r and the bs components of one gathered node come from
 * ONE load instruction (adjacent lanes, adjacent words).  Rows are stably
 * sorted by length inside windows of sigma rows (sigma % C == 0); entry k of
 * slice-row r sits at slice_ptr[s] + k*C + r; padding repeats the row's last
 * column with weight 0.  Weights are stored as fp32 -- exact for the dyadic
 * transfer weights (G6): mgi_tsell_fill returns 2 (nothing written) when some
 * weight is not exactly representable, and the caller keeps the fp64 SELL-32
 * layout.  w[e*wpe + t]; perm[n_slices*C] (-1 = padding). */
int mgi_tsell_size(int64_t n, const int64_t *row_ptr, int C, int sigma, int64_t *n_slices, int64_t *n_entries);
int mgi_tsell_fill(int64_t n, const int64_t *row_ptr, const int64_t *col_in, const double *w_in, int wpe, int C,
                   int sigma, int64_t *slice_ptr, int32_t *perm, int32_t *col, float *w);

/* Value-update map of a SELL-32-sigma layout (mg_update_matrix): map[k] = the
 * SELL entry e holding original CSR entry k (k < row_ptr[n]); row_pos[r] =
 * slice*32 + lane of row r (row_pos may be NULL). */
int mgi_sell_entry_map(int64_t n, const int64_t *row_ptr, const int64_t *slice_ptr, const int32_t *perm,
                       int64_t *map, int32_t *row_pos);

/* Stable counting-sort transpose (R = P^T): out_row_ptr[n_cols+1],
 * out_col[nnz], out_w[nnz*wpe]; entries of each output row in ascending
 * input-row order. */
int mgi_csr_transpose(int64_t n_rows, int64_t n_cols, const int64_t *row_ptr, const int64_t *col,
                      const double *w, int wpe, int64_t *out_row_ptr, int64_t *out_col,
                      double *out_w);

/* Inverse diagonal blocks D^-1 of a BSR matrix by Gauss-Jordan with partial
 * pivoting (max |a|, ties -> lowest row; reading Z10): dinv[n*bs*bs].
 * Returns 0, MG_ERR_STRUCTURE (missing diagonal) or MG_ERR_SINGULAR (-5). */
int mgi_block_diag_inverse(int64_t n, int bs, const int64_t *row_ptr, const int64_t *col,
                           const double *val, double *dinv);

/* Dense inverse of an N x N row-major matrix (Gauss-Jordan, partial
 * pivoting; OpenMP over rows).  a is overwritten; inv[N*N]. */
int mgi_dense_inverse(int64_t N, double *a, double *inv);

/* Expand owned BSR rows to a dense row-major (n*bs) x (n*bs) matrix. */
int mgi_bsr_to_dense(int64_t n, int bs, const int64_t *row_ptr, const int64_t *col,
                     const double *val, double *dense);

/* Multi-GPU row-partition plan: given the GLOBAL columns of
 * an n_rows-row local CSR operator whose column space is a level of which this
 * rank owns rows [col_begin, col_end), produce
 *   - local_col[nnz]: owned columns renumbered to c - col_begin, the g-th
 *     ghost (ghosts sorted by global index) to (col_end - col_begin) + g;
 *   - ghosts[*n_ghost] (capacity nnz): global indices of the ghost columns.
 * Returns 0. */
int mgi_localize_columns(int64_t n_rows, int64_t col_begin, int64_t col_end, const int64_t *row_ptr,
                         const int64_t *col, int64_t *local_col, int64_t *ghosts,
                         int64_t *n_ghost);

/* Owner rank of global row g under contiguous splitters
 * bounds[0..nranks] (bounds[r] <= g < bounds[r+1]). */
int mgi_owner(int64_t g, const int64_t *bounds, int nranks);

/* Rows of R = P^T owned by this rank, from the P entries every rank routed
 * to it (multi-GPU restriction setup).  Input: m entries (J = global coarse
 * row, i = global fine row, w[wpe]) in arrival order (source ranks ascending,
 * each in its CSR order); output: CSR rows r0 .. r0+nr-1 (out_row_ptr[nr+1]),
 * out_col = global fine rows, out_w[m*wpe].  Stable counting sort on J, so
 * each row lists fine rows ascending -- identical to the single-GPU
 * transpose.  Returns 0 or MG_ERR_STRUCTURE (J outside [r0, r0+nr)). */
int mgi_assemble_routed_rows(int64_t m, const int64_t *J, const int64_t *i, const double *w, int wpe, int64_t r0,
                             int64_t nr, int64_t *out_row_ptr, int64_t *out_col, double *out_w);

/* Number of device kernels the context has launched so far (eager launches
 * plus the kernel nodes of every CUDA-graph launch).  Bench accounting. */
typedef struct mg_ctx_s *mgi_ctx;
int64_t mgi_launch_count(mgi_ctx ctx);

/* The context's CUDA stream (as void*), device, level count and finest-level
 * row count (libns: the NS step runs on the pressure solver's stream). */
int mgi_stream_info(mgi_ctx ctx, void **stream, int *device, int *n_levels, int64_t *n_fine);

/* Agree on a status over all ranks of the context (collective; host-side
 * all-gather through the transport): *agreed = the status of the lowest rank
 * whose status is not MG_OK, else MG_OK.  Single GPU: *agreed = status.  Lets
 * a rank-local failure (e.g. a Newton assembly callback) fail every rank
 * together instead of leaving the others in a collective.  Returns an
 * mg_status of the agreement itself. */
int mgi_agree(mgi_ctx ctx, int status, int *agreed);

/* One V-cycle (eager, not graph-launched) with CUDA events between its
 * phases: out[l] = ms spent on level l's kernels (both legs; level 0 = the
 * coarse solve), out[n_levels + l] = ms in level l's halo exchanges,
 * out[2 n_levels] = ms in agglomeration all-gathers.  n_out >= 2 n_levels + 1.
 * Returns an mg_status. */
int mgi_vcycle_profile(mgi_ctx ctx, double *x, const double *b, int zero, double *out, int n_out);

/* Per-level sizes after setup: n rows, true nnzb, stored SELL entries of A,
 * nnz of P (into the level) and of R.  Returns 0 or MG_ERR_INVALID_ARG. */
int mgi_level_info(mgi_ctx ctx, int level, int64_t *n, int64_t *nnzb, int64_t *sell_entries, int64_t *nnz_p,
                   int64_t *sell_entries_p, int64_t *sell_entries_r);

#ifdef __cplusplus
}
#endif
#endif /* MGB200_MG_INTERNAL_H */
