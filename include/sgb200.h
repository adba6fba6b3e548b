/* sgb200.h — C ABI of the B200-native estimation-based SpGEMM (libsgb200.so).
 *
 * Drop-in boundary for the reference's `sketchgemm.spgemm` pipeline
 * (/root/reference/pkg/src/sketchgemm/engine.py:136-249).  The reference is a
 * pure-Python package with no FFI; these entry points are the stage operators
 * its engine calls, re-expressed as plain C over DEVICE pointers so that the
 * Python host (paper_2604_19004_b200/engine.py) binds them with ctypes exactly
 * as a maintainer would from sketchgemm.
 *
 * Conventions
 *  - every pointer is a device pointer unless named *_host;
 *  - CSR: row_ptr int64[n+1], col_idx int32[nnz], values f64 (dtype 0) or
 *    f32 (dtype 1); per-row arrays are int64 unless stated;
 *  - `stream` is a cudaStream_t (NULL = legacy default stream);
 *  - return 0 on success, else an SG_ERR_* code; sg_last_error() gives the
 *    message of the last failure on the calling thread;
 *  - no global mutable state besides the per-thread error string: scratch is
 *    passed in (`ws`, sized by sg_workspace_bytes), so calls are reentrant.
 */
#ifndef SGB200_H
#define SGB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SG_OK 0
#define SG_ERR_ARG 1
#define SG_ERR_CUDA 2
#define SG_ERR_WORKSPACE 3

#define SG_F64 0
#define SG_F32 1

/* prediction kinds (predict.py:27-30) */
#define SG_PRED_EXACT 0
#define SG_PRED_ESTIMATED 1
#define SG_PRED_UPPER 2

/* plan kinds (accumulate.py:39-44) */
#define SG_KIND_HASH 0
#define SG_KIND_ENHANCED_HASH 1
#define SG_KIND_DENSE 2
#define SG_KIND_ESC 3
#define SG_KIND_FALLBACK 4

/* Tier ladder (accumulate.py:47-61). */
typedef struct sg_tiers {
  int32_t n_hash;
  int32_t n_dense;
  int64_t hash_caps[8];
  int64_t dense_spans[8];
  int64_t enh_cap;
  int64_t esc_max;
  double coef;
} sg_tiers_t;

int sg_abi_version(void);
const char* sg_last_error(void);

/* Number of kernels this library has enqueued since load (diagnostic;
 * bench.py reports the count inside its timed region). */
unsigned long long sg_launch_count(void);

/* Per-kernel device timer (measurement only; bench.py's roofline).  Enabling
 * (or disabling) clears the record; while enabled, the dominant kernels
 * ("k_bmr", "k_expand", "k_hash_warp", "k_hash_block", "k_bitmap") are
 * bracketed by CUDA events on their launching stream.  sg_kernel_time
 * waits for the recorded launches of `name` and returns their summed
 * duration and count. */
int sg_kernel_timer(int enable);
int sg_kernel_time(const char* name, double* total_ms, int64_t* launches);

/* Scratch bytes needed by sg_symbolic / sg_numeric / sg_fallback / sg_scan
 * for a problem with `m` rows of A. */
size_t sg_workspace_bytes(int64_t m);

/* Replaces analysis.compute_row_stats (analysis.py:96-128): products per row,
 * output span [span_lo, span_hi] (sentinels b_ncols / -1 when a row has no
 * products); totals2[0] = total products, totals2[1] = max row products. */
int sg_row_stats(int64_t m, int64_t b_ncols, const int64_t* a_ptr, const int32_t* a_col,
                 const int64_t* b_ptr, const int32_t* b_col, int64_t* products,
                 int64_t* span_lo, int64_t* span_hi, int64_t* totals2, void* stream);

/* Replaces analysis.build_b_sketches (analysis.py:131-146) + hll.hash_ranks
 * (hll.py:64-76): regs is uint8[k * 2^p], one HLL sketch per row of B. */
int sg_hll_build(int64_t k, const int64_t* b_ptr, const int32_t* b_col, int p, uint8_t* regs,
                 void* stream);

/* Replaces analysis.merged_row_estimates (analysis.py:149-169) and
 * predict.estimate_pass (predict.py:87-103): per selected row of A (rows ==
 * NULL selects all nsel = m rows), max-merge the sketches of the B rows it
 * selects and estimate (hll.py:79-86).  lin_table[z] = m*ln(m/z) for z in
 * 1..m-1 (precomputed by the host with the reference's own log so the
 * linear-counting branch is bit-identical); alpha_mm = (alpha_m*m)*m. */
int sg_hll_estimate(int64_t nsel, const int64_t* rows, const int64_t* a_ptr,
                    const int32_t* a_col, const uint8_t* regs, int p, const double* lin_table,
                    double alpha_mm, double* est, void* stream);

/* Numeric windows of long rows, recorded by the count kernels (sg_symbolic,
 * sg_fallback mode 0) and consumed by sg_window_numeric.
 *  win_off  int64[m+1]  window-slot offsets (from sg_window_capacity)
 *  wins     int32[2*win_off[m]] (first column, rank in row) pairs, init -1
 *  nwin     int32[m]    slots used per row, init 0
 *  bm_off   int64[m+1]  64-column word offsets of saved key bitmaps, or NULL
 *  bm_save  16-byte words [bm_off[m]]: per 64 columns {bits 0-31, row rank
 *           of bit 0, bits 32-63, row rank of bit 32} (uint32 x 4), or NULL
 *           (then the numeric pass rebuilds each window's key bitmap from the
 *           products); lets the numeric pass skip the key pass and the
 *           prefix, and bulk-copy a window's words into shared memory
 *  pre_save unused (NULL)
 * Windows start on 4096-column tiles and hold at most 8192 distinct columns
 * over at most 131072 columns (greedy cuts in column order), so two windows'
 * bitmaps and values sit in one SM's shared memory. */
typedef struct sg_windows {
  const int64_t* win_off;
  int32_t* wins;
  int32_t* nwin;
  const int64_t* bm_off;
  uint64_t* bm_save;
  int32_t* pre_save;
  const int64_t* btile_off; /* B tile index (sg_btile_plan/build), or NULL */
  const int32_t* btile;
} sg_windows_t;

/* B tile index: for the longest B rows (as many as fit budget_bytes), the
 * offset within the row of the first column >= t*4096 for every tile t, so
 * the numeric windows (which start on 4096-column tiles) clip B rows with two
 * lookups instead of binary searches.  sg_btile_plan writes tbl_scan
 * int64[k+1] (exclusive scan of table sizes), totals_host[0] = table entries,
 * totals_host[1] = minimum indexed row length (-1: none); sg_btile_build then
 * fills tbl_off int64[k] (-1 for rows without a table) and tbl int32[]. */
int sg_btile_plan(int64_t k, int64_t b_ncols, const int64_t* b_ptr, int64_t budget_bytes,
                  int64_t* tbl_scan, int64_t* totals_host, void* ws, size_t ws_bytes, void* stream);
int sg_btile_build(int64_t k, int64_t b_ncols, const int64_t* b_ptr, const int32_t* b_col,
                   const int64_t* tbl_scan, int64_t* tbl_off, int32_t* tbl, void* stream);

/* Sizes the window tables for rows with select[row] != 0 (all rows when
 * select == NULL): writes win_off and, if bm_off != NULL, bm_off (both
 * int64[m+1] exclusive scans); totals_host[0] = win_off[m],
 * totals_host[1] = bm_off[m] (0 without bm_off). */
int sg_window_capacity(int64_t m, const int64_t* products, const int64_t* span_lo,
                       const int64_t* span_hi, const uint8_t* select, int64_t* win_off,
                       int64_t* bm_off, int64_t* totals_host, void* ws, size_t ws_bytes,
                       void* stream);

/* Replaces predict.symbolic_pass (predict.py:39-84): exact distinct output
 * columns per row of C (counts int64[m]).  With win != NULL, rows counted
 * with a bitmap also record their numeric windows (and save their bitmaps
 * when win->bm_save != NULL).  assist_cr > 1 enables assisted symbolic
 * binning: hash-counted rows are sized by
 * products / assist_cr (the conservative sampled CR, predict.py:111-118)
 * and rows whose table fills are recounted with product sizing; 1 = the
 * reference's product sizing.  Counts are exact either way.  Rows with
 * 0 < products <= min(skip_max_products, 1024) are not counted (counts = -2):
 * the caller accumulates them into a staging slab instead (0 = count all). */
int sg_symbolic(int64_t m, int64_t b_ncols, const int64_t* a_ptr, const int32_t* a_col,
                const int64_t* b_ptr, const int32_t* b_col, const int64_t* products,
                const int64_t* span_lo, const int64_t* span_hi, int64_t* counts,
                const sg_windows_t* win, double assist_cr, int64_t skip_max_products, void* ws,
                size_t ws_bytes, void* stream);

/* Long-row numeric pass over the recorded windows, work grouped by column
 * range so concurrent CTAs share B-row slabs in L2; values accumulated in
 * shared memory (fp64) and written sorted at out_off[row] + rank (out_off =
 * row_ptr of C).  Windows of rows with saved words: the warp-specialised
 * window kernel writes their columns (from the words) and values (optional
 * SG_LIGHT_LEN: light B rows through REDs at the saved ranks instead); other
 * windows: one CTA per window rebuilds the window's keys.  work_buf: scratch
 * of work_cap >= sg_window_work_bytes(m, nnz(A), total windows) bytes. */
int sg_window_numeric(int64_t m, int64_t b_ncols, int dtype, const int64_t* a_ptr,
                      const int32_t* a_col, const void* a_val, const int64_t* b_ptr,
                      const int32_t* b_col, const void* b_val, const int64_t* span_lo,
                      const int64_t* span_hi, const sg_windows_t* win, const int64_t* out_off,
                      int32_t* out_col, void* out_val, void* work_buf, int64_t work_cap, void* ws,
                      size_t ws_bytes, void* stream);

/* Deterministic values (EngineConfig(deterministic=True)): recomputes every
 * value of C -- whose structure (c_ptr, c_col, sorted) is final -- as a
 * sequential sum in the reference's stream order (A entries ascending, then
 * each B row's entries), one warp per row, no atomics: bit-identical run to
 * run (the reference's guarantee, engine.py:13-14).  acc: double[nnz(C)]
 * scratch (may be c_val itself when dtype is f64). */
int sg_det_values(int64_t m, int dtype, const int64_t* a_ptr, const int32_t* a_col, const void* a_val,
                  const int64_t* b_ptr, const int32_t* b_col, const void* b_val, const int64_t* c_ptr,
                  const int32_t* c_col, void* c_val, double* acc, void* stream);

/* Scratch bytes sg_window_numeric needs: window work items plus the heavy /
 * light entry tables of the windowed rows. */
int64_t sg_window_work_bytes(int64_t m, int64_t nnz_a, int64_t nwindows);

/* Replaces accumulate.plan_rows (accumulate.py:104-181) with the identical
 * integer rules.  pred is int64 (EXACT / UPPER) or f64 (ESTIMATED). */
int sg_plan(int64_t m, int pred_kind, const void* pred, const int64_t* products,
            const int64_t* span_lo, const int64_t* span_hi, const sg_tiers_t* tiers,
            int8_t* kind, int64_t* cap, int64_t* alloc, void* stream);

/* Exclusive prefix sum of int64 in[n] into out[n+1] (engine.py:256-258,349-350). */
int sg_scan(int64_t n, const int64_t* in, int64_t* out, void* ws, size_t ws_bytes, void* stream);

/* Replaces engine._numeric_phase (engine.py:252-309) with the batch kernels
 * accumulate_hash_like / accumulate_esc / accumulate_dense
 * (accumulate.py:335-430): every row whose plan kind is not FALLBACK and that
 * has products is accumulated and written SORTED at out_off[row] (hash rows
 * are sorted in-kernel: engine._sort_hash_rows, engine.py:331-343).
 * counts[row] = distinct count (0 if overflowed); overflow[row] = 1 when the
 * reference's tier limit is exceeded (hash: count > floor(0.8*cap); dense:
 * count > alloc).  Rows with skip_nwin[row] > 0 (nullable) are left to
 * sg_window_numeric.  exact (nullable): the rows' exact distinct counts
 * (symbolic workflow); hash tables are then sized by them instead of by the
 * tier capacity, and a row over its limit is flagged without accumulating
 * (same overflow set, same C).  escr_max > 0: rows of <= min(escr_max, 512)
 * products (columns < 2^23, not DENSE, within their limit) use the register
 * expand-sort-compress accumulator (low-CR short rows; 0 = off). */
int sg_numeric(int64_t m, int64_t b_ncols, int dtype, const int64_t* a_ptr, const int32_t* a_col,
               const void* a_val, const int64_t* b_ptr, const int32_t* b_col, const void* b_val,
               const int8_t* kind, const int64_t* cap, const int64_t* alloc,
               const int64_t* products, const int64_t* span_lo, const int64_t* span_hi,
               const int64_t* out_off, int32_t* out_col, void* out_val, int64_t* counts,
               uint8_t* overflow, const int32_t* skip_nwin, const int64_t* exact, int64_t escr_max,
               void* ws, size_t ws_bytes, void* stream);

/* Rows for the fallback pass (engine.py:202-203): overflow | (kind ==
 * FALLBACK & products > 0), ascending, minus rows with exclude_nwin[row] > 0
 * (nullable); *n_out_host receives the count. */
int sg_select_fallback(int64_t m, const int8_t* kind, const int64_t* products,
                       const uint8_t* overflow, const int32_t* exclude_nwin, int64_t* rows_out,
                       int64_t* n_out_host, void* ws, size_t ws_bytes, void* stream);

/* Replaces engine._fallback_phase (engine.py:312-328) /
 * accumulate.fallback_accumulate (accumulate.py:274-279): exact accumulation
 * of the given rows, which can never overflow.  mode 0 = count only
 * (counts[row] written; numeric windows recorded when win != NULL, as in
 * sg_symbolic), mode 1 = numeric, written sorted at out_off[row]. */
int sg_fallback(int mode, int64_t nrows, const int64_t* rows, int64_t b_ncols, int dtype,
                const int64_t* a_ptr, const int32_t* a_col, const void* a_val,
                const int64_t* b_ptr, const int32_t* b_col, const void* b_val,
                const int64_t* products, const int64_t* span_lo, const int64_t* span_hi,
                const int64_t* out_off, int32_t* out_col, void* out_val, int64_t* counts,
                const sg_windows_t* win, void* ws, size_t ws_bytes, void* stream);

/* Replaces engine.compact (engine.py:346-368): copy counts[row] entries of
 * every row with skip[row] == 0 from src_off[row] to dst_off[row]. */
int sg_compact(int64_t m, int dtype, const int64_t* counts, const uint8_t* skip,
               const int64_t* src_off, const int64_t* dst_off, const int32_t* src_col,
               const void* src_val, int32_t* dst_col, void* dst_val, void* stream);

/* Estimation error of per-row predictions (engine.py:218-226, the est-eval
 * harness cli.py:301-341): over rows with row_ptr[r+1] > row_ptr[r],
 * rel = |pred[r] - nnz_r| / nnz_r; out3 (host) = {live rows, mean rel,
 * population std of rel}.  Deterministic two-pass reduction; ws needs
 * 16 KB + 64 bytes of device scratch. */
int sg_est_errors(int64_t m, const double* pred, const int64_t* row_ptr, double* out3, void* ws, size_t ws_bytes,
                  void* stream);

/* ---- canonical CSR construction (the inputs' preparation on the device) */

/* Scratch bytes for sg_coo_to_csr / sg_transpose with `nnz` entries. */
size_t sg_build_workspace_bytes(int64_t nnz);

/* Replaces csr.from_triplets (csr.py:52-80): canonical CSR (rows ascending,
 * columns ascending within a row, duplicate coordinates summed in input
 * order) from nnz device triplets rows[i], cols[i] (int64) and vals[i]
 * (dtype SG_F64 / SG_F32).  col_out / val_out hold nnz slots; row_ptr holds
 * nrows + 1; *nnz_out_host receives the unique count.  SG_ERR_ARG for a
 * coordinate outside [0, nrows) x [0, ncols) or dimensions / nnz beyond the
 * 32-bit index limit (csr.py:57-63). */
int sg_coo_to_csr(int64_t nrows, int64_t ncols, int64_t nnz, const int64_t* rows, const int64_t* cols,
                  const void* vals, int dtype, int64_t* row_ptr, int32_t* col_out, void* val_out,
                  int64_t* nnz_out_host, void* ws, size_t ws_bytes, void* stream);

/* Replaces csr.transpose (csr.py:90-97): exact transpose of a canonical
 * nrows x ncols CSR into t_ptr[ncols + 1], t_col / t_val[nnz] (canonical,
 * rows ascending within every column).  Used by the AA^T mode
 * (engine.py:113-128). */
int sg_transpose(int64_t nrows, int64_t ncols, const int64_t* row_ptr, const int32_t* col, const void* val,
                 int dtype, int64_t* t_ptr, int32_t* t_col, void* t_val, void* ws, size_t ws_bytes,
                 void* stream);

/* ---- result download (the e2e path) */

/* Copies `bytes` from device memory to pageable host memory after the work
 * already enqueued on `stream`: the copy engine fills a ring of pinned
 * 64 MB staging buffers (allocated once per process) while `threads` native
 * workers (0 = 8) move them into host_dst, taking its page faults in
 * parallel.  Blocks until done.  Replaces the host copy-out of the reference
 * result (engine.py:214-215 returns host arrays). */
int sg_download(void* host_dst, const void* dev_src, size_t bytes, int threads, void* stream);

/* Page-lock (first touching in parallel) / release a page-aligned host range
 * in 256 MB registrations measured from p.  A destination pinned this way
 * from its first byte is downloaded by direct DMA (sg_download checks).
 * Used by the host result pool (device.py) that recycles C's host buffers
 * across calls. */
int sg_host_pin(void* p, size_t bytes, int threads);
int sg_host_unpin(void* p, size_t bytes, int threads);

#ifdef __cplusplus
}
#endif
#endif /* SGB200_H */
