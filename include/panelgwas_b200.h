/*
 * panelgwas_b200 — C ABI of the B200 (sm_100a) linear-association scan.
 *
 * This is the drop-in boundary for the hot path of the `panelgwas` reference
 * (/root/reference/pkg/src/panelgwas). The reference has no FFI of its own: its
 * boundary is Python. Each entry point below names the
 * reference interface it replaces; the Python host package
 * `paper_2604_21095_b200` (same names as panelgwas) binds them with ctypes,
 * and INTEGRATION.md shows the binding a panelgwas maintainer would add.
 *
 * Conventions
 *   - Every function returns a status code (PG_OK == 0). On failure the
 *     message is available from pg_last_error() (thread-local). Status codes
 *     map onto the reference exception classes (errors.py:4-17):
 *     PG_ERR_INVALID -> ValueError, PG_ERR_FORMAT -> FormatError,
 *     PG_ERR_CONFIG -> ConfigError, anything else -> PanelGwasError.
 *   - Host pointers are borrowed for the duration of the call. Device
 *     buffers, pinned staging and streams belong to the pg_ctx.
 *   - A pg_ctx is bound to one CUDA device; calls on one ctx are serialised
 *     by the caller (one ctx per GPU / per worker thread).
 *   - There is no CPU fallback: without a usable sm_100 device every compute
 *     entry point fails with PG_ERR_CUDA.
 */
#ifndef PANELGWAS_B200_H
#define PANELGWAS_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define PG_API __attribute__((visibility("default")))
#else
#define PG_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define PG_OK 0
#define PG_ERR_CUDA 1
#define PG_ERR_INVALID 2
#define PG_ERR_FORMAT 3
#define PG_ERR_NOMEM 4
#define PG_ERR_STATE 5
#define PG_ERR_CONFIG 6
/* not an error: pg_table_parse needs the generic (csv-module) path for this input */
#define PG_TABLE_GENERIC 100

/* Output modes (engine.py:41-44). */
#define PG_MODE_THRESHOLD 0
#define PG_MODE_TOPK 1
#define PG_MODE_FULL 2

/* Genotype encodings accepted by pg_scan_*. */
#define PG_GENO_BED 0       /* PLINK 2-bit codes, SNP-major rows (plink.py:29-61) */
#define PG_GENO_BGEN8 1     /* BGEN layout-2 probability pairs, 8-bit (bgen.py:238-249) */
#define PG_GENO_BGEN16 2    /* same, 16-bit */
#define PG_GENO_DENSE_F64 3 /* real dosages in [0,2], NaN = missing (dense.py:79-97) */

PG_API const char* pg_last_error(void);
PG_API int pg_abi_version(void);
/* Number of usable sm_100 devices (0 when none). */
PG_API int pg_device_count(int* n);

typedef struct pg_ctx pg_ctx;

/* Page-locked host memory for staging genotype blocks (cudaHostAlloc). */
PG_API int pg_host_alloc(int64_t bytes, void** out);
PG_API int pg_host_free(void* ptr);

/* Context lifetime. Replaces the panel-side state the reference shares
 * between workers, engine._Prepared (engine.py:154-167). */
PG_API int pg_ctx_create(int device, pg_ctx** out);
PG_API int pg_ctx_destroy(pg_ctx* ctx);
/* Synchronise the ctx stream (used before timing / teardown). */
PG_API int pg_ctx_sync(pg_ctx* ctx);
/* The ctx's cudaStream_t (as void*), for callers that time or order work on it. */
PG_API int pg_ctx_stream(pg_ctx* ctx, void** stream);

/* Device panel preparation: the reference's residualize + standardize_columns
 * (kernel.py:310-347, driven by engine.py:259-279) in fp64 on the GPU.
 *   y             host f64 [n_kept, ld] row-major (kept samples x phenotypes, missing
 *                 values already handled by the panel's missing policy)
 *   basis_q       host f64 [n_kept, rank] row-major orthonormal covariate basis
 *                 (kernel.build_covariate_basis; rank 0 = centring only)
 *   zero_variance out u8 [n_pheno]: 1 where sd <= 1e-12 max(1, |centre|) (kernel.py:344)
 *   sd            out f64 [n_pheno] (may be NULL)
 * The standardized panel stays on the device; pg_ctx_commit_panel quantizes the kept
 * columns into the resident limbs (same result as pg_ctx_set_panel on the host-prepared
 * matrix up to 1e-16 relative rounding). Non-finite input -> PG_ERR_INVALID. */
PG_API int pg_ctx_prepare_panel(pg_ctx* ctx, const double* y, int64_t n_kept, int64_t n_pheno, int64_t ld,
                                const double* basis_q, int64_t rank, uint8_t* zero_variance, double* sd);
/* Quantize prepared columns kept_cols[0..n_cols) (engine.py:271-279 drops zero-variance
 * columns) into the resident panel; geometry as pg_ctx_set_panel. */
PG_API int pg_ctx_commit_panel(pg_ctx* ctx, const int64_t* kept_cols, int64_t n_cols,
                               const int64_t* geno_row_index, int64_t n_samples_src);
/* Copy the prepared (standardized, uncompacted) panel back: out f64 [n_kept, n_pheno]. */
PG_API int pg_ctx_fetch_prepared_panel(pg_ctx* ctx, double* out);
/* Pipelined prepare + commit of ALL columns (the same reference steps as
 * pg_ctx_prepare_panel + pg_ctx_commit_panel with kept_cols = every column): `y` (page-locked
 * host memory) is uploaded in chunks of `chunk_cols` phenotypes (rounded up to 256), each
 * prepared and quantized as it lands, and the call returns at once. The next scan's GEMM
 * runs chunk by chunk as the chunks become ready, so the upload overlaps the first batch.
 * Without zero-variance columns the panel is bit-identical to the synchronous path; a
 * zero-variance column stays in the panel with r = 0 (the caller drops it, or uses the
 * synchronous path). pg_ctx_panel_async_wait returns the zero-variance flags and sd
 * (as pg_ctx_prepare_panel) once the preparation is complete; non-finite input ->
 * PG_ERR_INVALID there. */
PG_API int pg_ctx_set_panel_async(pg_ctx* ctx, const double* y, int64_t n_kept, int64_t n_pheno, int64_t ld,
                                  const double* basis_q, int64_t rank, const int64_t* geno_row_index,
                                  int64_t n_samples_src, int64_t chunk_cols);
PG_API int pg_ctx_panel_async_wait(pg_ctx* ctx, uint8_t* zero_variance, double* sd);
/* Multi-GPU panel preparation: as pg_ctx_set_panel_async for the panel geometry of all
 * n_pheno phenotypes, but this context uploads, prepares and quantizes only the columns
 * [col_begin, col_end) (a rank's share; multiples of 256, or ending at n_pheno), read from `y`
 * (page-locked, its column c at y[c - col_begin], `ld` per row); pg_ctx_panel_async_wait then
 * returns the flags / sd of those columns. The other rows arrive with
 * pg_ctx_import_panel_rows from the ranks that prepared them (pg_ctx_export_panel_rows; an
 * all-gather over NVLink in bench.py). pg_ctx_panel_rows_bytes: buffer size for n_rows rows. */
PG_API int pg_ctx_set_panel_async_cols(pg_ctx* ctx, const double* y, int64_t n_kept, int64_t n_pheno, int64_t ld,
                                       int64_t col_begin, int64_t col_end, const double* basis_q, int64_t rank,
                                       const int64_t* geno_row_index, int64_t n_samples_src, int64_t chunk_cols);
PG_API int pg_ctx_panel_rows_bytes(pg_ctx* ctx, int64_t n_rows, int64_t* bytes);
PG_API int pg_ctx_export_panel_rows(pg_ctx* ctx, void* d_dst, int64_t row_begin, int64_t row_end);
PG_API int pg_ctx_import_panel_rows(pg_ctx* ctx, const void* d_src, int64_t row_begin, int64_t row_end);
/* `follower` takes `leader`'s pipelined panel (pg_ctx_set_panel_async) chunk by chunk: each
 * chunk, once prepared on the leader, is copied device to device to the follower and marked
 * ready there, so both contexts' first scans run their GEMMs behind the one upload (two
 * contexts per GPU). Chunks are issued by whichever context needs the next
 * one. The leader must outlive the follower's use of the panel. */
PG_API int pg_ctx_follow_panel(pg_ctx* follower, pg_ctx* leader);
/* Copy `src`'s resident panel (limbs, scales, sample map) into `dst` on the same device, device
 * to device (export + import), so that two contexts can scan batches of one job in turn
 * ("two contexts per GPU"). Both must have the same precision mode. */
PG_API int pg_ctx_clone_panel(pg_ctx* dst, pg_ctx* src);

/* Upload the standardized phenotype panel once; it stays resident in HBM as
 * three int8 limb planes [P_pad, K_pad] (q = 32385 qH + 127 q1 + q0, 23-bit
 * per-phenotype quantization) plus per-phenotype scale and limb-sum vectors.
 * Replaces: engine._run_scan_open panel hand-off (engine.py:269-279) — the
 * `ytil` produced by kernel.standardize_columns (kernel.py:330-347).
 *   ytil            host f64, row i = kept sample i, `ld` elements per row
 *   geno_row_index  host i64 [n_kept]: genotype-file row of kept sample i
 *                   (phenotypes.align_samples, phenotypes.py:165-220)
 *   n_samples_src   samples in the genotype source (.fam rows) */
PG_API int pg_ctx_set_panel(pg_ctx* ctx, const double* ytil, int64_t n_kept, int64_t n_pheno, int64_t ld,
                     const int64_t* geno_row_index, int64_t n_samples_src);
/* Same, but `d_ytil` is a device pointer on the ctx device. */
PG_API int pg_ctx_set_panel_device(pg_ctx* ctx, const double* d_ytil, int64_t n_kept, int64_t n_pheno, int64_t ld,
                            const int64_t* geno_row_index, int64_t n_samples_src);
/* Export / import the resident split panel (device pointers, same layout and
 * size reported by *bytes) so it can be broadcast over NCCL between ranks. */
PG_API int pg_ctx_panel_bytes(pg_ctx* ctx, int64_t* bytes);
PG_API int pg_ctx_export_panel(pg_ctx* ctx, void* d_dst);
PG_API int pg_ctx_import_panel(pg_ctx* ctx, const void* d_src, int64_t n_kept, int64_t n_pheno,
                        const int64_t* geno_row_index, int64_t n_samples_src);

/* Extension mode (--residualize-genotypes; prepare_genotype_batch with
 * residualize_genotypes=True, kernel.py:409-410): project every genotype row off the
 * covariate basis Q (host f64 [n_kept, rank], kept-sample order, column 0 = the
 * normalised intercept as built by build_covariate_basis). Because the panel is already
 * orthogonal to Q only the per-marker variance changes: V_res = V - |Q^T g_c|^2, computed
 * by an exact side GEMM of the genotype codes against the quantized basis. rank <= 1
 * (or q == NULL) switches the extension off. Call after pg_ctx_set_panel. */
PG_API int pg_ctx_set_basis(pg_ctx* ctx, const double* q, int64_t n_kept, int64_t rank);

/* Scan parameters. `r_bar` (host f64 [n_pheno]) is the per-phenotype premask
 * bar on |r| — engine._abs_t_to_abs_r / premask_abs_r (engine.py:170-175,
 * 321-333) for THRESHOLD, the TopKWriter bar for TOPK (engine.py:205-211).
 * Candidates are pairs of non-skipped markers with |r| >= r_bar. */
PG_API int pg_ctx_set_scan(pg_ctx* ctx, double df, int mode, const double* r_bar);
/* Replace the premask bar between batches without resetting the scan (TOPK bar
 * tightening, engine.py:205-211 / output.py:199-200). */
PG_API int pg_ctx_set_rbar(pg_ctx* ctx, const double* r_bar);

/* Dosage sources (BGEN, real-valued dense) use the wide-digit GEMM (base-255 digits, 4 rows
 * per marker, 3 accumulators) by default; 0 selects the balanced-ternary planes (8 / 16 rows).
 * Both are exact integer contractions: results are bitwise identical (A/B switch). */
PG_API int pg_ctx_set_wide_digits(pg_ctx* ctx, int enable);
/* Tuning switch: decode PLINK rows inside the GEMM producer (default 1) or through
 * materialized int8 planes (0). Results are identical; exposed for A/B measurement. */
PG_API int pg_ctx_set_fused_decode(pg_ctx* ctx, int enable);
/* PLINK batches with missing calls (reference imputes them per marker, kernel.py:399-408):
 * 1 (default) keeps the fused one-row-per-marker GEMM and runs the missing-call mask rows of
 * only the markers that have any through a side GEMM; 0 sends the whole batch to the two-row
 * (dosage, mask) planes. Exact either way: results are bitwise identical (A/B switch). */
PG_API int pg_ctx_set_missing_side_gemm(pg_ctx* ctx, int enable);
/* Precision.F64 (engine.py:31-33: float64 storage end to end): 1 quantizes the panel at two
 * levels (y~ = s (q + q2 / 2^22), ~46 bits) and runs the exact GEMM once per level, summing
 * the int64 partials before the statistics; 0 (default, the reference's default f32 mode's
 * accuracy class) one 23-bit level. Call before the panel is uploaded (pg_ctx_set_panel /
 * pg_ctx_commit_panel / pg_ctx_import_panel); changing it drops the current panel. */
PG_API int pg_ctx_set_f64_panel(pg_ctx* ctx, int enable);
/* PLINK THRESHOLD / TOPK scans (default 1): the GEMM runs two of the three panel limbs (two
 * MMAs per 32 samples); the premask is widened by the rigorous bound |sum_k q0 u| <=
 * ||q0_p||_2 ||u_m||_2 on the deferred limb, and every candidate gets sum_k q0 u added
 * exactly before its fp64 r, t and p (results bitwise identical to 0 = all three limbs). */
PG_API int pg_ctx_set_two_limb_premask(pg_ctx* ctx, int enable);

/* Result summary of the last scan call. */
typedef struct pg_batch_info {
  int64_t n_markers;
  int64_t n_candidates; /* THRESHOLD/TOPK: candidate pairs held by the ctx */
  int64_t clamp_count;  /* |r| > 1 before clipping (kernel.py:455) */
  int64_t n_skipped_monomorphic;
  int64_t n_skipped_all_missing;
  double gemm_ms;       /* device time of the association kernel(s) */
  double decode_ms;     /* device time of the decode kernels */
  int64_t launches;     /* kernels of this library launched for the batch */
  int64_t rows_per_marker; /* GEMM rows per marker (1: PLINK, 2: + missing calls, 8/16: BGEN / real dosages) */
} pg_batch_info;

/* Scan one block of markers from HOST memory.
 * Replaces, fused: <Source>.read_marker_batch (plink.py:167-185, bgen.py:251-262,
 * dense.py:79-97) -> prepare_genotype_batch (kernel.py:376-421) ->
 * correlate (kernel.py:428-457) -> premask + t_from_r (engine.py:197-217) ->
 * p_from_t for candidates (output.py:129).
 *   geno_kind  PG_GENO_*
 *   data       BED: uint8 rows of `row_bytes` = ceil(n_samples_src/4)
 *              BGEN8/16: per marker, the inflated probability pairs
 *                        [n_samples_src x 2] (u8 or u16) then n_samples_src
 *                        ploidy bytes (bit 7 = missing)
 *              DENSE_F64: f64 rows of n_samples_src dosages
 *   row_bytes  bytes per marker row in `data` */
PG_API int pg_scan(pg_ctx* ctx, int geno_kind, const void* data, int64_t n_markers, int64_t row_bytes,
            pg_batch_info* info);
/* Same, with `d_data` already resident on the device (rows `row_pitch` bytes apart,
 * row_pitch a multiple of 16). */
PG_API int pg_scan_device(pg_ctx* ctx, int geno_kind, const void* d_data, int64_t n_markers, int64_t row_bytes,
                   int64_t row_pitch, pg_batch_info* info);

/* Stage a BGEN batch COMPRESSED: `blob` is the host byte range of the file holding the
 * batch's genotype blocks; block i = blob[block_off[i], +block_size[i]) (the u32
 * uncompressed length + zlib stream, bgen.py:183-196). The blocks are inflated on the GPU
 * (one warp per stream), validated with the reference reader's checks and repacked into
 * slot `slot` for pg_scan_staged (8- or 16-bit rows; mixed batches widened exactly).
 * On PG_ERR_FORMAT diag = {variant, reason, a, b} as pg_bgen_inflate; reason 2 (zlib
 * stream error or oversize output) carries no message: re-inflate that block with
 * pg_bgen_inflate on the host to obtain zlib's own text. */
PG_API int pg_stage_bgen(pg_ctx* ctx, int slot, const void* blob, int64_t blob_bytes, const int64_t* block_off,
                         const int64_t* block_size, int64_t count, int64_t* diag);
/* The same in two phases, so the H2D and inflate of batch i+1 overlap the scan of batch i:
 * _begin enqueues everything on the copy stream and returns (`blob` must stay valid and
 * unmodified until _end; pinned memory makes the copy asynchronous); _end waits for the
 * validation summary, reports errors like pg_stage_bgen, and enqueues the repack. */
PG_API int pg_stage_bgen_begin(pg_ctx* ctx, int slot, const void* blob, int64_t blob_bytes,
                               const int64_t* block_off, const int64_t* block_size, int64_t count);
PG_API int pg_stage_bgen_end(pg_ctx* ctx, int slot, int64_t* diag);

/* Asynchronous staging for pipelined scans (transfer of batch i+1 overlaps the
 * GEMM of batch i). pg_stage copies HOST rows into staging slot `slot` (0 or 1) on
 * the ctx's copy stream and returns immediately; `data` must stay valid (pinned
 * memory recommended) until pg_scan_staged(slot) returns. pg_scan_staged waits
 * for the slot's copy on the device, then scans it exactly like pg_scan. */
PG_API int pg_stage(pg_ctx* ctx, int slot, int geno_kind, const void* data, int64_t n_markers, int64_t row_bytes);
PG_API int pg_scan_staged(pg_ctx* ctx, int slot, pg_batch_info* info);

/* Per-marker QC of the last scan: StandardizedBatch.allele_frequency,
 * missing_count, variance_before_scaling, skip_reason (kernel.py:360-373). Any pointer may be NULL. */
PG_API int pg_fetch_marker_stats(pg_ctx* ctx, double* af, int64_t* missing_count, double* variance, int8_t* skip);
/* Candidates of the last scan in (marker, phenotype) order: BatchStats.cand_rows,
 * cand_cols, cand_r, cand_t (output.py:74-87) plus their two-sided p (fp64,
 * floored at P_FLOOR; kernel.py:192-209). Any pointer may be NULL. */
PG_API int pg_fetch_candidates(pg_ctx* ctx, int64_t* rows, int64_t* cols, double* r, double* t, double* p);
/* FULL mode: t of non-skipped markers, row-major [n_ok, n_pheno], f32 (elem=4)
 * or f64 (elem=8) — BatchStats.t_rows (engine.py:197-198). */
PG_API int pg_fetch_full(pg_ctx* ctx, void* out, int elem_bytes, int64_t* n_rows);
/* Per-phenotype max |r| (exact fp64 r of the maximizing pair) over all non-skipped markers
 * scanned since tracking was enabled: the minimum-p statistic. Tracking is off by default
 * (it costs the GEMM epilogue a compare per pair); pg_ctx_track_max_abs_r(ctx, 1) after
 * pg_ctx_set_scan enables it and clears the maxima. */
PG_API int pg_ctx_track_max_abs_r(pg_ctx* ctx, int enable);
PG_API int pg_fetch_max_abs_r(pg_ctx* ctx, double* out);

/* ---- effect sizes (north star: beta / t / -log10 p) ----
 * The reference engine reports R T P only (output.py:29-43); beta exists in its OLS oracle
 * (oracle.ols_single, oracle.py:35-90). With pheno_sd[j] = sd (1/N) of kept residualized
 * phenotype j (standardize_columns, kernel.py:330-347) and var = the marker's
 * variance_before_scaling (kernel.py:411), each scan also yields
 *   beta = r * pheno_sd / sqrt(var),  se = pheno_sd / sqrt(var) * sqrt((1 - r^2) / df),
 * the slope of y_res on g and its standard error (beta / se == t). With
 * residualize_genotypes + adjusted df these equal ols_single(y, g, C).beta / .se.
 * pheno_sd == NULL disables; a new panel disables. */
PG_API int pg_ctx_set_beta_scale(pg_ctx* ctx, const double* pheno_sd, int64_t n_pheno);
/* beta / se of the last scan's candidates, aligned with pg_fetch_candidates. NULL skips. */
PG_API int pg_fetch_candidate_beta(pg_ctx* ctx, double* beta, double* se);
/* FULL mode: beta rows aligned with pg_fetch_full (se = beta / t). */
PG_API int pg_fetch_full_beta(pg_ctx* ctx, void* out, int elem_bytes, int64_t* n_rows);
/* Test hook: the next scans start the 64-bit candidate counter at `base` instead of 0
 * (candidate slots are counter - base), so a test can drive the counter across 2^31
 * inside one launch without producing 2^31 candidates. */
PG_API int pg_ctx_debug_candidate_base(pg_ctx* ctx, uint64_t base);

/* ---- element-wise statistics on the device (host arrays in/out) ---- */
/* kernel.t_from_r (kernel.py:460-478) */
PG_API int pg_t_from_r(pg_ctx* ctx, const double* r, int64_t n, double df, double* t);
/* kernel.p_from_t (kernel.py:192-209); counts p <= P_FLOOR into *underflow (may be NULL) */
PG_API int pg_p_from_t(pg_ctx* ctx, const double* t, int64_t n, double df, double* p, int64_t* underflow);
/* kernel.reg_inc_beta (kernel.py:147-189), broadcast already applied by caller */
PG_API int pg_reg_inc_beta(pg_ctx* ctx, const double* a, const double* b, const double* x, int64_t n, double* out);
/* kernel.p_from_t for a scalar t: the reference's scalar path (kernel.py:201-204 ->
 * _reg_inc_beta_scalar, kernel.py:136-144), the form t_threshold_for_p bisects on */
PG_API int pg_p_from_t_scalar(pg_ctx* ctx, double t, double df, double* p);
/* kernel.reg_inc_beta with scalar a, b, x (kernel.py:156-163 -> _reg_inc_beta_scalar) */
PG_API int pg_reg_inc_beta_scalar(pg_ctx* ctx, double a, double b, double x, double* out);
/* kernel.t_threshold_for_p (kernel.py:212-235) */
PG_API int pg_t_threshold_for_p(pg_ctx* ctx, double p_threshold, double df, double* t_crit);

/* Native BGEN v1.2 variant index (host). Replaces BgenSource._index_variants
 * (genotypes/bgen.py:130-168): walks n_variants headers from byte first_variant of the
 * memory-mapped file. Per variant: block_offset/block_size of the compressed genotype
 * block, position, and 5 strings (variant id, rsid, chrom, allele1, allele2) as byte
 * ranges text[text_off[5v+s] .. text_off[5v+s+1]) (text_off has 5n+1 entries).
 * On PG_ERR_FORMAT diag = {variant, kind, detail, 0}: kind 1 truncated header field
 * (detail = field code), 2 n_alleles != 2 (detail = n), 3 payload past EOF (detail = size);
 * PG_ERR_INVALID with kind 4: text buffer too small. On success diag[0] = end offset. */
PG_API int pg_bgen_index(const char* path, int64_t first_variant, int64_t n_variants, int64_t* block_offset,
                         int64_t* block_size, uint32_t* position, char* text, int64_t text_cap, int64_t* text_off,
                         int64_t* diag);
/* Parallel zlib inflate + validation of `count` genotype blocks (host threads; replaces the
 * inflate half of BgenSource._decode_variant, genotypes/bgen.py:183-232) into device-staging
 * rows [2n probabilities (u8 | u16) | n ploidy bytes]. `rows` must hold count x row_cap
 * bytes with row_cap >= 5n; on success rows are packed at *out_row_bytes (3n or 5n) and
 * *out_bits is 8 or 16 (mixed batches are widened exactly, x257). On PG_ERR_FORMAT
 * diag = {variant, reason, a, b} (reasons: 1 block < 4 B, 2 zlib (message in pg_last_error),
 * 3 inflated size (a got, b want), 4 sample count (a), 5 alleles (a), 6 ploidy range (a, b),
 * 7 non-diploid, 8 phased, 9 bits (a), 10 block size (a got, b want), 11 past EOF). */
PG_API int pg_bgen_inflate(const char* path, const int64_t* block_offset, const int64_t* block_size, int64_t count,
                           int64_t n_samples, int n_threads, uint8_t* rows, int64_t row_cap, int* out_bits,
                           int64_t* out_row_bytes, int64_t* diag);

/* Native table-body parser (host). Replaces the cell loop of
 * phenotypes.load_table (phenotypes.py:67-138): records after the header line
 * (starting at byte body_offset, physical line number first_lineno), cells split on
 * `delim`, blank lines skipped, ID cell (field id_field) stripped, value cells ->
 * NaN for {"", "NA", "NaN", "nan", "-9"}, Python float() otherwise, unparseable or
 * non-finite -> NaN counted per column. Call once with values == NULL to get *n_rows,
 * then with values [n_rows, n_fields-1], id_off/id_len [n_rows] (byte ranges into buf),
 * missing/unparseable [n_fields-1]. A ragged record -> PG_ERR_FORMAT with *err_line /
 * *err_cells; PG_TABLE_GENERIC when quoting, '\r', non-ASCII or '_' appear. */
PG_API int pg_table_parse(const char* buf, int64_t len, int64_t body_offset, char delim, int64_t n_fields,
                          int64_t id_field, int n_threads, int64_t first_lineno, int64_t* n_rows, double* values,
                          int64_t* id_off, int64_t* id_len, int64_t* missing, int64_t* unparseable,
                          int64_t* err_line, int64_t* err_cells);

/* ---- native TSV emitter (host code; output.py:50-52, 106-113) ---- */
/* Python repr(float) of each value, one per line ('\n'-terminated). */
PG_API int pg_format_float_repr(const double* x, int64_t n, char* out, int64_t out_cap, int64_t* out_len);
/* THRESHOLD / TOPK record lines, byte-identical to the reference writer: per record
 * <prefix[row]>AF\tN_MISS<mid>R\tT\tP\t<pheno[col]>\n with repr() floats. prefix / pheno
 * strings are given as blobs + offset arrays (n_rows+1 / n_pheno+1 entries). */
PG_API int pg_format_tsv(int64_t n, const int64_t* rows, const int64_t* cols, const double* r, const double* t,
                         const double* p, const double* af, const int64_t* n_miss, const char* prefix_blob,
                         const int64_t* prefix_off, const char* pheno_blob, const int64_t* pheno_off,
                         const char* mid, int64_t mid_len, char* out, int64_t out_cap, int64_t* out_len);

/* n lines of ncols tab-separated doubles rendered as Python repr() (effect-size sidecar
 * BETA\tSE lines, aligned with the record lines). PG_ERR_INVALID when out_cap is too small. */
PG_API int pg_format_float_columns(int64_t n, int ncols, const double* const* cols, char* out, int64_t out_cap,
                                   int64_t* out_len);

/* TOPK writer merge (host; output.TopKWriter.emit, output.py:155-213): the held records
 * (sorted by phenotype, p, marker source index) and a batch's new candidates (any order, every
 * source index above the held ones) merged per phenotype, the first k of each kept. out_idx
 * (capacity n_pheno * k) receives indices into [held ++ fresh] in (phenotype, p, source index)
 * order, *n_out their count. Phenotypes are merged in parallel on host threads. */
PG_API int pg_topk_merge(int64_t n_pheno, int64_t k, const int64_t* held_col, const double* held_p,
                         const int64_t* held_src, int64_t n_held, const int64_t* fresh_col, const double* fresh_p,
                         const int64_t* fresh_src, int64_t n_fresh, int64_t* out_idx, int64_t* n_out);

/* The merge's column gather: out_cols[c][i] = held_cols[c][idx[i]] (idx[i] < n_held) or
 * fresh_cols[c][idx[i] - n_held], for n_cols columns of 8-byte elements, on host threads. */
PG_API int pg_topk_gather(int64_t n_out, const int64_t* idx, int64_t n_held, int n_cols, const void* const* held_cols,
                          const void* const* fresh_cols, void* const* out_cols);
/* out = src[starts[i] .. starts[i] + lens[i]) for i < n, concatenated (TOPK line prefixes). */
PG_API int pg_gather_spans(const char* src, const int64_t* starts, const int64_t* lens, int64_t n, char* out);

/* FULL-mode marker sidecar lines "SOURCE_INDEX CHR ID POS A1 A2 AF N_MISS" (tab-separated, LF) of
 * markers rows[0..n): replaces the per-marker f-string of FullMatrixWriter.emit
 * (/root/reference/pkg/src/panelgwas/output.py:245-252). prefix blob/offsets as in pg_format_tsv;
 * AF rendered as Python repr. PG_ERR_INVALID when out_cap is too small. */
PG_API int pg_format_marker_lines(int64_t n, const int64_t* rows, const int64_t* src_index,
                                  const char* prefix_blob, const int64_t* prefix_off, const double* af,
                                  const int64_t* n_miss, char* out, int64_t out_cap, int64_t* out_len);

/* PLINK .bim catalog (host). pg_bim_index validates the reference grammar
 * (/root/reference/pkg/src/panelgwas/genotypes/plink.py:64-90: 6 fields per non-blank line,
 * position an integer >= 0) and records per marker the byte spans of chrom / id / allele1 /
 * allele2 (tok_start, tok_len: [cap x 4]) and the position; *same counts markers with equal
 * alleles. PG_TABLE_GENERIC (100) when the file needs the line-by-line reader (non-ASCII, bare
 * CR, field-count or position errors: that reader raises the reference's message).
 * pg_bim_prefixes renders "CHR\tID\tPOS\tA1\tA2\t" for markers [first, first+count)
 * (alleles swapped when swap != 0) with out_off[count+1] byte offsets. */
PG_API int pg_bim_index(const char* buf, int64_t len, int64_t cap, int64_t* n, int64_t* tok_start,
                        int32_t* tok_len, int64_t* pos, int64_t* same);
PG_API int pg_bim_prefixes(const char* buf, const int64_t* tok_start, const int32_t* tok_len, const int64_t* pos,
                           int64_t first, int64_t count, int swap, char* out, int64_t out_cap, int64_t* out_off);

/* ---- genotype decode on the device (host arrays in/out) ---- */
/* PlinkSource.read_marker_batch / decode_bed_codes (plink.py:48-61, 167-185):
 * rows of `row_bytes` packed codes -> dosages (elem 4: f32, 8: f64) [n_markers, n_samples]
 * with NaN for missing, plus per-row NaN counts. */
PG_API int pg_decode_bed(pg_ctx* ctx, const uint8_t* packed, int64_t n_markers, int64_t row_bytes, int64_t n_samples,
                  int elem_bytes, void* dosages, int64_t* missing_count);
/* BgenSource._decode_variant probability -> dosage map (bgen.py:238-249). */
PG_API int pg_decode_bgen(pg_ctx* ctx, const void* probs, const uint8_t* ploidy, int64_t n_markers, int64_t n_samples,
                   int bits, double* dosages, int64_t* missing_count);

/* ---- library kernels (kernel.py public API) ---- */
/* prepare_genotype_batch (kernel.py:376-421) without genotype residualization
 * (or with it when q != NULL): f64 in, standardized rows out (elem 4 or 8). */
PG_API int pg_prepare_batch(pg_ctx* ctx, const double* dosages, int64_t n_markers, int64_t n_samples, const double* q,
                     int64_t rank, int elem_bytes, void* out, double* af, int64_t* missing_count, double* variance,
                     int8_t* skip);
/* correlate (kernel.py:428-457): fp64 R = G Y / N with clamp count. */
PG_API int pg_correlate_f64(pg_ctx* ctx, const double* gt, int64_t m, int64_t n, const double* yt, int64_t p, double* r,
                     int64_t* clamp_count);

/* Measurement hook: average device time (CUDA events on the ctx stream) of the per-marker
 * statistics kernel K1 alone over `reps` launches on a device block, for the HBM roofline
 * of the decode stage (bench.py). Same inputs as pg_scan_device; results are discarded. */
PG_API int pg_time_marker_stats(pg_ctx* ctx, int kind, const void* d_data, int64_t n_markers, int64_t row_pitch,
                                int reps, float* ms);

/* Test hook: inflate `count` zlib streams (stream i = blob[off[i] + skip, off[i] + size[i]))
 * with the GPU decoder used by pg_stage_bgen; out [count, out_stride], out_len and status
 * (0 ok, 1 malformed / bad checksum, 2 output larger than out_stride) per stream. */
PG_API int pg_debug_inflate(const void* blob, int64_t blob_bytes, const int64_t* off, const int64_t* size,
                            int64_t count, int64_t skip, void* out, int64_t out_stride, int64_t* out_len, int* status);

/* ---- test hooks (exercise single kernels with device pointers) ---- */
/* Raw association GEMM: X[c, p] = kWH * sum_k qh[p,k] v[c,k] + sum_k q1[p,k] v127[c,k] + q0[p,k] v[c,k]
 * (int8 operands, exact int32 accumulation, returned as f64 [c_pad, p_pad]).
 * p_pad % 128 == 0, c_pad % 256 == 0, k_pad % 64 == 0. */
PG_API int pg_debug_assoc_gemm(const void* d_qh, const void* d_q1, const void* d_q0, int64_t p_pad, const void* d_v,
                               const void* d_v127, int64_t c_pad, int64_t k_pad, double* d_x, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PANELGWAS_B200_H */
