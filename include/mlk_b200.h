/*
 * mlk_b200.h -- C ABI of the sm_100a per-histogram compress/decompress path.
 *
 * Drop-in boundary for the reference package `mlk` (arXiv 2212.10733,
 * /root/reference/pkg/src/mlk).  Two levels are exported:
 *
 *  (1) the reference's own operator API (mlk/kernels.py:20-32, implemented by
 *      _ckernels.pyx / _pykernels.py), batched: Newton solves, zigzag,
 *      LEB128 varints, fixed-width index packing, plus the DEFLATE stage the
 *      residual codec wraps around them (residual.py:60-98);
 *  (2) the stage API that replaces the per-shard numpy code in
 *      pipeline._compress_shard (pipeline.py:196-320) and
 *      pipeline._decode_shard (pipeline.py:397-427).
 *
 * Conventions: every pointer is DEVICE memory unless its name ends in `_h`;
 * every entry point is asynchronous on `stream` and returns MLK_OK or a
 * negative MLK_ERR_* code (the Python wrapper maps them to the reference's
 * exception classes, errors.py:4-34).  Newton outcomes are per-image status
 * codes, never errors (as in the reference).  No entry point keeps per-shard
 * state in globals, so shards may run concurrently on several streams.
 */
#ifndef MLK_B200_H
#define MLK_B200_H

#include <stdint.h>
#include <cuda_runtime.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define MLK_OK 0
#define MLK_ERR_DIM (-1)      /* DimensionError */
#define MLK_ERR_CONFIG (-2)   /* ConfigError */
#define MLK_ERR_FORMAT (-3)   /* FormatError */
#define MLK_ERR_SIZE (-4)     /* SizeMismatchError */
#define MLK_ERR_VALUE (-5)    /* ValueError (kernels.py codecs) */
#define MLK_ERR_CUDA (-6)     /* launch / runtime failure */

/* Newton status codes, _pykernels.py:11-13 */
#define MLK_NEWTON_CONVERGED 0
#define MLK_NEWTON_MAX_ITER 1
#define MLK_NEWTON_DEGENERATE 2

/* per-image flag bits written by the stage kernels */
#define MLK_F_SELECTED 1u     /* residual coded (pipeline.py:235) */
#define MLK_F_NONFINITE 2u    /* AE error not finite -> exception (pipeline.py:233) */
#define MLK_F_RECHECK 4u      /* AE-error decision needs the exact pass */
#define MLK_F_EXC_NEWTON 8u   /* Newton not converged (pipeline.py:268) */
#define MLK_F_EXC_OVERFLOW 16u/* lambda f32 overflow (pipeline.py:271) */
#define MLK_F_EXC_GATE 32u    /* final PD gate (pipeline.py:285) */
#define MLK_F_EXCEPTION (MLK_F_NONFINITE | MLK_F_EXC_NEWTON | MLK_F_EXC_OVERFLOW | MLK_F_EXC_GATE)

/* One shard of the node-range decomposition (decomp.py:73-105), or the
 * contiguous index range [j0, j0 + n_img) of it that one rank processes.
 * Image j of the table entry is shard member g = j0 + j, the D doubles at
 * f0 + base + (g / block) * plane_stride + (g % block) * D, i.e. plane-major
 * members exactly as partition() lists them (decomp.py:102). */
typedef struct {
    int64_t base;
    int64_t plane_stride;
    int32_t block;
    int32_t n_img;
    int32_t img_off;    /* first index of this shard in the per-image arrays */
    int32_t small_blas; /* n_img*L*D <= 1e6: OpenBLAS small-matrix kernel order */
    double mean, std;   /* AEModel normaliser (autoencoder.py:26-57) */
    double eb;          /* error bound chosen by the search (residual.py:129) */
    int32_t lossless;   /* search fell back to lossless payloads */
    int32_t w_off;      /* float offset of this shard's W (L x D) */
    int32_t j0;         /* member index of image 0 (0 unless the shard is split) */
    int32_t pad;
} MlkShard;

/* Grid tables, all DEVICE arrays of D = rows*cols doubles computed on the
 * host with the reference's numpy expressions (lagrange.py:68-80, 163-173,
 * 199-204; qoi.py:65-72). */
typedef struct {
    int32_t rows, cols, D, pad;
    double mass;
    const double* vol;      /* grid.vol (row-major) */
    const double* vpar;     /* v_par of each cell's column */
    const double* vperp2;   /* v_perp**2 of each cell's row */
    const double* hmvol;    /* (0.5*mass) * vol */
    const double* ash;      /* 3*D: base[r] / max|base[r]| for r = 0, 1, 2 */
    const uint8_t* tree_cols; /* D: decode bracketing probed from the host BLAS */
    double s0, s1, s2;      /* shared row scales */
    int32_t sep, pad2;      /* vol takes vcls[2*row_edge + col_edge] everywhere */
    double vcls[4];
} MlkGrid;

typedef struct {
    double step;
    int32_t max_iter;
    int32_t retry;
    double tol;
    double floor;
    double retry_step;
    int32_t retry_max_iter;
    int32_t lam_f32;        /* lambda_precision == "f32" */
    double tau;
} MlkNewton;

/* ---------------- library info ---------------- */
const char* mlk_version(void);
int mlk_device_check(void); /* MLK_OK when a sm_100 device is current */

/* ======================= (1) reference operator API ======================= */

/* kernels.newton_solve (kernels.py:26; _ckernels.pyx:62-137), batched over
 * n systems.  f_plus (n, d), a (n, 4, d), b (n, 4) -> lam (n, 4),
 * status (n), iters (n). */
int mlk_newton_solve_batch(const double* f_plus, const double* a, const double* b,
                           int64_t n, int32_t d, double step, int32_t max_iter, double tol,
                           double* lam, int32_t* status, int32_t* iters, cudaStream_t stream);

/* kernels.zigzag_map / zigzag_unmap (kernels.py:27-28; _ckernels.pyx:143-150) */
int mlk_zigzag_map(const int64_t* q, uint64_t* z, int64_t n, cudaStream_t stream);
int mlk_zigzag_unmap(const uint64_t* z, int64_t* q, int64_t n, cudaStream_t stream);

/* kernels.varint_encode (kernels.py:29; _ckernels.pyx:153-171) over n_streams
 * independent streams: stream s is values[off[s] .. off[s+1]).  Bytes go to
 * out + out_off[s] (capacity 10 values each); out_len[s] receives the length. */
int mlk_varint_encode_batch(const uint64_t* values, const int64_t* off, int32_t n_streams,
                            uint8_t* out, const int64_t* out_off, int64_t* out_len,
                            cudaStream_t stream);

/* kernels.varint_decode (kernels.py:30; _ckernels.pyx:174-211): stream s has
 * in_len[s] bytes at in + in_off[s] and decodes count[s] values into
 * values + val_off[s]; consumed[s] = bytes used, or -1 (truncated) /
 * -2 (exceeds 64 bits). */
int mlk_varint_decode_batch(const uint8_t* in, const int64_t* in_off, const int64_t* in_len,
                            int32_t n_streams, const int64_t* count, uint64_t* values,
                            const int64_t* val_off, int64_t* consumed, cudaStream_t stream);

/* kernels.pack_indices / unpack_indices (kernels.py:31-32; _ckernels.pyx:217-275).
 * pack returns MLK_ERR_VALUE via *bad (device int) when an index >= 2**bits. */
int mlk_pack_indices(const uint16_t* idx, int64_t n, int32_t bits, uint8_t* out,
                     int32_t* bad, cudaStream_t stream);
int mlk_unpack_indices(const uint8_t* buf, int64_t count, int32_t bits, uint16_t* out,
                       cudaStream_t stream);

/* zlib.compress(data, 6) (residual.py:70,77) for n streams: input s is
 * in_len[s] bytes at in + in_off[s]; output (2-byte zlib header, DEFLATE
 * stream reproducing zlib 1.3 deflate_slow level 6, Adler-32) goes to
 * out + out_off[s] with capacity out_cap each; out_len[s] = bytes written,
 * -1 if out_cap was too small, -2 if the input exceeds 32000 bytes.
 * `work` = n_workers * MLK_DEFLATE_WORK bytes, zero-filled before first use
 * (the kernel leaves it reusable).  Only streams longer than nmin bytes are
 * processed (the others are left to mlk_zlib_compress6_warp). */
#define MLK_DEFLATE_WORK (1u << 18)
int mlk_zlib_compress6(const uint8_t* in, const int64_t* in_off, const int64_t* in_len,
                       int32_t n, uint8_t* out, const int64_t* out_off, int64_t out_cap,
                       int64_t* out_len, uint8_t* work, int32_t n_workers, int64_t nmin,
                       cudaStream_t stream);

/* Same bytes as mlk_zlib_compress6, one warp per stream with the working set
 * in shared memory, for the streams with nmin < in_len <= nmax (<= 16000);
 * run it over the size tiers, then mlk_zlib_compress6 for larger streams.
 * Two launches on `stream`: the LZ77 parse, then the Huffman trees and the
 * bit stream (one fused launch when prof is given).  sym_scratch: n *
 * sym_cap bytes (sym_cap >= 3 * nmax + 19, a multiple of 16) for the LZ77
 * symbol buffers, whose last 16 bytes carry the parse's summary to the
 * second launch; prof (may be NULL): 16 u64 cycle/counter accumulators. */
int mlk_zlib_compress6_warp(const uint8_t* in, const int64_t* in_off, const int64_t* in_len,
                            int32_t n, int32_t nmin, int32_t nmax, uint8_t* out,
                            const int64_t* out_off, int64_t out_cap, int64_t* out_len,
                            int32_t n_blocks, uint8_t* sym_scratch, int64_t sym_cap,
                            uint64_t* prof, cudaStream_t stream);

/* dst[dst_off[i] .. + len[i]) = src[src_off[i] .. + len[i]) for n segments */
int mlk_gather_segments(const uint8_t* src, const int64_t* src_off, const int64_t* len,
                        int32_t n, uint8_t* dst, const int64_t* dst_off, cudaStream_t stream);

/* mlk_zlib_compress6_warp with dynamic balance: the warps claim streams one
 * at a time from *counter (device int, zero before the launch; one counter
 * per concurrently running tier). */
int mlk_zlib_compress6_warp_dyn(const uint8_t* in, const int64_t* in_off, const int64_t* in_len,
                                int32_t n, int32_t nmin, int32_t nmax, uint8_t* out,
                                const int64_t* out_off, int64_t out_cap, int64_t* out_len,
                                int32_t n_blocks, uint8_t* sym_scratch, int64_t sym_cap,
                                uint64_t* prof, int32_t* counter, cudaStream_t stream);

/* zlib.decompress (residual.py:86) for n streams; out_len[s] = bytes produced,
 * or -1 (corrupt) / -2 (output capacity exceeded). */
int mlk_zlib_decompress(const uint8_t* in, const int64_t* in_off, const int64_t* in_len,
                        int32_t n, uint8_t* out, const int64_t* out_off, int64_t out_cap,
                        int64_t* out_len, cudaStream_t stream);

/* fdata.gen_synthetic (fdata.py:322-347) on device, bit-identical: planes
 * plane0 .. plane0 + n_planes - 1 of the corpus, each nd = n_nodes * D
 * doubles, out[p * nd + e] = the numpy value.  base (nd doubles, device) is
 * the per-node image before the per-plane rho term; pcg_h (HOST, 8 x u64):
 * the Generator's PCG64 state and increment after seeding (hi, lo each),
 * then the affine map of 32 steps (A^32, c_32).  Only noise == 0 corpora. */
int mlk_synth_planes(const double* base, int64_t nd, int64_t plane0, int32_t n_planes,
                     const uint64_t* pcg_h, double rho, double value_min, double* out,
                     cudaStream_t stream);

/* ---- per-call operators of the reference's public stage API
 * (mlk/__init__.py:9-38), used by quantizer / residual / lagrange /
 * autoencoder here; every one is elementwise in the reference's order. */

/* quantizer._nearest (quantizer.py:91-93) over lat (n, L) with the
 * float64-upcast centroids cents (L, K) f32: first minimum, NaN first. */
int mlk_pq_nearest(const double* lat, int64_t n, int32_t L, const float* cents, int32_t K,
                   uint16_t* idx, cudaStream_t stream);
/* quantizer.pq_decode's lookup (quantizer.py:132-138): out (n, L) f64;
 * *bad = 1 when an index is >= K (SizeMismatchError). */
int mlk_pq_lookup(const uint16_t* idx, int64_t n, int32_t L, const float* cents, int32_t K,
                  double* out, int32_t* bad, cudaStream_t stream);
/* BuiltinCodec.compress's codes (residual.py:63-69): z = zigzag(rint(r / 2eb));
 * *err |= 1 for a non-finite residual, 2 for |q| >= 2**62. */
int mlk_quantize_codes(const double* r, int64_t n, double eb, uint64_t* z, int32_t* err,
                       cudaStream_t stream);
/* BuiltinCodec.decompress's values (residual.py:92-99): mode 0 = q * 2eb,
 * mode 1 = raw float64 bits. */
int mlk_dequantize(const uint64_t* z, int64_t n, double eb, int32_t mode, double* out,
                   cudaStream_t stream);
/* quantize_roundtrip (residual.py:100-102); with recon != NULL the corrected
 * images recon + roundtrip(a - recon) of find_error_bound (residual.py:149-155). */
int mlk_quantize_roundtrip(const double* a, const double* recon, int64_t n, double eb,
                           double* out, cudaStream_t stream);
/* lagrange.apply_lambda (lagrange.py:136-149) for n images f (n, D) with
 * lam (n, 4) and constraint rows a (4, D) at a + i * a_stride. */
int mlk_apply_lambda_rows(const double* f, int64_t n, int32_t D, const double* lam,
                          const double* a, int64_t a_stride, double floor_, double* out,
                          cudaStream_t stream);
/* autoencoder.decode_batch on raw f64 latents (autoencoder.py:106-110),
 * OpenBLAS bracketing per column from tree_cols (may be NULL). */
int mlk_ae_decode(const double* lat, int64_t n, int32_t L, const float* W, int32_t D,
                  double mean, double sd, const uint8_t* tree_cols, double* out,
                  cudaStream_t stream);

/* ======================= (2) stage API (one launch covers all shards) ====== */

/* Pass 1 over f0 (autoencoder.encode_batch autoencoder.py:99-103 in OpenBLAS
 * order; qoi.compute_qoi_batch qoi.py:60-76; per-image max/min/sum/sum-sq).
 * lat (total, L); stats (total, 4) = [max, min, sum, sumsq]; qoi (total, 4). */
int mlk_stage1(const double* f0, const MlkShard* shards, int32_t n_shards, int32_t total,
               const MlkGrid* grid_h, const float* W, int32_t L, double* lat, double* stats,
               double* qoi, cudaStream_t stream);

/* quantizer.pq_train (quantizer.py:99-108; kmeans_1d 53-91) for every
 * (shard, dim): first_idx / draws are the PCG64 draws kmeans_1d consumes
 * (one integers() then K-1 random(), computed by the host from the seed).
 * shards (device) and shards_h (the same table on the host, for validation).  cents (n_shards, L, K) float32, sorted;
 * scratch >= 4 * L * total doubles; info (n_shards, L, 4); cents64 (may be
 * NULL) receives the same centroids before the float32 cast (kmeans_1d's
 * float64 result). */
int mlk_kmeans(const double* lat, const MlkShard* shards, const MlkShard* shards_h,
               int32_t n_shards, int32_t L, int32_t K, const int64_t* first_idx,
               const double* draws, double* scratch, float* cents, double* cents64,
               int32_t* info, cudaStream_t stream);

/* diagnostics: cycles of CTA 0 of the last mlk_kmeans launch in its phases
 * (load + distinct test, k-means++ seeding, Lloyd), its Lloyd sweeps and six
 * sub-phase totals; out_h is a HOST array of 12. */
int mlk_kmeans_prof(int64_t* out_h, cudaStream_t stream);

/* pq_encode + AE-error decision (quantizer.py:111-120; pipeline.py:228-235):
 * codes (total, L) u8; flags gets SELECTED or RECHECK.  gram holds per shard
 * [W W^T (L*L), row sums (L), ||W_k||_2 (L), max|W_k| (L)] computed by the
 * host; recon_bound (total) bounds max|recon| for the probe's slack. */
int mlk_select(const double* lat, const double* stats, const MlkShard* shards,
               int32_t n_shards, int32_t total, const MlkGrid* grid_h, const float* cents,
               int32_t L, int32_t K, const double* gram, double tau, uint8_t* codes,
               uint8_t* flags, double* err_approx, double* recon_bound, cudaStream_t stream);

/* exact per-image NRMSE (qoi.py:107-119, numpy pairwise order) for images
 * flagged RECHECK; rewrites their flags to SELECTED / NONFINITE / 0. */
int mlk_recheck(const double* f0, const double* stats, const MlkShard* shards,
                int32_t n_shards, int32_t total, const MlkGrid* grid_h, const float* W,
                int32_t L, const float* cents, int32_t K, const uint8_t* codes, double tau,
                uint8_t* flags, double* err_exact, cudaStream_t stream);

/* one CTA per shard: sel[img_off + r] = r-th selected image (ascending, as
 * np.flatnonzero, pipeline.py:235), sel_rank[img] = r or -1, sel_by_range =
 * the same set ordered by range bucket, sel_count[s], eb_hi[s] = tau * max
 * range of the selection (residual.py:143-144). */
int mlk_compact(const uint8_t* flags, const double* stats, const MlkShard* shards,
                int32_t n_shards, double tau, int32_t* sel, int32_t* sel_rank,
                int32_t* sel_by_range, int32_t* sel_count, double* eb_hi, cudaStream_t stream);

/* residual.find_error_bound's predicate (residual.py:149-155) for `span`
 * (1 or 2) bisection levels of a lookahead tree per launch: cand
 * (n_shards, n_nodes) holds each shard's candidate bounds in heap order
 * (node 1 = the current query, 2i = next query if node i is accepted, 2i+1
 * if rejected; <= 0 / NaN = no query).  For every shard the launch walks
 * levels 0 .. level-1 through the flags of earlier launches, then evaluates
 * the node reached and, for span 2, both its children, in one pass over the
 * images; fail[s*n_nodes + i] becomes non-zero when a selected image of
 * shard s misses tau at node i.  Launches queue on one stream, so walking
 * the tree needs no host round trip.  The launch visits positions
 * act_start[s] .. act_start[s] + (act_off[s+1] - act_off[s]) of shard s's
 * range-ordered selection (smallest ranges fail first).  recon (may be
 * NULL): the reconstructions mlk_probe_bins stored, read instead of decoding
 * the latent codes again (sel_count and sel_rank then required). */
int mlk_probe(const double* f0, const double* stats, const MlkShard* shards,
              int32_t n_shards, const MlkGrid* grid_h, const float* W, int32_t L,
              const float* cents, int32_t K, const uint8_t* codes,
              const int32_t* sel_by_range, const int32_t* act_off, const int32_t* act_start,
              int32_t n_work,
              const double* recon_bound, double tau, const double* cand, int32_t n_nodes,
              int32_t level, int32_t span, int32_t* fail, const double* bins,
              const double* eb_hi, const int32_t* sel_count, const int32_t* sel_rank,
              const double* recon, cudaStream_t stream);

/* Residual-magnitude profile of every selected image (34 counts + 34 sums of
 * r^2 over log2 bins anchored at eb_hi[s]) at bins[(img_off + pos) * 68],
 * pos = the image's place in the range-ordered selection; mlk_probe uses it
 * (bins may be NULL) to certify passes without re-reading the image.
 * recon (may be NULL; n_sel rows of (D + 1) & ~1 doubles): each selected
 * image's decoder reconstruction at row sum(sel_count[0..s-1]) +
 * sel_rank[img] (= the projection's residual slot), for mlk_probe and
 * mlk_project. */
int mlk_probe_bins(const double* f0, const MlkShard* shards, int32_t n_shards,
                   const MlkGrid* grid_h, const float* W, int32_t L, const float* cents,
                   int32_t K, const uint8_t* codes, const int32_t* sel_by_range,
                   const int32_t* sel_count, int32_t n_sel, const double* eb_hi, double* bins,
                   const int32_t* sel_rank, double* recon, cudaStream_t stream);

/* Stage 4 encode + stage 5 (pipeline.py:239-292): residual q / zigzag /
 * varint for selected images into varint + (slot_base[s] + sel_rank) *
 * varint_cap; lagrange.project_batch + cast_lambda + apply_lambda_batch +
 * the final gate.  Per image: lam (cast; 0 for exceptions), qst (stored
 * QoIs; 0 for exceptions), status, iters, flags |= EXC_*, ferr (final
 * NRMSE), fqoi (moments of the final image), fsse (sum of squared final
 * errors).  *err_flag = MLK_ERR_CONFIG when |q| >= 2**62 (residual.py:67).
 * img_list (device, n_list entries) restricts the launch to those images
 * (NULL: all `total`), so the images without residuals can be projected
 * while the error-bound search of the others is still running.  recon (may
 * be NULL; needs slot_base): mlk_probe_bins' stored reconstructions, read
 * (one bulk copy per image) for the selected images instead of decoding. */
int mlk_project(const double* f0, const double* stats, const double* qoi,
                const MlkShard* shards, int32_t n_shards, int32_t total, const MlkGrid* grid_h,
                const float* W, int32_t L, const float* cents, int32_t K, const uint8_t* codes,
                const int32_t* sel_rank, const int32_t* slot_base, const MlkNewton* opts_h,
                uint8_t* flags, double* lam, double* qst, int32_t* status, int32_t* iters,
                double* ferr, double* fqoi, double* fsse, uint8_t* varint, int64_t varint_cap,
                int64_t* varint_len, int32_t* err_flag, const int32_t* img_list,
                int32_t n_list, const double* recon, cudaStream_t stream);

/* Decode path (pipeline.py:397-427) for all images of all shards: recon from
 * codes; + residual (res_slot[img] >= 0: D zigzag codes at res_codes +
 * slot * D, dequantised with res_eb[slot] unless res_mode[slot] == 1
 * (lossless f64 bits), BuiltinCodec.decompress residual.py:81-98); apply
 * lambda with the stored QoIs and floor_ (lamq (total, 8) = [lam, qoi]);
 * exceptions (exc_slot[img] >= 0) copied from exc_img.  Output images are
 * written at the shard addresses of `out`; *neg (device, may be NULL) is
 * OR-ed with 1 when a written value is < 0 (FDataset's check, fdata.py:70-
 * 103, without a second pass over the output). */
int mlk_decode(const MlkShard* shards, int32_t n_shards, int32_t total, const MlkGrid* grid_h,
               const float* W, int32_t L, const float* cents, int32_t K, const uint8_t* codes,
               const int32_t* res_slot, const uint64_t* res_codes, const double* res_eb,
               const uint8_t* res_mode, const double* lamq, const int32_t* exc_slot,
               const double* exc_img, double floor_, double* out, int32_t* neg,
               cudaStream_t stream);

/* image_nrmse_batch(a, b) (qoi.py:107-119, exact) + per-image squared-error
 * sums, moments of a and b (compute_qoi_batch; qa/qb may be NULL) and
 * ext = (max, min) of every image of a.  a, b: (total, D) contiguous. */
int mlk_compare(const double* a, const double* b, int32_t total, const MlkGrid* grid_h,
                double* err, double* sse, double* qa, double* qb, double* ext,
                cudaStream_t stream);

/* The report's reductions (pipeline._build_report, pipeline.py:367-391;
 * qoi.py:122-133) over the per-image arrays mlk_project leaves in HBM.  One
 * segment per CompressOut (DEVICE arrays of n images); order (device int64,
 * may be NULL) is each image's dataset index.  out (MLK_REPORT_NVALS doubles,
 * device) = [data max, data min, sum fsse, defined-QoI count, converged,
 * ae_ok, selected, exceptions, qoi d2 (4), qoi max (4), qoi min (4)] with
 * identities (-inf / +inf / 0) for empty input; per_image (may be NULL)
 * receives ferr in dataset order, 0 for exceptions.  scratch >= 20 * 296 *
 * n_segs doubles. */
#define MLK_REPORT_NVALS 20
typedef struct {
    const uint8_t* flags;
    const int32_t* status;
    const double* stats;   /* (n, 4) */
    const double* qoi;     /* (n, 4) */
    const double* fqoi;    /* (n, 4) */
    const double* fsse;    /* (n) */
    const double* ferr;    /* (n) */
    const int64_t* order;  /* (n) or NULL */
    int64_t n;
} MlkReportSeg;

int mlk_report(const MlkReportSeg* segs_h, int32_t n_segs, double* scratch,
               int64_t scratch_doubles, double* out, double* per_image, cudaStream_t stream);

/* HOST function: walk one shard's residual section (pipeline.py:140-156 and
 * the payload header of residual.py:81-98) over host memory `sec` (len
 * bytes).  For entry k: idx (image index), body_off = base + offset of its
 * zlib stream within sec, body_len, eb and mode from the payload header.
 * Returns MLK_ERR_FORMAT with *why = 1 truncated, 2 trailing bytes,
 * 3 payload shorter than its header, 4 payload dims != (rows, cols),
 * 5 unknown mode, 6 image index >= n_images, 7 more than cap entries. */
int mlk_parse_residual_section(const uint8_t* sec, int64_t len, int32_t n_images, int32_t rows,
                               int32_t cols, int64_t base, int32_t cap, int32_t* idx,
                               int64_t* body_off, int64_t* body_len, double* eb, uint8_t* mode,
                               int32_t* count_out, int32_t* why);

/* HOST: 1 if p lies in page-locked host memory (cudaHostAlloc/Register). */
int mlk_is_pinned(const void* p);

/* HOST: the next `depth` decisions of n error-bound searches as heap-ordered
 * nodes (residual.py:129-173; engine._Search): kind[i * 2^depth + v] in {0
 * ended, 1 eb_hi probe, 2 bisection, 3 floor probe} and the bisection
 * midpoint 0.5 * (lo + hi) in log space (the caller exponentiates). */
int mlk_search_tree(const int8_t* kind0, const int32_t* step0, const uint8_t* best0,
                    const double* lo0, const double* hi0, const double* lo_end,
                    const double* hi_end, int32_t n, int32_t depth, int32_t steps, int8_t* kind,
                    double* mid);

/* HOST: page-lock / release an existing host range (cudaHostRegister), e.g.
 * the shared mapping of an output file that device results are copied to. */
int mlk_host_register(void* p, int64_t bytes);
int mlk_host_unregister(void* p);

/* HOST memory only: exception entries <I idx[k]> + 8 D bytes of the host
 * histogram at src + src_off[k] (elements), back to back at dst
 * (pipeline.py:116-184, 281-292).  compress() fills the archive's exception
 * sections from its own input with it instead of a device -> host copy. */
int mlk_host_exception_entries(uint8_t* dst, const double* src, const int64_t* src_off,
                               const uint32_t* idx, int64_t n, int32_t D);

/* ---- shard-blob assembly on device (container.py:90-95, pipeline.py:116-184) */

/* list[img_off + r] = r-th image of shard s (ascending) with flags & mask;
 * count[s] = number of such images (the sorted exception list,
 * pipeline.py:287). */
int mlk_list_flags(const uint8_t* flags, const MlkShard* shards, int32_t n_shards, uint32_t mask,
                   int32_t* list, int32_t* count, cudaStream_t stream);

/* the images of [0, total) with (flags & mask) != 0 into `set` and the rest
 * into `clear`, both ascending; *n_set = the size of `set` (device).  flags
 * must be 4-byte aligned. */
int mlk_split_flags(const uint8_t* flags, int32_t total, uint32_t mask, int32_t* set,
                    int32_t* clear, int32_t* n_set, cudaStream_t stream);

/* residual section entries (pipeline.py:132-137): for payload e of shard
 * entry_shard[e] at out + dst_off[e]: <II> (index, 13 + zlen) then the
 * <BHHd> payload header (residual.py:33) then the zlib body zbuf[zoff[e]..]. */
int mlk_pack_residuals(const int32_t* sel, const MlkShard* shards, const int32_t* entry_shard,
                       const int64_t* dst_off, const int64_t* zoff, const int64_t* zlen,
                       const uint8_t* zbuf, const int32_t* slot_base, int32_t rows,
                       int32_t cols, int32_t n, uint8_t* out, cudaStream_t stream);

/* lambda section (pipeline.py:116-119): per image [lam, qoi] as <f4 or <f8 at
 * out + sec_off[shard] + record * j. */
int mlk_pack_lambdas(const double* lam, const double* qst, const MlkShard* shards,
                     int32_t n_shards, int32_t total, const int64_t* sec_off, int32_t f32,
                     uint8_t* out, cudaStream_t stream);

/* exception entries (pipeline.py:158-163): <I index> + the original histogram
 * read from f0, after the 4-byte count at out + sec_off[shard]. */
int mlk_pack_exceptions(const double* f0, const MlkShard* shards, int32_t n_shards,
                        const int32_t* exc_list, const int32_t* exc_off, const int64_t* sec_off,
                        int32_t n_exc_total, int32_t D, uint8_t* out, cudaStream_t stream);

/* ---- AE training (off the per-histogram path) ----
 * Replaces autoencoder.train (autoencoder.py:137-177) with fit_normalizer
 * (77-84) and _loss_and_grad_normalized (127-134), as compress() calls it per
 * shard (pipeline.py:209-218).  One job per shard: the training images are
 * base + row_off[i] (i < n, D doubles each, device), order is the epochs x n
 * table of rng.permutation draws (device int32), w (L x D f64, device) holds
 * the Glorot / warm-start weights on entry and the trained weights on exit,
 * mv is reserved (unused; NULL), xn n x D f64 scratch (the normalised
 * training images, written once per call).  bias (2T doubles, device) = [1 - beta1^t,
 * 1 - beta2^t] for t = 1..T, computed with Python floats.  norm (2 per job)
 * receives (mean, std); diag (2 per job) receives (-1, 0) or (epoch, mse) of
 * the first non-finite mse (TrainingDivergedError).  MLK_ERR_CONFIG when the
 * per-CTA column slice of W, its gradient and both Adam moments does not fit
 * shared memory even at the largest cluster size. */
#define MLK_STD_FLOOR 1e-30   /* autoencoder.STD_FLOOR */
typedef struct {
    const double* base;
    const int64_t* row_off;
    const int32_t* order;
    double* w;
    double* mv;
    double* xn;
    int32_t n;
    int32_t epochs;
} MlkTrainJob;

/* numpy's pairwise summation of a job's n*D training entries laid out as a
 * tree (autoencoder.pairwise_tree): leaves [leaf_start, +leaf_len) of <= 128
 * entries, then internal nodes level by level, deepest first (node
 * n_leaves + k = node child[2k] + node child[2k+1] for k in level_off[lv] ..
 * level_off[lv+1]); nodes is scratch for n_leaves + level_off[n_levels]
 * doubles.  fit_normalizer's mean and std are computed through it. */
typedef struct {
    const int64_t* leaf_start;
    const int32_t* leaf_len;
    const int32_t* child;
    const int32_t* level_off;
    double* nodes;
    int64_t n_total;
    int32_t n_leaves;
    int32_t n_levels;
} MlkPwTree;

int mlk_ae_train(const MlkTrainJob* jobs, const MlkTrainJob* jobs_h, const MlkPwTree* trees,
                 const MlkPwTree* trees_h, int32_t n_jobs, int32_t L,
                 int32_t D, int32_t batch, double lr, double beta1, double one_minus_beta1,
                 double beta2, double one_minus_beta2, double eps, const double* bias,
                 int32_t T, double* norm, double* diag, cudaStream_t stream);

/* diagnostics: {cluster size, rows per chunk, columns per CTA, shared-memory
 * bytes} of the last mlk_ae_train launch; out_h is a HOST array of 4. */
int mlk_ae_train_config(int32_t* out_h, cudaStream_t stream);

#ifdef __cplusplus
}
#endif
#endif
