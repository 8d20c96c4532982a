/*
 * undertext_b200.h -- C ABI of the B200-native CVA / PCA hot path.
 *
 * Drop-in boundary for the reference package `undertext`
 * (/root/reference/pkg/src/undertext).  The reference is pure Python + numpy;
 * its "plugin interface" for this path is the set of Python functions listed
 * next to each entry point below.  A maintainer binds these symbols with
 * ctypes; the in-tree Python mirror
 * (paper_1612_06457_b200/) does exactly that.
 *
 * Conventions:
 *   - every function returns a status: UT_OK, UT_EDATA (-> DataError),
 *     UT_ENUMERIC (-> NumericError), UT_ECUDA (-> RuntimeError); no C++
 *     exception crosses the ABI; ut_last_error() gives the message (per thread);
 *   - all array pointers are DEVICE pointers owned by the caller unless the
 *     parameter is documented as host; the library never frees them;
 *   - every call takes the caller's stream (a cudaStream_t passed as void*),
 *     enqueues asynchronously and never synchronizes, so calls are capturable
 *     in CUDA graphs; the device is the one current on the calling thread;
 *   - data-dependent failures (bad point, non-PD matrix) are reported through
 *     small device-side status words the caller reads when it needs them.
 *   - matrices are row-major: m[i*ld + j].
 */
#ifndef UNDERTEXT_B200_H
#define UNDERTEXT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define UT_OK 0
#define UT_EDATA 1
#define UT_ENUMERIC 2
#define UT_ECUDA 3

/* sample types of a spectral cube (SpectralStack.planes dtype, stack.py:43-49) */
enum { UT_U8 = 0, UT_U16 = 1, UT_F16 = 2, UT_F32 = 3, UT_F64 = 4 };

/* device-side info codes written by the solvers */
enum {
  UT_INFO_OK = 0,
  UT_INFO_ASYM_A = 1,      /* eigen.py:90  _check_symmetric(A) */
  UT_INFO_ASYM_M = 2,      /* eigen.py:91  _check_symmetric(M) */
  UT_INFO_NOT_PD = 3,      /* eigen.py:94-104 cholesky failed (aux = eig(M')) */
  UT_INFO_NO_CONVERGE = 4  /* Jacobi sweep cap reached (never seen in tests) */
};

/* A band-sequential cube (or a row shard of one), SpectralStack.planes (B,H,W). */
typedef struct {
  const void* data;      /* device pointer to element (band 0, local row 0, col 0) */
  int32_t dtype;         /* UT_U8 .. UT_F64 */
  int32_t bands;         /* B, 1..32 */
  int64_t rows;          /* local rows */
  int64_t cols;          /* W */
  int64_t band_stride;   /* elements between bands */
  int64_t row_stride;    /* elements between rows */
  int64_t row0;          /* global row index of local row 0 (row sharding) */
} ut_cube;

/* Outputs of ut_cva_solve (all device pointers, B = bands, C = classes). */
typedef struct {
  double* within;        /* B*B  ScatterPair.within   (projection.py:199) */
  double* between;       /* B*B  ScatterPair.between  (projection.py:200) */
  double* class_means;   /* C*B  ScatterPair.class_means */
  double* counts;        /* C    ScatterPair.counts (exact integers) */
  double* grand_mean;    /* B    ScatterPair.grand_mean = ProjectionModel.mean */
  double* evals;         /* B    descending (eigen.py:111) */
  double* evecs;         /* B*B  column j = eigenvector j, M'-orthonormal, sign-normalized */
  double* aux;           /* B    eig(M') when info == UT_INFO_NOT_PD */
  int32_t* info;         /* 1 */
} ut_cva_out;

/* Outputs of ut_pca_solve (projection.py:335-338 + _pca_from_covariance :263-270). */
typedef struct {
  double* mean;          /* B */
  double* std;           /* B  (0 -> 1 as projection.py:336) */
  double* corr;          /* B*B correlation matrix that is diagonalized */
  double* evals;         /* B descending */
  double* evecs;         /* B*B orthonormal, sign-normalized */
  int32_t* info;         /* 1 */
} ut_pca_out;

/* ---------------------------------------------------------------- misc */
int ut_version(void);
/* SHA-256 prefix (32 hex digits) of the sources this library was built from
 * (paper_1612_06457_b200/build.py: source_hash); the loader refuses a mismatch. */
const char* ut_build_hash(void);
const char* ut_last_error(void);
/* number of doubles in one class-moment record: 1 + B + B*B */
int64_t ut_moment_len(int32_t bands);

/* ------------------------------------------------- K1: training gather
 * Replaces annotations.assemble_matrix's point loop (annotations.py:195-215):
 * values[b*ld + j] = (double) cube[b, y_j - row0, x_j] for the n points
 * xy = [x0,y0,x1,y1,...] (global coordinates).  first_bad receives the lowest
 * index of an out-of-bounds point, or -1 (DataError in the reference,
 * annotations.py:208-212). */
int ut_gather(const ut_cube* cube, const int32_t* xy, int64_t n,
              double* values, int64_t ld, int64_t* first_bad, void* stream);

/* ------------------------------------------------- K1: class moments
 * Per-class count, mean and centred scatter M2 of a B x n design matrix
 * (two-pass, like compute_scatter's per-class loop, projection.py:187-198).
 * cls[j] in [0, classes) is the class *index* of point j (index into the sorted
 * unique labels).  moments: classes records of ut_moment_len(B) doubles:
 * [count, mean(B), M2(B*B)].  pivots: optional device array of C point
 * indices (the first point of each class; NULL = found on the device) used
 * as per-class shifts.  ws: ut_class_moments_ws(n, B, C) bytes. */
size_t ut_class_moments_ws(int64_t n, int32_t bands, int32_t classes);
int ut_class_moments(const double* values, int64_t ld, const int32_t* cls,
                     int64_t n, int32_t bands, int32_t classes, const int32_t* pivots,
                     double* moments, void* ws, size_t ws_bytes, void* stream);

/* standardize(dm) (projection.py:152-169): out[b, j] = (x[b, j] - mean_b) / std_b
 * with the N - 1 divisor and std = 1 for a constant row; n >= 2 (DataError
 * otherwise).  values / out: B x n fp64, row strides ld / ld_out (elements);
 * may alias when ld == ld_out.  Feeds fit_lda (projection.py:240-260). */
int ut_standardize(const double* values, int64_t ld, int32_t bands, int64_t n, double* out,
                   int64_t ld_out, double* mean, double* std, void* stream);

/* Fused gather + class moments straight from the cube (the pipeline form of
 * assemble_matrix + compute_scatter): xy as for ut_gather; points outside the
 * (shard of the) cube are skipped and reported in first_bad (-1 if none). */
int ut_cube_class_moments(const ut_cube* cube, const int32_t* xy, const int32_t* cls,
                          int64_t n, int32_t classes, const int32_t* pivots,
                          double* moments, int64_t* first_bad, void* ws, size_t ws_bytes,
                          void* stream);

/* ------------------------------------------------- K3: CVA solve
 * Combines `groups` partial moment sets (rank-major [groups][classes][len],
 * e.g. all-gathered from row shards) with the parallel-axis rule, builds the
 * symmetrized within / between scatter (projection.py:190-200), then solves
 * between v = lambda (within + ridge*tr/B*I) v in one CTA (eigen.py:63-113).
 * want = number of leading eigenvectors the caller needs (<= 0: all).  When
 * want <= (classes with points) - 1 the rank of S_b is exploited: only a C x C
 * eigenproblem is solved, evals beyond C are exact zeros and evecs columns
 * >= want are zero; otherwise all B pairs are computed. */
int ut_cva_solve(const double* moments, int32_t groups, int32_t bands,
                 int32_t classes, double ridge, int32_t want, const ut_cva_out* out,
                 void* stream);

/* ------------------------------------------------- K3: eigensolver
 * solve_gen_eig_sym(A, M, ridge) (eigen.py:75-113).  M == NULL selects the
 * plain symmetric problem with no ridge and orthonormal vectors (the
 * np.linalg.eigh + sign_normalize of _pca_from_covariance, projection.py:263). */
int ut_gen_eig_sym(const double* A, const double* M, int32_t bands, double ridge,
                   double* evals, double* evecs, double* aux, int32_t* info,
                   void* stream);

/* ------------------------------------------------- K2: region moments
 * One pass over a region (x0, y0, w, h) in *local* row coordinates:
 * moments = [n, mean(B), M2(B*B)] (projection.py:325-334, shifted one-pass
 * form; shift = mean of a fixed strided sample).  ws: ut_region_moments_ws. */
size_t ut_region_moments_ws(int32_t bands);
int ut_region_moments(const ut_cube* cube, int64_t x0, int64_t y0, int64_t w,
                      int64_t h, double* moments, void* ws, size_t ws_bytes,
                      void* stream);
/* Diagnostics for tests: the path the calling thread's last ut_region_moments
 * took (UT_REGION_PATH_*), and the byte offset in the workspace of the int32
 * flag the integer path raises when a sample left its fixed-point range (the
 * fp64 path then redid the region). */
enum { UT_REGION_PATH_DFMA = 0, UT_REGION_PATH_DMMA = 1, UT_REGION_PATH_IMMA = 2 };
int32_t ut_region_last_path(void);
int64_t ut_region_flag_offset(void);

/* ------------------------------------------------- K3: PCA solve
 * Combines `groups` region-moment records, then std / correlation /
 * eigh / top-k / sign-normalize (projection.py:335-338, :263-270). */
int ut_pca_solve(const double* moments, int32_t groups, int32_t bands,
                 const ut_pca_out* out, void* stream);

/* ------------------------------------------------- K4: projector
 * project_stack / _project_rows (projection.py:371-439) fused with the global
 * min/max of rescale_full (rendering.py:126-127).
 * coef: B x ld_coef row-major (ProjectionModel.coefficients, or evecs);
 * components (HOST array of k indices into coef columns); mean (B); std (B or
 * NULL for methods without standardization).  scores: k planes of rows*cols
 * float32, dense.  minmax: 2k floats [-min_0..-min_{k-1}, max_0..max_{k-1}]
 * (negated mins so a MAX all-reduce combines shards).  nonfinite: 1 int set
 * non-zero if any score is NaN/Inf (ScorePlane check, rendering.py:49-50).
 * precision: 0 = fp32 FMA on centred samples with an fp64-exact mean split,
 *            1 = fp64 throughout.  ws: ut_project_ws(). */
size_t ut_project_ws(void);
int ut_project_minmax(const ut_cube* cube, const double* coef, int32_t ld_coef,
                      const int32_t* components, int32_t k, const double* mean,
                      const double* std, int32_t precision, float* scores,
                      float* minmax, int32_t* nonfinite, void* ws, size_t ws_bytes,
                      void* stream);

/* ------------------------------------------------- K5: stretch
 * rescale_full -> linear_to_codes -> round_half_away (rendering.py:124-130,
 * quantize.py:13-46) for k dense planes of npix float32 scores, using the
 * minmax record produced by ut_project_minmax (possibly all-reduced):
 * plane c uses lo = -minmax[c], hi = minmax[ld_minmax + c].
 * depth 8 -> uint8 codes, 16 -> uint16.  lo == hi renders zeros. */
int ut_stretch(const float* scores, const float* minmax, int32_t k, int32_t ld_minmax,
               int64_t npix, int32_t depth, void* codes, void* stream);

/* ------------------------------------------------- single planes
 * rescale_full on an arbitrary float32/float64 plane (e.g. a host ScorePlane):
 * lohi[0] = min, lohi[1] = max (rendering.py:126-127); nonfinite set if a
 * NaN/Inf is present (ScorePlane check, rendering.py:49-50). */
size_t ut_plane_minmax_ws(void);
int ut_plane_minmax(const void* plane, int32_t dtype, int64_t n, double* lohi,
                    int32_t* nonfinite, void* ws, size_t ws_bytes, void* stream);
/* linear_to_codes(values, lo, hi, depth) (quantize.py:36-46) with device
 * lohi = {lo, hi}; lo == hi (constant plane) gives zeros. */
int ut_linear_to_codes(const void* plane, int32_t dtype, int64_t n, const double* lohi,
                       int32_t depth, void* codes, void* stream);

/* Order statistics for rescale_percentile (rendering.py:146-179): out[j] =
 * the value of 1-based rank ranks[j] (HOST int64[2]) of the ascending
 * float32/float64 plane, exact (radix select; no copy of the plane). */
size_t ut_plane_select_ws(void);
int ut_plane_select(const void* plane, int32_t dtype, int64_t n, const int64_t* ranks,
                    double* out, void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------- normalize_stack
 * stack.py:180-213: scope 0 = per-band, 1 = global min/max; out = uint8
 * planes [bands][rows][cols] contiguous, round_half_away(255 (v - lo) /
 * (hi - lo)) bit-identical to numpy.  lohi (device, 2*bands doubles) returns
 * each band's lo, hi; constant[b] = 1 where lo == hi (band -> zeros; the
 * reference warns).  NaN in a band (scope) gives lo = hi = NaN and zeros. */
size_t ut_normalize_ws(void);
int ut_normalize_stack(const ut_cube* cube, int32_t scope, void* out, double* lohi,
                       int32_t* constant, void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------- synthetic cubes
 * Seeded generator for the BASELINE.json configs: class map
 * from `nshapes` shapes (rects kind 0: [y0,x0,y1,x1); ellipses kind 1:
 * [cy,cx,ry,rx]) evaluated in integer arithmetic, later shapes win; pixel =
 * means[c] + chol[c] z (z ~ N(0,1) from a counter hash of seed/pixel/band),
 * clipped to [0,1] and cast (u16: round_half_away(4095 v)).
 * means: C*B doubles, chol: C*B*B doubles (row-major lower), shapes: HOST
 * int64 [nshapes][6] = {kind, class, a, b, c, d}.  Rows [row0, row0+rows). */
int ut_synth_cube(const ut_cube* cube, int64_t height, const double* means,
                  const double* chol, int32_t classes, const int64_t* shapes,
                  int32_t nshapes, uint64_t seed, void* stream);

/* class index of pixels (x_j, y_j): for host-side training-point sampling
 * checks (device version of the same integer class map). */
int ut_class_of(const int64_t* shapes, int32_t nshapes, const int32_t* xy,
                int64_t n, int32_t* cls, void* stream);

/* ------------------------------------------------- composites
 * compose_rgb (rendering.py:206-225): out[3 i + c] = plane_c[i] for three
 * device code planes of npix samples (depth 8: uint8, 16: uint16), the
 * recipe's channel choice and swap already applied by the caller. */
int ut_compose_rgb(const void* r, const void* g, const void* b, int32_t depth, int64_t npix,
                   void* out, void* stream);

/* ------------------------------------------------- image encoders
 * save_image (rendering.py:303-331) replaces cv2.imwrite (libpng / libtiff).
 * img: device, (rows, cols, channels) C-contiguous uint8 (depth 8) or uint16
 * (depth 16), channels 1 (gray) or 3 (RGB).  format 0 = PNG, 1 = TIFF.
 * ut_encode_png writes the PNG's IDAT chunks (zlib stream of the row-filtered
 * image, chunk CRCs included) to `out`; the caller frames them with the
 * signature, IHDR and IEND.  ut_encode_tiff writes the strips back to back
 * (compression 1 = raw, 8 = one zlib stream per strip over Predictor-2
 * samples) with strip_bytes[s] (device, ceil(rows / rows_per_strip) entries);
 * the caller adds the header and IFD.  *out_len (device) = bytes written.
 * Output bytes depend only on the image (deterministic). */
size_t ut_encode_ws(int64_t rows, int64_t cols, int32_t channels, int32_t depth, int32_t format,
                    int64_t rows_per_strip);
int64_t ut_encode_bound(int64_t rows, int64_t cols, int32_t channels, int32_t depth,
                        int32_t format, int64_t rows_per_strip);
int ut_encode_png(const void* img, int64_t rows, int64_t cols, int32_t channels, int32_t depth,
                  uint8_t* out, int64_t out_cap, int64_t* out_len, void* ws, size_t ws_bytes,
                  void* stream);
int ut_encode_tiff(const void* img, int64_t rows, int64_t cols, int32_t channels, int32_t depth,
                   int32_t compression, int64_t rows_per_strip, uint8_t* out, int64_t out_cap,
                   int64_t* strip_bytes, int64_t* out_len, void* ws, size_t ws_bytes,
                   void* stream);

/* ------------------------------------------------- image decode
 * load_stack / load_image (stack.py:119-177, rendering.py:334-343) replace
 * cv2.imread for TIFF bands.  src: the file's bytes in device memory; strip i
 * is in_len[i] bytes at in_off[i] and decodes to out_len[i] bytes at
 * dst + out_off[i] (all four arrays device).  compression 1 = raw strips,
 * 5 = TIFF LZW, 8 = one zlib stream per strip (Adler-32 checked).  status[i]
 * (device) = 0, or nonzero if strip i is malformed / too short / too long.
 * Tiles of a tiled TIFF and the IDAT stream of a PNG are streams too.
 * ut_unpredict undoes TIFF Predictor 2 (horizontal differencing per channel)
 * in place, after swapping the bytes of big-endian 16-bit samples if asked.
 * ut_untile scatters decoded tiles (tile t = row-major (ty, tx), tile_rows x
 * tile_row_bytes bytes each, contiguous) into the image rows.
 * ut_png_unfilter reconstructs n PNGs' inflated scanlines in place and writes
 * the images: table (device) holds, per image, work_off, out_off, rows, cols,
 * channels (1 / 3), depth (8 / 16); 16-bit samples come out little endian;
 * status[i] != 0 if image i has an invalid filter byte. */
int ut_decode_strips(const uint8_t* src, const int64_t* in_off, const int64_t* in_len, int64_t nstrips,
                     int32_t compression, uint8_t* dst, const int64_t* out_off, const int64_t* out_len,
                     int32_t* status, void* stream);
/* ut_decode_streams: the same with a promise about the largest out_len of the batch
 * (0 = unknown); deflate streams of <= 8 KB each take a small-window kernel. */
int ut_decode_streams(const uint8_t* src, const int64_t* in_off, const int64_t* in_len, int64_t nstreams,
                      int32_t compression, uint8_t* dst, const int64_t* out_off, const int64_t* out_len,
                      int64_t max_out_len, int32_t* status, void* stream);
int ut_unpredict(void* img, int32_t depth, int64_t rows, int64_t cols, int32_t channels,
                 int32_t predictor, int32_t swap_bytes, void* stream);
int ut_untile(const uint8_t* tiles, uint8_t* img, int64_t rows, int64_t row_bytes, int64_t tile_rows,
              int64_t tile_row_bytes, int64_t tiles_across, int64_t ntiles, void* stream);
int ut_png_unfilter(uint8_t* work, const int64_t* table, int64_t n, uint8_t* out, int32_t* status,
                    void* stream);

/* ------------------------------------------------- collectives (row shards)
 * SURVEY.md §8(b) ut_allreduce_f64 / §8(e): the sharded path's two exchange
 * steps, issued as NCCL collectives on the caller's stream so a rank's step
 * (kernels + collectives) is one capturable stream of work.  Replaces the
 * reference's single-process numpy reductions (projection.py:186-199 -- the
 * per-class sums -- and rendering.py:126-127 -- the global min / max), which
 * have no multi-process form.  NCCL is loaded at run time (torch's
 * libnccl.so.2, or UT_NCCL_LIB); ut_comm_available returns its version code
 * or 0.  comm: the handle ut_comm_init returns (an ncclComm_t); id: 128 bytes
 * from ut_comm_unique_id on one rank, shared by the caller (e.g. over the
 * torch.distributed store).  op: UT_OP_SUM / UT_OP_MIN / UT_OP_MAX, in place.
 * ut_allgather_f64: recv[r*n .. r*n+n) = rank r's send[0..n). */
enum { UT_OP_SUM = 0, UT_OP_MIN = 1, UT_OP_MAX = 2 };
int32_t ut_comm_available(void);
int ut_comm_unique_id(void* id_out);
int ut_comm_init(const void* id, int32_t nranks, int32_t rank, int32_t device, void** comm_out);
int ut_comm_destroy(void* comm);
int ut_allreduce_f64(void* comm, double* buf, int64_t n, int32_t op, void* stream);
int ut_allreduce_f32(void* comm, float* buf, int64_t n, int32_t op, void* stream);
int ut_allgather_f64(void* comm, const double* send, double* recv, int64_t n, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* UNDERTEXT_B200_H */
