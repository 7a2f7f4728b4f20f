/*
 * pastila.h -- C-ABI of the B200-native PaSTiLa hot path (libpastila.so).
 *
 * The reference (sniplab, /root/reference/pkg/src/sniplab) is pure Python and
 * has no FFI of its own; this ABI is the boundary under its Python API.  Each
 * entry point names the reference function whose semantics it provides
 * (file:line), and the Python package paper_2401_13680_b200 binds exactly
 * these symbols through ctypes.
 *
 * Conventions
 *   - every function returns 0 on success, a negative PST_E* code on error;
 *     pst_last_error() returns the message of the last failure on the
 *     calling thread (ValueError-class messages reuse the reference wording);
 *   - "host" pointers are ordinary CPU memory (pinned or pageable), "dev"
 *     pointers are device memory of the context's GPU;
 *   - all values are IEEE binary64, indices/labels int64;
 *   - a context owns one GPU (one process per GPU; multi-GPU goes through
 *     torch.distributed/NCCL above this layer).
 */
#ifndef PASTILA_H
#define PASTILA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PST_OK 0
#define PST_EINVAL -1   /* bad argument (maps to ValueError)   */
#define PST_ECUDA -2    /* CUDA runtime failure (RuntimeError) */
#define PST_ENOMEM -3   /* device allocation failed           */
#define PST_ESTATE -4   /* missing prerequisite (no series)   */

typedef struct pst_ctx pst_ctx;

/* Snippet-search output (select_snippets, snippets.py:154-244).
 * Caller-owned host buffers; sizes: K for the snippet arrays, N = n-m+1 for
 * curve / nearest, K*N for profiles (row-major, in frac order), S = n/m for
 * counts.  Any pointer may be NULL to skip that output.                    */
typedef struct pst_snippets {
  int64_t* indices;        /* [K] segment index, frac order               */
  double* fracs;           /* [K]                                         */
  double* curve;           /* [N] representativeness curve                */
  double* profiles;        /* [K*N] chosen profiles, frac order           */
  int64_t* counts;         /* [S] windows per nearest segment             */
  int32_t* nearest;        /* [N] nearest segment of every window         */
  int64_t* labels;         /* [n] per-point labels (labeling.py:91-119)   */
  double profile_area;     /* out: sum(curve)                             */
  double profile_max;      /* out: max over all S profiles                */
  double criterion;        /* out: Eq. 18 score (length_select.py:56-87), 0 if K<2 */
  int64_t unassigned;      /* out: windows whose nearest is not chosen    */
} pst_snippets;

/* ---- context (no reference counterpart: the reference is host-only; one
 * context per process and GPU owns the uploaded series and device buffers;
 * pst_last_error is per thread and carries the reference's ValueError text) */
int pst_create(int device, pst_ctx** out);
int pst_destroy(pst_ctx* ctx);
const char* pst_last_error(void);
int pst_device_count(int* out);

/* Upload a series and build its exact prefix sums (series.py:152-190,
 * the sequential np.cumsum order).  Replaces TimeSeries ingestion for the
 * device path.  x: host, n >= 2.                                          */
int pst_set_series(pst_ctx* ctx, const double* x, int64_t n);
/* Same from a device pointer (bench: input already resident in HBM).      */
int pst_set_series_dev(pst_ctx* ctx, const double* x_dev, int64_t n);

/* compute_sliding_stats (series.py:152-190): bit-identical to the reference
 * on the same input.  Outputs are host arrays of n-l+1 entries (NULL ok).  */
int pst_sliding_stats(pst_ctx* ctx, int64_t l, double* means, double* stds, double* vars);

/* segment_distance_matrix / distance_row (zdist.py:138-225): distance rows
 * for queries q0 .. q0+rows-1 against every length-l window.
 * method 0 = sliding (correlation identity), 1 = direct z-normalization.
 * out: host [rows * (n-l+1)].                                             */
int pst_distance_rows(pst_ctx* ctx, int64_t l, int64_t q0, int64_t rows, int method, double* out);

/* mpdist_profile / segment_profiles (mpdist.py:179-232, snippets.py:119-128):
 * MPdist profiles of segments [seg_lo, seg_hi) at snippet size m, inner
 * window l, order statistic k.  out: host [(seg_hi-seg_lo) * (n-m+1)].    */
int pst_mpdist_profiles(pst_ctx* ctx, int64_t m, int64_t l, int64_t k,
                        int64_t seg_lo, int64_t seg_hi, double* out);

/* select_snippets + label_series + criterion_score for one length:
 * all S profiles are computed on the device and never leave it; only the
 * outputs in *res are copied back.                                        */
int pst_select_snippets(pst_ctx* ctx, int64_t m, int64_t l, int64_t k, int64_t K, pst_snippets* res);
/* select_length (length_select.py:116-182): one search per grid length, in
 * grid order; l = ls[i] (ls NULL: ceil(m/2)), k = ceil(m/10); Eq. 18 score
 * per length; m_best = argmax (score, -m).  indices/fracs [nm*K] in frac
 * order, scores/areas [nm]; any output may be NULL.  Errors as the reference:
 * "length grid is empty", "... duplicates", "... at least 2 snippets".     */
int pst_sweep(pst_ctx* ctx, const int64_t* ms, const int64_t* ls, int64_t nm, int64_t K,
              int64_t* indices, double* fracs, double* scores, double* areas, int64_t* m_best);

/* select_snippets(..., profiles=...) on caller-supplied host profiles
 * D [S*N] of a series of length n (snippets.py:191-244).                  */
int pst_select_from_profiles(pst_ctx* ctx, const double* D, int64_t S, int64_t N, int64_t n, int64_t K,
                             pst_snippets* res);

/* criterion_score (length_select.py:56-87) on host profiles P [K*N] (snippet
 * order); out = sum over pairs of sum|P_a-P_b| / profile_max (0 if max==0). */
int pst_criterion(pst_ctx* ctx, const double* P, int64_t K, int64_t N, double profile_max, double* out);
/* label_series (labeling.py:91-119) on host profiles P [K*N]; labels [n].   */
int pst_labels(pst_ctx* ctx, const double* P, int64_t K, int64_t N, int64_t n, int64_t* labels);

/* ---- device-level API (multi-GPU sharding / benchmark) ----------------
 * segment_profiles (snippets.py:119-128, mpdist.py:179-232) for segments
 * [seg_lo, seg_hi), written to a caller-owned device matrix D_dev (row
 * stride ld >= n-m+1).                                                     */
int pst_profiles_dev(pst_ctx* ctx, int64_t m, int64_t l, int64_t k,
                     int64_t seg_lo, int64_t seg_hi, double* D_dev, int64_t ld);
/* Greedy-step areas sum_j min(D[s][j], curve[j]) for rows of D_dev
 * (snippets.py:201-206; curve_dev == NULL means +inf, i.e. plain row sums).
 * areas_dev [rows].                                                        */
int pst_areas_dev(pst_ctx* ctx, const double* D_dev, int64_t rows, int64_t N, int64_t ld,
                  const double* curve_dev, double* areas_dev);
/* Per-window minimum value and first argmin over rows (snippets.py:212,
 * ties -> lower row), row indices offset by row_base.  minval_dev [N],
 * argmin_dev [N].                                                          */
int pst_colmin_dev(pst_ctx* ctx, const double* D_dev, int64_t rows, int64_t N, int64_t ld,
                   int64_t row_base, double* minval_dev, int32_t* argmin_dev);
/* Max over a rows x N device matrix (profile_max of a rank's segment rows,
 * snippets.py:241); out_dev receives one double.                          */
int pst_max_dev(pst_ctx* ctx, const double* D_dev, int64_t rows, int64_t N, int64_t ld, double* out_dev);
/* Profiles of segments [seg_lo, seg_hi) computed in device-sized chunks and
 * reduced without being stored (S x N larger than HBM, C4: n = 1e7):
 * areas_dev[s-seg_lo] = sum_j min(D[s][j], curve_dev[j]) (curve NULL: +inf);
 * if minval_dev/argmin_dev are given, running per-window minimum and first
 * argmin (segment index, caller initialises minval to +inf); if rowmax_dev
 * is given, running max (caller initialises it to 0.0).  Serves the greedy
 * rounds of select_snippets (snippets.py:201-213) and segment-row sharding. */
int pst_profile_reduce_dev(pst_ctx* ctx, int64_t m, int64_t l, int64_t k, int64_t seg_lo, int64_t seg_hi,
                           const double* curve_dev, double* areas_dev, double* minval_dev,
                           int32_t* argmin_dev, double* rowmax_dev);
/* ---- key path evidence (no reference counterpart; the reference computes
 * every profile value in fp64, mpdist.py:179-232) -------------------------
 * Profile keys of segments [seg_lo, seg_hi): the high 32-bit word of the e
 * value (e = d^2/2l) of each window's k-th smallest P_ABBA element, as the
 * fast pass stores them; the exact profile value lies in
 * [f(key:00000000), f(key:ffffffff)], f(e) = sqrt(2l * e).  out: host
 * [(seg_hi-seg_lo) * (n-m+1)].                                             */
int pst_profile_keys(pst_ctx* ctx, int64_t m, int64_t l, int64_t k, int64_t seg_lo, int64_t seg_hi,
                     int32_t* out);
/* Exact MPdist profile values D[seg[i]][win[i]] (mpdist.py:179-232 at one
 * window), bit-identical to pst_mpdist_profiles; host arrays of cnt.      */
int pst_window_exact(pst_ctx* ctx, int64_t m, int64_t l, int64_t k, const int64_t* seg, const int64_t* win,
                     int64_t cnt, double* out);
/* Certification counters of key-path selections since the last reset:
 * [lengths, greedy candidates evaluated exactly, greedy steps with >1
 * candidate, uncertain attribution windows, exact window evaluations,
 * profile_max candidates, fallbacks to the exact path, windows].         */
int pst_cert_stats(pst_ctx* ctx, int64_t* out8, int reset);
/* Streamed key path (profile keys larger than HBM, e.g. C4): greedy passes
 * after the second recompute only the segments whose area lower bound (from
 * per-block key minima kept since pass 0) can still win (snippets.py:201-210
 * decides the same argmin).  Counters since the last reset: [pruned passes,
 * rows recomputed in them, pruned passes that fell back to a full pass,
 * rows of those].                                                          */
int pst_prune_stats(pst_ctx* ctx, int64_t* out4, int reset);
/* ---- multi-GPU data plane (segment-row sharding; the
 * reference has none: its workers are processes, scheduler.py:373-405) ----
 * One NCCL communicator per context (NCCL is dlopen'ed).  Rank 0 creates the
 * 128-byte id, the caller distributes it, every rank calls pst_comm_init.
 * Collectives are in place on device buffers on the context stream:
 * dtype 0 = f64, 1 = i64, 2 = i32; op 0 = min, 1 = max, 2 = sum.          */
int pst_comm_unique_id(char* out128);
int pst_comm_init(pst_ctx* ctx, const char* id128, int nranks, int rank);
int pst_comm_destroy(pst_ctx* ctx);
int pst_comm_allreduce(pst_ctx* ctx, void* buf_dev, int64_t count, int dtype, int op);
int pst_comm_broadcast(pst_ctx* ctx, void* buf_dev, int64_t bytes, int root);
int pst_comm_allgather(pst_ctx* ctx, const void* send_dev, void* recv_dev, int64_t bytes_per_rank);
/* Device glue of the sharded greedy (snippets.py:201-213 split over ranks):
 * best available local row as (area, global index) [2 doubles]; global pick
 * among nranks gathered pairs (marks it taken if local); attribution tie
 * indices idx[j] = local_arg[j] + base where the local minimum equals the
 * global one, else INT64_MAX; curve = row (first) or min(curve, row).     */
int pst_local_best_dev(pst_ctx* ctx, const double* areas_dev, const uint8_t* taken_dev, int64_t rows,
                       int64_t base, double* out2_dev);
int pst_pick_global_dev(pst_ctx* ctx, const double* pairs_dev, int nranks, int64_t base, int64_t rows,
                        uint8_t* taken_dev, double* out2_dev);
int pst_tie_index_dev(pst_ctx* ctx, const double* lmin_dev, const double* gmin_dev, const int32_t* larg_dev,
                      int64_t base, int64_t N, int64_t* out_dev);
int pst_curve_min_dev(pst_ctx* ctx, double* curve_dev, const double* row_dev, int64_t N, int first);
/* Instrumentation: milliseconds of the profile row-loop and selection
 * kernels since the last call (needs PASTILA_KTIME=1 and pst_timing on).  */
int pst_kernel_times(pst_ctx* ctx, double* out2);
/* The context's CUDA stream (cudaStream_t) for caller-side event timing.  */
int pst_stream(pst_ctx* ctx, void** stream_out);
/* Profile-kernel timing: pst_timing(ctx,1) enables + resets; pst_timing_read
 * returns device milliseconds and launches of profile kernels since.      */
int pst_timing(pst_ctx* ctx, int enable);
int pst_timing_read(pst_ctx* ctx, double* ms, int64_t* launches);
/* Wait for all work queued on the context stream.                        */
int pst_sync(pst_ctx* ctx);
/* Kernel launches issued on the context since creation (instrumentation). */
int64_t pst_launch_count(pst_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* PASTILA_H */
