// Shared definitions for libpastila (B200 / sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>
#include <cstring>
#include <string>

#include "../../include/pastila.h"

#define PST_INF __longlong_as_double(0x7ff0000000000000LL)
#define FULLMASK 0xffffffffu

// thread-local last error (pst_last_error)
void pst_set_error(const char* fmt, ...);

#define PST_CUDA(call)                                                         \
  do {                                                                         \
    cudaError_t _e = (call);                                                   \
    if (_e != cudaSuccess) {                                                   \
      pst_set_error("CUDA error %s at %s:%d: %s", cudaGetErrorName(_e),        \
                    __FILE__, __LINE__, cudaGetErrorString(_e));               \
      return PST_ECUDA;                                                        \
    }                                                                          \
  } while (0)

#define PST_TRY(expr)            \
  do {                           \
    int _r = (expr);             \
    if (_r != PST_OK) return _r; \
  } while (0)

// Order-preserving 64-bit key of a NON-NEGATIVE double (callers clamp).
__device__ __forceinline__ long long dkey(double v) { return __double_as_longlong(v); }
__device__ __forceinline__ double kdbl(long long k) { return __longlong_as_double(k); }
// clamp at +0 (also maps -0.0 and tiny negatives from rounding to +0.0)
__device__ __forceinline__ double clamp0(double v) { return v > 0.0 ? v : 0.0; }

// Per-length derived window data (all n-l+1 long except df/dg: n-l).
struct LenData {
  int64_t l = -1, Nl = 0;
  double* mu = nullptr;     // window means (series.py:179)
  double* var = nullptr;    // clamped variances (series.py:180-187)
  double* sd = nullptr;     // sqrt(var)
  double* nrm = nullptr;    // 1/sqrt(l*var), 0 for constant windows
  double* bias = nullptr;   // e for a constant column vs non-constant query: 0.5, else 1.0
  double* cbias = nullptr;  // e for a constant query: 0 (constant column) / 0.5
  double* df = nullptr;     // (x[i+l]-x[i])/2
  double* dg = nullptr;     // (x[i+l]-mc[i+1]) + (x[i]-mc[i])
  double* mc = nullptr;     // direct window mean sum(x)/l (centering of the distance kernels)
  unsigned long long* hash = nullptr;  // 64-bit polynomial hash of the window's bit patterns (exact repeats)
  bool has_rep = false;     // two windows share a hash (possible exact repeat): the rule must run
};

struct pst_ctx {
  int dev = 0;
  cudaStream_t st = nullptr;
  cudaStream_t st2 = nullptr;   // selection stream (overlaps the next batch's row loop)
  cudaEvent_t ev_rows[2] = {nullptr, nullptr}, ev_sel[2] = {nullptr, nullptr};
  int64_t n = 0, cap_n = 0;
  double* x = nullptr;
  double* csum = nullptr;   // [n+1] sequential prefix sum of x
  double* csq = nullptr;    // [n+1] sequential prefix sum of x*x
  int64_t* chg = nullptr;   // [n] #{t in [1,i] : x[t] != x[t-1]}
  LenData L;
  int64_t cap_l = 0;
  // scratch for the MPdist tile kernel (AB matrices of in-flight tiles)
  double* scratch = nullptr;
  size_t scratch_bytes = 0;
  // profile matrix D (S x N) + greedy buffers
  double* D = nullptr;
  size_t D_bytes = 0;
  // key path: S x N profile keys, exact rows of greedy candidates, certification lists
  int* Dk = nullptr;
  size_t Dk_bytes = 0;
  void* cert = nullptr;
  size_t cert_bytes = 0;
  // certification counters of the last key-path selections (pst_cert_stats):
  // [0] lengths, [1] greedy candidates evaluated exactly, [2] greedy steps with >1
  // candidate, [3] uncertain attribution windows, [4] exact (segment, window)
  // evaluations, [5] max candidates, [6] fallbacks to the exact path, [7] windows
  int64_t cert_stats[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  void* work = nullptr;
  size_t work_bytes = 0;
  void* aux = nullptr;       // per-length preparation scratch (hash sort); never holds live results
  size_t aux_bytes = 0;
  // streamed key path: per-block key minima of every profile row + greedy-pass
  // lower-bound scratch (pruned greedy passes); freed after each length
  void* prune = nullptr;
  size_t prune_bytes = 0;
  // [0] pruned greedy passes, [1] rows recomputed in them, [2] pruned passes
  // that fell back to a full pass (too many candidates), [3] rows of those passes
  int64_t prune_stats[4] = {0, 0, 0, 0};
  int64_t launches = 0;
  double* dbg = nullptr;
  size_t dbg_bytes = 0;
  int64_t dbg_T = 0, dbg_NC = 0, dbg_w = 0;
  // kernel timing (profile kernel): events around each launch_mpdist call
  bool timing = false;
  void* tev = nullptr;  // std::vector<std::pair<cudaEvent_t,cudaEvent_t>>*
  double t_ms = 0.0;
  int64_t t_calls = 0, t_launch = 0;
  // per-kernel-class event timing (PASTILA_KTIME=1, instrumentation): row loop vs selection
  void* kev = nullptr;  // std::vector<KEv>*
  double k_ms[2] = {0.0, 0.0};
  int num_sms = 148;
  size_t smem_optin = 0;
  // NCCL communicator of the sharded search (comm.cu), one per context
  void* comm = nullptr;
  int comm_size = 1, comm_rank = 0;
};

int pst_ensure(void** p, size_t* cap, size_t bytes);
int pst_ensure_len(pst_ctx* c, int64_t l);

// kernels launched from several translation units.  The profile kernels are
// templated on the value type V of their minima / order statistics: double
// (exact e values) or int (32-bit key = high word of e, see mpdist.cu).
struct MPArgs {
  const double *x, *mu /* centering means (LenData::mc) */, *nrm, *bias, *cbias, *df, *dg;
  const unsigned long long* hash;  // window hashes (exact-repeat zeros, see same_window in mpdist.cu)
  int rep;                         // apply the exact-repeat rule (always, except the A/B test knob)
  int64_t n, l, m, w, k, Nl, N, T;
  int64_t seg0;      // segment of blockIdx.y == 0 (segs: its position in the list)
  const int64_t* segs;  // optional device list of segment indices (nullptr: seg0 + blockIdx.y)
  void* D;           // output rows (segment seg0+blockIdx.y -> row rowD0+blockIdx.y): double d / int key
  int64_t ldD, rowD0;
  void* ab;          // scratch, w*Tp values V per CTA, lane-run order (see mpdist.cu)
  int64_t R, Tp;     // lane-run length (odd) and AB row stride Tp = 32*R >= T
  void* dbg_ba;      // optional: allP_BA of CTA (0,0) (debug)
  void* ba;          // scratch: allP_BA per CTA (NCmax values V)
  int dbg_flags;     // debug (PASTILA_DBGF, timing experiments only, wrong results):
                     //   1 = selection: skip unsettled-window solves, 2 = selection: skip count pass,
                     //   4 = selection: skip the run-start solves
};

// Tile geometry of the profile kernels for one (m, l) on one series length:
// shared by the exact (double) and key (int) paths and by the exact
// single-window evaluator, so that all three compute bit-identical e values.
struct TileGeom {
  int64_t w, N, NCmax, T, ntile, R, Tp;
  int nt, P, chm;
  bool rows2;
  bool v2;         // k_rowsP (thread-owned windows) instead of k_mpdist / k_mpdist2
  size_t smem_d;   // dynamic smem of the one-row kernel with V = double (geometry decisions)
};
int tile_geom(pst_ctx* c, int64_t m, int64_t l, TileGeom& g);

int launch_mpdist(pst_ctx* c, int64_t m, int64_t l, int64_t k, int64_t seg_lo, int64_t seg_hi,
                  double* D_dev, int64_t ld);
// key path: Dk rows receive the 32-bit key (high word of e) of the k-th smallest
// P_ABBA element instead of the distance (exact d lies in [f(lo(key)), f(hi(key))]).
int launch_mpdist_keys(pst_ctx* c, int64_t m, int64_t l, int64_t k, int64_t seg_lo, int64_t seg_hi,
                       int* Dk_dev, int64_t ld);
int launch_mpdist_keys_list(pst_ctx* c, int64_t m, int64_t l, int64_t k, const int64_t* segs, int64_t cnt,
                            int* Dk_dev, int64_t ld);
// exact profile values at single (segment, window) pairs, bit-identical to the
// full profile kernels: out[i] = D[seg[i]][win[i]] (device arrays, cnt entries).
int kernel_times_read(pst_ctx* c, double* out2);
int launch_window_exact(pst_ctx* c, int64_t m, int64_t l, int64_t k, const int64_t* seg_dev,
                        const int64_t* win_dev, int64_t cnt, double* out_dev);
