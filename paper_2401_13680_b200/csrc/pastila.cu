// libpastila: context, sliding statistics, distance rows, greedy snippet
// selection, nearest-segment attribution, labels, Eq. 18 criterion, C-ABI.
#include "common.cuh"

#include <cub/cub.cuh>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <numeric>
#include <vector>

static thread_local std::string g_err;

void pst_set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
}

int pst_ensure(void** p, size_t* cap, size_t bytes) {
  if (bytes <= *cap && *p) return PST_OK;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *cap = 0;
  if (bytes == 0) return PST_OK;
  cudaError_t e = cudaMalloc(p, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    pst_set_error("device allocation of %zu bytes failed: %s", bytes, cudaGetErrorString(e));
    *p = nullptr;
    return PST_ENOMEM;
  }
  *cap = bytes;
  return PST_OK;
}

namespace {

// ----------------------------------------------------------------- kernels
// Exact sequential prefix sums (np.cumsum order, series.py:177-178) and the
// running count of value changes (constant-window test, series.py:183-187).
// The summation order must be strictly sequential to be bit-identical with
// numpy, so one thread runs the dependent DADD chain; the other threads stage
// chunks of x into shared memory (double-buffered, coalesced) and write the
// results back, keeping global-memory latency off the chain.
constexpr int PFX_CH = 1024;
__global__ void __launch_bounds__(256) k_prefix(const double* __restrict__ x, int64_t n, double* csum, double* csq,
                                                int64_t* chg) {
  __shared__ double xin[2][PFX_CH];
  __shared__ double os[PFX_CH], oq[PFX_CH];
  __shared__ int64_t oc[PFX_CH];
  const int tid = threadIdx.x;
  double s = 0.0, q = 0.0, prev = 0.0;
  int64_t c = 0;
  if (tid == 0) {
    csum[0] = 0.0;
    csq[0] = 0.0;
  }
  const int64_t nch = (n + PFX_CH - 1) / PFX_CH;
  for (int i = tid; i < PFX_CH && i < n; i += 256) xin[0][i] = x[i];
  __syncthreads();
  for (int64_t ch = 0; ch < nch; ++ch) {
    const int cur = (int)(ch & 1);
    const int64_t base = ch * PFX_CH;
    const int cnt = (int)min((int64_t)PFX_CH, n - base);
    if (tid == 0) {
      const double* xv = xin[cur];
      for (int i = 0; i < cnt; ++i) {
        const double v = xv[i];
        s = __dadd_rn(s, v);
        q = __dadd_rn(q, __dmul_rn(v, v));
        if (base + i > 0 && v != prev) ++c;
        prev = v;
        os[i] = s;
        oq[i] = q;
        oc[i] = c;
      }
    } else if (ch + 1 < nch) {  // prefetch the next chunk meanwhile
      const int64_t nb = base + PFX_CH;
      const int ncnt = (int)min((int64_t)PFX_CH, n - nb);
      for (int i = tid - 1; i < ncnt; i += 255) xin[cur ^ 1][i] = x[nb + i];
    }
    __syncthreads();
    for (int i = tid; i < cnt; i += 256) {
      csum[base + i + 1] = os[i];
      csq[base + i + 1] = oq[i];
      chg[base + i] = oc[i];
    }
    __syncthreads();
  }
}

__device__ __forceinline__ double win_mean(const double* csum, int64_t i, int64_t l) {
  return __ddiv_rn(__dsub_rn(csum[i + l], csum[i]), (double)l);
}

// Per-length window statistics, bit-identical to series.py:179-189, plus the
// derived arrays of the distance recurrence (see mpdist.cu header).
__global__ void k_stats(const double* __restrict__ x, const double* __restrict__ csum,
                        const double* __restrict__ csq, const int64_t* __restrict__ chg, int64_t n,
                        int64_t l, LenData L) {
  const int64_t Nl = n - l + 1;
  const double dl = (double)l;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < Nl; i += (int64_t)gridDim.x * blockDim.x) {
    const double mu = win_mean(csum, i, l);
    double v = __dsub_rn(__ddiv_rn(__dsub_rn(csq[i + l], csq[i]), dl), __dmul_rn(mu, mu));
    v = v > 0.0 ? v : 0.0;                        // np.maximum(var, 0)
    if (chg[i + l - 1] - chg[i] == 0) v = 0.0;    // sliding max == sliding min
    L.mu[i] = mu;
    L.var[i] = v;
    L.sd[i] = __dsqrt_rn(v);
    const bool cst = (v == 0.0);
    // Distance kernels center with the direct window mean and normalize with the
    // centered sum of squares (two-pass): accurate even where the prefix-sum
    // variance cancels.  The constant flag keeps the reference rule above.
    double sx = 0.0;
    for (int64_t t = 0; t < l; ++t) sx += x[i + t];
    const double mc = sx / dl;
    L.mc[i] = mc;
    double css = 0.0;
    if (!cst)
      for (int64_t t = 0; t < l; ++t) {
        const double d = x[i + t] - mc;
        css = fma(d, d, css);
      }
    L.nrm[i] = (cst || css <= 0.0) ? 0.0 : __drcp_rn(__dsqrt_rn(css));
    L.bias[i] = cst ? 0.5 : 1.0;
    L.cbias[i] = cst ? 0.0 : 0.5;

  }
}

__global__ void k_dfdg(const double* __restrict__ x, int64_t n, int64_t l, LenData L) {
  const int64_t Nl = n - l + 1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i + 1 < Nl; i += (int64_t)gridDim.x * blockDim.x) {
    L.df[i] = (x[i + l] - x[i]) * 0.5;
    L.dg[i] = (x[i + l] - L.mc[i + 1]) + (x[i] - L.mc[i]);
  }
}

// Window hashes for the exact-repeat rule (zdist.py:98-106: bit-equal windows are
// at distance 0 wherever they sit): Horner over the l sample bit patterns, mod 2^64.
__global__ void k_hash(const double* __restrict__ x, int64_t n, int64_t l, unsigned long long* hash) {
  const int64_t Nl = n - l + 1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < Nl; i += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long h = 0;
    for (int64_t t = 0; t < l; ++t) h = h * 0x9E3779B97F4A7C15ull + (unsigned long long)__double_as_longlong(x[i + t]);
    hash[i] = h;
  }
}

__global__ void k_adjacent_equal(const unsigned long long* __restrict__ v, int64_t n, int* flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i + 1 < n; i += (int64_t)gridDim.x * blockDim.x)
    if (v[i] == v[i + 1]) *flag = 1;
}

// Distance rows for queries q0..q0+rows-1 (zdist.py:191-225): one thread per
// diagonal; diagonals entering at row 0 (column c0 >= 0) or at column 0
// (row r0 > 0) start from a fresh centered dot product.
__global__ void k_rows(const double* __restrict__ x, LenData L, int64_t n, int64_t l, int64_t q0,
                       int64_t rows, double* __restrict__ out) {
  const int64_t Nl = n - l + 1;
  const int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x - (rows - 1);  // column - row
  if (d >= Nl) return;
  int64_t r = d >= 0 ? 0 : -d;
  int64_t c = d >= 0 ? d : 0;
  if (r >= rows) return;
  int64_t q = q0 + r;
  double cov = 0.0;
  {
    const double mq = L.mc[q], mc = L.mc[c];
    double acc = 0.0, sq = 0.0;
    for (int64_t t = 0; t < l; ++t) {
      const double xq = x[q + t] - mq;
      acc = fma(xq, x[c + t], acc);
      sq += xq;
    }
    cov = fma(-mc, sq, acc);
  }
  const double twol = 2.0 * (double)l;
  for (;;) {
    double e;
    const double nq = L.nrm[q];
    if (nq == 0.0)
      e = L.cbias[c];
    else
      e = fma(-(cov * nq), L.nrm[c], L.bias[c]);
    if (nq != 0.0 && c != q && L.hash[q] == L.hash[c]) {  // exact repeat (bit-equal windows): d = 0
      bool same = true;
      for (int64_t t = 0; t < l && same; ++t) same = __double_as_longlong(x[q + t]) == __double_as_longlong(x[c + t]);
      if (same) e = 0.0;
    }
    if (c == q) e = 0.0;
    e = clamp0(e);
    if (e < 1e-15) e = 0.0;
    if (e > 2.0) e = 2.0;
    out[r * Nl + c] = sqrt(twol * e);
    if (++r >= rows || c + 1 >= Nl) break;
    cov = fma(L.df[q], L.dg[c], fma(L.dg[q], L.df[c], cov));
    ++q;
    ++c;
  }
}

// Direct z-normalized distances (zdist.py:126-135): explicit per-window
// mean/std (two-pass), constant windows z-normalize to zeros.
__global__ void k_rows_direct(const double* __restrict__ x, int64_t n, int64_t l, int64_t q0, int64_t rows,
                              double* __restrict__ out) {
  const int64_t Nl = n - l + 1;
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t r = blockIdx.y;
  if (c >= Nl || r >= rows) return;
  const int64_t q = q0 + r;
  auto stat = [&](int64_t s0, double& mean, double& sdv, bool& flat) {
    double s = 0.0, mn = x[s0], mx = x[s0];
    for (int64_t t = 0; t < l; ++t) {
      s += x[s0 + t];
      mn = fmin(mn, x[s0 + t]);
      mx = fmax(mx, x[s0 + t]);
    }
    mean = s / (double)l;
    double ss = 0.0;
    for (int64_t t = 0; t < l; ++t) {
      const double dv = x[s0 + t] - mean;
      ss += dv * dv;
    }
    sdv = sqrt(ss / (double)l);
    flat = (mn == mx) || sdv == 0.0;
  };
  double mq, sq, mc, sc;
  bool fq, fc;
  stat(q, mq, sq, fq);
  stat(c, mc, sc, fc);
  double acc = 0.0;
  for (int64_t t = 0; t < l; ++t) {
    const double zq = fq ? 0.0 : (x[q + t] - mq) / sq;
    const double zc = fc ? 0.0 : (x[c + t] - mc) / sc;
    acc += (zq - zc) * (zq - zc);
  }
  out[r * Nl + c] = (c == q) ? 0.0 : sqrt(acc);
}

// Deterministic block reduction helpers (fixed order: per-thread strided
// sequential sum, then a fixed shuffle tree) -- identical rows give
// bit-identical sums, as numpy row sums do (snippets.py:205).
template <int NT>
__device__ double block_sum(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULLMASK, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int wv = 0; wv < NT / 32; ++wv) t += sh[wv];
  __syncthreads();
  return t;
}

// areas[r] = sum_j min(D[r][j], curve[j])  (curve == nullptr: +inf)
__global__ void __launch_bounds__(256) k_areas(const double* __restrict__ D, int64_t N, int64_t ld,
                                               const double* __restrict__ curve, double* areas) {
  __shared__ double sh[8];
  const double* row = D + blockIdx.x * ld;
  double acc = 0.0;
  if (curve) {
    for (int64_t j = threadIdx.x; j < N; j += 256) acc += fmin(row[j], curve[j]);
  } else {
    for (int64_t j = threadIdx.x; j < N; j += 256) acc += row[j];
  }
  const double t = block_sum<256>(acc, sh);
  if (threadIdx.x == 0) areas[blockIdx.x] = t;
}

// argmin over available rows (ties -> lowest index, snippets.py:207); marks it taken,
// folds it into the curve in a follow-up kernel.
__global__ void __launch_bounds__(1024) k_pick(const double* __restrict__ areas, uint8_t* taken, int64_t S,
                                               int64_t* best_out) {
  __shared__ double bv[32];
  __shared__ int64_t bi[32];
  double v = PST_INF;
  int64_t idx = INT64_MAX;
  for (int64_t s = threadIdx.x; s < S; s += blockDim.x) {
    if (taken[s]) continue;
    const double a = areas[s];
    if (a < v || (a == v && s < idx)) {
      v = a;
      idx = s;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(FULLMASK, v, o);
    const int64_t oi = __shfl_xor_sync(FULLMASK, idx, o);
    if (ov < v || (ov == v && oi < idx)) {
      v = ov;
      idx = oi;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    bv[threadIdx.x >> 5] = v;
    bi[threadIdx.x >> 5] = idx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int wv = 1; wv < (int)(blockDim.x >> 5); ++wv)
      if (bv[wv] < v || (bv[wv] == v && bi[wv] < idx)) {
        v = bv[wv];
        idx = bi[wv];
      }
    if (idx == INT64_MAX) {  // all taken or all +inf areas: lowest available index
      for (int64_t s = 0; s < S; ++s)
        if (!taken[s]) {
          idx = s;
          break;
        }
    }
    *best_out = idx;
    taken[idx] = 1;
  }
}

__global__ void k_curve(double* curve, const double* __restrict__ D, int64_t ld, const int64_t* best, int64_t N) {
  const double* row = D + (*best) * ld;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < N; j += (int64_t)gridDim.x * blockDim.x)
    curve[j] = fmin(curve[j], row[j]);
}

__global__ void k_fill(double* p, double v, int64_t N) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < N; j += (int64_t)gridDim.x * blockDim.x) p[j] = v;
}

// Per-window first argmin over rows (snippets.py:212, labeling.py:115).
__global__ void k_colmin(const double* __restrict__ D, int64_t rows, int64_t N, int64_t ld, int64_t base,
                         double* minval, int32_t* arg) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < N; j += (int64_t)gridDim.x * blockDim.x) {
    double b = D[j];
    int64_t bi = 0;
    for (int64_t r = 1; r < rows; ++r) {
      const double v = D[r * ld + j];
      if (v < b) {
        b = v;
        bi = r;
      }
    }
    if (minval) minval[j] = b;
    arg[j] = (int32_t)(bi + base);
  }
}

// Running per-window minimum over successive row chunks (streamed selection):
// strict '<' keeps the first (lowest) segment index, chunks arrive in order.
__global__ void k_colmin_acc(const double* __restrict__ D, int64_t rows, int64_t N, int64_t ld, int64_t base,
                             double* minval, int32_t* arg) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < N; j += (int64_t)gridDim.x * blockDim.x) {
    double b = minval[j];
    int64_t bi = -1;
    for (int64_t r = 0; r < rows; ++r) {
      const double v = D[r * ld + j];
      if (v < b) {
        b = v;
        bi = r;
      }
    }
    if (bi >= 0) {
      minval[j] = b;
      arg[j] = (int32_t)(bi + base);
    }
  }
}

__global__ void k_count(const int32_t* __restrict__ arg, int64_t N, unsigned long long* counts) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < N; j += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&counts[arg[j]], 1ull);
}

// max over the S x N matrix (profile_max, snippets.py:241): order independent.
__global__ void k_max(const double* __restrict__ D, int64_t rows, int64_t N, int64_t ld, unsigned long long* out) {
  double m = 0.0;
  for (int64_t r = blockIdx.y; r < rows; r += gridDim.y)
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < N; j += (int64_t)gridDim.x * blockDim.x)
      m = fmax(m, D[r * ld + j]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(FULLMASK, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

// Eq. 18 pair sums: sum_j |P_a[j] - P_b[j]| for one (a, b) pair per CTA.
__global__ void __launch_bounds__(256) k_pairdiff(const double* __restrict__ P, int64_t N, int64_t K,
                                                  double* out) {
  __shared__ double sh[8];
  int64_t a = 0, b = 0, t = blockIdx.x;
  for (a = 0; a < K; ++a) {
    const int64_t cnt = K - 1 - a;
    if (t < cnt) {
      b = a + 1 + t;
      break;
    }
    t -= cnt;
  }
  const double* pa = P + a * N;
  const double* pb = P + b * N;
  double acc = 0.0;
  for (int64_t j = threadIdx.x; j < N; j += 256) acc += fabs(pa[j] - pb[j]);
  const double s = block_sum<256>(acc, sh);
  if (threadIdx.x == 0) out[blockIdx.x] = s;
}

// labels (labeling.py:114-118): argmin over K ordered profiles, tail copies the last window.
__global__ void k_labels(const double* __restrict__ P, int64_t K, int64_t N, int64_t n, int64_t* labels) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = i < N ? i : N - 1;
    double b = P[j];
    int64_t bi = 0;
    for (int64_t r = 1; r < K; ++r) {
      const double v = P[r * N + j];
      if (v < b) {
        b = v;
        bi = r;
      }
    }
    labels[i] = bi;
  }
}

__global__ void k_gather_rows(const double* __restrict__ D, int64_t ld, const int64_t* __restrict__ idx, int64_t K,
                              int64_t N, double* out) {
  const int64_t r = blockIdx.y;
  const double* row = D + idx[r] * ld;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < N; j += (int64_t)gridDim.x * blockDim.x)
    out[r * N + j] = row[j];
}

// ------------------------------------------------------------ key path
// The fast profile pass (launch_mpdist_keys) stores, for every (segment,
// window), the 32-bit key K of the k-th smallest e (high word of its bit
// pattern).  The exact path's value is d* = f(e*) with f = e_to_dist
// (monotone) and e* in the bucket [lo(K), hi(K)] (same tiles and fma order:
// e* is the exact path's own value, not an approximation of it).  Every
// decision below is taken from monotone interval bounds of d* and is
// certified; the ones the bounds cannot decide are resolved with exact
// values (exact profiles of greedy candidates, k_window_exact for single
// windows), so the outputs equal the all-exact pipeline's bit for bit.
__device__ __forceinline__ double e2d(double ev, double twol) {  // == e_to_dist (mpdist.cu)
  if (ev < 1e-15) ev = 0.0;
  if (ev > 2.0) ev = 2.0;
  return sqrt(twol * ev);
}
// exact interval [f(lo(K)), f(hi(K))]; K < 0 <=> e* < 0 <=> d* = 0
__host__ __device__ inline double hilo2d(int hi, unsigned lo) {
  const unsigned long long b = ((unsigned long long)(unsigned)hi << 32) | lo;
  double d;
  memcpy(&d, &b, 8);
  return d;
}
__device__ __forceinline__ void kb_exact(int K, double twol, double& lo, double& hi) {
  if (K < 0) {
    lo = hi = 0.0;
    return;
  }
  lo = e2d(hilo2d(K, 0u), twol);
  hi = e2d(hilo2d(K, 0xffffffffu), twol);
}
constexpr int KEY_TWO = 0x40000000;
constexpr int NEAR_M = 8;  // nearest (key, segment) pairs kept per window on the streamed path  // key of e = 2.0 (rho clip): f is constant from here on
// largest key whose interval can reach below hi(K1): every segment whose key at
// the window is above it is certified farther than the best one
__device__ int near_kthr(int K1, double twol, int K15) {
  double l1, h1, lo, hi;
  kb_exact(K1, twol, l1, h1);
  if (h1 == 0.0) return K15;         // d* = 0 <=> key < K15, and lo(K15) = 0
  if (K1 >= KEY_TWO) return INT_MAX;  // f is constant from the clip on
  int kthr = K1;                      // adjacent buckets differ by ~2^-21 relative in d: a step or two
  for (;;) {
    kb_exact(kthr + 1, twol, lo, hi);
    if (lo > h1) return kthr;
    if (kthr + 1 >= KEY_TWO) return INT_MAX;
    ++kthr;
  }
}

// Cheap outer bounds in fp32 for the greedy area sums: the bucket edges lo(K)
// and lo(K+1) >= hi(K) are exact floats for 2^-126 <= e <= 2; fp32 product and
// sqrt errors (<= 3 ulp = 2^-22.4) are covered by the 2^-20 margins.
// K15 = key of 1e-15 (the snap): below it d* = 0, its bucket straddles it.
__device__ __forceinline__ void kb_fast(int K, float twolf, int K15, double dclip, double& lo, double& hi) {
  if (K < K15) {
    lo = hi = 0.0;
    return;
  }
  if (K >= KEY_TWO) {
    lo = hi = dclip;
    return;
  }
  const float elo = __int_as_float((K - (896 << 20)) << 3);
  const float ehi = __int_as_float((K + 1 - (896 << 20)) << 3);
  lo = (K == K15) ? 0.0 : (double)(__fsqrt_rn(__fmul_rn(twolf, elo)) * (1.0f - 0x1p-20f));
  hi = (double)(__fsqrt_rn(__fmul_rn(twolf, ehi)) * (1.0f + 0x1p-20f));
}

// Greedy-step area bounds, same reduction structure as k_areas (per-thread
// strided fp64 sums + block_sum), so that fp-monotonicity makes
// alo[s] <= area*[s] <= ahi[s] hold for the rounded sums too.
// segs != nullptr: row blockIdx.x holds segment segs[blockIdx.x] (taken/alo/ahi index)
__global__ void __launch_bounds__(256) k_areas_kb(const int* __restrict__ Dk, int64_t N, int64_t ld,
                                                  const double* __restrict__ curve, const uint8_t* __restrict__ taken,
                                                  float twolf, int K15, double dclip, double* alo, double* ahi,
                                                  const int64_t* __restrict__ segs = nullptr) {
  __shared__ double sh[8];
  const int64_t s = segs ? segs[blockIdx.x] : blockIdx.x;
  if (taken[s]) {
    if (threadIdx.x == 0) alo[s] = ahi[s] = PST_INF;
    return;
  }
  const int* row = Dk + blockIdx.x * ld;
  double al = 0.0, ah = 0.0;
  for (int64_t j = threadIdx.x; j < N; j += 256) {
    double lo, hi;
    kb_fast(row[j], twolf, K15, dclip, lo, hi);
    if (curve) {
      const double c = curve[j];
      lo = fmin(lo, c);
      hi = fmin(hi, c);
    }
    al += lo;
    ah += hi;
  }
  const double tl = block_sum<256>(al, sh);
  const double th = block_sum<256>(ah, sh);
  if (threadIdx.x == 0) {
    alo[s] = tl;
    ahi[s] = th;
  }
}

// ---- pruned greedy passes of the streamed key path -------------------------
// Pass 0 keeps, per profile row s and block b of B windows, the smallest key
// Bm[s][b].  A later greedy pass (curve fixed) then has, for every segment,
//   LB[s] = sum_b sum_{j in b} min(curve_j, lo(Bm[s][b])) <= area*[s]
// (lo = kb_fast's lower bound, monotone in the key), and only the segments
// with LB[s] <= (an exact upper bound of the winner's area) are recomputed.
// (also the maximum key of every row, Rx: profile_max candidates)
__global__ void k_block_min(const int* __restrict__ Dk, int64_t rows, int64_t N, int B, int64_t NB,
                            int* __restrict__ Bm, int* __restrict__ Rx) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < rows * NB;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / NB, b = t - r * NB;
    const int* p = Dk + r * N + b * B;
    const int e = (int)((int64_t)B < N - b * B ? (int64_t)B : N - b * B);
    int mn = INT_MAX, mx = INT_MIN;
    for (int i = 0; i < e; ++i) {
      mn = min(mn, p[i]);
      mx = max(mx, p[i]);
    }
    Bm[t] = mn;
    atomicMax(Rx + r, mx);
  }
}
__global__ void k_fill_i32(int* p, int v, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}
// Pass-1 candidate pairs without the key rows: a superset of k_pairs' lists.
// Attribution (mode 0): k_pairs' exact list when the window's near list
// (k_near_keys_acc) is complete, else key(s, j) >= Bm[s][j / B], so Bm > kthr
// excludes s.
// Maximum (mode 1): key(s, j) <= Rx[s], so Rx < thr excludes s.
__global__ void k_pairs_sum(const int* __restrict__ Bm, const int* __restrict__ Rx, int64_t S, int64_t NB, int B,
                            const int* __restrict__ TK, const int32_t* __restrict__ TS, int64_t Nw,
                            const int64_t* __restrict__ wins, int nwin, const int* __restrict__ K1w, int thr,
                            int mode, double twol, int K15, int cap, int64_t* pseg, int64_t* pwin, int* cnt) {
  const int lane = threadIdx.x & 31;
  const int wv = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  if (wv >= nwin) return;
  const int64_t j = wins[wv];
  const int kthr = mode == 0 ? near_kthr(K1w[j], twol, K15) : thr;
  if (mode == 0 && TK[(NEAR_M - 1) * Nw + j] > kthr) {  // the near list holds every key <= kthr: exact pairs
    if (lane < NEAR_M && TK[lane * Nw + j] <= kthr) {
      const int i = atomicAdd(cnt, 1);
      if (i < cap) {
        pseg[i] = TS[lane * Nw + j];
        pwin[i] = j;
      }
    }
    return;
  }
  const int64_t b = j / B;
  for (int64_t s = lane; s < S; s += 32) {
    if (mode == 0 ? Bm[s * NB + b] <= kthr : Rx[s] >= kthr) {
      const int i = atomicAdd(cnt, 1);
      if (i < cap) {
        pseg[i] = s;
        pwin[i] = j;
      }
    }
  }
}
// per block: the curve values sorted ascending (Cs[b*B ..]) and their
// exclusive prefix sums (Cp[b*(B+1) ..], B+1 entries)
constexpr int PRUNE_BMAX = 64;
__global__ void k_curve_blocks(const double* __restrict__ curve, int64_t N, int B, int64_t NB, double* Cs,
                               double* Cp) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < NB; b += (int64_t)gridDim.x * blockDim.x) {
    const int e = (int)((int64_t)B < N - b * B ? (int64_t)B : N - b * B);
    double v[PRUNE_BMAX];
    for (int i = 0; i < e; ++i) {
      const double x = curve[b * B + i];
      int j = i;
      while (j > 0 && v[j - 1] > x) {
        v[j] = v[j - 1];
        --j;
      }
      v[j] = x;
    }
    double acc = 0.0;
    Cp[b * (B + 1)] = 0.0;
    for (int i = 0; i < e; ++i) {
      Cs[b * B + i] = v[i];
      acc += v[i];
      Cp[b * (B + 1) + i + 1] = acc;
    }
  }
}
// LB[s] (taken rows: +inf).  These sums round differently from k_areas', so
// the bound is lowered by 1e-7 relative: an fp64 sum of N non-negative terms
// is within (N-1) * 2^-53 relative of its exact value (1.1e-9 at C4's N = 1e7),
// which covers both sums for N up to ~4e8.
__global__ void __launch_bounds__(256) k_lb(const int* __restrict__ Bm, int64_t NB, int B, int64_t N,
                                            const double* __restrict__ Cs, const double* __restrict__ Cp,
                                            const uint8_t* __restrict__ taken, float twolf, int K15, double dclip,
                                            double* LB) {
  __shared__ double sh[8];
  const int64_t s = blockIdx.x;
  if (taken[s]) {
    if (threadIdx.x == 0) LB[s] = PST_INF;
    return;
  }
  double acc = 0.0;
  for (int64_t b = threadIdx.x; b < NB; b += 256) {
    double lo, hi;
    kb_fast(Bm[s * NB + b], twolf, K15, dclip, lo, hi);
    const int e = (int)((int64_t)B < N - b * B ? (int64_t)B : N - b * B);
    const double* cs = Cs + b * B;
    int a = 0, z = e;  // #(curve values < lo)
    while (a < z) {
      const int mid = (a + z) >> 1;
      if (cs[mid] < lo) a = mid + 1;
      else z = mid;
    }
    acc += Cp[b * (B + 1) + a] + (double)(e - a) * lo;
  }
  const double t = block_sum<256>(acc, sh);
  if (threadIdx.x == 0) LB[s] = t * (1.0 - 1e-7);
}
__global__ void k_set_bounds(const double* __restrict__ LB, int64_t S, double* alo, double* ahi) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < S; s += (int64_t)gridDim.x * blockDim.x) {
    alo[s] = LB[s];
    ahi[s] = PST_INF;
  }
}

// greedy candidates: available s with alo[s] <= min over available of ahi
__global__ void __launch_bounds__(1024) k_greedy_cands(const double* __restrict__ alo, const double* __restrict__ ahi,
                                                       const uint8_t* __restrict__ taken, int64_t S, int cap,
                                                       int64_t* list, int* cnt) {
  __shared__ double wm[32];
  double m = PST_INF;
  for (int64_t s = threadIdx.x; s < S; s += blockDim.x)
    if (!taken[s]) m = fmin(m, ahi[s]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmin(m, __shfl_xor_sync(FULLMASK, m, o));
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
  __syncthreads();
  m = PST_INF;
  for (int v = 0; v < (int)(blockDim.x >> 5); ++v) m = fmin(m, wm[v]);
  for (int64_t s = threadIdx.x; s < S; s += blockDim.x)
    if (!taken[s] && alo[s] <= m) {
      const int i = atomicAdd(cnt, 1);
      if (i < cap) list[i] = s;
    }
}

// Attribution from keys: per window the smallest key K1, its first segment,
// its multiplicity and the next larger key K2; certified iff K1 is unique and
// lo(K2) > hi(K1) (then the first argmin of d* is that segment).  Also the
// per-window maximum key (profile_max candidates).
__global__ void k_near_keys(const int* __restrict__ Dk, int64_t S, int64_t N, int64_t ld, double twol,
                            int32_t* nearest, uint8_t* unc, int* kmaxw, int* K1w) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < N; j += (int64_t)gridDim.x * blockDim.x) {
    int K1 = INT_MAX, K2 = INT_MAX, KM = INT_MIN, n1 = 0;
    int64_t s1 = 0;
    for (int64_t s = 0; s < S; ++s) {
      const int K = Dk[s * ld + j];
      KM = max(KM, K);
      if (K < K1) {
        K2 = K1;
        K1 = K;
        s1 = s;
        n1 = 1;
      } else if (K == K1) {
        ++n1;
      } else {
        K2 = min(K2, K);
      }
    }
    bool ok = n1 == 1;
    if (ok && K2 != INT_MAX) {
      double l1, h1, l2, h2;
      kb_exact(K1, twol, l1, h1);
      kb_exact(K2, twol, l2, h2);
      ok = l2 > h1;
    }
    nearest[j] = (int32_t)s1;
    unc[j] = ok ? 0 : 1;
    kmaxw[j] = KM;
    K1w[j] = K1;
  }
}

// k_near_keys over chunks of segment rows [base, base+rows) arriving in order
// (streamed key path): running smallest key, first segment, multiplicity,
// next key and max key per window; finalize with k_near_finalize.  Also the
// NEAR_M smallest (key, segment) pairs of every window, TK/TS [NEAR_M][N],
// ascending, ties in segment order: a pruned pass 1 takes an uncertain
// window's candidate pairs from them when the list is complete.
__global__ void k_near_keys_acc(const int* __restrict__ Dk, int64_t rows, int64_t N, int64_t ld, int64_t base,
                                int first, int* K1w, int32_t* s1w, int* n1w, int* K2w, int* kmaxw, int* TK,
                                int32_t* TS) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < N; j += (int64_t)gridDim.x * blockDim.x) {
    int K1 = INT_MAX, K2 = INT_MAX, KM = INT_MIN, n1 = 0;
    int64_t s1 = 0;
    int tk[NEAR_M], ts[NEAR_M];
#pragma unroll
    for (int i = 0; i < NEAR_M; ++i) {
      tk[i] = first ? INT_MAX : TK[i * N + j];
      ts[i] = first ? -1 : TS[i * N + j];
    }
    if (!first) {
      K1 = K1w[j];
      K2 = K2w[j];
      KM = kmaxw[j];
      n1 = n1w[j];
      s1 = s1w[j];
    }
    for (int64_t r = 0; r < rows; ++r) {
      const int K = Dk[r * ld + j];
      KM = max(KM, K);
      if (K < K1) {
        K2 = K1;
        K1 = K;
        s1 = base + r;
        n1 = 1;
      } else if (K == K1) {
        ++n1;
      } else {
        K2 = min(K2, K);
      }
      if (K < tk[NEAR_M - 1]) {  // stable insert: after the equal keys already held
        int pos = NEAR_M - 1;
#pragma unroll
        for (int i = NEAR_M - 2; i >= 0; --i)
          if (tk[i] > K) pos = i;
#pragma unroll
        for (int i = NEAR_M - 1; i > 0; --i)
          if (i > pos) {
            tk[i] = tk[i - 1];
            ts[i] = ts[i - 1];
          }
#pragma unroll
        for (int i = 0; i < NEAR_M; ++i)
          if (i == pos) {
            tk[i] = K;
            ts[i] = (int)(base + r);
          }
      }
    }
    K1w[j] = K1;
    K2w[j] = K2;
    kmaxw[j] = KM;
    n1w[j] = n1;
    s1w[j] = (int32_t)s1;
#pragma unroll
    for (int i = 0; i < NEAR_M; ++i) {
      TK[i * N + j] = tk[i];
      TS[i * N + j] = ts[i];
    }
  }
}
__global__ void k_near_finalize(int64_t N, double twol, const int* __restrict__ K1w, const int32_t* __restrict__ s1w,
                                const int* __restrict__ n1w, const int* __restrict__ K2w, int32_t* nearest,
                                uint8_t* unc) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < N; j += (int64_t)gridDim.x * blockDim.x) {
    bool ok = n1w[j] == 1;
    if (ok && K2w[j] != INT_MAX) {
      double l1, h1, l2, h2;
      kb_exact(K1w[j], twol, l1, h1);
      kb_exact(K2w[j], twol, l2, h2);
      ok = l2 > h1;
    }
    nearest[j] = s1w[j];
    unc[j] = ok ? 0 : 1;
  }
}

// windows with a flag set -> compact list (unordered)
__global__ void k_flag_list(const uint8_t* __restrict__ flag, int64_t N, int cap, int64_t* list, int* cnt) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < N; j += (int64_t)gridDim.x * blockDim.x)
    if (flag[j]) {
      const int i = atomicAdd(cnt, 1);
      if (i < cap) list[i] = j;
    }
}
__global__ void k_kmax_flag(const int* __restrict__ kmaxw, int64_t N, int thr, uint8_t* flag) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < N; j += (int64_t)gridDim.x * blockDim.x)
    flag[j] = kmaxw[j] >= thr ? 1 : 0;
}
__global__ void k_max_int(const int* __restrict__ v, int64_t N, int* out) {
  int m = INT_MIN;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < N; j += (int64_t)gridDim.x * blockDim.x)
    m = max(m, v[j]);
  m = __reduce_max_sync(FULLMASK, m);
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// Candidate (segment, window) pairs of listed windows, one warp per window:
// mode 0 (attribution): segments whose lower bound lo(K) <= hi(K1w[j]);
// mode 1 (profile_max): segments with K >= thr.
__global__ void k_pairs(const int* __restrict__ Dk, int64_t S, int64_t ld, int64_t base,
                        const int64_t* __restrict__ wins, int nwin, const int* __restrict__ K1w, int thr, int mode,
                        double twol, int K15, int cap, int64_t* pseg, int64_t* pwin, int* cnt) {
  const int lane = threadIdx.x & 31;
  const int wv = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  if (wv >= nwin) return;
  const int64_t j = wins[wv];
  const int kthr = mode == 0 ? near_kthr(K1w[j], twol, K15) : thr;
  for (int64_t s = lane; s < S; s += 32) {
    const int K = Dk[s * ld + j];
    if (mode == 0 ? K <= kthr : K >= kthr) {
      const int i = atomicAdd(cnt, 1);
      if (i < cap) {
        pseg[i] = base + s;
        pwin[i] = j;
      }
    }
  }
}

__global__ void k_set_nearest(const int64_t* __restrict__ win, const int64_t* __restrict__ seg, int cnt,
                              int32_t* nearest) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < cnt) nearest[win[i]] = (int32_t)seg[i];
}
__global__ void k_mark_taken(uint8_t* taken, int64_t s) { taken[s] = 1; }
__global__ void k_curve_row(double* curve, const double* __restrict__ row, int64_t N) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < N; j += (int64_t)gridDim.x * blockDim.x)
    curve[j] = fmin(curve[j], row[j]);
}

int grid_for(int64_t n, int threads, int cap = 148 * 16) {
  int64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

bool valid(pst_ctx* c) {
  if (!c) {
    pst_set_error("null context");
    return false;
  }
  return true;
}

int need_series(pst_ctx* c) {
  if (c->n <= 0) {
    pst_set_error("no series uploaded (call pst_set_series first)");
    return PST_ESTATE;
  }
  return PST_OK;
}

}  // namespace

int pst_ensure_len(pst_ctx* c, int64_t l) {
  PST_TRY(need_series(c));
  if (l < 1 || l > c->n) {
    pst_set_error("window length %lld out of range [1, %lld]", (long long)l, (long long)c->n);
    return PST_EINVAL;
  }
  if (c->L.l == l) return PST_OK;
  const int64_t Nl = c->n - l + 1;
  if (Nl > c->cap_l) {
    double** arrs[] = {&c->L.mu, &c->L.var, &c->L.sd, &c->L.nrm, &c->L.bias, &c->L.cbias, &c->L.df, &c->L.dg, &c->L.mc,
                       (double**)&c->L.hash};
    for (double** a : arrs) {
      if (*a) cudaFree(*a);
      *a = nullptr;
      cudaError_t e = cudaMalloc((void**)a, (size_t)(Nl + 1) * sizeof(double));
      if (e != cudaSuccess) {
        cudaGetLastError();
        pst_set_error("device allocation for window statistics failed: %s", cudaGetErrorString(e));
        c->cap_l = 0;
        c->L.l = -1;
        return PST_ENOMEM;
      }
    }
    c->cap_l = Nl;
  }
  k_stats<<<grid_for(Nl, 256), 256, 0, c->st>>>(c->x, c->csum, c->csq, c->chg, c->n, l, c->L);
  k_dfdg<<<grid_for(Nl, 256), 256, 0, c->st>>>(c->x, c->n, l, c->L);
  k_hash<<<grid_for(Nl, 256), 256, 0, c->st>>>(c->x, c->n, l, c->L.hash);
  c->launches += 3;
  PST_CUDA(cudaGetLastError());
  {  // any two equal window hashes?  (sorted copy, adjacent compare); if none, no exact repeat exists
    size_t tmp = 0;
    PST_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, (const unsigned long long*)nullptr,
                                            (unsigned long long*)nullptr, (int)Nl, 0, 64, c->st));
    const size_t kb = ((size_t)Nl * 8 + 255) & ~(size_t)255;
    PST_TRY(pst_ensure(&c->aux, &c->aux_bytes, kb + 256 + tmp));
    unsigned long long* sorted = (unsigned long long*)c->aux;
    int* flag = (int*)((char*)c->aux + kb);
    void* tmpp = (char*)c->aux + kb + 256;
    PST_CUDA(cub::DeviceRadixSort::SortKeys(tmpp, tmp, c->L.hash, sorted, (int)Nl, 0, 64, c->st));
    PST_CUDA(cudaMemsetAsync(flag, 0, 4, c->st));
    k_adjacent_equal<<<grid_for(Nl, 256), 256, 0, c->st>>>(sorted, Nl, flag);
    c->launches += 2;
    int h = 0;
    PST_CUDA(cudaMemcpyAsync(&h, flag, 4, cudaMemcpyDeviceToHost, c->st));
    PST_CUDA(cudaStreamSynchronize(c->st));
    c->L.has_rep = h != 0;
  }
  c->L.l = l;
  c->L.Nl = Nl;
  return PST_OK;
}

// ================================================================== C-ABI
extern "C" {

const char* pst_last_error(void) { return g_err.c_str(); }

int pst_device_count(int* out) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    cudaGetLastError();
    *out = 0;
    pst_set_error("cudaGetDeviceCount: %s", cudaGetErrorString(e));
    return PST_ECUDA;
  }
  *out = n;
  return PST_OK;
}

int pst_create(int device, pst_ctx** out) {
  *out = nullptr;
  int nd = 0;
  PST_TRY(pst_device_count(&nd));
  if (device < 0 || device >= nd) {
    pst_set_error("device %d out of range [0, %d)", device, nd);
    return PST_EINVAL;
  }
  PST_CUDA(cudaSetDevice(device));
  pst_ctx* c = new pst_ctx();
  c->dev = device;
  cudaError_t e = cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete c;
    pst_set_error("cudaStreamCreate: %s", cudaGetErrorString(e));
    return PST_ECUDA;
  }
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  int optin = 0;
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  c->smem_optin = (size_t)optin;
  *out = c;
  return PST_OK;
}

int pst_destroy(pst_ctx* c) {
  if (!c) return PST_OK;
  cudaSetDevice(c->dev);
  cudaStreamSynchronize(c->st);
  pst_comm_destroy(c);
  void* ptrs[] = {c->x, c->csum, c->csq, c->chg, c->L.mu, c->L.var, c->L.sd, c->L.nrm, c->L.bias,
                  c->L.cbias, c->L.df, c->L.dg, c->L.mc, c->scratch, c->D, c->work, c->dbg, c->Dk, c->cert,
                  c->L.hash, c->aux, c->prune};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (c->st2) {
    cudaStreamSynchronize(c->st2);
    for (int bi = 0; bi < 2; ++bi) {
      cudaEventDestroy(c->ev_rows[bi]);
      cudaEventDestroy(c->ev_sel[bi]);
    }
    cudaStreamDestroy(c->st2);
  }
  cudaStreamDestroy(c->st);
  delete c;
  return PST_OK;
}

static int set_series_common(pst_ctx* c, const double* x, int64_t n, cudaMemcpyKind kind) {
  if (!valid(c)) return PST_EINVAL;
  if (n < 2) {
    pst_set_error("series needs at least 2 samples, got %lld", (long long)n);
    return PST_EINVAL;
  }
  PST_CUDA(cudaSetDevice(c->dev));
  if (n > c->cap_n) {
    void** arrs[] = {(void**)&c->x, (void**)&c->csum, (void**)&c->csq, (void**)&c->chg};
    for (void** a : arrs) {
      if (*a) cudaFree(*a);
      *a = nullptr;
    }
    c->cap_n = 0;
    size_t cap = 0;
    PST_TRY(pst_ensure((void**)&c->x, &cap, (size_t)(n + 8) * sizeof(double)));  // padded: 16-byte bulk copies
    cap = 0;
    PST_TRY(pst_ensure((void**)&c->csum, &cap, (size_t)(n + 1) * sizeof(double)));
    cap = 0;
    PST_TRY(pst_ensure((void**)&c->csq, &cap, (size_t)(n + 1) * sizeof(double)));
    cap = 0;
    PST_TRY(pst_ensure((void**)&c->chg, &cap, (size_t)(n + 1) * sizeof(int64_t)));
    c->cap_n = n;
  }
  PST_CUDA(cudaMemcpyAsync(c->x, x, (size_t)n * sizeof(double), kind, c->st));
  c->n = n;
  c->L.l = -1;
  k_prefix<<<1, 256, 0, c->st>>>(c->x, n, c->csum, c->csq, c->chg);
  c->launches++;
  PST_CUDA(cudaGetLastError());
  return PST_OK;
}

int pst_set_series(pst_ctx* c, const double* x, int64_t n) {
  return set_series_common(c, x, n, cudaMemcpyHostToDevice);
}

int pst_set_series_dev(pst_ctx* c, const double* x, int64_t n) {
  return set_series_common(c, x, n, cudaMemcpyDeviceToDevice);
}

int pst_sync(pst_ctx* c) {
  if (!valid(c)) return PST_EINVAL;
  PST_CUDA(cudaStreamSynchronize(c->st));
  return PST_OK;
}

int64_t pst_launch_count(pst_ctx* c) { return c ? c->launches : -1; }

int pst_sliding_stats(pst_ctx* c, int64_t l, double* means, double* stds, double* vars) {
  if (!valid(c)) return PST_EINVAL;
  PST_CUDA(cudaSetDevice(c->dev));
  PST_TRY(pst_ensure_len(c, l));
  const size_t b = (size_t)c->L.Nl * sizeof(double);
  if (means) PST_CUDA(cudaMemcpyAsync(means, c->L.mu, b, cudaMemcpyDeviceToHost, c->st));
  if (stds) PST_CUDA(cudaMemcpyAsync(stds, c->L.sd, b, cudaMemcpyDeviceToHost, c->st));
  if (vars) PST_CUDA(cudaMemcpyAsync(vars, c->L.var, b, cudaMemcpyDeviceToHost, c->st));
  PST_CUDA(cudaStreamSynchronize(c->st));
  return PST_OK;
}

int pst_distance_rows(pst_ctx* c, int64_t l, int64_t q0, int64_t rows, int method, double* out) {
  if (!valid(c)) return PST_EINVAL;
  PST_CUDA(cudaSetDevice(c->dev));
  PST_TRY(pst_ensure_len(c, l));
  const int64_t Nl = c->n - l + 1;
  if (rows < 1 || q0 < 0 || q0 + rows > Nl) {
    pst_set_error("query window [%lld, %lld) is outside a series of length %lld", (long long)(q0 + rows - 1),
                  (long long)(q0 + rows - 1 + l), (long long)c->n);
    return PST_EINVAL;
  }
  const size_t bytes = (size_t)rows * Nl * sizeof(double);
  PST_TRY(pst_ensure(&c->work, &c->work_bytes, bytes));
  double* d = (double*)c->work;
  if (method == 0) {
    const int64_t nd = Nl + rows - 1;
    k_rows<<<(unsigned)((nd + 255) / 256), 256, 0, c->st>>>(c->x, c->L, c->n, l, q0, rows, d);
  } else if (method == 1) {
    dim3 g((unsigned)((Nl + 255) / 256), (unsigned)rows);
    k_rows_direct<<<g, 256, 0, c->st>>>(c->x, c->n, l, q0, rows, d);
  } else {
    pst_set_error("unknown method %d, expected 0 (sliding) or 1 (direct)", method);
    return PST_EINVAL;
  }
  c->launches++;
  PST_CUDA(cudaGetLastError());
  PST_CUDA(cudaMemcpyAsync(out, d, bytes, cudaMemcpyDeviceToHost, c->st));
  PST_CUDA(cudaStreamSynchronize(c->st));
  return PST_OK;
}

static int check_mkl(pst_ctx* c, int64_t m, int64_t l, int64_t k) {
  PST_TRY(need_series(c));
  if (m < 2) {
    pst_set_error("snippet size must be at least 2, got %lld", (long long)m);
    return PST_EINVAL;
  }
  if (m > c->n) {
    pst_set_error("snippet size %lld exceeds series length %lld", (long long)m, (long long)c->n);
    return PST_EINVAL;
  }
  if (l < 1 || l > m) {
    pst_set_error("window size %lld out of range [1, %lld]", (long long)l, (long long)m);
    return PST_EINVAL;
  }
  if (k < 1) {
    pst_set_error("order statistic must be at least 1, got %lld", (long long)k);
    return PST_EINVAL;
  }
  return PST_OK;
}

int pst_profiles_dev(pst_ctx* c, int64_t m, int64_t l, int64_t k, int64_t seg_lo, int64_t seg_hi, double* D_dev,
                     int64_t ld) {
  if (!valid(c)) return PST_EINVAL;
  PST_CUDA(cudaSetDevice(c->dev));
  PST_TRY(check_mkl(c, m, l, k));
  const int64_t S = c->n / m;
  if (seg_lo < 0 || seg_hi > S || seg_lo >= seg_hi) {
    pst_set_error("segment index %lld out of range [0, %lld)", (long long)(seg_lo < 0 ? seg_lo : seg_hi - 1),
                  (long long)S);
    return PST_EINVAL;
  }
  if (ld < c->n - m + 1) {
    pst_set_error("row stride %lld smaller than the window count %lld", (long long)ld, (long long)(c->n - m + 1));
    return PST_EINVAL;
  }
  return launch_mpdist(c, m, l, k, seg_lo, seg_hi, D_dev, ld);
}

int pst_mpdist_profiles(pst_ctx* c, int64_t m, int64_t l, int64_t k, int64_t seg_lo, int64_t seg_hi, double* out) {
  if (!valid(c)) return PST_EINVAL;
  PST_CUDA(cudaSetDevice(c->dev));
  PST_TRY(check_mkl(c, m, l, k));
  const int64_t N = c->n - m + 1;
  const size_t bytes = (size_t)(seg_hi - seg_lo) * N * sizeof(double);
  PST_TRY(pst_ensure((void**)&c->D, &c->D_bytes, bytes > 0 ? bytes : 8));
  PST_TRY(pst_profiles_dev(c, m, l, k, seg_lo, seg_hi, c->D, N));
  PST_CUDA(cudaMemcpyAsync(out, c->D, bytes, cudaMemcpyDeviceToHost, c->st));
  PST_CUDA(cudaStreamSynchronize(c->st));
  return PST_OK;
}

int pst_areas_dev(pst_ctx* c, const double* D, int64_t rows, int64_t N, int64_t ld, const double* curve,
                  double* areas) {
  if (!valid(c)) return PST_EINVAL;
  if (rows <= 0) return PST_OK;
  k_areas<<<(unsigned)rows, 256, 0, c->st>>>(D, N, ld, curve, areas);
  c->launches++;
  PST_CUDA(cudaGetLastError());
  return PST_OK;
}

// max over rows x N of a device matrix (profile_max of a rank's rows, snippets.py:241); out_dev: 1 double
int pst_max_dev(pst_ctx* c, const double* D, int64_t rows, int64_t N, int64_t ld, double* out_dev) {
  if (!valid(c)) return PST_EINVAL;
  PST_CUDA(cudaMemsetAsync(out_dev, 0, 8, c->st));
  if (rows > 0) {
    dim3 g((unsigned)grid_for(N, 256, 64), (unsigned)std::min<int64_t>(rows, 64));
    k_max<<<g, 256, 0, c->st>>>(D, rows, N, ld, (unsigned long long*)out_dev);
    c->launches++;
    PST_CUDA(cudaGetLastError());
  }
  return PST_OK;
}

int pst_colmin_dev(pst_ctx* c, const double* D, int64_t rows, int64_t N, int64_t ld, int64_t base, double* minval,
                   int32_t* arg) {
  if (!valid(c)) return PST_EINVAL;
  if (rows <= 0) return PST_OK;
  k_colmin<<<grid_for(N, 256), 256, 0, c->st>>>(D, rows, N, ld, base, minval, arg);
  c->launches++;
  PST_CUDA(cudaGetLastError());
  return PST_OK;
}

static int run_select(pst_ctx* c, const double* D, int64_t S, int64_t N, int64_t n, int64_t K,
                      pst_snippets* res);
static int run_select_streamed(pst_ctx* c, int64_t m, int64_t l, int64_t k, int64_t S, int64_t N, int64_t n,
                               int64_t K, int64_t chunk, pst_snippets* res);

// Rows of D that fit the device next to the profile-kernel scratch; the
// whole S x N matrix when it fits (PASTILA_STREAM_ROWS forces a chunk size).
static int64_t profile_chunk_rows(pst_ctx* c, int64_t S, int64_t N, int64_t w) {
  if (const char* e = getenv("PASTILA_STREAM_ROWS")) {
    const int64_t v = atoll(e);
    if (v >= 1 && v < S) return v;
  }
  size_t fr = 0, tot = 0;
  if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) return S;
  const size_t have = fr + c->D_bytes;  // D is reallocated in place
  // profile-kernel scratch: two buffers of at least one segment's AB tiles (w x Tp per tile, Tp <= 1.1 T)
  // plus column minima, or 2 x 6 GB; work buffers; slack
  const size_t seg_scratch = (size_t)N * 8 * (size_t)(w + w / 10 + 2);
  const size_t reserve = std::max((size_t)12 << 30, 2 * seg_scratch) + (size_t)N * 8 * 16 + ((size_t)2 << 30);
  if (have <= reserve) return 1;
  const int64_t rows = (int64_t)((have - reserve) / ((size_t)N * 8));
  return rows >= S ? S : (rows < 1 ? 1 : rows);
}

// Profiles of segments [seg_lo, seg_hi) computed chunk by chunk and reduced
// without keeping them: areas_dev[s - seg_lo] = sum_j min(D[s][j], curve[j])
// (curve NULL: plain sums); optional running per-window minimum + first
// argmin (segment index; caller initialises minval to +inf) and running max
// (caller initialises *rowmax_dev to 0 as unsigned 64-bit bits).
int pst_profile_reduce_dev(pst_ctx* c, int64_t m, int64_t l, int64_t k, int64_t seg_lo, int64_t seg_hi,
                           const double* curve_dev, double* areas_dev, double* minval_dev, int32_t* argmin_dev,
                           double* rowmax_dev) {
  if (!valid(c)) return PST_EINVAL;
  PST_CUDA(cudaSetDevice(c->dev));
  PST_TRY(check_mkl(c, m, l, k));
  const int64_t S = c->n / m, N = c->n - m + 1;
  if (seg_lo < 0 || seg_hi > S || seg_lo >= seg_hi) {
    pst_set_error("segment index %lld out of range [0, %lld)", (long long)(seg_lo < 0 ? seg_lo : seg_hi - 1),
                  (long long)S);
    return PST_EINVAL;
  }
  int64_t chunk = profile_chunk_rows(c, seg_hi - seg_lo, N, m - l + 1);
  PST_TRY(pst_ensure((void**)&c->D, &c->D_bytes, (size_t)chunk * N * sizeof(double)));
  for (int64_t s0 = seg_lo; s0 < seg_hi; s0 += chunk) {
    const int64_t rows = std::min(chunk, seg_hi - s0);
    PST_TRY(launch_mpdist(c, m, l, k, s0, s0 + rows, c->D, N));
    k_areas<<<(unsigned)rows, 256, 0, c->st>>>(c->D, N, N, curve_dev, areas_dev + (s0 - seg_lo));
    c->launches++;
    if (minval_dev && argmin_dev) {
      k_colmin_acc<<<grid_for(N, 256), 256, 0, c->st>>>(c->D, rows, N, N, s0, minval_dev, argmin_dev);
      c->launches++;
    }
    if (rowmax_dev) {
      dim3 g((unsigned)grid_for(N, 256, 64), (unsigned)std::min<int64_t>(rows, 64));
      k_max<<<g, 256, 0, c->st>>>(c->D, rows, N, N, (unsigned long long*)rowmax_dev);
      c->launches++;
    }
    PST_CUDA(cudaGetLastError());
  }
  return PST_OK;
}

static int run_select_keys(pst_ctx* c, const int* Dk, int64_t m, int64_t l, int64_t k, int64_t S, int64_t N,
                           int64_t n, int64_t K, pst_snippets* res);

// Key path (launch_mpdist_keys + certified selection) when the S x N key matrix
// fits next to the profile-kernel scratch; PASTILA_EXACT=1 forces the exact
// path (A/B and parity tests), PASTILA_STREAM_ROWS the streamed exact path.
static bool use_keys(pst_ctx* c, int64_t S, int64_t N, int64_t w) {
  if (const char* e = getenv("PASTILA_EXACT"))
    if (atoi(e) > 0) return false;
  if (getenv("PASTILA_STREAM_ROWS")) return false;
  size_t fr = 0, tot = 0;
  if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) return false;
  const size_t have = fr + c->Dk_bytes + c->D_bytes;
  // profile-kernel scratch of the exact single-segment profiles of greedy candidates (f64 AB tiles, two buffers)
  const size_t seg_scratch = (size_t)N * 8 * (size_t)(w + w / 10 + 2);
  const size_t reserve = std::max((size_t)8 << 30, 2 * seg_scratch) + (size_t)N * 8 * (24 + 16) + ((size_t)3 << 30);
  return have > reserve && (size_t)S * N * sizeof(int) <= have - reserve;
}

struct PruneBufs {
  int* Bm = nullptr;  // [S][NB] per-block minimum keys
  double *Cs = nullptr, *Cp = nullptr, *LB = nullptr;
  int64_t* segl = nullptr;  // [S] segments to recompute
  int* Rx = nullptr;        // [S] maximum key of every row
  int B = 0;
  int64_t NB = 0;
};
static int run_select_keys_streamed(pst_ctx* c, int64_t m, int64_t l, int64_t k, int64_t S, int64_t N,
                                    int64_t n, int64_t K, int64_t chunk, const PruneBufs& pb, pst_snippets* res);
static int prune_alloc(pst_ctx* c, int64_t S, int64_t N, int64_t K, PruneBufs& pb);
static void prune_free(pst_ctx* c);

// Streamed key path: the key matrix does not fit (or PASTILA_STREAM_KEYS forces it).
static bool use_keys_streamed(pst_ctx* c, int64_t S, int64_t N, int64_t w) {
  if (const char* e = getenv("PASTILA_EXACT"))
    if (atoi(e) > 0) return false;
  if (getenv("PASTILA_STREAM_ROWS")) return false;
  if (getenv("PASTILA_STREAM_KEYS")) return true;
  return !use_keys(c, S, N, w);
}
// segments of keys per chunk: the free memory after the scratch reserve, at most S
static int64_t key_chunk_rows(pst_ctx* c, int64_t S, int64_t N, int64_t w) {
  size_t fr = 0, tot = 0;
  if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) return 1;
  const size_t have = fr + c->Dk_bytes + c->D_bytes;
  // profile-kernel scratch of the exact single-segment profiles of greedy candidates (f64 AB tiles, two buffers)
  const size_t seg_scratch = (size_t)N * 8 * (size_t)(w + w / 10 + 2);
  const size_t reserve = std::max((size_t)12 << 30, 2 * seg_scratch) + (size_t)N * 8 * (24 + 16 + 8) +
                         ((size_t)4 << 30);
  if (have <= reserve) return 1;
  const int64_t rows = (int64_t)((have - reserve) / ((size_t)N * sizeof(int)));
  return rows >= S ? S : (rows < 1 ? 1 : rows);
}

int pst_select_snippets(pst_ctx* c, int64_t m, int64_t l, int64_t k, int64_t K, pst_snippets* res) {
  if (!valid(c)) return PST_EINVAL;
  PST_CUDA(cudaSetDevice(c->dev));
  PST_TRY(check_mkl(c, m, l, k));
  const int64_t n = c->n, S = n / m, N = n - m + 1;
  if (S < 2) {
    pst_set_error("snippet size %lld leaves only %lld segment(s) of a series of length %lld; need at least 2",
                  (long long)m, (long long)S, (long long)n);
    return PST_EINVAL;
  }
  if (K < 1 || K > S) {
    pst_set_error("snippet count %lld out of range [1, %lld]", (long long)K, (long long)S);
    return PST_EINVAL;
  }
  if (use_keys_streamed(c, S, N, m - l + 1)) {  // key matrix does not fit: streamed key path
    if (c->D) {  // the exact matrix is not needed on this path
      cudaFree(c->D);
      c->D = nullptr;
      c->D_bytes = 0;
    }
    PruneBufs pb;  // block minima first: the key chunk is sized from what is left
    int r = prune_alloc(c, S, N, K, pb);
    if (r == PST_OK) {
      const char* sk = getenv("PASTILA_STREAM_KEYS");
      const int64_t chunk = sk ? std::max<int64_t>(1, atoll(sk)) : key_chunk_rows(c, S, N, m - l + 1);
      r = run_select_keys_streamed(c, m, l, k, S, N, n, K, chunk, pb, res);
    }
    prune_free(c);
    if (r != 1) return r;
    c->cert_stats[6]++;  // a certification cap was exceeded: recompute this length exactly
  } else if (use_keys(c, S, N, m - l + 1)) {
    if (c->D) {  // the exact matrix is not needed on this path
      cudaFree(c->D);
      c->D = nullptr;
      c->D_bytes = 0;
    }
    PST_TRY(pst_ensure((void**)&c->Dk, &c->Dk_bytes, (size_t)S * N * sizeof(int)));
    PST_TRY(launch_mpdist_keys(c, m, l, k, 0, S, c->Dk, N));
    const int r = run_select_keys(c, c->Dk, m, l, k, S, N, n, K, res);
    if (r != 1) return r;
    c->cert_stats[6]++;  // a certification cap was exceeded: recompute this length exactly
  }
  if (c->Dk) {
    cudaFree(c->Dk);
    c->Dk = nullptr;
    c->Dk_bytes = 0;
  }
  const int64_t chunk = profile_chunk_rows(c, S, N, m - l + 1);
  if (chunk < S) return run_select_streamed(c, m, l, k, S, N, n, K, chunk, res);
  PST_TRY(pst_ensure((void**)&c->D, &c->D_bytes, (size_t)S * N * sizeof(double)));
  PST_TRY(launch_mpdist(c, m, l, k, 0, S, c->D, N));
  return run_select(c, c->D, S, N, n, K, res);
}

// select_length (length_select.py:116-182) through the C-ABI: one search per
// grid length in grid order (l = ls[i], or ceil(m/2) when ls is NULL; k is the
// default ceil(m/10), length_select.py:163), Eq. 18 score per length, and
// m_best = argmax (score, -m).  Outputs: indices/fracs [nm*K] (frac order),
// scores/areas [nm], *m_best.
int pst_sweep(pst_ctx* c, const int64_t* ms, const int64_t* ls, int64_t nm, int64_t K, int64_t* indices,
              double* fracs, double* scores, double* areas, int64_t* m_best) {
  if (!valid(c)) return PST_EINVAL;
  if (nm < 1 || !ms) {
    pst_set_error("length grid is empty");
    return PST_EINVAL;
  }
  for (int64_t i = 0; i < nm; ++i)
    for (int64_t j = 0; j < i; ++j)
      if (ms[i] == ms[j]) {
        pst_set_error("length grid has duplicates: m=%lld", (long long)ms[i]);
        return PST_EINVAL;
      }
  if (K < 2) {
    pst_set_error("length selection needs at least 2 snippets per search, got %lld", (long long)K);
    return PST_EINVAL;
  }
  int64_t best = -1;
  double best_score = 0.0;
  for (int64_t i = 0; i < nm; ++i) {
    const int64_t m = ms[i];
    const int64_t l = ls ? ls[i] : (m + 1) / 2;
    const int64_t k = (m + 9) / 10 > 1 ? (m + 9) / 10 : 1;
    pst_snippets r;
    memset(&r, 0, sizeof(r));
    r.indices = indices ? indices + i * K : nullptr;
    r.fracs = fracs ? fracs + i * K : nullptr;
    PST_TRY(pst_select_snippets(c, m, l, k, K, &r));
    if (scores) scores[i] = r.criterion;
    if (areas) areas[i] = r.profile_area;
    if (best < 0 || r.criterion > best_score || (r.criterion == best_score && m < ms[best])) {
      best = i;
      best_score = r.criterion;
    }
  }
  if (m_best) *m_best = ms[best];
  return PST_OK;
}

// select_snippets(..., profiles=...) (snippets.py:191-196): greedy + attribution on
// caller-supplied host profiles D [S*N].
int pst_select_from_profiles(pst_ctx* c, const double* Dh, int64_t S, int64_t N, int64_t n, int64_t K,
                             pst_snippets* res) {
  if (!valid(c)) return PST_EINVAL;
  PST_CUDA(cudaSetDevice(c->dev));
  if (S < 1 || N < 1 || n < N || K < 1 || K > S) {
    pst_set_error("snippet count %lld out of range [1, %lld]", (long long)K, (long long)S);
    return PST_EINVAL;
  }
  PST_TRY(pst_ensure((void**)&c->D, &c->D_bytes, (size_t)S * N * sizeof(double)));
  PST_CUDA(cudaMemcpyAsync(c->D, Dh, (size_t)S * N * sizeof(double), cudaMemcpyHostToDevice, c->st));
  return run_select(c, c->D, S, N, n, K, res);
}

// Device work buffers of one selection.
struct SelBufs {
  double *curve, *areas, *prof, *pair, *nearval, *rows;
  uint8_t* taken;
  int64_t *best, *labels, *ord, *zero;
  unsigned long long *counts, *dmax;
  int32_t* nearest;
};

static int sel_bufs(pst_ctx* c, int64_t S, int64_t N, int64_t n, int64_t K, bool streamed, SelBufs& b) {
  const int64_t npair = K * (K - 1) / 2;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 255) & ~(size_t)255;
    return o;
  };
  const size_t o_curve = take(N * 8), o_areas = take(S * 8), o_taken = take(S), o_best = take(K * 8),
               o_counts = take(S * 8), o_near = take(N * 4), o_prof = take(K * N * 8), o_lab = take(n * 8),
               o_pair = take((npair + 1) * 8), o_max = take(8), o_ord = take(K * 8), o_zero = take(8),
               o_nv = streamed ? take(N * 8) : 0, o_rows = streamed ? take(K * N * 8) : 0;
  PST_TRY(pst_ensure(&c->work, &c->work_bytes, off));
  char* wb = (char*)c->work;
  b.curve = (double*)(wb + o_curve);
  b.areas = (double*)(wb + o_areas);
  b.taken = (uint8_t*)(wb + o_taken);
  b.best = (int64_t*)(wb + o_best);
  b.counts = (unsigned long long*)(wb + o_counts);
  b.nearest = (int32_t*)(wb + o_near);
  b.prof = (double*)(wb + o_prof);
  b.labels = (int64_t*)(wb + o_lab);
  b.pair = (double*)(wb + o_pair);
  b.dmax = (unsigned long long*)(wb + o_max);
  b.ord = (int64_t*)(wb + o_ord);
  b.zero = (int64_t*)(wb + o_zero);
  b.nearval = streamed ? (double*)(wb + o_nv) : nullptr;
  b.rows = streamed ? (double*)(wb + o_rows) : nullptr;
  return PST_OK;
}

// Common tail: counts, (-frac, index) ordering, ordered profiles, labels,
// criterion pair sums, curve area and the host copies.  src/ld/src_row[step]
// locate the chosen profiles (rows of D, or the streamed row buffer).
static int finish_select(pst_ctx* c, SelBufs& b, int64_t S, int64_t N, int64_t n, int64_t K, const double* src,
                         const std::vector<int64_t>& src_row, pst_snippets* res) {
  const int64_t npair = K * (K - 1) / 2;
  PST_CUDA(cudaMemsetAsync(b.counts, 0, S * 8, c->st));
  k_count<<<grid_for(N, 256), 256, 0, c->st>>>(b.nearest, N, b.counts);
  c->launches++;
  PST_CUDA(cudaGetLastError());
  // host: chosen order by (-frac, index)  (snippets.py:228)
  std::vector<int64_t> chosen(K);
  std::vector<unsigned long long> hcounts(S);
  unsigned long long hmax = 0;
  PST_CUDA(cudaMemcpyAsync(chosen.data(), b.best, K * 8, cudaMemcpyDeviceToHost, c->st));
  PST_CUDA(cudaMemcpyAsync(hcounts.data(), b.counts, S * 8, cudaMemcpyDeviceToHost, c->st));
  PST_CUDA(cudaMemcpyAsync(&hmax, b.dmax, 8, cudaMemcpyDeviceToHost, c->st));
  PST_CUDA(cudaStreamSynchronize(c->st));
  std::vector<int64_t> order(K);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t bb) {
    const double fa = (double)hcounts[chosen[a]] / (double)N, fb = (double)hcounts[chosen[bb]] / (double)N;
    if (fa != fb) return fa > fb;
    return chosen[a] < chosen[bb];
  });
  std::vector<int64_t> ordidx(K), ordsrc(K);
  for (int64_t r = 0; r < K; ++r) {
    ordidx[r] = chosen[order[r]];
    ordsrc[r] = src_row[order[r]];
  }
  PST_CUDA(cudaMemcpyAsync(b.ord, ordsrc.data(), K * 8, cudaMemcpyHostToDevice, c->st));
  {
    dim3 g((unsigned)grid_for(N, 256, 256), (unsigned)K);
    k_gather_rows<<<g, 256, 0, c->st>>>(src, N, b.ord, K, N, b.prof);
    c->launches++;
  }
  if (res->labels) {
    k_labels<<<grid_for(n, 256), 256, 0, c->st>>>(b.prof, K, N, n, b.labels);
    c->launches++;
  }
  if (npair > 0) {
    k_pairdiff<<<(unsigned)npair, 256, 0, c->st>>>(b.prof, N, K, b.pair);
    c->launches++;
  }
  // curve area: deterministic device sum
  k_areas<<<1, 256, 0, c->st>>>(b.curve, N, N, nullptr, b.areas);
  c->launches++;
  PST_CUDA(cudaGetLastError());
  double area = 0.0;
  std::vector<double> hpair(npair > 0 ? npair : 1);
  PST_CUDA(cudaMemcpyAsync(&area, b.areas, 8, cudaMemcpyDeviceToHost, c->st));
  if (npair > 0) PST_CUDA(cudaMemcpyAsync(hpair.data(), b.pair, npair * 8, cudaMemcpyDeviceToHost, c->st));
  if (res->curve) PST_CUDA(cudaMemcpyAsync(res->curve, b.curve, N * 8, cudaMemcpyDeviceToHost, c->st));
  if (res->profiles) PST_CUDA(cudaMemcpyAsync(res->profiles, b.prof, K * N * 8, cudaMemcpyDeviceToHost, c->st));
  if (res->nearest) PST_CUDA(cudaMemcpyAsync(res->nearest, b.nearest, N * 4, cudaMemcpyDeviceToHost, c->st));
  if (res->labels) PST_CUDA(cudaMemcpyAsync(res->labels, b.labels, n * 8, cudaMemcpyDeviceToHost, c->st));
  PST_CUDA(cudaStreamSynchronize(c->st));
  res->profile_area = area;
  double pm;
  memcpy(&pm, &hmax, 8);
  res->profile_max = pm;
  double tot = 0.0;
  for (int64_t p = 0; p < npair; ++p) tot += hpair[p];  // itertools.combinations order
  res->criterion = (K < 2 || pm == 0.0) ? 0.0 : tot / pm;
  int64_t covered = 0;
  for (int64_t r = 0; r < K; ++r) {
    if (res->indices) res->indices[r] = ordidx[r];
    if (res->fracs) res->fracs[r] = (double)hcounts[ordidx[r]] / (double)N;
    covered += (int64_t)hcounts[ordidx[r]];
  }
  if (res->counts)
    for (int64_t s = 0; s < S; ++s) res->counts[s] = (int64_t)hcounts[s];
  res->unassigned = N - covered;
  return PST_OK;
}

// Greedy + attribution on the resident S x N matrix D.
static int run_select(pst_ctx* c, const double* D, int64_t S, int64_t N, int64_t n, int64_t K,
                      pst_snippets* res) {
  SelBufs b;
  PST_TRY(sel_bufs(c, S, N, n, K, false, b));
  // profile_max
  PST_CUDA(cudaMemsetAsync(b.dmax, 0, 8, c->st));
  {
    dim3 g((unsigned)grid_for(N, 256, 64), (unsigned)std::min<int64_t>(S, 64));
    k_max<<<g, 256, 0, c->st>>>(D, S, N, N, b.dmax);
    c->launches++;
  }
  // greedy (snippets.py:201-210)
  PST_CUDA(cudaMemsetAsync(b.taken, 0, S, c->st));
  k_fill<<<grid_for(N, 256), 256, 0, c->st>>>(b.curve, HUGE_VAL, N);
  c->launches++;
  for (int64_t step = 0; step < K; ++step) {
    k_areas<<<(unsigned)S, 256, 0, c->st>>>(D, N, N, step == 0 ? nullptr : b.curve, b.areas);
    k_pick<<<1, 1024, 0, c->st>>>(b.areas, b.taken, S, b.best + step);
    k_curve<<<grid_for(N, 256), 256, 0, c->st>>>(b.curve, D, N, b.best + step, N);
    c->launches += 3;
  }
  PST_CUDA(cudaGetLastError());
  // attribution (snippets.py:212-213)
  k_colmin<<<grid_for(N, 256), 256, 0, c->st>>>(D, S, N, N, 0, nullptr, b.nearest);
  c->launches++;
  std::vector<int64_t> chosen(K);
  PST_CUDA(cudaMemcpyAsync(chosen.data(), b.best, K * 8, cudaMemcpyDeviceToHost, c->st));
  PST_CUDA(cudaStreamSynchronize(c->st));
  return finish_select(c, b, S, N, n, K, D, chosen, res);
}

// Same greedy when S x N does not fit the device (C4: n = 1e7): profiles are
// recomputed chunk by chunk for every greedy round and reduced on the fly
// (pst_profile_reduce_dev); only the K chosen rows are kept.  The first pass
// also produces the attribution minima and profile_max.  Profiles do not
// depend on the chunking, so the result is identical to the resident path.
static int run_select_streamed(pst_ctx* c, int64_t m, int64_t l, int64_t k, int64_t S, int64_t N, int64_t n,
                               int64_t K, int64_t chunk, pst_snippets* res) {
  (void)chunk;
  SelBufs b;
  PST_TRY(sel_bufs(c, S, N, n, K, true, b));
  PST_CUDA(cudaMemsetAsync(b.dmax, 0, 8, c->st));
  PST_CUDA(cudaMemsetAsync(b.taken, 0, S, c->st));
  PST_CUDA(cudaMemsetAsync(b.zero, 0, 8, c->st));
  k_fill<<<grid_for(N, 256), 256, 0, c->st>>>(b.curve, HUGE_VAL, N);
  k_fill<<<grid_for(N, 256), 256, 0, c->st>>>(b.nearval, HUGE_VAL, N);
  c->launches += 2;
  std::vector<int64_t> steps(K);
  for (int64_t step = 0; step < K; ++step) {
    if (step == 0)
      PST_TRY(pst_profile_reduce_dev(c, m, l, k, 0, S, nullptr, b.areas, b.nearval, b.nearest, (double*)b.dmax));
    else
      PST_TRY(pst_profile_reduce_dev(c, m, l, k, 0, S, b.curve, b.areas, nullptr, nullptr, nullptr));
    k_pick<<<1, 1024, 0, c->st>>>(b.areas, b.taken, S, b.best + step);
    c->launches++;
    int64_t best = 0;
    PST_CUDA(cudaMemcpyAsync(&best, b.best + step, 8, cudaMemcpyDeviceToHost, c->st));
    PST_CUDA(cudaStreamSynchronize(c->st));
    double* row = b.rows + step * N;
    PST_TRY(launch_mpdist(c, m, l, k, best, best + 1, row, N));  // the chosen profile, recomputed
    k_curve<<<grid_for(N, 256), 256, 0, c->st>>>(b.curve, row, N, b.zero, N);
    c->launches++;
    PST_CUDA(cudaGetLastError());
    steps[step] = step;
  }
  return finish_select(c, b, S, N, n, K, b.rows, steps, res);
}

// ---------------------------------------------------------------- key path
static double e2d_h(double ev, double twol) {  // host twin of e2d / e_to_dist (IEEE ops, same order)
  if (ev < 1e-15) ev = 0.0;
  if (ev > 2.0) ev = 2.0;
  return sqrt(twol * ev);
}
static void kb_exact_h(int K, double twol, double& lo, double& hi) {
  if (K < 0) {
    lo = hi = 0.0;
    return;
  }
  lo = e2d_h(hilo2d(K, 0u), twol);
  hi = e2d_h(hilo2d(K, 0xffffffffu), twol);
}

// caps of the exact work one key-path selection may need; beyond them the
// length is recomputed on the exact path (degenerate inputs: many exact ties)
constexpr int CAP_G = 16;        // exact greedy candidates per step
constexpr int CAP_W = 1 << 16;   // uncertain attribution / max windows
constexpr int CAP_P = 1 << 18;   // exact (segment, window) evaluations

struct CertBufs {
  double *alo, *ahi, *crow, *carea, *pval, *pval2;
  int64_t *glist, *wins, *pseg, *pwin, *mwins, *pseg2, *pwin2;
  int *cnt, *kmaxw, *K1w, *n1w, *K2w;
  int32_t* s1w;
  uint8_t* unc;
  int* TK;  // [NEAR_M][N] streamed path: smallest keys per window
  int32_t* TS;
};
static int cert_bufs(pst_ctx* c, int64_t S, int64_t N, CertBufs& b) {
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 255) & ~(size_t)255;
    return o;
  };
  const size_t o_alo = take(S * 8), o_ahi = take(S * 8), o_crow = take((size_t)CAP_G * N * 8),
               o_carea = take(CAP_G * 8), o_pval = take((size_t)CAP_P * 8), o_gl = take(CAP_G * 8),
               o_w = take((size_t)CAP_W * 8), o_ps = take((size_t)CAP_P * 8), o_pw = take((size_t)CAP_P * 8),
               o_cnt = take(4 * 4), o_km = take(N * 4), o_k1 = take(N * 4), o_unc = take(N),
               o_mw = take((size_t)CAP_W * 8), o_ps2 = take((size_t)CAP_P * 8), o_pw2 = take((size_t)CAP_P * 8),
               o_pv2 = take((size_t)CAP_P * 8), o_s1 = take(N * 4), o_n1 = take(N * 4), o_k2 = take(N * 4),
               o_tk = take((size_t)NEAR_M * N * 4), o_ts = take((size_t)NEAR_M * N * 4);
  PST_TRY(pst_ensure(&c->cert, &c->cert_bytes, off));
  char* p = (char*)c->cert;
  b.alo = (double*)(p + o_alo);
  b.ahi = (double*)(p + o_ahi);
  b.crow = (double*)(p + o_crow);
  b.carea = (double*)(p + o_carea);
  b.pval = (double*)(p + o_pval);
  b.glist = (int64_t*)(p + o_gl);
  b.wins = (int64_t*)(p + o_w);
  b.pseg = (int64_t*)(p + o_ps);
  b.pwin = (int64_t*)(p + o_pw);
  b.cnt = (int*)(p + o_cnt);
  b.kmaxw = (int*)(p + o_km);
  b.K1w = (int*)(p + o_k1);
  b.unc = (uint8_t*)(p + o_unc);
  b.mwins = (int64_t*)(p + o_mw);
  b.pseg2 = (int64_t*)(p + o_ps2);
  b.pwin2 = (int64_t*)(p + o_pw2);
  b.pval2 = (double*)(p + o_pv2);
  b.s1w = (int32_t*)(p + o_s1);
  b.n1w = (int*)(p + o_n1);
  b.K2w = (int*)(p + o_k2);
  b.TK = (int*)(p + o_tk);
  b.TS = (int32_t*)(p + o_ts);
  return PST_OK;
}

// exact values of the listed (segment, window) pairs -> host vectors
static int eval_pairs_at(pst_ctx* c, int64_t m, int64_t l, int64_t k, const int64_t* dseg, const int64_t* dwin,
                         double* dval, int cnt, std::vector<int64_t>& seg, std::vector<int64_t>& win,
                         std::vector<double>& val) {
  seg.resize(cnt);
  win.resize(cnt);
  val.resize(cnt);
  if (cnt == 0) return PST_OK;
  PST_TRY(launch_window_exact(c, m, l, k, dseg, dwin, cnt, dval));
  PST_CUDA(cudaMemcpyAsync(seg.data(), dseg, (size_t)cnt * 8, cudaMemcpyDeviceToHost, c->st));
  PST_CUDA(cudaMemcpyAsync(win.data(), dwin, (size_t)cnt * 8, cudaMemcpyDeviceToHost, c->st));
  PST_CUDA(cudaMemcpyAsync(val.data(), dval, (size_t)cnt * 8, cudaMemcpyDeviceToHost, c->st));
  PST_CUDA(cudaStreamSynchronize(c->st));
  c->cert_stats[4] += cnt;
  return PST_OK;
}
static int eval_pairs(pst_ctx* c, int64_t m, int64_t l, int64_t k, CertBufs& cb, int cnt, std::vector<int64_t>& seg,
                      std::vector<int64_t>& win, std::vector<double>& val) {
  return eval_pairs_at(c, m, l, k, cb.pseg, cb.pwin, cb.pval, cnt, seg, win, val);
}

// exact nearest-segment fixes from evaluated (segment, window, value) triples:
// per window the first argmin (value, then lowest segment)
static int apply_nearest_fixes(pst_ctx* c, CertBufs& cb, const std::vector<int64_t>& ps,
                               const std::vector<int64_t>& pw, const std::vector<double>& pv, int32_t* nearest) {
  const size_t np = ps.size();
  std::vector<size_t> ord(np);
  std::iota(ord.begin(), ord.end(), 0);
  std::sort(ord.begin(), ord.end(), [&](size_t a, size_t bb) {
    if (pw[a] != pw[bb]) return pw[a] < pw[bb];
    if (pv[a] != pv[bb]) return pv[a] < pv[bb];
    return ps[a] < ps[bb];
  });
  std::vector<int64_t> fw, fs;
  for (size_t i = 0; i < np; ++i)
    if (i == 0 || pw[ord[i]] != pw[ord[i - 1]]) {
      fw.push_back(pw[ord[i]]);
      fs.push_back(ps[ord[i]]);
    }
  const int nf = (int)fw.size();
  if (nf > 0) {
    PST_CUDA(cudaMemcpyAsync(cb.wins, fw.data(), (size_t)nf * 8, cudaMemcpyHostToDevice, c->st));
    PST_CUDA(cudaMemcpyAsync(cb.pseg, fs.data(), (size_t)nf * 8, cudaMemcpyHostToDevice, c->st));
    k_set_nearest<<<(nf + 255) / 256, 256, 0, c->st>>>(cb.wins, cb.pseg, nf, nearest);
    c->launches++;
    PST_CUDA(cudaStreamSynchronize(c->st));  // fw / fs are host vectors
  }
  return PST_OK;
}

static int read_cnt(pst_ctx* c, const int* dcnt, int& h) {
  PST_CUDA(cudaMemcpyAsync(&h, dcnt, 4, cudaMemcpyDeviceToHost, c->st));
  PST_CUDA(cudaStreamSynchronize(c->st));
  return PST_OK;
}

// Greedy + attribution + profile_max on the resident key matrix Dk (S x N).
// Returns PST_OK, or 1 when a cap is exceeded (caller falls back to the exact path).
static int run_select_keys(pst_ctx* c, const int* Dk, int64_t m, int64_t l, int64_t k, int64_t S, int64_t N,
                           int64_t n, int64_t K, pst_snippets* res) {
  const double twol = 2.0 * (double)l;
  const float twolf = (float)twol;
  int K15;
  {
    const double t = 1e-15;
    unsigned long long bits;
    memcpy(&bits, &t, 8);
    K15 = (int)(bits >> 32);
  }
  const double dclip = e2d_h(2.0, twol);
  SelBufs b;
  PST_TRY(sel_bufs(c, S, N, n, K, true, b));  // rows: the K chosen exact profiles
  CertBufs cb;
  PST_TRY(cert_bufs(c, S, N, cb));
  c->cert_stats[0]++;
  c->cert_stats[7] += N;

  // ---- greedy (snippets.py:201-210)
  PST_CUDA(cudaMemsetAsync(b.taken, 0, S, c->st));
  k_fill<<<grid_for(N, 256), 256, 0, c->st>>>(b.curve, HUGE_VAL, N);
  c->launches++;
  std::vector<int64_t> chosen(K);
  for (int64_t step = 0; step < K; ++step) {
    const double* cur = step == 0 ? nullptr : b.curve;
    k_areas_kb<<<(unsigned)S, 256, 0, c->st>>>(Dk, N, N, cur, b.taken, twolf, K15, dclip, cb.alo, cb.ahi);
    PST_CUDA(cudaMemsetAsync(cb.cnt, 0, 4, c->st));
    k_greedy_cands<<<1, 1024, 0, c->st>>>(cb.alo, cb.ahi, b.taken, S, CAP_G, cb.glist, cb.cnt);
    c->launches += 2;
    PST_CUDA(cudaGetLastError());
    int nc = 0;
    PST_TRY(read_cnt(c, cb.cnt, nc));
    if (nc > CAP_G || nc < 1) return 1;
    std::vector<int64_t> cand(nc);
    PST_CUDA(cudaMemcpyAsync(cand.data(), cb.glist, (size_t)nc * 8, cudaMemcpyDeviceToHost, c->st));
    PST_CUDA(cudaStreamSynchronize(c->st));
    std::sort(cand.begin(), cand.end());
    c->cert_stats[1] += nc;
    if (nc > 1) c->cert_stats[2]++;
    for (int i = 0; i < nc; ++i) {  // exact profiles and exact areas (k_areas, as the exact path)
      double* row = cb.crow + (size_t)i * N;
      PST_TRY(launch_mpdist(c, m, l, k, cand[i], cand[i] + 1, row, N));
      k_areas<<<1, 256, 0, c->st>>>(row, N, N, cur, cb.carea + i);
      c->launches++;
    }
    std::vector<double> ca(nc);
    PST_CUDA(cudaMemcpyAsync(ca.data(), cb.carea, (size_t)nc * 8, cudaMemcpyDeviceToHost, c->st));
    PST_CUDA(cudaStreamSynchronize(c->st));
    int bi = 0;
    for (int i = 1; i < nc; ++i)
      if (ca[i] < ca[bi]) bi = i;  // ties -> lowest index (cand sorted)
    chosen[step] = cand[bi];
    double* keep = b.rows + step * N;
    PST_CUDA(cudaMemcpyAsync(keep, cb.crow + (size_t)bi * N, (size_t)N * 8, cudaMemcpyDeviceToDevice, c->st));
    k_mark_taken<<<1, 1, 0, c->st>>>(b.taken, cand[bi]);
    k_curve_row<<<grid_for(N, 256), 256, 0, c->st>>>(b.curve, keep, N);
    c->launches += 2;
  }
  PST_CUDA(cudaMemcpyAsync(b.best, chosen.data(), K * 8, cudaMemcpyHostToDevice, c->st));

  // ---- attribution (snippets.py:212-213) and profile_max (snippets.py:241)
  k_near_keys<<<grid_for(N, 256), 256, 0, c->st>>>(Dk, S, N, N, twol, b.nearest, cb.unc, cb.kmaxw, cb.K1w);
  PST_CUDA(cudaMemsetAsync(cb.cnt, 0, 16, c->st));
  k_flag_list<<<grid_for(N, 256), 256, 0, c->st>>>(cb.unc, N, CAP_W, cb.wins, cb.cnt);
  c->launches += 2;
  PST_CUDA(cudaGetLastError());
  int nw = 0;
  PST_TRY(read_cnt(c, cb.cnt, nw));
  if (nw > CAP_W) return 1;
  c->cert_stats[3] += nw;
  std::vector<int64_t> ps, pw;
  std::vector<double> pv;
  if (nw > 0) {
    k_pairs<<<(unsigned)((nw * 32 + 255) / 256), 256, 0, c->st>>>(Dk, S, N, 0, cb.wins, nw, cb.K1w, 0, 0, twol, K15, CAP_P,
                                                                cb.pseg, cb.pwin, cb.cnt + 1);
    c->launches++;
    int np = 0;
    PST_TRY(read_cnt(c, cb.cnt + 1, np));
    if (np > CAP_P) return 1;
    PST_TRY(eval_pairs(c, m, l, k, cb, np, ps, pw, pv));
    // per window: first argmin of the exact values
    std::vector<size_t> ord(np);
    std::iota(ord.begin(), ord.end(), 0);
    std::sort(ord.begin(), ord.end(), [&](size_t a, size_t bb) {
      if (pw[a] != pw[bb]) return pw[a] < pw[bb];
      if (pv[a] != pv[bb]) return pv[a] < pv[bb];
      return ps[a] < ps[bb];
    });
    std::vector<int64_t> fw, fs;
    for (size_t i = 0; i < ord.size(); ++i)
      if (i == 0 || pw[ord[i]] != pw[ord[i - 1]]) {
        fw.push_back(pw[ord[i]]);
        fs.push_back(ps[ord[i]]);
      }
    const int nf = (int)fw.size();
    if (nf > 0) {
      PST_CUDA(cudaMemcpyAsync(cb.wins, fw.data(), (size_t)nf * 8, cudaMemcpyHostToDevice, c->st));
      PST_CUDA(cudaMemcpyAsync(cb.pseg, fs.data(), (size_t)nf * 8, cudaMemcpyHostToDevice, c->st));
      k_set_nearest<<<(nf + 255) / 256, 256, 0, c->st>>>(cb.wins, cb.pseg, nf, b.nearest);
      c->launches++;
    }
  }
  double pmax = 0.0;
  {
    static const int kIntMin = INT_MIN;
    PST_CUDA(cudaMemcpyAsync(cb.cnt + 2, &kIntMin, 4, cudaMemcpyHostToDevice, c->st));
    k_max_int<<<grid_for(N, 256, 1024), 256, 0, c->st>>>(cb.kmaxw, N, cb.cnt + 2);
    c->launches++;
    int kmax = 0;
    PST_TRY(read_cnt(c, cb.cnt + 2, kmax));
    double lo, hi;
    kb_exact_h(kmax, twol, lo, hi);
    if (lo == hi) {
      pmax = lo;
    } else {  // candidates: every (segment, window) whose interval reaches lo(kmax)
      // keys below K15 are exactly 0 and cannot exceed a candidate; adjacent
      // buckets differ by ~2^-21 relative, so the loop takes a step or two
      int thr = kmax, guard = 0;
      while (thr > K15) {
        double l2, h2;
        kb_exact_h(thr - 1, twol, l2, h2);
        if (h2 < lo) break;
        --thr;
        if (++guard > 1024) return 1;
      }
      k_kmax_flag<<<grid_for(N, 256), 256, 0, c->st>>>(cb.kmaxw, N, thr, cb.unc);
      PST_CUDA(cudaMemsetAsync(cb.cnt, 0, 8, c->st));
      k_flag_list<<<grid_for(N, 256), 256, 0, c->st>>>(cb.unc, N, CAP_W, cb.wins, cb.cnt);
      c->launches += 2;
      int nmw = 0;
      PST_TRY(read_cnt(c, cb.cnt, nmw));
      if (nmw > CAP_W || nmw < 1) return 1;
      k_pairs<<<(unsigned)((nmw * 32 + 255) / 256), 256, 0, c->st>>>(Dk, S, N, 0, cb.wins, nmw, cb.K1w, thr, 1,
                                                                   twol, K15, CAP_P, cb.pseg, cb.pwin, cb.cnt + 1);
      c->launches++;
      int np = 0;
      PST_TRY(read_cnt(c, cb.cnt + 1, np));
      if (np > CAP_P || np < 1) return 1;
      PST_TRY(eval_pairs(c, m, l, k, cb, np, ps, pw, pv));
      c->cert_stats[5] += np;
      for (double v : pv) pmax = std::max(pmax, v);
    }
  }
  {
    unsigned long long bits;
    memcpy(&bits, &pmax, 8);
    PST_CUDA(cudaMemcpyAsync(b.dmax, &bits, 8, cudaMemcpyHostToDevice, c->st));
    PST_CUDA(cudaStreamSynchronize(c->st));  // &bits is a stack variable
  }
  std::vector<int64_t> steps(K);
  std::iota(steps.begin(), steps.end(), 0);
  return finish_select(c, b, S, N, n, K, b.rows, steps, res);
}

// ---- streamed key path (S x N keys do not fit: C4, n = 1e7) -------------------
// One certified greedy step from the area bounds of all S rows (alo/ahi filled).
static int greedy_step_keys(pst_ctx* c, int64_t m, int64_t l, int64_t k, int64_t S, int64_t N, SelBufs& b,
                            CertBufs& cb, int64_t step, std::vector<int64_t>& chosen) {
  const double* cur = step == 0 ? nullptr : b.curve;
  PST_CUDA(cudaMemsetAsync(cb.cnt, 0, 4, c->st));
  k_greedy_cands<<<1, 1024, 0, c->st>>>(cb.alo, cb.ahi, b.taken, S, CAP_G, cb.glist, cb.cnt);
  c->launches++;
  PST_CUDA(cudaGetLastError());
  int nc = 0;
  PST_TRY(read_cnt(c, cb.cnt, nc));
  if (nc > CAP_G || nc < 1) return 1;
  std::vector<int64_t> cand(nc);
  PST_CUDA(cudaMemcpyAsync(cand.data(), cb.glist, (size_t)nc * 8, cudaMemcpyDeviceToHost, c->st));
  PST_CUDA(cudaStreamSynchronize(c->st));
  std::sort(cand.begin(), cand.end());
  c->cert_stats[1] += nc;
  if (nc > 1) c->cert_stats[2]++;
  for (int i = 0; i < nc; ++i) {
    double* row = cb.crow + (size_t)i * N;
    PST_TRY(launch_mpdist(c, m, l, k, cand[i], cand[i] + 1, row, N));
    k_areas<<<1, 256, 0, c->st>>>(row, N, N, cur, cb.carea + i);
    c->launches++;
  }
  std::vector<double> ca(nc);
  PST_CUDA(cudaMemcpyAsync(ca.data(), cb.carea, (size_t)nc * 8, cudaMemcpyDeviceToHost, c->st));
  PST_CUDA(cudaStreamSynchronize(c->st));
  int bi = 0;
  for (int i = 1; i < nc; ++i)
    if (ca[i] < ca[bi]) bi = i;
  chosen[step] = cand[bi];
  double* keep = b.rows + step * N;
  PST_CUDA(cudaMemcpyAsync(keep, cb.crow + (size_t)bi * N, (size_t)N * 8, cudaMemcpyDeviceToDevice, c->st));
  k_mark_taken<<<1, 1, 0, c->st>>>(b.taken, cand[bi]);
  k_curve_row<<<grid_for(N, 256), 256, 0, c->st>>>(b.curve, keep, N);
  c->launches += 2;
  return PST_OK;
}

// Profiles are recomputed chunk by chunk (chunk segments of keys at a time) in
// max(K, 2) passes: pass t feeds greedy step t's area bounds; pass 0 also
// accumulates the per-window attribution state and maxima; pass 1 collects the
// candidate (segment, window) pairs of the windows pass 0 left uncertain and
// of profile_max.  Certification and exact resolution as run_select_keys.
// Block minima for the pruned passes (1 and later): the smallest block (16, 32
// or 64 windows) whose S x NB keys take at most a third of the device memory
// left for this length.  PASTILA_PRUNE=0 disables.
static int PRUNE_MEM_PCT = 55;
static int prune_alloc(pst_ctx* c, int64_t S, int64_t N, int64_t K, PruneBufs& pb) {
  if (const char* e = getenv("PASTILA_PRUNE_MEM_PCT")) PRUNE_MEM_PCT = atoi(e);  // tuning experiments
  pb = PruneBufs();
  (void)K;  // max(K, 2) >= 2 passes: pass 1 and later can be pruned
  if (const char* e = getenv("PASTILA_PRUNE"))
    if (atoi(e) == 0) return PST_OK;
  size_t fr = 0, tot = 0;
  if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) return PST_OK;
  const size_t have = fr + c->Dk_bytes + c->prune_bytes;
  for (int B : {16, 32, 64}) {
    const int64_t NB = (N + B - 1) / B;
    const size_t need = (size_t)S * NB * 4 + (size_t)NB * (2 * B + 1) * 8 + (size_t)S * 20 + 4096;
    if (need > have / 100 * PRUNE_MEM_PCT) continue;
    if (c->Dk) {  // the chunk buffer is sized after this allocation
      cudaFree(c->Dk);
      c->Dk = nullptr;
      c->Dk_bytes = 0;
    }
    PST_TRY(pst_ensure(&c->prune, &c->prune_bytes, need));
    char* p = (char*)c->prune;
    pb.B = B;
    pb.NB = NB;
    pb.Bm = (int*)p;
    size_t o = ((size_t)S * NB * 4 + 255) & ~(size_t)255;
    pb.Cs = (double*)(p + o);
    o += ((size_t)NB * B * 8 + 255) & ~(size_t)255;
    pb.Cp = (double*)(p + o);
    o += ((size_t)NB * (B + 1) * 8 + 255) & ~(size_t)255;
    pb.LB = (double*)(p + o);
    o += ((size_t)S * 8 + 255) & ~(size_t)255;
    pb.segl = (int64_t*)(p + o);
    o += ((size_t)S * 8 + 255) & ~(size_t)255;
    pb.Rx = (int*)(p + o);
    return PST_OK;
  }
  return PST_OK;
}
static void prune_free(pst_ctx* c) {
  if (c->prune) cudaFree(c->prune);
  c->prune = nullptr;
  c->prune_bytes = 0;
}
// Key-bucket area bounds (k_areas_kb with the current curve) of the listed
// segments: their key rows are recomputed from a device list, up to `chunk`
// rows per profile launch (so the row loop and the selection of consecutive
// batches still overlap).
static int rows_bounds(pst_ctx* c, int64_t m, int64_t l, int64_t k, int64_t N, int64_t chunk,
                       const std::vector<int64_t>& segs, const PruneBufs& pb, const SelBufs& b, const CertBufs& cb,
                       float twolf, int K15, double dclip) {
  if (segs.empty()) return PST_OK;
  PST_CUDA(cudaMemcpyAsync(pb.segl, segs.data(), segs.size() * 8, cudaMemcpyHostToDevice, c->st));
  for (size_t i = 0; i < segs.size(); i += (size_t)chunk) {
    const int64_t cnt = std::min<int64_t>(chunk, (int64_t)(segs.size() - i));
    PST_TRY(launch_mpdist_keys_list(c, m, l, k, pb.segl + i, cnt, c->Dk, N));
    k_areas_kb<<<(unsigned)cnt, 256, 0, c->st>>>(c->Dk, N, N, b.curve, b.taken, twolf, K15, dclip, cb.alo, cb.ahi,
                                                 pb.segl + i);
    c->launches++;
    PST_CUDA(cudaGetLastError());
  }
  PST_CUDA(cudaStreamSynchronize(c->st));  // the host list is reused by the caller
  return PST_OK;
}
// Greedy area bounds of a pass >= 2 without recomputing every row.  Every
// segment gets alo = LB (a rigorous lower bound), ahi = +inf; the PROBES
// segments with the smallest LB get their key-bucket bounds, whose smallest
// upper bound U bounds the winner's exact area from above; every segment with
// LB <= U is recomputed (the winner, and every segment tied with it, has
// LB <= area* <= U).  k_greedy_cands then sees exactly the candidates the full
// pass would give it, or a superset: the exact areas decide as before.
// done = false: too many candidates, the caller runs the full pass.
static int pruned_bounds(pst_ctx* c, int64_t m, int64_t l, int64_t k, int64_t S, int64_t N, int64_t chunk,
                         const PruneBufs& pb, const SelBufs& b, const CertBufs& cb, float twolf, int K15,
                         double dclip, bool& done, int64_t& rows) {
  constexpr int PROBES = 32;
  done = false;
  rows = 0;
  k_curve_blocks<<<grid_for(pb.NB, 128), 128, 0, c->st>>>(b.curve, N, pb.B, pb.NB, pb.Cs, pb.Cp);
  k_lb<<<(unsigned)S, 256, 0, c->st>>>(pb.Bm, pb.NB, pb.B, N, pb.Cs, pb.Cp, b.taken, twolf, K15, dclip, pb.LB);
  k_set_bounds<<<grid_for(S, 256), 256, 0, c->st>>>(pb.LB, S, cb.alo, cb.ahi);
  c->launches += 3;
  PST_CUDA(cudaGetLastError());
  std::vector<double> lb(S);
  PST_CUDA(cudaMemcpyAsync(lb.data(), pb.LB, (size_t)S * 8, cudaMemcpyDeviceToHost, c->st));
  PST_CUDA(cudaStreamSynchronize(c->st));
  std::vector<int64_t> order;
  order.reserve(S);
  for (int64_t s = 0; s < S; ++s)
    if (lb[s] < HUGE_VAL) order.push_back(s);
  if (order.empty()) return PST_OK;  // nothing available: the full pass reports it
  const size_t np = std::min<size_t>(PROBES, order.size());
  std::partial_sort(order.begin(), order.begin() + np, order.end(),
                    [&](int64_t a, int64_t z) { return lb[a] < lb[z] || (lb[a] == lb[z] && a < z); });
  std::vector<int64_t> probes(order.begin(), order.begin() + np);
  std::sort(probes.begin(), probes.end());
  PST_TRY(rows_bounds(c, m, l, k, N, chunk, probes, pb, b, cb, twolf, K15, dclip));
  std::vector<double> hi(np);
  for (size_t i = 0; i < np; ++i)
    PST_CUDA(cudaMemcpyAsync(&hi[i], cb.ahi + probes[i], 8, cudaMemcpyDeviceToHost, c->st));
  PST_CUDA(cudaStreamSynchronize(c->st));
  const double U = *std::min_element(hi.begin(), hi.end());
  std::vector<int64_t> rest;
  for (int64_t s = 0; s < S; ++s)
    if (lb[s] <= U && !std::binary_search(probes.begin(), probes.end(), s)) rest.push_back(s);
  rows = (int64_t)np;
  if ((int64_t)(rest.size() + np) > S / 2) return PST_OK;  // a full pass is as cheap
  PST_TRY(rows_bounds(c, m, l, k, N, chunk, rest, pb, b, cb, twolf, K15, dclip));
  rows += (int64_t)rest.size();
  if (getenv("PASTILA_DEBUG"))
    fprintf(stderr, "[pastila] pruned pass: B=%d, %lld of %lld rows recomputed (U=%.17g)\n", pb.B,
            (long long)rows, (long long)S, U);
  done = true;
  return PST_OK;
}
// Pass 1's candidate pairs from the block minima / row maxima (k_pairs_sum),
// instead of from the key rows; ok = false when either list exceeds LIM pairs
// (the exact evaluation of a long superset costs more than a full pass).
static int pruned_pairs(pst_ctx* c, int64_t S, int64_t N, const PruneBufs& pb, const CertBufs& cb, int nw,
                        bool need_max, int nmw, int thr, double twol, int K15, bool& ok) {
  constexpr int LIM = 32768;
  ok = false;
  if (nw > 0) {
    k_pairs_sum<<<(unsigned)((nw * 32 + 255) / 256), 256, 0, c->st>>>(pb.Bm, pb.Rx, S, pb.NB, pb.B, cb.TK, cb.TS,
                                                                      N, cb.wins, nw,
                                                                      cb.K1w, 0, 0, twol, K15, CAP_P, cb.pseg,
                                                                      cb.pwin, cb.cnt + 1);
    c->launches++;
  }
  if (need_max) {
    k_pairs_sum<<<(unsigned)((nmw * 32 + 255) / 256), 256, 0, c->st>>>(pb.Bm, pb.Rx, S, pb.NB, pb.B, cb.TK, cb.TS,
                                                                       N, cb.mwins,
                                                                       nmw, cb.K1w, thr, 1, twol, K15, CAP_P,
                                                                       cb.pseg2, cb.pwin2, cb.cnt + 3);
    c->launches++;
  }
  PST_CUDA(cudaGetLastError());
  int n1 = 0, n3 = 0;
  PST_TRY(read_cnt(c, cb.cnt + 1, n1));
  PST_TRY(read_cnt(c, cb.cnt + 3, n3));
  ok = n1 <= LIM && n3 <= LIM;
  if (getenv("PASTILA_DEBUG"))
    fprintf(stderr, "[pastila] pass-1 pairs from block summaries: %d attribution, %d maximum (limit %d)\n", n1, n3,
            LIM);
  return PST_OK;
}

static int run_select_keys_streamed(pst_ctx* c, int64_t m, int64_t l, int64_t k, int64_t S, int64_t N, int64_t n,
                                    int64_t K, int64_t chunk, const PruneBufs& pb, pst_snippets* res) {
  const double twol = 2.0 * (double)l;
  const float twolf = (float)twol;
  int K15;
  {
    const double t = 1e-15;
    unsigned long long bits;
    memcpy(&bits, &t, 8);
    K15 = (int)(bits >> 32);
  }
  const double dclip = e2d_h(2.0, twol);
  SelBufs b;
  PST_TRY(sel_bufs(c, S, N, n, K, true, b));
  CertBufs cb;
  PST_TRY(cert_bufs(c, S, N, cb));
  PST_TRY(pst_ensure((void**)&c->Dk, &c->Dk_bytes, (size_t)chunk * N * sizeof(int)));
  c->cert_stats[0]++;
  c->cert_stats[7] += N;
  PST_CUDA(cudaMemsetAsync(b.taken, 0, S, c->st));
  k_fill<<<grid_for(N, 256), 256, 0, c->st>>>(b.curve, HUGE_VAL, N);
  c->launches++;
  std::vector<int64_t> chosen(K);
  int nw = 0, nmw = 0, thr = 0;
  double pmax = 0.0;
  bool need_max = false;
  const int64_t passes = std::max<int64_t>(K, 2);
  for (int64_t pass = 0; pass < passes; ++pass) {
    const bool greedy = pass < K;
    const double* cur = pass == 0 ? nullptr : b.curve;
    if (pass == 1) PST_CUDA(cudaMemsetAsync(cb.cnt + 1, 0, 12, c->st));  // pair counters [1] and [3]
    // passes >= 1: recompute only the rows whose greedy area can still win, and
    // take pass 1's candidate pairs from the block summaries of pass 0
    bool pruned = false;
    if (pass >= 1 && pb.Bm) {
      bool pairs_ok = true;  // the cheap check first: a failed one costs no recomputed rows
      if (pass == 1) PST_TRY(pruned_pairs(c, S, N, pb, cb, nw, need_max, nmw, thr, twol, K15, pairs_ok));
      bool areas_ok = !greedy;
      int64_t prow = 0;
      if (greedy && pairs_ok)
        PST_TRY(pruned_bounds(c, m, l, k, S, N, chunk, pb, b, cb, twolf, K15, dclip, areas_ok, prow));
      pruned = areas_ok && pairs_ok;
      if (pruned) {
        c->prune_stats[0]++;
        c->prune_stats[1] += prow;
      } else {
        c->prune_stats[2]++;
        c->prune_stats[3] += S;
        if (pass == 1) PST_CUDA(cudaMemsetAsync(cb.cnt + 1, 0, 12, c->st));  // the full pass collects them again
      }
    }
    if (pass == 0 && pb.Bm) {
      k_fill_i32<<<grid_for(S, 256), 256, 0, c->st>>>(pb.Rx, INT_MIN, S);
      c->launches++;
    }
    for (int64_t s0 = 0; s0 < S && !pruned; s0 += chunk) {
      const int64_t rows = std::min(chunk, S - s0);
      PST_TRY(launch_mpdist_keys(c, m, l, k, s0, s0 + rows, c->Dk, N));
      if (pass == 0 && pb.Bm) {
        k_block_min<<<grid_for(rows * pb.NB, 256), 256, 0, c->st>>>(c->Dk, rows, N, pb.B, pb.NB,
                                                                   pb.Bm + s0 * pb.NB, pb.Rx + s0);
        c->launches++;
      }
      if (greedy) {
        k_areas_kb<<<(unsigned)rows, 256, 0, c->st>>>(c->Dk, N, N, cur, b.taken + s0, twolf, K15, dclip,
                                                       cb.alo + s0, cb.ahi + s0);
        c->launches++;
      }
      if (pass == 0) {
        k_near_keys_acc<<<grid_for(N, 256), 256, 0, c->st>>>(c->Dk, rows, N, N, s0, s0 == 0 ? 1 : 0, cb.K1w,
                                                            cb.s1w, cb.n1w, cb.K2w, cb.kmaxw, cb.TK, cb.TS);
        c->launches++;
      }
      if (pass == 1) {
        if (nw > 0) {
          k_pairs<<<(unsigned)((nw * 32 + 255) / 256), 256, 0, c->st>>>(c->Dk, rows, N, s0, cb.wins, nw, cb.K1w, 0,
                                                                      0, twol, K15, CAP_P, cb.pseg, cb.pwin,
                                                                      cb.cnt + 1);
          c->launches++;
        }
        if (need_max) {
          k_pairs<<<(unsigned)((nmw * 32 + 255) / 256), 256, 0, c->st>>>(c->Dk, rows, N, s0, cb.mwins, nmw,
                                                                       cb.K1w, thr, 1, twol, K15, CAP_P,
                                                                       cb.pseg2, cb.pwin2, cb.cnt + 3);
          c->launches++;
        }
      }
      PST_CUDA(cudaGetLastError());
    }
    if (greedy) {
      const int r = greedy_step_keys(c, m, l, k, S, N, b, cb, pass, chosen);
      if (r != PST_OK) return r;
    }
    if (pass == 0) {  // attribution state complete: certified windows and the lists for pass 1
      k_near_finalize<<<grid_for(N, 256), 256, 0, c->st>>>(N, twol, cb.K1w, cb.s1w, cb.n1w, cb.K2w, b.nearest,
                                                          cb.unc);
      PST_CUDA(cudaMemsetAsync(cb.cnt, 0, 4, c->st));
      k_flag_list<<<grid_for(N, 256), 256, 0, c->st>>>(cb.unc, N, CAP_W, cb.wins, cb.cnt);
      c->launches += 2;
      PST_TRY(read_cnt(c, cb.cnt, nw));
      if (nw > CAP_W) return 1;
      c->cert_stats[3] += nw;
      static const int kIntMin = INT_MIN;
      PST_CUDA(cudaMemcpyAsync(cb.cnt + 2, &kIntMin, 4, cudaMemcpyHostToDevice, c->st));
      k_max_int<<<grid_for(N, 256, 1024), 256, 0, c->st>>>(cb.kmaxw, N, cb.cnt + 2);
      c->launches++;
      int kmax = 0;
      PST_TRY(read_cnt(c, cb.cnt + 2, kmax));
      double lo, hi;
      kb_exact_h(kmax, twol, lo, hi);
      if (lo == hi) {
        pmax = lo;
      } else {
        need_max = true;
        thr = kmax;
        int guard = 0;
        while (thr > K15) {
          double l2, h2;
          kb_exact_h(thr - 1, twol, l2, h2);
          if (h2 < lo) break;
          --thr;
          if (++guard > 1024) return 1;
        }
        k_kmax_flag<<<grid_for(N, 256), 256, 0, c->st>>>(cb.kmaxw, N, thr, cb.unc);
        PST_CUDA(cudaMemsetAsync(cb.cnt, 0, 4, c->st));
        k_flag_list<<<grid_for(N, 256), 256, 0, c->st>>>(cb.unc, N, CAP_W, cb.mwins, cb.cnt);
        c->launches += 2;
        PST_TRY(read_cnt(c, cb.cnt, nmw));
        if (nmw > CAP_W || nmw < 1) return 1;
      }
    }
  }
  PST_CUDA(cudaMemcpyAsync(b.best, chosen.data(), K * 8, cudaMemcpyHostToDevice, c->st));
  std::vector<int64_t> ps, pw;
  std::vector<double> pv;
  if (nw > 0) {
    int np = 0;
    PST_TRY(read_cnt(c, cb.cnt + 1, np));
    if (np > CAP_P) return 1;
    PST_TRY(eval_pairs(c, m, l, k, cb, np, ps, pw, pv));
    PST_TRY(apply_nearest_fixes(c, cb, ps, pw, pv, b.nearest));
  }
  if (need_max) {
    int np = 0;
    PST_TRY(read_cnt(c, cb.cnt + 3, np));
    if (np > CAP_P || np < 1) return 1;
    PST_TRY(eval_pairs_at(c, m, l, k, cb.pseg2, cb.pwin2, cb.pval2, np, ps, pw, pv));
    c->cert_stats[5] += np;
    for (double v : pv) pmax = std::max(pmax, v);
  }
  {
    unsigned long long bits;
    memcpy(&bits, &pmax, 8);
    PST_CUDA(cudaMemcpyAsync(b.dmax, &bits, 8, cudaMemcpyHostToDevice, c->st));
    PST_CUDA(cudaStreamSynchronize(c->st));
  }
  std::vector<int64_t> steps(K);
  std::iota(steps.begin(), steps.end(), 0);
  return finish_select(c, b, S, N, n, K, b.rows, steps, res);
}

// criterion_score on caller-supplied profiles (length_select.py:56-87):
// P host [K*N] in snippet order, pairs summed in itertools.combinations order.
int pst_criterion(pst_ctx* c, const double* P, int64_t K, int64_t N, double profile_max, double* out) {
  if (!valid(c)) return PST_EINVAL;
  PST_CUDA(cudaSetDevice(c->dev));
  if (K < 2) {
    pst_set_error("separation needs at least 2 snippets, got %lld", (long long)K);
    return PST_EINVAL;
  }
  if (profile_max == 0.0) {
    *out = 0.0;
    return PST_OK;
  }
  const int64_t npair = K * (K - 1) / 2;
  const size_t bp = (size_t)K * N * 8;
  PST_TRY(pst_ensure(&c->work, &c->work_bytes, bp + npair * 8 + 256));
  double* dP = (double*)c->work;
  double* dpair = (double*)((char*)c->work + ((bp + 255) & ~(size_t)255));
  PST_CUDA(cudaMemcpyAsync(dP, P, bp, cudaMemcpyHostToDevice, c->st));
  k_pairdiff<<<(unsigned)npair, 256, 0, c->st>>>(dP, N, K, dpair);
  c->launches++;
  PST_CUDA(cudaGetLastError());
  std::vector<double> h(npair);
  PST_CUDA(cudaMemcpyAsync(h.data(), dpair, npair * 8, cudaMemcpyDeviceToHost, c->st));
  PST_CUDA(cudaStreamSynchronize(c->st));
  double tot = 0.0;
  for (int64_t i = 0; i < npair; ++i) tot += h[i];
  *out = tot / profile_max;
  return PST_OK;
}

// label_series on caller-supplied ordered profiles (labeling.py:91-119).
int pst_labels(pst_ctx* c, const double* P, int64_t K, int64_t N, int64_t n, int64_t* labels) {
  if (!valid(c)) return PST_EINVAL;
  PST_CUDA(cudaSetDevice(c->dev));
  if (K < 1 || N < 1 || n < N) {
    pst_set_error("bad label shapes K=%lld N=%lld n=%lld", (long long)K, (long long)N, (long long)n);
    return PST_EINVAL;
  }
  const size_t bp = ((size_t)K * N * 8 + 255) & ~(size_t)255;
  PST_TRY(pst_ensure(&c->work, &c->work_bytes, bp + (size_t)n * 8));
  double* dP = (double*)c->work;
  int64_t* dl = (int64_t*)((char*)c->work + bp);
  PST_CUDA(cudaMemcpyAsync(dP, P, (size_t)K * N * 8, cudaMemcpyHostToDevice, c->st));
  k_labels<<<grid_for(n, 256), 256, 0, c->st>>>(dP, K, N, n, dl);
  c->launches++;
  PST_CUDA(cudaGetLastError());
  PST_CUDA(cudaMemcpyAsync(labels, dl, (size_t)n * 8, cudaMemcpyDeviceToHost, c->st));
  PST_CUDA(cudaStreamSynchronize(c->st));
  return PST_OK;
}

// Pruned-pass counters of the streamed key path (see pst_ctx::prune_stats).
int pst_prune_stats(pst_ctx* c, int64_t* out, int reset) {
  if (!valid(c)) return PST_EINVAL;
  if (out)
    for (int i = 0; i < 4; ++i) out[i] = c->prune_stats[i];
  if (reset)
    for (int i = 0; i < 4; ++i) c->prune_stats[i] = 0;
  return PST_OK;
}

// Certification counters of the key path (see pst_ctx::cert_stats); reset != 0 clears them.
int pst_cert_stats(pst_ctx* c, int64_t* out, int reset) {
  if (!valid(c)) return PST_EINVAL;
  if (out)
    for (int i = 0; i < 8; ++i) out[i] = c->cert_stats[i];
  if (reset)
    for (int i = 0; i < 8; ++i) c->cert_stats[i] = 0;
  return PST_OK;
}

// Key-path profile keys of segments [seg_lo, seg_hi) (host out [(hi-lo) * N]):
// out = high word of the exact path's e_k (test / certification evidence).
int pst_profile_keys(pst_ctx* c, int64_t m, int64_t l, int64_t k, int64_t seg_lo, int64_t seg_hi, int32_t* out) {
  if (!valid(c)) return PST_EINVAL;
  PST_CUDA(cudaSetDevice(c->dev));
  PST_TRY(check_mkl(c, m, l, k));
  const int64_t S = c->n / m, N = c->n - m + 1;
  if (seg_lo < 0 || seg_hi > S || seg_lo >= seg_hi) {
    pst_set_error("segment index %lld out of range [0, %lld)", (long long)(seg_lo < 0 ? seg_lo : seg_hi - 1),
                  (long long)S);
    return PST_EINVAL;
  }
  const size_t bytes = (size_t)(seg_hi - seg_lo) * N * sizeof(int);
  PST_TRY(pst_ensure((void**)&c->Dk, &c->Dk_bytes, bytes));
  PST_TRY(launch_mpdist_keys(c, m, l, k, seg_lo, seg_hi, c->Dk, N));
  PST_CUDA(cudaMemcpyAsync(out, c->Dk, bytes, cudaMemcpyDeviceToHost, c->st));
  PST_CUDA(cudaStreamSynchronize(c->st));
  return PST_OK;
}

// Exact profile values at single (segment, window) pairs (host arrays of cnt).
int pst_window_exact(pst_ctx* c, int64_t m, int64_t l, int64_t k, const int64_t* seg, const int64_t* win,
                     int64_t cnt, double* out) {
  if (!valid(c)) return PST_EINVAL;
  PST_CUDA(cudaSetDevice(c->dev));
  PST_TRY(check_mkl(c, m, l, k));
  const int64_t S = c->n / m, N = c->n - m + 1;
  for (int64_t i = 0; i < cnt; ++i)
    if (seg[i] < 0 || seg[i] >= S || win[i] < 0 || win[i] >= N) {
      pst_set_error("pair %lld (segment %lld, window %lld) out of range", (long long)i, (long long)seg[i],
                    (long long)win[i]);
      return PST_EINVAL;
    }
  if (cnt <= 0) return PST_OK;
  PST_TRY(pst_ensure_len(c, l));  // before taking c->work: a new length rebuilds its arrays through it
  const size_t b = (size_t)cnt * 8;
  PST_TRY(pst_ensure(&c->work, &c->work_bytes, 3 * ((b + 255) & ~(size_t)255)));
  char* w = (char*)c->work;
  int64_t* ds = (int64_t*)w;
  int64_t* dw = (int64_t*)(w + ((b + 255) & ~(size_t)255));
  double* dv = (double*)(w + 2 * ((b + 255) & ~(size_t)255));
  PST_CUDA(cudaMemcpyAsync(ds, seg, b, cudaMemcpyHostToDevice, c->st));
  PST_CUDA(cudaMemcpyAsync(dw, win, b, cudaMemcpyHostToDevice, c->st));
  PST_TRY(launch_window_exact(c, m, l, k, ds, dw, cnt, dv));
  PST_CUDA(cudaMemcpyAsync(out, dv, b, cudaMemcpyDeviceToHost, c->st));
  PST_CUDA(cudaStreamSynchronize(c->st));
  return PST_OK;
}

// Row-loop / selection kernel milliseconds since the last read (PASTILA_KTIME=1 and
// pst_timing enabled; instrumentation only: events around every launch).
int pst_kernel_times(pst_ctx* c, double* out2) {
  if (!valid(c)) return PST_EINVAL;
  return kernel_times_read(c, out2);
}

// The context's CUDA stream (cudaStream_t), for event timing by callers.
int pst_stream(pst_ctx* c, void** out) {
  if (!valid(c)) return PST_EINVAL;
  *out = (void*)c->st;
  return PST_OK;
}

// Profile-kernel timing: enable(1)/disable(0) and reset; read accumulated
// device milliseconds and kernel launches of all profile computations since.
int pst_timing(pst_ctx* c, int enable) {
  if (!valid(c)) return PST_EINVAL;
  c->timing = enable != 0;
  c->t_ms = 0.0;
  c->t_calls = 0;
  c->t_launch = 0;
  if (c->tev) {
    auto* v = (std::vector<std::pair<cudaEvent_t, cudaEvent_t>>*)c->tev;
    for (auto& p : *v) {
      cudaEventDestroy(p.first);
      cudaEventDestroy(p.second);
    }
    v->clear();
  }
  return PST_OK;
}

int pst_timing_read(pst_ctx* c, double* ms, int64_t* launches) {
  if (!valid(c)) return PST_EINVAL;
  PST_CUDA(cudaStreamSynchronize(c->st));
  if (c->tev) {
    auto* v = (std::vector<std::pair<cudaEvent_t, cudaEvent_t>>*)c->tev;
    for (auto& p : *v) {
      float f = 0.f;
      PST_CUDA(cudaEventElapsedTime(&f, p.first, p.second));
      c->t_ms += f;
      c->t_calls++;
      cudaEventDestroy(p.first);
      cudaEventDestroy(p.second);
    }
    v->clear();
  }
  *ms = c->t_ms;
  *launches = c->t_launch;
  return PST_OK;
}

// debug: rank-move histogram of the selection (PASTILA_DBGF=16): 8 counters, read and cleared
int pst_debug_hist(pst_ctx* c, int64_t* out8) {
  if (!c->dbg) { pst_set_error("PASTILA_DBGF=16 not set"); return PST_ESTATE; }
  PST_CUDA(cudaDeviceSynchronize());
  PST_CUDA(cudaMemcpy(out8, c->dbg, 64, cudaMemcpyDeviceToHost));
  PST_CUDA(cudaMemset(c->dbg, 0, 64));
  return PST_OK;
}

// debug: AB matrix (w x T) and allP_BA (NC) of the first tile of the last profile launch
int pst_debug_last_tile(pst_ctx* c, double* ab, double* ba, int64_t* dims) {
  if (!c->dbg) { pst_set_error("PASTILA_DEBUG not set"); return PST_ESTATE; }
  PST_CUDA(cudaStreamSynchronize(c->st));
  dims[0] = c->dbg_w; dims[1] = c->dbg_T; dims[2] = c->dbg_NC;
  if (ab) PST_CUDA(cudaMemcpy(ab, c->scratch, (size_t)c->dbg_w * c->dbg_T * 8, cudaMemcpyDeviceToHost));
  if (ba) PST_CUDA(cudaMemcpy(ba, c->dbg, (size_t)c->dbg_NC * 8, cudaMemcpyDeviceToHost));
  return PST_OK;
}

}  // extern "C"
