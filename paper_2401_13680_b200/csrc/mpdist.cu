// MPdist profile tile kernel (north_star items 2+3): z-normalized distance
// rows by the centered diagonal recurrence, column minima (allP_BA), row
// sliding minima (allP_AB, van Herk / Gil-Werman blocks of width w), and the
// exact k-th smallest of the 2w-element P_ABBA multiset of every window.
//
// Reference semantics: zdist.py:74-123 (distances, constant-window and
// self-column conventions), mpdist.py:146-151 (sliding minima),
// mpdist.py:224-231 (column minima, concatenation, k-th smallest / max).
//
// One CTA = one segment s x one tile of T consecutive windows j in
// [J0, J0+T).  It sweeps the w query rows q = s*m + i; the tile needs columns
// [J0, J0+T+w-1).  All arithmetic is IEEE binary64.
//
// Work is expressed in "e-space": e = 1 - rho = d^2 / (2l).  d is monotone in
// e, so minima / order statistics are taken on e and the single sqrt is
// applied to the selected value (bit-exact monotone map).
//   cov(q,c)   centered covariance, SCAMP-style update:
//              cov(q+1,c+1) = cov(q,c) + df[q]*dg[c] + df[c]*dg[q]
//   e(q,c)     = bias[c] - cov*nrm[q]*nrm[c]         (non-constant query)
//              = cbias[c]                            (constant query)
//              = 0                                   (c == q, self column)
#include "common.cuh"
#include <algorithm>
#include <cstdlib>

namespace {

__device__ __forceinline__ double dmin(double a, double b) { return fmin(a, b); }

// k-th smallest (1-based) of the 2w keys of one window.  Keys are the bit
// patterns of non-negative doubles (order preserving).  A: w values in global
// scratch (stride ldA), B: w values in shared memory.  Exact: bracketing by
// counting passes; first pivot = previous window's answer (adjacent windows
// share most of their multiset), then interpolation, then key bisection.
__device__ long long select_kth(const double* __restrict__ A, int64_t ldA, const double* __restrict__ B,
                                int64_t w, int64_t k, long long pivot) {
  const int64_t M2 = 2 * w;
  if (M2 <= k) {  // mpdist.py:230-231: max fallback
    long long mx = 0;
    for (int64_t i = 0; i < w; ++i) {
      long long a = dkey(clamp0(A[i * ldA])), b = dkey(B[i]);
      mx = max(mx, max(a, b));
    }
    return mx;
  }
  long long lo = -1, hi = 0x7ff0000000000000LL;  // answer in (lo, hi]
  int64_t clo = 0, chi = M2;
  long long p = pivot;
  for (int it = 0; it < 200; ++it) {
    int64_t lt = 0, le = 0;
    long long mb = -1, ma = 0x7fffffffffffffffLL;
    for (int64_t i = 0; i < w; ++i) {
      long long v = dkey(clamp0(A[i * ldA]));
      lt += (v < p);
      le += (v <= p);
      if (v < p && v > mb) mb = v;
      if (v > p && v < ma) ma = v;
    }
    for (int64_t i = 0; i < w; ++i) {
      long long v = dkey(B[i]);
      lt += (v < p);
      le += (v <= p);
      if (v < p && v > mb) mb = v;
      if (v > p && v < ma) ma = v;
    }
    if (lt < k && k <= le) return p;
    if (k <= lt) {
      if (k == lt) return mb;
      hi = mb;
      chi = lt;
    } else {
      if (k == le + 1) return ma;
      lo = p;
      clo = le;
    }
    // next pivot in (lo, hi]
    long long np;
    if (it < 6 && hi < 0x7ff0000000000000LL) {
      double lv = lo < 0 ? 0.0 : kdbl(lo);
      double hv = kdbl(hi);
      double f = ((double)(k - clo) - 0.5) / (double)(chi - clo);
      double pv = lv + (hv - lv) * f;
      np = dkey(pv);
      if (np <= lo) np = lo + 1;
      if (np > hi) np = hi;
    } else if (hi >= 0x7ff0000000000000LL) {
      // no finite upper bracket yet: grow geometrically from the lower one
      double lv = lo < 0 ? 0.0 : kdbl(lo);
      np = dkey(lv > 0.0 ? lv * 2.0 : 1.0);
      if (np <= lo) np = lo + 1;
    } else {
      np = lo + (long long)(((unsigned long long)(hi - lo) + 1ull) >> 1);
      if (np <= lo) np = lo + 1;
    }
    p = np;
  }
  return p;  // unreachable in practice (bisection converges in <= 64 steps)
}

template <int P, int NT>
__global__ void __launch_bounds__(NT) k_mpdist(const MPArgs a) {
  extern __shared__ double sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = NT / 32;
  const int64_t l = a.l, w = a.w, T = a.T;
  const int64_t s = a.seg0 + blockIdx.y;
  const int64_t q0 = s * a.m;
  const int64_t J0 = (int64_t)blockIdx.x * T;
  const int64_t NJ = min(T, a.N - J0);
  const int64_t NC = NJ + w - 1;
  const int64_t NCmax = (int64_t)NT * P;
  double* xs = sm;             // [l]
  double* edge = xs + l;       // [w]
  double* E = edge + w;        // [NCmax] row e-values, later allP_BA
  double* SUF = E + NCmax;     // [NCmax]
  double* PRE = SUF + NCmax;   // [NCmax]
  double* xfer = PRE + NCmax;  // [64]
  double* red = xfer + 64;     // [2]
  double* ab = a.ab + ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * (w * T);
  const double* __restrict__ x = a.x;

  // ---- row-0 fresh dots: cov(q0, c) = sum_t (x[q0+t]-mu[q0]) * x[c+t] - mu[c]*sum_t(x[q0+t]-mu[q0])
  {
    const double mq = a.mu[q0];
    for (int64_t t = tid; t < l; t += NT) xs[t] = x[q0 + t] - mq;
    __syncthreads();
    if (tid == 0) {
      double s1 = 0.0;
      for (int64_t t = 0; t < l; ++t) s1 += xs[t];
      red[0] = s1;
    }
    __syncthreads();
  }
  double cov[P];
  {
    const double sx = red[0];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const int64_t cl = (int64_t)tid * P + p;
      double acc = 0.0;
      if (cl < NC) {
        const double* xc = x + J0 + cl;
        for (int64_t t = 0; t < l; ++t) acc = fma(xs[t], xc[t], acc);
        acc = fma(-a.mu[J0 + cl], sx, acc);
      }
      cov[p] = acc;
    }
  }
  __syncthreads();
  // ---- left edge (column J0) for rows 1..w-1: fresh dots against the centered column window
  {
    const double mc = a.mu[J0];
    for (int64_t t = tid; t < l; t += NT) xs[t] = x[J0 + t] - mc;
    __syncthreads();
    if (tid == 0) {
      double s1 = 0.0;
      for (int64_t t = 0; t < l; ++t) s1 += xs[t];
      red[1] = s1;
    }
    __syncthreads();
    const double sx = red[1];
    for (int64_t i = 1 + tid; i < w; i += NT) {
      const double* xq = x + q0 + i;
      double acc = 0.0;
      for (int64_t t = 0; t < l; ++t) acc = fma(xq[t], xs[t], acc);
      edge[i] = fma(-a.mu[q0 + i], sx, acc);
    }
  }
  // ---- per-column constants
  double dgc[P], dfc[P], nrmc[P], bic[P], colmin[P];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const int64_t cl = (int64_t)tid * P + p, c = J0 + cl;
    const bool ok = cl < NC;
    dgc[p] = (ok && c > 0) ? a.dg[c - 1] : 0.0;
    dfc[p] = (ok && c > 0) ? a.df[c - 1] : 0.0;
    nrmc[p] = ok ? a.nrm[c] : 0.0;
    bic[p] = ok ? a.bias[c] : 0.0;
    colmin[p] = PST_INF;
  }
  __syncthreads();

  const int64_t nblk = (NJ + w - 1) / w;  // van Herk blocks that contain windows
  const int64_t CH = (w + 31) / 32;
  for (int64_t i = 0; i < w; ++i) {
    const int64_t q = q0 + i;
    if (i > 0) {
      const double dfq = a.df[q - 1], dgq = a.dg[q - 1];
      double left = __shfl_up_sync(FULLMASK, cov[P - 1], 1);
      if (lane == 0 && warp > 0) left = xfer[((i - 1) & 1) * 32 + warp - 1];
#pragma unroll
      for (int p = P - 1; p >= 1; --p) cov[p] = fma(dfq, dgc[p], fma(dgq, dfc[p], cov[p - 1]));
      cov[0] = (tid == 0) ? edge[i] : fma(dfq, dgc[0], fma(dgq, dfc[0], left));
    }
    if (lane == 31) xfer[(i & 1) * 32 + warp] = cov[P - 1];
    const double nq = a.nrm[q];
    const bool qconst = (nq == 0.0);
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const int64_t cl = (int64_t)tid * P + p, c = J0 + cl;
      double e;
      if (qconst)
        e = (cl < NC) ? a.cbias[c] : 0.0;
      else
        e = fma(-(cov[p] * nq), nrmc[p], bic[p]);
      if (c == q) e = 0.0;
      if (cl >= NC) e = PST_INF;
      colmin[p] = dmin(colmin[p], e);
      E[cl] = e;
    }
    __syncthreads();
    // van Herk: warp per block pair (b, b+1); SUF over block b, PRE over block b+1
    for (int64_t b = warp; b < nblk; b += NW) {
      const int64_t bb = b * w, bn = bb + w;
      {
        const int64_t endb = min(bb + w, NC);
        const int64_t u0 = bb + lane * CH, u1 = min(u0 + CH, endb);
        double run = PST_INF;
        for (int64_t c = u1 - 1; c >= u0; --c) {
          run = dmin(run, E[c]);
          SUF[c] = run;
        }
        double tot = run;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) tot = dmin(tot, __shfl_down_sync(FULLMASK, tot, off));
        double carry = __shfl_down_sync(FULLMASK, tot, 1);
        if (lane == 31) carry = PST_INF;
        for (int64_t c = u0; c < u1; ++c) SUF[c] = dmin(SUF[c], carry);
      }
      {
        const int64_t endn = min(bn + w, NC);
        const int64_t u0 = bn + lane * CH, u1 = min(u0 + CH, endn);
        double run = PST_INF;
        for (int64_t c = u0; c < u1; ++c) {
          run = dmin(run, E[c]);
          PRE[c] = run;
        }
        double tot = run;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) tot = dmin(tot, __shfl_up_sync(FULLMASK, tot, off));
        double carry = __shfl_up_sync(FULLMASK, tot, 1);
        if (lane == 0) carry = PST_INF;
        for (int64_t c = u0; c < u1; ++c) PRE[c] = dmin(PRE[c], carry);
      }
      __syncwarp();
      double* abrow = ab + i * T;
      for (int64_t u = lane; u < w && bb + u < NJ; u += 32) {
        double v = SUF[bb + u];
        if (u > 0) v = dmin(v, PRE[bn + u - 1]);
        abrow[bb + u] = v;
      }
    }
    __syncthreads();
  }

  // ---- allP_BA (column minima), clamped at 0
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const int64_t cl = (int64_t)tid * P + p;
    if (cl < NC) E[cl] = clamp0(colmin[p]);
  }
  __syncthreads();
  if (a.dbg_ba && blockIdx.x == 0 && blockIdx.y == 0)
    for (int64_t c = tid; c < NC; c += NT) a.dbg_ba[c] = E[c];

  // ---- k-th smallest of P_ABBA per window; thread owns R consecutive windows
  const int64_t R = (NJ + NT - 1) / NT;
  const double twol = 2.0 * (double)l;
  double* Drow = a.D + (a.rowD0 + blockIdx.y) * a.ldD + J0;
  long long prev = -1;
  for (int64_t r = 0; r < R; ++r) {
    const int64_t j = (int64_t)tid * R + r;
    if (j >= NJ) break;
    long long piv = prev >= 0 ? prev : dkey(E[j + w / 2]);
    long long kk = select_kth(ab + j, T, E + j, w, a.k, piv);
    prev = kk;
    double ev = kdbl(kk);
    if (ev < 1e-15) ev = 0.0;  // rounding noise of an exact match (rho == 1)
    if (ev > 2.0) ev = 2.0;    // rho clipped at -1 (zdist.py:117)
    Drow[j] = sqrt(twol * ev);
  }
}

template <int P, int NT>
int launch_p(pst_ctx* c, const MPArgs& a, dim3 grid, size_t smem) {
  auto kern = k_mpdist<P, NT>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) {
    pst_set_error("cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    return PST_ECUDA;
  }
  kern<<<grid, NT, smem, c->st>>>(a);
  c->launches++;
  PST_CUDA(cudaGetLastError());
  return PST_OK;
}

template <int NT>
int launch_nt(pst_ctx* c, const MPArgs& a, dim3 grid, int P, size_t smem) {
  switch (P) {
    case 8: return launch_p<8, NT>(c, a, grid, smem);
    case 7: return launch_p<7, NT>(c, a, grid, smem);
    case 6: return launch_p<6, NT>(c, a, grid, smem);
    case 5: return launch_p<5, NT>(c, a, grid, smem);
    case 4: return launch_p<4, NT>(c, a, grid, smem);
    case 3: return launch_p<3, NT>(c, a, grid, smem);
    case 2: return launch_p<2, NT>(c, a, grid, smem);
    default: return launch_p<1, NT>(c, a, grid, smem);
  }
}

}  // namespace

// Profiles of segments [seg_lo, seg_hi) into D_dev rows 0.. (row stride ld).
int launch_mpdist(pst_ctx* c, int64_t m, int64_t l, int64_t k, int64_t seg_lo, int64_t seg_hi,
                  double* D_dev, int64_t ld) {
  PST_TRY(pst_ensure_len(c, l));
  const int64_t n = c->n, w = m - l + 1, Nl = n - l + 1, N = n - m + 1;
  // tile geometry: NC = NT*P columns, T = NC - w + 1 windows; aim for T >= 4w
  int P = 8, nt = (5 * w > 256 * 8) ? 512 : 256;
  const size_t smax = c->smem_optin ? c->smem_optin : 232448;
  auto smem_for = [&](int pp, int tt) {
    return (size_t)(l + w + 3 * (int64_t)tt * pp + 64 + 2) * sizeof(double);
  };
  while (P > 1 && smem_for(P, nt) > smax) P--;
  if (smem_for(P, nt) > smax || (int64_t)nt * P < w) {
    pst_set_error("snippet size %lld too large for shared-memory tiles", (long long)m);
    return PST_EINVAL;
  }
  const int64_t NCmax = (int64_t)nt * P;
  int64_t T = NCmax - w + 1;
  if (T > N) T = N;
  if (const char* tt = getenv("PASTILA_TILE_T")) { int64_t v = atoll(tt); if (v >= 1 && v < T) T = v; }
  const int64_t ntile = (N + T - 1) / T;
  // scratch: w*T doubles per CTA; bound CTAs per launch by the scratch budget
  const size_t per_cta = (size_t)w * (size_t)T * sizeof(double);
  size_t budget = (size_t)4 << 30;
  {
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) == cudaSuccess) budget = std::min(budget, fr / 4 + c->scratch_bytes);
  }
  int64_t segs_per = (int64_t)(budget / (per_cta * (size_t)ntile));
  if (segs_per < 1) segs_per = 1;
  if (segs_per > 65535) segs_per = 65535;
  if (segs_per > seg_hi - seg_lo) segs_per = seg_hi - seg_lo;
  PST_TRY(pst_ensure((void**)&c->scratch, &c->scratch_bytes, per_cta * (size_t)ntile * (size_t)segs_per));
  MPArgs a;
  a.x = c->x; a.mu = c->L.mc; a.nrm = c->L.nrm; a.bias = c->L.bias; a.cbias = c->L.cbias;
  a.df = c->L.df; a.dg = c->L.dg;
  a.n = n; a.l = l; a.m = m; a.w = w; a.k = k; a.Nl = Nl; a.N = N; a.T = T;
  a.D = D_dev; a.ldD = ld; a.ab = c->scratch;
  a.dbg_ba = nullptr;
  if (getenv("PASTILA_DEBUG")) {
    PST_TRY(pst_ensure((void**)&c->dbg, &c->dbg_bytes, (size_t)NCmax * 8));
    a.dbg_ba = c->dbg;
    c->dbg_T = T; c->dbg_NC = std::min(T, N) + w - 1; c->dbg_w = w;
  }
  if (const char* tt = getenv("PASTILA_TILE_T")) { int64_t v = atoll(tt); if (v >= 1 && v < T) T = v; a.T = T; }
  const size_t smem = smem_for(P, nt);
  for (int64_t s0 = seg_lo; s0 < seg_hi; s0 += segs_per) {
    const int64_t ns = std::min(segs_per, seg_hi - s0);
    a.seg0 = s0;
    a.rowD0 = s0 - seg_lo;
    dim3 grid((unsigned)ntile, (unsigned)ns);
    int r = (nt == 512) ? launch_nt<512>(c, a, grid, P, smem) : launch_nt<256>(c, a, grid, P, smem);
    if (r != PST_OK) return r;
  }
  return PST_OK;
}
