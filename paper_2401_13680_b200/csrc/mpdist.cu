// MPdist profile tile kernel (north_star items 2+3): z-normalized distance
// rows by the centered diagonal recurrence, column minima (allP_BA), row
// sliding minima (allP_AB, van Herk / Gil-Werman blocks of width w), and the
// k-th smallest of the 2w-element P_ABBA multiset of every window.
//
// Reference semantics: zdist.py:74-123 (distances, constant-window and
// self-column conventions), mpdist.py:146-151 (sliding minima),
// mpdist.py:224-231 (column minima, concatenation, k-th smallest / max).
//
// Two kernels per batch of segments, double-buffered over two streams:
//  * row loop (k_mpdist / k_mpdist2 / long-window layout): one CTA = one
//    segment s x one tile of T consecutive windows j in [J0, J0+T).  It sweeps
//    the w query rows q = s*m + i (one or two rows per barrier); the tile
//    needs columns [J0, J0+T+w-1).  Per row: distances, column minima, van Herk
//    row minima, and the AB row stored to HBM in lane-run order.
//  * selection (k_select_run): k-th smallest of every window's 2w values,
//    lanes sweeping runs of consecutive windows with the previous answer as
//    pivot (coalesced per-lane counts, warp-cooperative exact solves).
// The distance arithmetic is IEEE binary64.
//
// Work is expressed in "e-space": e = 1 - rho = d^2 / (2l).  d is monotone in
// e, so minima / order statistics are taken on e and the single sqrt is
// applied to the selected value (bit-exact monotone map).
//   cov(q,c)   centered covariance, SCAMP-style update:
//              cov(q+1,c+1) = cov(q,c) + df[q]*dg[c] + df[c]*dg[q]
//   e(q,c)     = bias[c] - cov*nrm[q]*nrm[c]         (non-constant query)
//              = cbias[c]                            (constant query)
//              = 0                                   (c == q, self column)
//
// Value type V of the minima and the order statistic (template parameter):
//  * double: the exact path -- profiles are d = sqrt(2l * e_k);
//  * int:    the key path -- every e is replaced by its 32-bit key, the high
//    word of its IEEE bit pattern read as a signed int.  For e >= +0 the key
//    is monotone non-decreasing in e; negative e (rounding residue of an exact
//    match, mapped to d = 0 anyway) get negative keys, below every e >= 0.
//    Minima commute with a monotone map, so every column minimum, sliding
//    minimum and the k-th smallest key are exactly key(exact value): the key
//    path returns key(e_k) of the exact path's e_k, i.e. e_k lies in the
//    2^-20-relative bucket [lo(key), hi(key)].  Same tiles, same fma order,
//    bit-identical e values; half the shared-memory / scratch bytes, and every
//    compare-and-select is one integer instruction instead of DSETP + 2 FSEL.
//    pastila.cu certifies every downstream decision from these buckets and
//    resolves the uncertain ones with exact values (k_window_exact below).
#include "common.cuh"
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <utility>
#include <vector>

namespace {

// NaN-free min/max (values are finite or +inf): 1 DSETP + 2 FSEL instead of the
// ~8-instruction IEEE fmin/fmax sequence; ints: one VIMNMX.
__device__ __forceinline__ double vmin(double a, double b) { return a < b ? a : b; }
__device__ __forceinline__ double vmax(double a, double b) { return a > b ? a : b; }
__device__ __forceinline__ int vmin(int a, int b) { return min(a, b); }
__device__ __forceinline__ int vmax(int a, int b) { return max(a, b); }

template <class V>
struct VT;
template <>
struct VT<double> {
  static __device__ __forceinline__ double inf() { return PST_INF; }
  static __device__ __forceinline__ double ninf() { return -PST_INF; }
  static __device__ __forceinline__ double of(double e) { return e; }
  static __device__ __forceinline__ double from_d(double v) { return v; }
  static __device__ __forceinline__ double quarter(double v) { return v * 0.25; }
};
template <>
struct VT<int> {
  static __device__ __forceinline__ int inf() { return INT_MAX; }
  static __device__ __forceinline__ int ninf() { return INT_MIN; }
  static __device__ __forceinline__ int of(double e) { return __double2hiint(e); }
  static __device__ __forceinline__ int from_d(double v) {  // key-space pivot arithmetic
    if (!(v > -2147483648.0)) return INT_MIN;
    if (v >= 2147483647.0) return INT_MAX;
    return (int)floor(v);
  }
  static __device__ __forceinline__ int quarter(int v) { return v - (2 << 20); }  // e/4: exponent - 2
};

// Exact repeats: bit-equal windows at different positions are at distance 0
// wherever they sit (zdist.py:98-106); the correlation path would leave a
// rounding residue there (up to ~1e-13 for long windows).  Each CTA marks,
// once, the columns whose window hash may equal one of its w query-window
// hashes (a 16384-bit, two-probe filter of the query hashes in shared
// memory); only marked columns are checked per row (hash, then samples).
constexpr int REP_WORDS = 512;
__device__ __noinline__ bool same_window(const double* __restrict__ x, const unsigned long long* __restrict__ hash,
                                         int64_t q, int64_t c, int l) {
  if (q == c || hash[q] != hash[c]) return false;
  for (int t = 0; t < l; ++t)
    if (__double_as_longlong(x[q + t]) != __double_as_longlong(x[c + t])) return false;
  return true;
}
__device__ __forceinline__ bool rep_probe(const unsigned* rmap, unsigned long long h) {
  const unsigned i1 = (unsigned)(h & 16383u), i2 = (unsigned)((h >> 20) & 16383u);
  return ((rmap[i1 >> 5] >> (i1 & 31)) & (rmap[i2 >> 5] >> (i2 & 31)) & 1u) != 0u;
}
// build the filter of the query hashes hash[q0 .. q0+w) (all threads; ends with a barrier)
__device__ __forceinline__ void rep_build(unsigned* rmap, const unsigned long long* __restrict__ hash, int64_t q0,
                                          int w, int tid, int nt) {
  for (int b = tid; b < REP_WORDS; b += nt) rmap[b] = 0u;
  __syncthreads();
  for (int i = tid; i < w; i += nt) {
    const unsigned long long h = hash[q0 + i];
    const unsigned i1 = (unsigned)(h & 16383u), i2 = (unsigned)((h >> 20) & 16383u);
    atomicOr(&rmap[i1 >> 5], 1u << (i1 & 31));
    atomicOr(&rmap[i2 >> 5], 1u << (i2 & 31));
  }
  __syncthreads();
}
// apply the rule to the marked columns of one row (rare path)
template <int P>
__device__ __noinline__ void rep_apply(double (&ed)[P], unsigned mask, const MPArgs& a, int64_t q, int64_t c0) {
#pragma unroll
  for (int p = 0; p < P; ++p)
    if ((mask >> p) & 1u)
      if (same_window(a.x, a.hash, q, c0 + p, (int)a.l)) ed[p] = 0.0;
}

// ---------------------------------------------------------------- selection
// Exact k-th smallest (1-based) of the 2w-element P_ABBA multiset of one
// window (mpdist.py:224-231): A = w row minima (AB scratch), B = w column
// minima (shared memory).  Helpers for the warp-cooperative exact path used
// for run starts and rare large rank moves (k_select_run below).
//
// exact warp max / min of doubles via two 32-bit REDUX steps on the
// order-preserving 64-bit key (sign-flipped bit pattern): tiny negative
// rounding residues of e = 1 - rho order correctly.  Keys: one REDUX.
__device__ __forceinline__ unsigned long long okey(double v) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double ukey(unsigned long long k) {
  const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)b);
}
__device__ __forceinline__ double warp_max(double v) {
  const unsigned long long k = okey(v);
  const unsigned kh = (unsigned)(k >> 32), kl = (unsigned)k;
  const unsigned h = __reduce_max_sync(FULLMASK, kh);
  const unsigned l = __reduce_max_sync(FULLMASK, kh == h ? kl : 0u);
  return ukey(((unsigned long long)h << 32) | l);
}
__device__ __forceinline__ double warp_min(double v) {
  const unsigned long long k = okey(v);
  const unsigned kh = (unsigned)(k >> 32), kl = (unsigned)k;
  const unsigned h = __reduce_min_sync(FULLMASK, kh);
  const unsigned l = __reduce_min_sync(FULLMASK, kh == h ? kl : 0xffffffffu);
  return ukey(((unsigned long long)h << 32) | l);
}
__device__ __forceinline__ int warp_max(int v) { return __reduce_max_sync(FULLMASK, v); }
__device__ __forceinline__ int warp_min(int v) { return __reduce_min_sync(FULLMASK, v); }

template <int TM, class V>
struct WinVals {
  V a[TM], b[TM];
};

template <int TM, class V>
__device__ __forceinline__ void count2(const WinVals<TM, V>& v, V p, int& lt, int& le) {
  int l1 = 0, l2 = 0;
#pragma unroll
  for (int t = 0; t < TM; ++t) {
    l1 += (v.a[t] < p) + (v.b[t] < p);
    l2 += (v.a[t] <= p) + (v.b[t] <= p);
  }
  lt = __reduce_add_sync(FULLMASK, l1);
  le = __reduce_add_sync(FULLMASK, l2);
}
template <int TM, class V>
__device__ __forceinline__ V below_max(const WinVals<TM, V>& v, V p) {  // largest element < p (or -inf)
  V m = VT<V>::ninf();
#pragma unroll
  for (int t = 0; t < TM; ++t) {
    m = vmax(m, v.a[t] < p ? v.a[t] : VT<V>::ninf());
    m = vmax(m, v.b[t] < p ? v.b[t] : VT<V>::ninf());
  }
  return warp_max(m);
}
template <int TM, class V>
__device__ __forceinline__ V above_min(const WinVals<TM, V>& v, V p) {  // smallest element > p (or +inf)
  V m = VT<V>::inf();
#pragma unroll
  for (int t = 0; t < TM; ++t) {
    m = vmin(m, v.a[t] > p ? v.a[t] : VT<V>::inf());
    m = vmin(m, v.b[t] > p ? v.b[t] : VT<V>::inf());
  }
  return warp_min(m);
}

// Next pivot of the exact bracketing search (heuristic only: correctness comes
// from the counts).  dist = rank distance from the current pivot to k.  Moves
// of 1-2 ranks take adjacent-value steps; longer moves extrapolate from the
// local spacing (pivot minus its neighbouring value, times the ranks still to
// go, doubled on every further one-sided step) until both brackets are known,
// then rank interpolation, then bisection.  Keys: the same arithmetic in key
// units (log-linear in e).
template <class V>
__device__ __forceinline__ V next_pivot(int it, bool down, int dist, V p, V nv, V lov, V hi, int clo, int chi,
                                        int k, bool haveLo, bool haveHi, int& grow) {
  double np;
  const double dp = (double)p, dnv = (double)nv, dlo = (double)lov, dhi = (double)hi;
  if (dist <= 2 && it < 6) {
    np = dnv;  // adjacent value (the bracket just found)
  } else if (haveLo && haveHi) {
    if (it < 12) {
      const float f = __fdividef((float)(k - clo) - 0.5f, (float)(chi - clo));
      np = dlo + (dhi - dlo) * (double)f;
    } else {
      np = 0.5 * (dlo + dhi);
    }
  } else {
    const double step = fabs(dp - dnv) * (double)(dist - 1) * (double)(1 << grow);
    grow = grow < 20 ? grow + 1 : grow;
    np = down ? dnv - step : dnv + step;
  }
  V r = VT<V>::from_d(np);
  if (haveLo) r = vmax(r, lov);
  if (haveHi) r = vmin(r, hi);
  if (r == p) r = nv;
  return r;
}

// lt0/le0 >= 0: the counts of p are already known (skip the first pass).
// Every iteration removes at least one element from the bracket [lov, hi]
// (both ends are elements), so 2w + 2 iterations always reach the answer.
template <int TM, class V>
__device__ V warp_select(const WinVals<TM, V>& v, int w, int k, V p, int lt0 = -1, int le0 = -1) {
  V lov = VT<V>::ninf(), hi = VT<V>::inf();
  int clo = 0, chi = 2 * w, grow = 0;
  bool haveLo = false, haveHi = false;
  for (int it = 0; it < 2 * w + 2; ++it) {
    int lt, le;
    if (it == 0 && lt0 >= 0) {
      lt = lt0;
      le = le0;
    } else {
      count2<TM, V>(v, p, lt, le);
    }
    if (lt < k && k <= le) return p;
    const bool down = k <= lt;
    V nv;
    int dist;
    if (down) {
      nv = below_max<TM, V>(v, p);  // #(<= nv) = lt
      if (k == lt) return nv;
      hi = nv;
      chi = lt;
      haveHi = true;
      dist = lt - k;
    } else {
      nv = above_min<TM, V>(v, p);  // smallest element > p
      if (k == le + 1) return nv;
      lov = nv;
      clo = le;
      haveLo = true;
      dist = k - le - 1;
    }
    p = next_pivot<V>(it, down, dist, p, nv, lov, hi, clo, chi, k, haveLo, haveHi, grow);
  }
  return p;
}

// van Herk row sliding minima for one row, register version.
// Blocks of w columns; a group of LPB lanes owns block b (SUF) and block b+1
// (PRE); lane chunks of CH (odd) consecutive columns; the combine
//   AB[u] = min(SUF_b[u], PRE_{b+1}[u-1])
// is done in registers (4 mins per element).  Results go to the CTA's row
// buffer srow[j] (window j of the tile); store_ab_row moves it to HBM.
struct VHGeom {
  int LPB, bpw, sub, ll, nblk, u0;
};

// E holds +inf beyond the tile's last column (rows never read past NC + w).
template <int CH, class V>
__device__ __forceinline__ void vh_row_reg(const V* __restrict__ E, int w, const VHGeom& g, int warp, int nw,
                                           V* __restrict__ srow) {
  for (int b0 = warp * g.bpw; b0 < g.nblk; b0 += nw * g.bpw) {  // warp-uniform trip count
    const bool live = b0 + g.sub < g.nblk;  // lane group has a block this iteration
    const int bb = (b0 + g.sub) * w, bn = bb + w;
    // positions past the block end read the block's last column instead of +inf:
    // it lies in every suffix of the block, and prefix values past the end are
    // never stored, so the minima are unchanged (groups without a block read block 0)
    const V* Es = E + (live ? bb : 0) + g.u0;
    const V* Ep = E + (live ? bn : w) + g.u0;
    const int tlim = w - 1 - g.u0;
    V sf[CH], pr[CH];
    V run = VT<V>::inf();
#pragma unroll
    for (int t = CH - 1; t >= 0; --t) {
      run = vmin(run, Es[min(t, tlim)]);
      sf[t] = run;
    }
    V totS = run;
    run = VT<V>::inf();
#pragma unroll
    for (int t = 0; t < CH; ++t) {
      run = vmin(run, Ep[min(t, tlim)]);
      pr[t] = run;
    }
    V totP = run;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      if (off < g.LPB) {
        const V ds = __shfl_down_sync(FULLMASK, totS, off, g.LPB);
        const V dp = __shfl_up_sync(FULLMASK, totP, off, g.LPB);
        totS = vmin(totS, ds);
        totP = vmin(totP, dp);
      }
    }
    V cs = __shfl_down_sync(FULLMASK, totS, 1, g.LPB);
    V cp = __shfl_up_sync(FULLMASK, totP, 1, g.LPB);
    if (g.ll == g.LPB - 1) cs = VT<V>::inf();
    if (g.ll == 0) cp = VT<V>::inf();
    const V C = vmin(cs, cp);
    if (live) {
      V* st = srow + bb;
#pragma unroll
      for (int t = 0; t < CH; ++t) {
        const int u = g.u0 + t;
        if (u < w) st[u] = (t > 0) ? vmin(vmin(sf[t], C), pr[t - 1]) : vmin(sf[t], C);
      }
    }
  }
}

// Two rows per barrier: 2*nblk (row, block) tasks over the lane groups, so
// that long windows (few blocks per tile) keep more warps busy.
template <int CH, class V>
__device__ __forceinline__ void vh_rows2_reg(const V* __restrict__ E0, const V* __restrict__ E1, int ntask, int w,
                                             const VHGeom& g, int warp, int nw, V* __restrict__ S0,
                                             V* __restrict__ S1) {
  for (int t0 = warp * g.bpw; t0 < ntask; t0 += nw * g.bpw) {  // warp-uniform trip count
    const int tau = t0 + g.sub;
    const bool live = tau < ntask;
    const bool second = tau >= g.nblk;
    const V* E = second ? E1 : E0;
    const int bb = (second ? tau - g.nblk : tau) * w, bn = bb + w;
    const V* Es = E + (live ? bb : 0) + g.u0;  // clamped reads, as in vh_row_reg
    const V* Ep = E + (live ? bn : w) + g.u0;
    const int tlim = w - 1 - g.u0;
    V sf[CH], pr[CH];
    V run = VT<V>::inf();
#pragma unroll
    for (int t = CH - 1; t >= 0; --t) {
      run = vmin(run, Es[min(t, tlim)]);
      sf[t] = run;
    }
    V totS = run;
    run = VT<V>::inf();
#pragma unroll
    for (int t = 0; t < CH; ++t) {
      run = vmin(run, Ep[min(t, tlim)]);
      pr[t] = run;
    }
    V totP = run;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      if (off < g.LPB) {
        const V ds = __shfl_down_sync(FULLMASK, totS, off, g.LPB);
        const V dp = __shfl_up_sync(FULLMASK, totP, off, g.LPB);
        totS = vmin(totS, ds);
        totP = vmin(totP, dp);
      }
    }
    V cs = __shfl_down_sync(FULLMASK, totS, 1, g.LPB);
    V cp = __shfl_up_sync(FULLMASK, totP, 1, g.LPB);
    if (g.ll == g.LPB - 1) cs = VT<V>::inf();
    if (g.ll == 0) cp = VT<V>::inf();
    const V C = vmin(cs, cp);
    if (live) {
      V* st = (second ? S1 : S0) + bb;
#pragma unroll
      for (int t = 0; t < CH; ++t) {
        const int u = g.u0 + t;
        if (u < w) st[u] = (t > 0) ? vmin(vmin(sf[t], C), pr[t - 1]) : vmin(sf[t], C);
      }
    }
  }
}

// One AB row from the CTA row buffer to HBM in lane-run order: window
// j = L*R + r (L = 0..31, r = 0..R-1) is stored at r*32 + L, so that the 32
// lanes of a selection warp, which sweep windows L*R + r for r = 0, 1, ...,
// read one contiguous 32-value line per row and step.  Thread tid always
// moves the same positions (lane L = tid%32, r = tid/32 + c*NT/32), so the
// offsets are set up once per tile and each element is one LDS + one STG;
// shared reads srow[L*R + r] have odd stride R (bank-conflict free), global
// stores are contiguous.  At most MAXC = P+1 elements per thread (T <= NT*P).
struct AbStore {
  int src, dst, cnt;
};
template <int NT>
__device__ __forceinline__ AbStore ab_store_setup(int NJ, int R, int tid) {
  const int L = tid & 31, r0 = tid >> 5;
  const int j0 = L * R + r0, jend = min(NJ, (L + 1) * R);
  AbStore s;
  s.src = j0;
  s.dst = r0 * 32 + L;
  s.cnt = j0 < jend ? (jend - j0 + NT / 32 - 1) / (NT / 32) : 0;
  return s;
}
template <int NT, int MAXC, class V>
__device__ __forceinline__ void store_ab_row(const AbStore& g, const V* __restrict__ srow, V* __restrict__ dst) {
  const V* s = srow + g.src;
  V* d = dst + g.dst;
#pragma unroll
  for (int c = 0; c < MAXC; ++c)
    if (c < g.cnt) d[c * NT] = s[c * (NT / 32)];
}

// ---- long windows: van Herk with every block split over several warps ----
// Scans per row: the suffix minima SUF of blocks 0..nblk-1 and the prefix
// minima PRE of blocks 0..nblk (block b = columns [b*w, (b+1)*w) of the tile,
// clipped to NC).  Each scan is cut into Q parts; a warp scans one part
// (phase 1: part-local scan + part total), and after a barrier adds the carry
// from the other parts' totals (phase 2).  The window combine
// AB[j] = min(SUF[j], PRE[j+w-1]) happens when the row is stored (PRE of
// block b ends in min(block b) = SUF_b[b*w], so u = 0 needs no special case).
struct SplitGeom {
  int nblk, Q, L, ntask;  // L = part length
};
__device__ __forceinline__ void split_task(const SplitGeom& sg, int t, int w, int NC, bool& suf, int& b, int& q,
                                           int& lo, int& hi) {
  const int nS = sg.nblk * sg.Q;
  suf = t < nS;
  const int tt = suf ? t : t - nS;
  b = tt / sg.Q;
  q = tt - b * sg.Q;
  const int bb = b * w;
  const int end = min(bb + w, NC);
  lo = min(bb + q * sg.L, end);
  hi = min(lo + sg.L, end);
}
// phase 1: part-local scans; TOT[(suf ? 0 : 1) * 32 * 16 + b * 16 + q] = part minimum
template <class V>
__device__ __forceinline__ void vh_split_scan(const V* __restrict__ E, V* __restrict__ SUF, V* __restrict__ PRE,
                                              V* __restrict__ TOT, const SplitGeom& sg, int w, int NC, int warp,
                                              int lane, int nw) {
  for (int t = warp; t < sg.ntask; t += nw) {
    bool suf;
    int b, q, lo, hi;
    split_task(sg, t, w, NC, suf, b, q, lo, hi);
    const int len = hi - lo;
    const int ch = (len + 31) >> 5;
    const int u0 = lo + lane * ch, u1 = min(u0 + ch, hi);
    V run = VT<V>::inf();
    if (suf) {
      for (int c = u1 - 1; c >= u0; --c) {
        run = vmin(run, E[c]);
        SUF[c] = run;
      }
    } else {
      for (int c = u0; c < u1; ++c) {
        run = vmin(run, E[c]);
        PRE[c] = run;
      }
    }
    V tot = run;  // carry between lanes of the part
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const V o = suf ? __shfl_down_sync(FULLMASK, tot, off) : __shfl_up_sync(FULLMASK, tot, off);
      if (suf ? lane + off < 32 : lane >= off) tot = vmin(tot, o);
    }
    V carry = suf ? __shfl_down_sync(FULLMASK, tot, 1) : __shfl_up_sync(FULLMASK, tot, 1);
    if (suf ? lane == 31 : lane == 0) carry = VT<V>::inf();
    if (suf)
      for (int c = u0; c < u1; ++c) SUF[c] = vmin(SUF[c], carry);
    else
      for (int c = u0; c < u1; ++c) PRE[c] = vmin(PRE[c], carry);
    // part minimum: lane 0 holds the suffix over the whole part, lane 31 the prefix
    const V pm = __shfl_sync(FULLMASK, tot, suf ? 0 : 31);
    if (lane == 0) TOT[(suf ? 0 : 512) + b * 16 + q] = pm;
  }
}
// phase 2: carries from the other parts of the same block
template <class V>
__device__ __forceinline__ void vh_split_carry(V* __restrict__ SUF, V* __restrict__ PRE, const V* __restrict__ TOT,
                                               const SplitGeom& sg, int w, int NC, int warp, int lane, int nw) {
  for (int t = warp; t < sg.ntask; t += nw) {
    bool suf;
    int b, q, lo, hi;
    split_task(sg, t, w, NC, suf, b, q, lo, hi);
    if (suf ? q == sg.Q - 1 : q == 0) continue;  // no parts beyond (SUF) / before (PRE)
    V v = VT<V>::inf();
    if (lane < sg.Q && (suf ? lane > q : lane < q)) v = TOT[(suf ? 0 : 512) + b * 16 + lane];
    const V carry = warp_min(v);
    if (suf)
      for (int c = lo + lane; c < hi; c += 32) SUF[c] = vmin(SUF[c], carry);
    else
      for (int c = lo + lane; c < hi; c += 32) PRE[c] = vmin(PRE[c], carry);
  }
}
// deferred store of a long-window row: AB[j] = min(SUF[j], PRE[j + w - 1]) in lane-run order
template <int NT, int MAXC, class V>
__device__ __forceinline__ void store_ab_combine(const AbStore& g, const V* __restrict__ SUF,
                                                 const V* __restrict__ PREw, V* __restrict__ dst) {
  const V* s = SUF + g.src;
  const V* p = PREw + g.src;
  V* d = dst + g.dst;
#pragma unroll
  for (int c = 0; c < MAXC; ++c)
    if (c < g.cnt) d[c * NT] = vmin(s[c * (NT / 32)], p[c * (NT / 32)]);
}

__host__ __device__ constexpr size_t align16(size_t b) { return (b + 15) & ~(size_t)15; }

// ---- TMA bulk staging of a tile's series samples (cp.async.bulk + mbarrier) --
// The row-0 and left-edge fresh dot products read the tile's column samples
// x[J0 .. J0+NC+l-1) and the segment's samples x[q0 .. q0+m); one elected
// thread copies both ranges global -> shared with 1-D bulk copies completing on
// an mbarrier (16-byte granularity: the ranges are widened to 16-byte aligned
// boundaries; the series buffer is padded, pastila.cu set_series).
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
struct BulkStage {
  const double* xt;  // tile samples: xt[t] = x[J0 + t]
  const double* xq;  // segment samples: xq[t] = x[q0 + t]
};
// stage [J0, J0+nt) and [q0, q0+nq) into buf (doubles, 16-byte aligned, room for nt+nq+4); all threads
// call it; returns views valid after the call (ends with the mbarrier wait)
__device__ __forceinline__ BulkStage bulk_stage(double* buf, unsigned long long* mbar, const double* x, int64_t J0,
                                                int nt, int64_t q0, int nq, int tid) {
  const int64_t a0 = J0 & ~1ll, a1 = q0 & ~1ll;                     // 16-byte aligned starts
  const int n0 = (int)(((J0 + nt) - a0 + 1) & ~1), n1 = (int)(((q0 + nq) - a1 + 1) & ~1);  // even counts
  double* b0 = buf;
  double* b1 = buf + n0;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(mbar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    const unsigned bytes = (unsigned)(n0 + n1) * 8u;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mbar)), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(b0)),
        "l"(x + a0), "r"((unsigned)n0 * 8u), "r"(smem_u32(mbar))
        : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(b1)),
        "l"(x + a1), "r"((unsigned)n1 * 8u), "r"(smem_u32(mbar))
        : "memory");
  }
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_u32(mbar))
        : "memory");
  }
  BulkStage st;
  st.xt = b0 + (J0 - a0);
  st.xq = b1 + (q0 - a1);
  return st;
}
__host__ __device__ inline size_t bulk_bytes(int64_t ncmax, int64_t l, int64_t m) {
  return (size_t)(ncmax + l + m + 8) * 8 + 16;  // both ranges + alignment slack + mbarrier
}

// Dynamic shared memory of the one-row kernel (k_mpdist): doubles first
// (row-0 staging xs[l], left-edge dots, per-row scalars, warp exchange), then
// the V arrays (e rows, AB row buffers; long windows: split van Herk buffers).
__host__ __device__ inline size_t smem_row1(bool klong, int64_t l, int64_t w, int64_t ncm, size_t sv) {
  if (!klong) return align16(align16((size_t)(l + 4 * w + 66) * 8) + (size_t)(4 * ncm) * sv) + bulk_bytes(ncm, l, l + w - 1);
  size_t b = align16((size_t)(w + 66) * 8) + (size_t)(6 * ncm + 1024) * sv;
  if ((size_t)l * 8 > (size_t)ncm * sv) b = align16(b) + (size_t)l * 8;  // xs does not fit E1
  return b;
}
// two rows per barrier (k_mpdist2)
__host__ __device__ inline size_t smem_row2(int64_t l, int64_t w, int64_t ncm, size_t sv) {
  return align16(align16((size_t)(l + 4 * w + 130) * 8) + (size_t)(8 * ncm) * sv) + bulk_bytes(ncm, l, l + w - 1);
}

// Row-0 fresh dots of a thread's P consecutive columns c0..c0+P-1:
//   cov[p] = fma(-mu[c], sum xs, sum_t fma(xs[t], x[c+t], .))   (t sequential per column)
// with the P chains interleaved and the x window sliding through registers
// (one new sample per step).  Same per-column operation order as a plain loop.
template <int P>
__device__ __forceinline__ void row0_dots(double (&cov)[P], const double* __restrict__ xs,
                                          const double* __restrict__ xJ, const double* __restrict__ muJ, double sx,
                                          int c0, int NC, int l) {
  double xw[P];
  const int lim = NC + l - 1;  // samples x[J0 + 0 .. J0 + NC + l - 2] exist
#pragma unroll
  for (int p = 0; p < P; ++p) {
    cov[p] = 0.0;
    xw[p] = (c0 + p < lim) ? xJ[c0 + p] : 0.0;
  }
#pragma unroll 4
  for (int t = 0; t < l; ++t) {
    const double xt = xs[t];
#pragma unroll
    for (int p = 0; p < P; ++p) cov[p] = fma(xt, xw[p], cov[p]);
#pragma unroll
    for (int p = 0; p < P - 1; ++p) xw[p] = xw[p + 1];
    xw[P - 1] = (c0 + P + t < lim) ? xJ[c0 + P + t] : 0.0;
  }
#pragma unroll
  for (int p = 0; p < P; ++p) cov[p] = (c0 + p < NC) ? fma(-muJ[c0 + p], sx, cov[p]) : 0.0;
}

template <int P, int NT, int CHM, class V>
__global__ void __launch_bounds__(NT, (NT <= 128 ? 4 : P <= 3 && NT <= 256 ? 3 : P <= 5 && NT <= 256 ? 2 : 1))
    k_mpdist(const MPArgs a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = NT / 32;
  constexpr int NCmax = NT * P;
  const int l = (int)a.l, w = (int)a.w, T = (int)a.T;
  const int64_t q0 = (a.segs ? a.segs[a.seg0 + blockIdx.y] : a.seg0 + blockIdx.y) * a.m;
  const int64_t J0 = (int64_t)blockIdx.x * a.T;
  const int NJ = (int)min(a.T, a.N - J0);
  const int NC = NJ + w - 1;
  // Long windows (CHM == 0, shared-memory van Herk) keep only edge[] of the
  // per-row arrays in shared memory -- their row scalars come from global
  // memory (L1 broadcast) -- and stage xs in E1 (unused until row 1) when it
  // fits, so a tile can hold P = 7 columns per thread.
  constexpr bool kLong = (CHM == 0);
  double *xs = nullptr, *edge, *rdf = nullptr, *rdg = nullptr, *rnq = nullptr, *xfer, *red;
  {
    double* db = (double*)smraw;
    if constexpr (!kLong) {
      xs = db;               // [l]
      edge = xs + l;         // [w]
      rdf = edge + w;        // [w] df[q-1] per row
      rdg = rdf + w;         // [w] dg[q-1] per row
      rnq = rdg + w;         // [w] nrm[q] per row
      xfer = rnq + w;        // [64]
    } else {
      edge = db;
      xfer = edge + w;
    }
    red = xfer + 64;         // [2]
  }
  V* E0 = (V*)(smraw + align16((size_t)((kLong ? w : l + 4 * w) + 66) * 8));  // [NCmax] e rows (even), later allP_BA
  V* E1 = E0 + NCmax;        // [NCmax] row e-values (odd rows)
  V* SR0 = E1 + NCmax;       // [NCmax] AB row buffer (even rows)
  V* SR1 = SR0 + NCmax;      // [NCmax] AB row buffer (odd rows)
  V* SUF = SR1 + NCmax;      // [NCmax] (shared-memory van Herk only)
  V* PRE = SUF + NCmax;      // [NCmax]
  V* TOT = PRE + NCmax;      // [1024] part minima of the split van Herk (long windows)
  if constexpr (kLong)
    xs = ((size_t)l * 8 <= (size_t)NCmax * sizeof(V)) ? (double*)E1
                                                       : (double*)((unsigned char*)smraw + align16(
                                                             align16((size_t)(w + 66) * 8) +
                                                             (size_t)(6 * NCmax + 1024) * sizeof(V)));
  V* E = E0;
  // AB scratch of this CTA: [w][Tp], each row in lane-run order (store_ab_row)
  const int R = (int)a.R, Tp = (int)a.Tp;
  V* ab = (V*)a.ab + ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * ((int64_t)w * Tp);
  const double* __restrict__ xJ = a.x + J0;
  const double* __restrict__ xQ = a.x + q0;
  const double* __restrict__ muJ = a.mu + J0;
  const double* __restrict__ muQ = a.mu + q0;
  if constexpr (!kLong) {  // samples of the fresh dots staged in shared memory by TMA bulk copies
    double* buf = (double*)align16((size_t)(SR1 + NCmax));
    const BulkStage st = bulk_stage(buf, (unsigned long long*)(buf + NCmax + l + a.m + 8), a.x, J0, NC + l - 1,
                                    q0, (int)a.m, tid);
    xJ = st.xt;
    xQ = st.xq;
  }

  // ---- row-0 fresh dots: cov(q0, c) = sum_t (x[q0+t]-mu[q0]) x[c+t] - mu[c] sum_t (x[q0+t]-mu[q0])
  {
    const double mq = muQ[0];
    for (int t = tid; t < l; t += NT) xs[t] = xQ[t] - mq;
    __syncthreads();
    if (tid == 0) {
      double s1 = 0.0;
      for (int t = 0; t < l; ++t) s1 += xs[t];
      red[0] = s1;
    }
    __syncthreads();
  }
  double cov[P];
  row0_dots<P>(cov, xs, xJ, muJ, red[0], tid * P, NC, l);
  __syncthreads();
  // ---- left edge (column J0) for rows 1..w-1: fresh dots against the centered column window
  {
    const double mc = muJ[0];
    for (int t = tid; t < l; t += NT) xs[t] = xJ[t] - mc;
    __syncthreads();
    if (tid == 0) {
      double s1 = 0.0;
      for (int t = 0; t < l; ++t) s1 += xs[t];
      red[1] = s1;
    }
    __syncthreads();
    const double sx = red[1];
    for (int i = 1 + tid; i < w; i += NT) {
      const double* xq = xQ + i;
      double acc = 0.0;
      for (int t = 0; t < l; ++t) acc = fma(xq[t], xs[t], acc);
      edge[i] = fma(-muQ[i], sx, acc);
    }
  }
  if constexpr (!kLong) {
    for (int i = tid; i < w; i += NT) {
      rdf[i] = i > 0 ? a.df[q0 + i - 1] : 0.0;
      rdg[i] = i > 0 ? a.dg[q0 + i - 1] : 0.0;
      rnq[i] = a.nrm[q0 + i];
    }
  }
  // ---- per-column constants
  double dgc[P], dfc[P], nrmc[P], bic[P];
  V colmin[P];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const int cl = tid * P + p;
    const bool ok = cl < NC;
    const int64_t c = J0 + cl;
    dgc[p] = (ok && c > 0) ? a.dg[c - 1] : 0.0;
    dfc[p] = (ok && c > 0) ? a.df[c - 1] : 0.0;
    nrmc[p] = ok ? a.nrm[c] : 0.0;
    bic[p] = ok ? a.bias[c] : PST_INF;
    colmin[p] = VT<V>::inf();
  }
  __shared__ unsigned rmap[REP_WORDS];
  if (a.rep)
    rep_build(rmap, a.hash, q0, w, tid, NT);  // ends with a barrier
  else
    __syncthreads();
  unsigned repm = 0;
#pragma unroll
  for (int p = 0; p < P; ++p)
    if (a.rep && tid * P + p < NC && rep_probe(rmap, a.hash[J0 + tid * P + p])) repm |= 1u << p;

  const int qloc = (int)(q0 - J0) - tid * P;  // my local index of the self column at row 0
  VHGeom g;
  {
    int LPB = 1;
    while (LPB < 32 && LPB * (CHM > 0 ? CHM : 1) < w) LPB *= 2;
    if (LPB < 8) LPB = 8;
    g.LPB = LPB;
    g.bpw = 32 / LPB;
    g.sub = lane / LPB;
    g.ll = lane % LPB;
    g.nblk = (NJ + w - 1) / w;
    g.u0 = g.ll * (CHM > 0 ? CHM : 1);
  }
  const bool tail = (tid + 1) * P > NC;  // this thread owns columns past the tile's last one
  const AbStore abst = ab_store_setup<NT>(NJ, R, tid);
  SplitGeom sg;
  {
    sg.nblk = (NJ + w - 1) / w;
    const int scans = 2 * sg.nblk + 1;
    sg.Q = max(1, min(16, NW / scans));
    sg.L = (w + sg.Q - 1) / sg.Q;
    sg.ntask = scans * sg.Q;
  }
  for (int i = 0; i < w; ++i) {
    double left = __shfl_up_sync(FULLMASK, cov[P - 1], 1);
    if (i > 0) {
      const double dfq = kLong ? __ldg(a.df + q0 + i - 1) : rdf[i];
      const double dgq = kLong ? __ldg(a.dg + q0 + i - 1) : rdg[i];
      if (lane == 0 && warp > 0) left = xfer[((i - 1) & 1) * 32 + warp - 1];
#pragma unroll
      for (int p = P - 1; p >= 1; --p) cov[p] = fma(dfq, dgc[p], fma(dgq, dfc[p], cov[p - 1]));
      cov[0] = (tid == 0) ? edge[i] : fma(dfq, dgc[0], fma(dgq, dfc[0], left));
    }
    if (lane == 31) xfer[(i & 1) * 32 + warp] = cov[P - 1];
    const double nq = kLong ? __ldg(a.nrm + q0 + i) : rnq[i];
    E = (i & 1) ? E1 : E0;
    V* Et = E + tid * P;
    if (nq != 0.0) {
      const double mnq = -nq;
      double ed[P];
#pragma unroll
      for (int p = 0; p < P; ++p) ed[p] = fma(cov[p] * mnq, nrmc[p], bic[p]);
      if (repm) rep_apply<P>(ed, repm, a, q0 + i, J0 + tid * P);
#pragma unroll
      for (int p = 0; p < P; ++p) {
        const V e = VT<V>::of(ed[p]);
        colmin[p] = vmin(colmin[p], e);
        Et[p] = e;
      }
      if (tail) {
#pragma unroll
        for (int p = 0; p < P; ++p)
          if (tid * P + p >= NC) Et[p] = VT<V>::inf();
      }
    } else {  // constant query window (row-uniform branch): zdist.py:111-112
#pragma unroll
      for (int p = 0; p < P; ++p) {
        const int cl = tid * P + p;
        const V e = (cl < NC) ? VT<V>::of(a.cbias[J0 + cl]) : VT<V>::inf();
        colmin[p] = vmin(colmin[p], e);
        Et[p] = e;
      }
    }
    {  // self column (zdist.py:121-122)
      const int ql = qloc + i;
      if (ql >= 0 && ql < P) Et[ql] = VT<V>::of(0.0);
    }
    __syncthreads();
    if constexpr (CHM > 0) {
      // the previous row's AB values are complete (written before this barrier)
      if (i > 0) store_ab_row<NT, P + 1, V>(abst, (i & 1) ? SR0 : SR1, ab + (int64_t)(i - 1) * Tp);
      vh_row_reg<CHM, V>(E, w, g, warp, NW, (i & 1) ? SR1 : SR0);
    } else {
      // buffers by row parity: (SUF, PRE) = (SUF, PRE) for even rows, (SR0, SR1) for odd rows
      if (i > 0) {
        const bool po = (i - 1) & 1;
        store_ab_combine<NT, P + 1, V>(abst, po ? SR0 : SUF, (po ? SR1 : PRE) + (w - 1),
                                       ab + (int64_t)(i - 1) * Tp);
      }
      V* sufc = (i & 1) ? SR0 : SUF;
      V* prec = (i & 1) ? SR1 : PRE;
      vh_split_scan<V>(E, sufc, prec, TOT, sg, w, NC, warp, lane, NW);
      __syncthreads();  // part totals complete
      vh_split_carry<V>(sufc, prec, TOT, sg, w, NC, warp, lane, NW);
    }
    // no trailing barrier: the next row writes the other E / row buffers; the
    // barrier after that row's writes orders this row's reads before row i+2's writes.
    // (TOT is rewritten only after the next row's first barrier.)
  }
  __syncthreads();
  if constexpr (CHM > 0) {
    store_ab_row<NT, P + 1, V>(abst, ((w - 1) & 1) ? SR1 : SR0, ab + (int64_t)(w - 1) * Tp);
  } else {
    const bool po = (w - 1) & 1;
    store_ab_combine<NT, P + 1, V>(abst, po ? SR0 : SUF, (po ? SR1 : PRE) + (w - 1), ab + (int64_t)(w - 1) * Tp);
  }
  E = E0;

  // ---- allP_BA (column minima), clamped; self columns [q0, q0+w) are exactly 0
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const int cl = tid * P + p;
    const int64_t c = J0 + cl;
    if (cl < NC) E[cl] = (c >= q0 && c < q0 + w) ? VT<V>::of(0.0) : colmin[p];
  }
  __syncthreads();
  {
    V* bag = (V*)a.ba + ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * NCmax;
    for (int c = tid; c < NC; c += NT) bag[c] = E[c];
    if (a.dbg_ba && !(a.dbg_flags & 16) && blockIdx.x == 0 && blockIdx.y == 0)
      for (int c = tid; c < NC; c += NT) ((V*)a.dbg_ba)[c] = E[c];
  }
}

// Row loop, two query rows per barrier (register van Herk only).  Each thread
// also carries one ghost column (its left neighbour's last column), so the
// second row of a pair needs no cross-warp exchange: at the start of a pair
// the neighbour's last two covariances arrive by shuffle (or, for lane 0, via
// shared memory from the previous warp), the ghost is advanced with the first
// row, and the second row uses it.  Same arithmetic as k_mpdist (bit-identical
// e values); half the barriers and twice the van Herk tasks per phase.
template <int P, int NT, int CHM, class V>
__global__ void __launch_bounds__(NT, (P <= 5 && NT <= 256 ? 2 : 1)) k_mpdist2(const MPArgs a) {
  static_assert(CHM > 0, "two-row kernel uses the register van Herk");
  extern __shared__ __align__(16) unsigned char smraw[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = NT / 32;
  constexpr int NCmax = NT * P;
  const int l = (int)a.l, w = (int)a.w;
  const int64_t q0 = (a.segs ? a.segs[a.seg0 + blockIdx.y] : a.seg0 + blockIdx.y) * a.m;
  const int64_t J0 = (int64_t)blockIdx.x * a.T;
  const int NJ = (int)min(a.T, a.N - J0);
  const int NC = NJ + w - 1;
  double* xs = (double*)smraw;   // [l]
  double* edge = xs + l;         // [w]
  double* rdf = edge + w;        // [w] df[q-1] per row
  double* rdg = rdf + w;         // [w] dg[q-1] per row
  double* rnq = rdg + w;         // [w] nrm[q] per row
  double* xfer = rnq + w;        // [2 parity][2][32] last two covariances of each warp
  double* red = xfer + 128;      // [2]
  V* EB = (V*)(smraw + align16((size_t)(l + 4 * w + 130) * 8));  // [4][NCmax] e rows; later allP_BA
  V* SRB = EB + 4 * NCmax;       // [4][NCmax] AB row buffers
  const int R = (int)a.R, Tp = (int)a.Tp;
  V* ab = (V*)a.ab + ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * ((int64_t)w * Tp);
  const double* __restrict__ muJ = a.mu + J0;
  const double* __restrict__ muQ = a.mu + q0;
  // samples of the fresh dots staged in shared memory by TMA bulk copies
  double* sbuf = (double*)align16((size_t)(SRB + 4 * NCmax));
  const BulkStage stg = bulk_stage(sbuf, (unsigned long long*)(sbuf + NCmax + l + a.m + 8), a.x, J0, NC + l - 1,
                                   q0, (int)a.m, tid);
  const double* __restrict__ xJ = stg.xt;
  const double* __restrict__ xQ = stg.xq;

  // ---- row-0 fresh dots (as k_mpdist)
  {
    const double mq = muQ[0];
    for (int t = tid; t < l; t += NT) xs[t] = xQ[t] - mq;
    __syncthreads();
    if (tid == 0) {
      double s1 = 0.0;
      for (int t = 0; t < l; ++t) s1 += xs[t];
      red[0] = s1;
    }
    __syncthreads();
  }
  double cov[P];
  row0_dots<P>(cov, xs, xJ, muJ, red[0], tid * P, NC, l);
  __syncthreads();
  {  // left edge (column J0) for rows 1..w-1
    const double mc = muJ[0];
    for (int t = tid; t < l; t += NT) xs[t] = xJ[t] - mc;
    __syncthreads();
    if (tid == 0) {
      double s1 = 0.0;
      for (int t = 0; t < l; ++t) s1 += xs[t];
      red[1] = s1;
    }
    __syncthreads();
    const double sx = red[1];
    for (int i = 1 + tid; i < w; i += NT) {
      const double* xq = xQ + i;
      double acc = 0.0;
      for (int t = 0; t < l; ++t) acc = fma(xq[t], xs[t], acc);
      edge[i] = fma(-muQ[i], sx, acc);
    }
  }
  for (int i = tid; i < w; i += NT) {
    rdf[i] = i > 0 ? a.df[q0 + i - 1] : 0.0;
    rdg[i] = i > 0 ? a.dg[q0 + i - 1] : 0.0;
    rnq[i] = a.nrm[q0 + i];
  }
  double dgc[P], dfc[P], nrmc[P], bic[P];
  V colmin[P];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const int cl = tid * P + p;
    const bool ok = cl < NC;
    const int64_t c = J0 + cl;
    dgc[p] = (ok && c > 0) ? a.dg[c - 1] : 0.0;
    dfc[p] = (ok && c > 0) ? a.df[c - 1] : 0.0;
    nrmc[p] = ok ? a.nrm[c] : 0.0;
    bic[p] = ok ? a.bias[c] : PST_INF;
    colmin[p] = VT<V>::inf();
  }
  // ghost column c0-1 (c0 = J0 + tid*P): its recurrence constants
  double dgG = 0.0, dfG = 0.0;
  if (tid > 0) {
    const int64_t cg = J0 + tid * P - 1;
    if (cg > 0 && tid * P - 1 < NC) {
      dgG = a.dg[cg - 1];
      dfG = a.df[cg - 1];
    }
  }
  if (lane == 31) {  // row-0 covariances for the next warp's lane 0
    xfer[0 * 64 + 0 * 32 + warp] = cov[P - 2 >= 0 ? P - 2 : 0];
    xfer[0 * 64 + 1 * 32 + warp] = cov[P - 1];
  }
  __shared__ unsigned rmap[REP_WORDS];
  if (a.rep)
    rep_build(rmap, a.hash, q0, w, tid, NT);  // ends with a barrier
  else
    __syncthreads();  // ends with a barrier
  unsigned repm = 0;
#pragma unroll
  for (int p = 0; p < P; ++p)
    if (a.rep && tid * P + p < NC && rep_probe(rmap, a.hash[J0 + tid * P + p])) repm |= 1u << p;

  const int qloc = (int)(q0 - J0) - tid * P;
  VHGeom g;
  {
    int LPB = 1;
    while (LPB < 32 && LPB * CHM < w) LPB *= 2;
    if (LPB < 8) LPB = 8;
    g.LPB = LPB;
    g.bpw = 32 / LPB;
    g.sub = lane / LPB;
    g.ll = lane % LPB;
    g.nblk = (NJ + w - 1) / w;
    g.u0 = g.ll * CHM;
  }
  const bool tail = (tid + 1) * P > NC;
  const AbStore abst = ab_store_setup<NT>(NJ, R, tid);

  // e-values of one row from its covariances -> shared row, column minima
  auto emit_row = [&](const double* cv, int i, V* Et) {
    const double nq = rnq[i];
    if (nq != 0.0) {
      const double mnq = -nq;
      double ed[P];
#pragma unroll
      for (int p = 0; p < P; ++p) ed[p] = fma(cv[p] * mnq, nrmc[p], bic[p]);
      if (repm) rep_apply<P>(ed, repm, a, q0 + i, J0 + tid * P);
#pragma unroll
      for (int p = 0; p < P; ++p) {
        const V e = VT<V>::of(ed[p]);
        colmin[p] = vmin(colmin[p], e);
        Et[p] = e;
      }
      if (tail) {
#pragma unroll
        for (int p = 0; p < P; ++p)
          if (tid * P + p >= NC) Et[p] = VT<V>::inf();
      }
    } else {  // constant query window (row-uniform branch): zdist.py:111-112
#pragma unroll
      for (int p = 0; p < P; ++p) {
        const int cl = tid * P + p;
        const V e = (cl < NC) ? VT<V>::of(a.cbias[J0 + cl]) : VT<V>::inf();
        colmin[p] = vmin(colmin[p], e);
        Et[p] = e;
      }
    }
    const int ql = qloc + i;  // self column (zdist.py:121-122)
    if (ql >= 0 && ql < P) Et[ql] = VT<V>::of(0.0);
  };

  const int npair = (w + 1) / 2;
  for (int it = 0; it < npair; ++it) {
    const int i0 = 2 * it, i1 = i0 + 1;
    const bool has1 = i1 < w;
    const int par = it & 1;
    // neighbour's last two covariances of the current state (row i0-1, or row 0 when it == 0)
    double g1 = __shfl_up_sync(FULLMASK, cov[P - 1], 1);
    double g2 = __shfl_up_sync(FULLMASK, cov[P >= 2 ? P - 2 : 0], 1);
    if (lane == 0 && warp > 0) {
      g2 = xfer[par * 64 + 0 * 32 + warp - 1];
      g1 = xfer[par * 64 + 1 * 32 + warp - 1];
    }
    double r0v[P];
    double gh;  // ghost column (c0-1) at row i0
    if (it == 0) {
#pragma unroll
      for (int p = 0; p < P; ++p) r0v[p] = cov[p];
      gh = g1;
    } else {
      const double dfq = rdf[i0], dgq = rdg[i0];
#pragma unroll
      for (int p = P - 1; p >= 1; --p) r0v[p] = fma(dfq, dgc[p], fma(dgq, dfc[p], cov[p - 1]));
      r0v[0] = (tid == 0) ? edge[i0] : fma(dfq, dgc[0], fma(dgq, dfc[0], g1));
      gh = fma(dfq, dgG, fma(dgq, dfG, g2));
    }
    emit_row(r0v, i0, EB + (par * 2 + 0) * NCmax + tid * P);
    if (has1) {
      const double dfq = rdf[i1], dgq = rdg[i1];
#pragma unroll
      for (int p = P - 1; p >= 1; --p) cov[p] = fma(dfq, dgc[p], fma(dgq, dfc[p], r0v[p - 1]));
      cov[0] = (tid == 0) ? edge[i1] : fma(dfq, dgc[0], fma(dgq, dfc[0], gh));
      emit_row(cov, i1, EB + (par * 2 + 1) * NCmax + tid * P);
      if (lane == 31) {
        xfer[(par ^ 1) * 64 + 0 * 32 + warp] = cov[P >= 2 ? P - 2 : 0];
        xfer[(par ^ 1) * 64 + 1 * 32 + warp] = cov[P - 1];
      }
    }
    __syncthreads();
    if (it > 0) {  // AB rows of the previous pair are complete
      const int pp = par ^ 1;
      store_ab_row<NT, P + 1, V>(abst, SRB + (pp * 2 + 0) * NCmax, ab + (int64_t)(i0 - 2) * Tp);
      store_ab_row<NT, P + 1, V>(abst, SRB + (pp * 2 + 1) * NCmax, ab + (int64_t)(i0 - 1) * Tp);
    }
    vh_rows2_reg<CHM, V>(EB + (par * 2 + 0) * NCmax, EB + (par * 2 + 1) * NCmax, g.nblk * (has1 ? 2 : 1), w, g,
                         warp, NW, SRB + (par * 2 + 0) * NCmax, SRB + (par * 2 + 1) * NCmax);
  }
  __syncthreads();
  {
    const int it = npair - 1, par = it & 1, i0 = 2 * it;
    store_ab_row<NT, P + 1, V>(abst, SRB + (par * 2 + 0) * NCmax, ab + (int64_t)i0 * Tp);
    if (i0 + 1 < w) store_ab_row<NT, P + 1, V>(abst, SRB + (par * 2 + 1) * NCmax, ab + (int64_t)(i0 + 1) * Tp);
  }
  V* E = EB;  // allP_BA (column minima), clamped; self columns [q0, q0+w) are exactly 0
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const int cl = tid * P + p;
    const int64_t c = J0 + cl;
    if (cl < NC) E[cl] = (c >= q0 && c < q0 + w) ? VT<V>::of(0.0) : colmin[p];
  }
  __syncthreads();
  {
    V* bag = (V*)a.ba + ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * NCmax;
    for (int c = tid; c < NC; c += NT) bag[c] = E[c];
    if (a.dbg_ba && !(a.dbg_flags & 16) && blockIdx.x == 0 && blockIdx.y == 0)
      for (int c = tid; c < NC; c += NT) ((V*)a.dbg_ba)[c] = E[c];
  }
}

// ---- row loop, thread-owned windows (w - 1 divisible by P) ------------------
// Deterministic sum of xs[0..l) by one warp: lane-strided partial sums, an
// xor tree, lane 0's result broadcast (the same procedure in k_window_exact).
__device__ __forceinline__ double warp_sum_fixed(const double* xs, int l, int lane) {
  double s = 0.0;
  for (int t = lane; t < l; t += 32) s += xs[t];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(FULLMASK, s, o);
  return __shfl_sync(FULLMASK, s, 0);
}

// Thread t owns columns [tP, tP+P) of the tile and windows [tP, tP+P).  With
// w - 1 = D*P, window tP+u ends at column (t+D)P + u, so its row minimum is
//   AB = min(SUF_t[u], MID_t, PRE_{t+D}[u]),  MID_t = min(bm[t+1 .. t+D-1]),
// where SUF/PRE are the thread-local suffix/prefix minima of a thread's P
// keys and bm its block minimum: 2 minima per key in registers, one 3-way
// minimum per window, vector shared-memory stores/loads of the PRE blocks, and
// the D-1 block minima (level 2) from shared memory -- read directly for
// D-1 <= 8, else through minima of 8 consecutive blocks (G).  No cross-lane
// scans.  AB rows go straight to the lane-run scratch layout of k_select_run.
// e values: same per-cell arithmetic as k_mpdist (row-0 and left-edge fresh
// dots in the same per-column fma order, same recurrence and e formula); the
// centered-window sums use warp_sum_fixed.
template <int P, int NT, class V>
__global__ void __launch_bounds__(NT, sizeof(V) == 4 ? 2 : 1) k_rowsP(const MPArgs a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NCmax = NT * P;
  const int l = (int)a.l, w = (int)a.w;
  const int D = (w - 1) / P, L2 = D - 1;
  const int64_t q0 = (a.segs ? a.segs[a.seg0 + blockIdx.y] : a.seg0 + blockIdx.y) * a.m;
  const int64_t J0 = (int64_t)blockIdx.x * a.T;
  const int NJ = (int)min(a.T, a.N - J0);
  const int NC = NJ + w - 1;
  double* xs = (double*)smraw;  // [l]
  double* edge = xs + l;        // [w]
  double* rdf = edge + w;       // [w]
  double* rdg = rdf + w;        // [w]
  double* rnq = rdg + w;        // [w]
  double* xfer = rnq + w;       // [2][32]
  double* red = xfer + 64;      // [2]
  constexpr int PS = P + 1;  // per-thread stride of the prefix-minima rows (odd: conflict-free)
  V* PREB = (V*)(smraw + align16((size_t)(l + 4 * w + 66) * 8));  // [2][NT*PS + 8*PS] prefix minima by row parity
  V* BMB = PREB + 2 * (NT * PS + 8 * PS);                          // [2][NT + 40] block minima
  V* GB = BMB + 2 * (NT + 40);                                     // [NT + 40] minima of 8 blocks
  V* BAs = GB;                                                     // allP_BA staging at the end (reuses GB..)
  const int R = (int)a.R, Tp = (int)a.Tp;
  V* ab = (V*)a.ab + ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * ((int64_t)w * Tp);
  const double* __restrict__ xJ = a.x + J0;
  const double* __restrict__ xQ = a.x + q0;
  const double* __restrict__ muJ = a.mu + J0;
  const double* __restrict__ muQ = a.mu + q0;
  const int c0 = tid * P;

  // ---- row-0 fresh dots (register-blocked: x window slides through registers)
  {
    const double mq = muQ[0];
    for (int t = tid; t < l; t += NT) xs[t] = xQ[t] - mq;
    __syncthreads();
    if (warp == 0) {
      const double s1 = warp_sum_fixed(xs, l, lane);
      if (lane == 0) red[0] = s1;
    }
    __syncthreads();
  }
  double cov[P];
  {
    const double sx = red[0];
    double xw[P];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      cov[p] = 0.0;
      xw[p] = (c0 + p < NC + l - 1) ? xJ[c0 + p] : 0.0;  // samples (not columns) of the window
    }
#pragma unroll 4
    for (int t = 0; t < l; ++t) {
      const double xt = xs[t];
#pragma unroll
      for (int p = 0; p < P; ++p) cov[p] = fma(xt, xw[p], cov[p]);
#pragma unroll
      for (int p = 0; p < P - 1; ++p) xw[p] = xw[p + 1];
      xw[P - 1] = (c0 + P + t < NC + l - 1) ? xJ[c0 + P + t] : 0.0;
    }
#pragma unroll
    for (int p = 0; p < P; ++p) cov[p] = (c0 + p < NC) ? fma(-muJ[c0 + p], sx, cov[p]) : 0.0;
  }
  __syncthreads();
  // ---- left edge (column J0) for rows 1..w-1
  {
    const double mc = muJ[0];
    for (int t = tid; t < l; t += NT) xs[t] = xJ[t] - mc;
    __syncthreads();
    if (warp == 0) {
      const double s1 = warp_sum_fixed(xs, l, lane);
      if (lane == 0) red[1] = s1;
    }
    __syncthreads();
    const double sx = red[1];
    for (int i = 1 + tid; i < w; i += NT) {
      const double* xq = xQ + i;
      double acc = 0.0;
      for (int t = 0; t < l; ++t) acc = fma(xq[t], xs[t], acc);
      edge[i] = fma(-muQ[i], sx, acc);
    }
  }
  for (int i = tid; i < w; i += NT) {
    rdf[i] = i > 0 ? a.df[q0 + i - 1] : 0.0;
    rdg[i] = i > 0 ? a.dg[q0 + i - 1] : 0.0;
    rnq[i] = a.nrm[q0 + i];
  }
  double dgc[P], dfc[P], nrmc[P];
  V colmin[P];
  double bic[P];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const int cl = c0 + p;
    const bool ok = cl < NC;
    const int64_t c = J0 + cl;
    dgc[p] = (ok && c > 0) ? a.dg[c - 1] : 0.0;
    dfc[p] = (ok && c > 0) ? a.df[c - 1] : 0.0;
    nrmc[p] = ok ? a.nrm[c] : 0.0;
    bic[p] = ok ? a.bias[c] : 1.0;
    colmin[p] = VT<V>::inf();
  }
  bool cst = false;  // a constant column (bias 0.5) among mine
#pragma unroll
  for (int p = 0; p < P; ++p) cst |= bic[p] != 1.0 && c0 + p < NC;
  const bool cst_tile = __syncthreads_or(cst);  // rare: constant windows in the tile
  const bool tail = c0 + P > NC;
  const bool self_tile = (q0 + w > J0) && (q0 < J0 + NC);
  const int qloc = (int)(q0 - J0) - c0;
  // lane-run scratch positions of my windows (window j -> (j % R) * 32 + j / R)
  int pos[P];
  const int nwok = min(P, max(0, NJ - c0));  // my valid windows
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const int j = c0 + p;
    pos[p] = (j % R) * 32 + j / R;
  }
  const bool rem_ok = tid + D < NT;  // my windows' last columns exist in this tile
  __shared__ unsigned rmap[REP_WORDS];
  if (a.rep)
    rep_build(rmap, a.hash, q0, w, tid, NT);  // ends with a barrier
  else
    __syncthreads();  // ends with a barrier
  unsigned repm = 0;
#pragma unroll
  for (int p = 0; p < P; ++p)
    if (a.rep && c0 + p < NC && rep_probe(rmap, a.hash[J0 + c0 + p])) repm |= 1u << p;

  for (int i = 0; i < w; ++i) {
    const int par = i & 1;
    double left = __shfl_up_sync(FULLMASK, cov[P - 1], 1);
    if (i > 0) {
      const double dfq = rdf[i], dgq = rdg[i];
      if (lane == 0 && warp > 0) left = xfer[((i - 1) & 1) * 32 + warp - 1];
#pragma unroll
      for (int p = P - 1; p >= 1; --p) cov[p] = fma(dfq, dgc[p], fma(dgq, dfc[p], cov[p - 1]));
      cov[0] = (tid == 0) ? edge[i] : fma(dfq, dgc[0], fma(dgq, dfc[0], left));
    }
    if (lane == 31) xfer[par * 32 + warp] = cov[P - 1];
    const double nq = rnq[i];
    V kk[P];
    if (nq != 0.0) {
      const double mnq = -nq;
      double ed[P];
      if (!cst_tile) {  // every column non-constant: bias 1.0
#pragma unroll
        for (int p = 0; p < P; ++p) ed[p] = fma(cov[p] * mnq, nrmc[p], 1.0);
      } else {
#pragma unroll
        for (int p = 0; p < P; ++p) ed[p] = fma(cov[p] * mnq, nrmc[p], (c0 + p < NC) ? a.bias[J0 + c0 + p] : PST_INF);
      }
      if (repm) rep_apply<P>(ed, repm, a, q0 + i, J0 + c0);
#pragma unroll
      for (int p = 0; p < P; ++p) kk[p] = VT<V>::of(ed[p]);
    } else {  // constant query window (row-uniform branch): zdist.py:111-112
#pragma unroll
      for (int p = 0; p < P; ++p) kk[p] = (c0 + p < NC) ? VT<V>::of(a.cbias[J0 + c0 + p]) : VT<V>::inf();
    }
    if (tail) {
#pragma unroll
      for (int p = 0; p < P; ++p)
        if (c0 + p >= NC) kk[p] = VT<V>::inf();
    }
    if (self_tile) {  // self column (zdist.py:121-122)
      const int ql = qloc + i;
#pragma unroll
      for (int p = 0; p < P; ++p)
        if (ql == p) kk[p] = VT<V>::of(0.0);
    }
    V sf[P], pr[P];
    sf[P - 1] = kk[P - 1];
#pragma unroll
    for (int p = P - 2; p >= 0; --p) sf[p] = vmin(kk[p], sf[p + 1]);
    pr[0] = kk[0];
#pragma unroll
    for (int p = 1; p < P; ++p) pr[p] = vmin(pr[p - 1], kk[p]);
#pragma unroll
    for (int p = 0; p < P; ++p) colmin[p] = vmin(colmin[p], kk[p]);
    V* PRE = PREB + par * (NT * PS + 8 * PS);
    V* BM = BMB + par * (NT + 40);
#pragma unroll
    for (int p = 0; p < P; ++p) PRE[tid * PS + p] = pr[p];
    BM[tid] = sf[0];
    __syncthreads();
    V mid = VT<V>::inf();
    if (L2 <= 8) {
      for (int d = 1; d <= L2; ++d) mid = vmin(mid, BM[tid + d]);
    } else {
      V g = BM[tid];
#pragma unroll
      for (int d = 1; d < 8; ++d) g = vmin(g, BM[min(tid + d, NT - 1)]);
      GB[tid] = g;
      __syncthreads();
      int d = 1;
      for (; d + 8 <= L2; d += 8) mid = vmin(mid, GB[min(tid + d, NT - 1)]);
      mid = vmin(mid, GB[min(tid + L2 - 7, NT - 1)]);
    }
    if (rem_ok) {
      const V* rp = PRE + (tid + D) * PS;
      V* abrow = ab + (int64_t)i * Tp;
#pragma unroll
      for (int p = 0; p < P; ++p)
        if (p < nwok) abrow[pos[p]] = vmin(vmin(sf[p], mid), rp[p]);
    }
  }
  // ---- allP_BA (column minima); self columns [q0, q0+w) are exactly 0
  __syncthreads();
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const int cl = c0 + p;
    const int64_t c = J0 + cl;
    if (cl < NC) BAs[cl] = (c >= q0 && c < q0 + w) ? VT<V>::of(0.0) : colmin[p];
  }
  __syncthreads();
  {
    V* bag = (V*)a.ba + ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * NCmax;
    for (int c = tid; c < NC; c += NT) bag[c] = BAs[c];
    if (a.dbg_ba && !(a.dbg_flags & 16) && blockIdx.x == 0 && blockIdx.y == 0)
      for (int c = tid; c < NC; c += NT) ((V*)a.dbg_ba)[c] = BAs[c];
  }
}
__host__ __device__ inline size_t smem_rowsP(int64_t l, int64_t w, int NT, int P, size_t sv) {
  // doubles, then PREB [2][NCmax + 8P], BMB [2][NT + 40], GB / BA staging [max(NT + 40, NCmax)]
  const size_t ncm = (size_t)NT * P;
  return align16((size_t)(l + 4 * w + 66) * 8) + (2 * ((size_t)NT * (P + 1) + 8 * (P + 1)) + 2 * (NT + 40) +
                                                 std::max((size_t)NT + 40, ncm)) * sv;
}

// Generic (memory-resident) variant of the warp selection for 2w > 32*2*16.
template <class V>
struct MemWin {
  const V* A;  // row minima, stride sa
  const V* B;  // column minima, contiguous
  int w;
  int64_t sa;
};
template <class V>
__device__ __forceinline__ void count2m(const MemWin<V>& v, int lane, V p, int& lt, int& le) {
  int l1 = 0, l2 = 0;
  for (int i = lane; i < v.w; i += 32) {
    const V x = v.A[i * v.sa], y = v.B[i];
    l1 += (x < p) + (y < p);
    l2 += (x <= p) + (y <= p);
  }
  lt = __reduce_add_sync(FULLMASK, l1);
  le = __reduce_add_sync(FULLMASK, l2);
}
template <class V>
__device__ __forceinline__ V below_maxm(const MemWin<V>& v, int lane, V p) {
  V m = VT<V>::ninf();
  for (int i = lane; i < v.w; i += 32) {
    const V x = v.A[i * v.sa], y = v.B[i];
    m = vmax(m, x < p ? x : VT<V>::ninf());
    m = vmax(m, y < p ? y : VT<V>::ninf());
  }
  return warp_max(m);
}
template <class V>
__device__ __forceinline__ V above_minm(const MemWin<V>& v, int lane, V p) {
  V m = VT<V>::inf();
  for (int i = lane; i < v.w; i += 32) {
    const V x = v.A[i * v.sa], y = v.B[i];
    m = vmin(m, x > p ? x : VT<V>::inf());
    m = vmin(m, y > p ? y : VT<V>::inf());
  }
  return warp_min(m);
}
template <class V>
__device__ V warp_select_mem(const MemWin<V>& v, int lane, int k, V p, int lt0 = -1, int le0 = -1) {
  const int w = v.w;
  V lov = VT<V>::ninf(), hi = VT<V>::inf();
  int clo = 0, chi = 2 * w, grow = 0;
  bool haveLo = false, haveHi = false;
  for (int it = 0; it < 2 * w + 2; ++it) {  // >= 1 element leaves the bracket per iteration
    int lt, le;
    if (it == 0 && lt0 >= 0) {
      lt = lt0;
      le = le0;
    } else {
      count2m<V>(v, lane, p, lt, le);
    }
    if (lt < k && k <= le) return p;
    const bool down = k <= lt;
    V nv;
    int dist;
    if (down) {
      nv = below_maxm<V>(v, lane, p);
      if (k == lt) return nv;
      hi = nv;
      chi = lt;
      haveHi = true;
      dist = lt - k;
    } else {
      nv = above_minm<V>(v, lane, p);
      if (k == le + 1) return nv;
      lov = nv;
      clo = le;
      haveLo = true;
      dist = k - le - 1;
    }
    p = next_pivot<V>(it, down, dist, p, nv, lov, hi, clo, chi, k, haveLo, haveHi, grow);
  }
  return p;
}

// Selection kernel: one CTA per (tile, segment) of the row kernel's scratch,
// NWS warps.  Lane L of a warp owns the run of consecutive windows
// j = L*R + r, r in [r0, r1) (the warp's share of the run length R); the AB
// scratch is stored in lane-run order, so at step r the warp's 32 lanes read
// one contiguous line per row, and lane L's column-minima window
// BA[j .. j+w) in shared memory has lane stride R (odd: conflict free).
//
// Step r: every lane counts #(< p) and #(<= p) of its own 2w values with the
// previous window's answer p as pivot: the w row minima in one coalesced pass
// (~4 instructions per element), the w column minima incrementally (the B
// window slides by one; recounted whenever p changes).  Where p is still the k-th smallest (53-75% of windows,
// depending on m) the window is done; the other lanes' windows are solved
// one after another by the whole warp (warp_select: the column is gathered
// into registers, lane l holding elements l, l+32, ...; the known counts seed
// the bracketing search).  Each lane's first window is solved the same way.
__device__ __forceinline__ double e_to_dist(double ev, double twol) {
  if (ev < 1e-15) ev = 0.0;  // rounding noise of an exact match (rho == 1)
  if (ev > 2.0) ev = 2.0;    // rho clipped at -1 (zdist.py:117)
  return sqrt(twol * ev);
}
// profile output: exact path d = f(e) (double rows), key path: the key itself (int rows)
__device__ __forceinline__ void put_out(double* row, int64_t j, double v, double twol) { row[j] = e_to_dist(v, twol); }
__device__ __forceinline__ void put_out(int* row, int64_t j, int v, double) { row[j] = v; }
template <class V>
struct OutT {
  using type = double;
};
template <>
struct OutT<int> {
  using type = int;
};

// exact k-th smallest of window (lane L, step r), whole warp; TM = 0: long
// windows, values re-read from memory on every pass.  fresh: no pivot yet
// (answers may be tiny negative residues, so no sentinel value is used).
// Also returns #(B < ans) and #(B <= ans) for the lane's incremental B counts.
template <int TM, class V>
__device__ __forceinline__ V solve_col(const V* __restrict__ Ac, const V* Bc, int Tp, int w, int k, int lane,
                                       bool fresh, V piv, int lt0, int le0, int& ltB, int& leB, V* colbuf) {
  V x;
  int b1 = 0, b2 = 0;
  if constexpr (TM > 0) {
    WinVals<TM, V> v;
#pragma unroll
    for (int t = 0; t < TM; ++t) {
      const int i = lane + 32 * t;
      const bool ok = i < w;
      v.a[t] = ok ? __ldg(Ac + (int64_t)i * Tp) : VT<V>::inf();
      v.b[t] = ok ? Bc[i] : VT<V>::inf();
    }
    if (fresh)
      piv = vmax(VT<V>::quarter(warp_max(v.a[0] < VT<V>::inf() ? v.a[0] : VT<V>::ninf())), VT<V>::of(0.0));
    x = warp_select<TM, V>(v, w, k, piv, lt0, le0);
#pragma unroll
    for (int t = 0; t < TM; ++t) {
      b1 += v.b[t] < x;
      b2 += v.b[t] <= x;
    }
  } else {  // long windows: the gathered column is staged once in the warp's shared buffer
#pragma unroll 8
    for (int i = lane; i < w; i += 32) colbuf[i] = __ldg(Ac + (int64_t)i * Tp);
    __syncwarp();
    MemWin<V> v{colbuf, Bc, w, 1};
    if (fresh) piv = vmax(VT<V>::quarter(warp_max(lane < w ? colbuf[lane] : VT<V>::ninf())), VT<V>::of(0.0));
    x = warp_select_mem<V>(v, lane, k, piv, lt0, le0);
    for (int i = lane; i < w; i += 32) {
      b1 += Bc[i] < x;
      b2 += Bc[i] <= x;
    }
    __syncwarp();  // colbuf is rewritten by the next solve
  }
  ltB = __reduce_add_sync(FULLMASK, b1);
  leB = __reduce_add_sync(FULLMASK, b2);
  return x;
}
template <int TM, class V>
__device__ __forceinline__ V solve_window(const V* __restrict__ ab, const V* BA, int w, int k, int R, int Tp, int L,
                                          int r, int lane, bool fresh, V piv, int lt0, int le0, int& ltB, int& leB,
                                          V* colbuf) {
  return solve_col<TM, V>(ab + r * 32 + L, BA + L * R + r, Tp, w, k, lane, fresh, piv, lt0, le0, ltB, leB, colbuf);
}

// Lane pass of one window: counts of the pivot p and the two nearest values
// on each side of it (multisets: duplicates kept), so that rank moves of one
// or two resolve without the warp-cooperative solve.
template <class V>
__device__ __forceinline__ void lane_acc(V v, V p, int& lt, int& le, V& b1, V& b2, V& a1, V& a2) {
  const bool l = v < p, e = v <= p;
  lt += l;
  le += e;
  const V vb = l ? v : VT<V>::ninf();
  const V va = e ? VT<V>::inf() : v;
  b2 = vmax(b2, vmin(b1, vb));
  b1 = vmax(b1, vb);
  a2 = vmin(a2, vmax(a1, va));
  a1 = vmin(a1, va);
}

template <int NWS, int TM, class V, bool LP>
__global__ void __launch_bounds__(NWS * 32, 1) k_select_run(const MPArgs a, int NCmax) {
  using O = typename OutT<V>::type;
  extern __shared__ __align__(16) unsigned char smsel[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int w = (int)a.w, R = (int)a.R, Tp = (int)a.Tp, k = (int)a.k;
  const int64_t J0 = (int64_t)blockIdx.x * a.T;
  const int NJ = (int)min(a.T, a.N - J0);
  const int NC = NJ + w - 1;
  const int64_t cta = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;
  const V* __restrict__ ab = (const V*)a.ab + cta * ((int64_t)w * Tp);
  const V* __restrict__ bag = (const V*)a.ba + cta * NCmax;
  V* BA = (V*)smsel;
  V* colbuf = BA + NCmax + warp * w;  // [w] per warp, long windows (TM == 0) only
  for (int c = tid; c < NC; c += NWS * 32) BA[c] = bag[c];
  __syncthreads();
  const double twol = 2.0 * (double)a.l;
  O* Drow = (O*)a.D + (a.rowD0 + blockIdx.y) * a.ldD + J0;
  const int rper = (R + NWS - 1) / NWS;
  const int r0 = warp * rper, r1 = min(R, r0 + rper);
  if (r0 >= r1) return;
  const int jl = lane * R;  // first window of this lane's run

  if (2 * w <= k) {  // the k-th smallest is the maximum (mpdist.py:229-230)
    for (int r = r0; r < r1; ++r) {
      const int j = jl + r;
      const bool ok = j < NJ;
      const V* Ap = ab + r * 32 + lane;
      const V* Bp = BA + (ok ? j : 0);
      V mx = VT<V>::ninf();
#pragma unroll 8
      for (int i = 0; i < w; ++i) mx = vmax(mx, vmax(__ldg(Ap + (int64_t)i * Tp), Bp[i]));
      if (ok) put_out(Drow, j, mx, twol);
    }
    return;
  }

  // first window of every lane's run, lanes in turn; lane L starts from lane
  // L-1's answer (its window lies R to the left).  ltB/leB: this lane's counts
  // of its B window (BA[j .. j+w)) below / at-or-below p, kept incrementally.
  V p = VT<V>::of(0.0);
  int ltB = 0, leB = 0;
  {
    V prev = VT<V>::of(0.0);
    for (int L = 0; L < 32; ++L) {
      if (L * R + r0 >= NJ || (a.dbg_flags & 4)) break;  // warp-uniform
      int b1, b2;
      prev = solve_window<TM, V>(ab, BA, w, k, R, Tp, L, r0, lane, L == 0, prev, -1, -1, b1, b2, colbuf);
      if (lane == L) {
        p = prev;
        ltB = b1;
        leB = b2;
      }
    }
    if (jl + r0 < NJ) put_out(Drow, jl + r0, p, twol);
  }
  if constexpr (LP) {
    // every window: one lane-local pass over its 2w values (A from the scratch,
    // B from shared memory); only rank moves beyond 2 go to the warp
    for (int r = r0 + 1; r < r1; ++r) {
      const int j = jl + r;
      const bool ok = j < NJ;
      const V* Ap = ab + r * 32 + lane;
      const V* Bp = BA + (ok ? j : 0);
      int lt = 0, le = 0;
      V b1 = VT<V>::ninf(), b2 = VT<V>::ninf(), a1 = VT<V>::inf(), a2 = VT<V>::inf();
      constexpr int kUn = TM >= 7 || TM == 0 ? 16 : 8;
#pragma unroll kUn
      for (int i = 0; i < w; ++i) {
        lane_acc<V>(__ldg(Ap + (int64_t)i * Tp), p, lt, le, b1, b2, a1, a2);
        lane_acc<V>(Bp[i], p, lt, le, b1, b2, a1, a2);
      }
      V ans = p;
      bool done = lt < k && k <= le;
      if (a.dbg_ba && (a.dbg_flags & 16) && ok) {  // instrumentation: rank-move histogram (PASTILA_DBGF=16)
        const int mv = (lt < k && k <= le) ? 0 : (k <= lt ? lt - k + 1 : k - le);
        const int b = mv == 0 ? 0 : mv == 1 ? 1 : mv == 2 ? 2 : mv <= 4 ? 3 : mv <= 8 ? 4 : mv <= 16 ? 5 : 6;
        atomicAdd((unsigned long long*)a.dbg_ba + b, 1ull);
      }
      if (!done) {
        if (k <= lt) {
          const int need = lt - k + 1;  // rank from the top among the values below p
          if (need == 1) { ans = b1; done = true; }
          else if (need == 2) { ans = b2; done = true; }
        } else {
          const int need = k - le;  // rank among the values above p
          if (need == 1) { ans = a1; done = true; }
          else if (need == 2) { ans = a2; done = true; }
        }
      }
      unsigned pend = __ballot_sync(FULLMASK, ok && !done);
      if (a.dbg_flags & 1) pend = 0;
      while (pend) {
        const int L = __ffs(pend) - 1;
        pend &= pend - 1;
        const V pl = __shfl_sync(FULLMASK, p, L);
        const int ltl = __shfl_sync(FULLMASK, lt, L), lel = __shfl_sync(FULLMASK, le, L);
        int b1c, b2c;
        const V x = solve_window<TM, V>(ab, BA, w, k, R, Tp, L, r, lane, false, pl, ltl, lel, b1c, b2c, colbuf);
        if (lane == L) ans = x;
      }
      p = ans;
      if (ok) put_out(Drow, j, p, twol);
    }
    return;
  }
  for (int r = r0 + 1; r < r1; ++r) {
    const int j = jl + r;
    const bool ok = j < NJ;
    const V* Ap = ab + r * 32 + lane;
    if (ok) {  // slide the B window: BA[j-1] leaves, BA[j+w-1] enters
      const V out = BA[j - 1], in = BA[j + w - 1];
      ltB += (in < p) - (out < p);
      leB += (in <= p) - (out <= p);
    }
    int lt = ltB, le = leB;
    if (!(a.dbg_flags & 2)) {
      // loads in flight per lane: the pass is a chain of HBM round trips (measured best)
      constexpr int kSelUnroll = TM >= 7 || TM == 0 ? 32 : TM >= 4 ? 16 : 8;
#pragma unroll kSelUnroll
      for (int i = 0; i < w; ++i) {
        const V va = __ldg(Ap + (int64_t)i * Tp);
        lt += va < p;
        le += va <= p;
      }
    }
    unsigned pend = __ballot_sync(FULLMASK, ok && !(lt < k && k <= le));
    if (a.dbg_flags & 1) pend = 0;
    while (pend) {
      const int L = __ffs(pend) - 1;
      pend &= pend - 1;
      const V pl = __shfl_sync(FULLMASK, p, L);
      const int ltl = __shfl_sync(FULLMASK, lt, L), lel = __shfl_sync(FULLMASK, le, L);
      int b1, b2;
      const V x = solve_window<TM, V>(ab, BA, w, k, R, Tp, L, r, lane, false, pl, ltl, lel, b1, b2, colbuf);
      if (lane == L) {
        p = x;
        ltB = b1;
        leB = b2;
      }
    }
    if (ok) put_out(Drow, j, p, twol);
  }
}

// ---- exact profile values at single (segment, window) pairs ----------------
// D[s][j] of the exact path, bit-identical: the window's tile (J0 = floor(j/T)*T
// of the same TileGeom) is replayed over the diagonals that reach the w x w
// square rows [0, w) x columns [j, j+w): row-0 fresh dots and left-edge fresh
// dots exactly as k_mpdist computes them (same sequential sums, same fma
// order), then the same recurrence and e formula.  One CTA per pair; the
// diagonal state lives in a double-buffered shared row (a barrier per row).
// Used to resolve the decisions the key path cannot certify (pastila.cu).
struct WinArgs {
  const double *x, *mu, *nrm, *bias, *cbias, *df, *dg;
  const unsigned long long* hash;
  int64_t l, m, w, k, N, T;
  int sumfixed;  // 1: centered-window sums by warp_sum_fixed (k_rowsP tiles), 0: sequential (k_mpdist)
  const int64_t *seg, *win;
  double* out;
};
constexpr int WX_NT = 256;
__global__ void __launch_bounds__(WX_NT) k_window_exact(const WinArgs a) {
  extern __shared__ __align__(16) unsigned char smw[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int l = (int)a.l, w = (int)a.w, k = (int)a.k;
  const int64_t s = a.seg[blockIdx.x], j = a.win[blockIdx.x];
  const int64_t q0 = s * a.m;
  const int64_t J0 = (j / a.T) * a.T;
  const int jl = (int)(j - J0);
  const int C0 = max(0, jl - w + 1);  // region columns [C0, jl + w) (tile-local)
  const int NCW = jl + w - C0;
  double* xs = (double*)smw;              // [l]
  double* cv = xs + l;                    // [2][NCW] covariances by row parity
  double* edge = cv + 2 * NCW;            // [w]
  double* ABr = edge + w;                 // [w] row minima over the window
  double* BAc = ABr + w;                  // [w] column minima of the window's columns
  double* wmin = BAc + w;                 // [2][WX_NT/32] per-warp row minima
  double* red = wmin + 2 * (WX_NT / 32);  // [2]
  const double* __restrict__ xJ = a.x + J0;
  const double* __restrict__ xQ = a.x + q0;
  // row-0 dots (k_mpdist: acc = sum_t fma(xs[t], x[c+t]); cov = fma(-mu[c], sum xs, acc))
  {
    const double mq = a.mu[q0];
    for (int t = tid; t < l; t += WX_NT) xs[t] = xQ[t] - mq;
    __syncthreads();
    if (a.sumfixed) {
      if (warp == 0) {
        const double s1 = warp_sum_fixed(xs, l, lane);
        if (lane == 0) red[0] = s1;
      }
    } else if (tid == 0) {
      double s1 = 0.0;
      for (int t = 0; t < l; ++t) s1 += xs[t];
      red[0] = s1;
    }
    __syncthreads();
    const double sx = red[0];
    for (int u = tid; u < NCW; u += WX_NT) {
      const int cl = C0 + u;
      const double* xc = xJ + cl;
      double acc = 0.0;
      for (int t = 0; t < l; ++t) acc = fma(xs[t], xc[t], acc);
      cv[u] = fma(-a.mu[J0 + cl], sx, acc);
    }
    __syncthreads();
  }
  if (C0 == 0) {  // left edge column J0, rows 1..w-1
    const double mc = a.mu[J0];
    for (int t = tid; t < l; t += WX_NT) xs[t] = xJ[t] - mc;
    __syncthreads();
    if (a.sumfixed) {
      if (warp == 0) {
        const double s1 = warp_sum_fixed(xs, l, lane);
        if (lane == 0) red[1] = s1;
      }
    } else if (tid == 0) {
      double s1 = 0.0;
      for (int t = 0; t < l; ++t) s1 += xs[t];
      red[1] = s1;
    }
    __syncthreads();
    const double sx = red[1];
    for (int i = 1 + tid; i < w; i += WX_NT) {
      const double* xq = xQ + i;
      double acc = 0.0;
      for (int t = 0; t < l; ++t) acc = fma(xq[t], xs[t], acc);
      edge[i] = fma(-a.mu[q0 + i], sx, acc);
    }
  }
  for (int u = tid; u < w; u += WX_NT) BAc[u] = PST_INF;
  __syncthreads();
  for (int i = 0; i < w; ++i) {
    const double* prv = cv + ((i - 1) & 1) * NCW;
    double* cur = cv + (i & 1) * NCW;
    const int64_t q = q0 + i;
    const double nq = a.nrm[q];
    const double dfq = i > 0 ? a.df[q - 1] : 0.0, dgq = i > 0 ? a.dg[q - 1] : 0.0;
    double rm = PST_INF;
    for (int u = tid; u < NCW; u += WX_NT) {
      const int cl = C0 + u;
      const int64_t c = J0 + cl;
      double cvv;
      if (i == 0) {
        cvv = cv[u];
      } else if (cl == 0) {
        cvv = edge[i];
      } else {
        const double left = u > 0 ? prv[u - 1] : 0.0;  // u == 0 (cl > 0): off the needed diagonals
        const double dgc = c > 0 ? a.dg[c - 1] : 0.0, dfc = c > 0 ? a.df[c - 1] : 0.0;
        cvv = fma(dfq, dgc, fma(dgq, dfc, left));
      }
      if (i > 0) cur[u] = cvv;
      if (cl >= jl) {
        double e = (nq != 0.0) ? fma(cvv * (-nq), a.nrm[c], a.bias[c]) : a.cbias[c];
        if (nq != 0.0 && a.hash[q] == a.hash[c] && same_window(a.x, a.hash, q, c, l)) e = 0.0;
        if (c == q) e = 0.0;
        rm = vmin(rm, e);
        BAc[cl - jl] = vmin(BAc[cl - jl], e);  // column owned by this thread
      }
    }
    rm = warp_min(rm);
    if (lane == 0) wmin[(i & 1) * (WX_NT / 32) + warp] = rm;
    __syncthreads();
    if (tid == 0) {
      double m = PST_INF;
      for (int v = 0; v < WX_NT / 32; ++v) m = vmin(m, wmin[(i & 1) * (WX_NT / 32) + v]);
      ABr[i] = m;
    }
  }
  __syncthreads();
  for (int u = tid; u < w; u += WX_NT) {
    const int64_t c = j + u;
    if (c >= q0 && c < q0 + w) BAc[u] = 0.0;  // self columns (k_mpdist allP_BA clamp)
  }
  __syncthreads();
  if (warp == 0) {
    double ans;
    if (2 * w <= k) {
      double mx = -PST_INF;
      for (int u = lane; u < w; u += 32) mx = vmax(mx, vmax(ABr[u], BAc[u]));
      ans = warp_max(mx);
    } else {
      MemWin<double> v{ABr, BAc, w, 1};
      ans = warp_select_mem<double>(v, lane, k, ABr[0], -1, -1);
    }
    if (lane == 0) a.out[blockIdx.x] = e_to_dist(ans, 2.0 * (double)a.l);
  }
}

// Grouped lane-run selection (lane pass): one CTA per (G consecutive tiles,
// segment), so each lane's run of consecutive windows spans G tiles -- G times
// fewer cold run starts (each is a warp-cooperative solve from scratch) than
// one run per tile.  Window jg of the group lives in tile g = jg / T at
// tile-local jl; its row minima are in that tile's lane-run scratch, its
// column-minima window in that tile's BA (all G BA arrays in shared memory).
template <int NWS, int TM, class V>
__global__ void __launch_bounds__(NWS * 32, 1) k_select_grp(const MPArgs a, int NCmax, int G, int ntile) {
  using O = typename OutT<V>::type;
  extern __shared__ __align__(16) unsigned char smsel[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int w = (int)a.w, R = (int)a.R, Tp = (int)a.Tp, k = (int)a.k, T = (int)a.T;
  const int t0 = blockIdx.x * G;
  const int ntl = min(G, ntile - t0);
  const int64_t J0g = (int64_t)t0 * T;
  const int NJg = (int)min((int64_t)ntl * T, a.N - J0g);
  V* BAs = (V*)smsel;                        // [G][NCmax]
  V* colbuf = BAs + G * NCmax + warp * w;    // [w] per warp, long windows (TM == 0) only
  const int64_t cta0 = (int64_t)blockIdx.y * ntile + t0;
  for (int g = 0; g < ntl; ++g) {
    const int NJt = (int)min((int64_t)T, a.N - (J0g + (int64_t)g * T));
    const int NCt = NJt + w - 1;
    const V* bag = (const V*)a.ba + (cta0 + g) * NCmax;
    for (int c = tid; c < NCt; c += NWS * 32) BAs[g * NCmax + c] = bag[c];
  }
  __syncthreads();
  const double twol = 2.0 * (double)a.l;
  O* Drow = (O*)a.D + (a.rowD0 + blockIdx.y) * a.ldD + J0g;
  const int Rg = (NJg + 31) / 32;
  const int rper = (Rg + NWS - 1) / NWS;
  const int r0 = warp * rper, r1 = min(Rg, r0 + rper);
  if (r0 >= r1) return;
  const V* abase = (const V*)a.ab + cta0 * ((int64_t)w * Tp);
  const int64_t tstride = (int64_t)w * Tp;
  // column pointers of group window jg: AB column base and BA window base
  auto col = [&](int jg, const V*& Ac, const V*& Bc) {
    const int g = jg / T, jl = jg - g * T;
    Ac = abase + g * tstride + (jl % R) * 32 + jl / R;
    Bc = BAs + g * NCmax + jl;
  };
  const int jl0 = lane * Rg;  // first window of this lane's run
  if (2 * w <= k) {           // the k-th smallest is the maximum (mpdist.py:229-230)
    for (int r = r0; r < r1; ++r) {
      const int jg = jl0 + r;
      if (jg >= NJg) continue;
      const V *Ac, *Bc;
      col(jg, Ac, Bc);
      V mx = VT<V>::ninf();
      for (int i = 0; i < w; ++i) mx = vmax(mx, vmax(__ldg(Ac + (int64_t)i * Tp), Bc[i]));
      put_out(Drow, jg, mx, twol);
    }
    return;
  }
  // run starts, lanes in turn, each seeded with the previous lane's answer
  V p = VT<V>::of(0.0);
  {
    V prev = VT<V>::of(0.0);
    for (int L = 0; L < 32; ++L) {
      const int jg = L * Rg + r0;
      if (jg >= NJg) break;  // warp-uniform
      const V *Ac, *Bc;
      col(jg, Ac, Bc);
      int b1, b2;
      prev = solve_col<TM, V>(Ac, Bc, Tp, w, k, lane, L == 0, prev, -1, -1, b1, b2, colbuf);
      if (lane == L) p = prev;
    }
    if (jl0 + r0 < NJg) put_out(Drow, jl0 + r0, p, twol);
  }
  for (int r = r0 + 1; r < r1; ++r) {
    const int jg = jl0 + r;
    const bool ok = jg < NJg;
    const V *Ap, *Bp;
    col(ok ? jg : jl0 + r0, Ap, Bp);
    int lt = 0, le = 0;
    V b1 = VT<V>::ninf(), b2 = VT<V>::ninf(), a1 = VT<V>::inf(), a2 = VT<V>::inf();
    constexpr int kUn = TM >= 7 || TM == 0 ? 16 : 8;
#pragma unroll kUn
    for (int i = 0; i < w; ++i) {
      lane_acc<V>(__ldg(Ap + (int64_t)i * Tp), p, lt, le, b1, b2, a1, a2);
      lane_acc<V>(Bp[i], p, lt, le, b1, b2, a1, a2);
    }
    V ans = p;
    bool done = lt < k && k <= le;
    if (!done) {
      if (k <= lt) {
        const int need = lt - k + 1;
        if (need == 1) { ans = b1; done = true; }
        else if (need == 2) { ans = b2; done = true; }
      } else {
        const int need = k - le;
        if (need == 1) { ans = a1; done = true; }
        else if (need == 2) { ans = a2; done = true; }
      }
    }
    unsigned pend = __ballot_sync(FULLMASK, ok && !done);
    while (pend) {
      const int L = __ffs(pend) - 1;
      pend &= pend - 1;
      const V pl = __shfl_sync(FULLMASK, p, L);
      const int ltl = __shfl_sync(FULLMASK, lt, L), lel = __shfl_sync(FULLMASK, le, L);
      const V *Ac, *Bc;
      col(L * Rg + r, Ac, Bc);
      int b1c, b2c;
      const V x = solve_col<TM, V>(Ac, Bc, Tp, w, k, lane, false, pl, ltl, lel, b1c, b2c, colbuf);
      if (lane == L) ans = x;
    }
    p = ans;
    if (ok) put_out(Drow, jg, p, twol);
  }
}

template <int NWS, int TM, class V>
int launch_grp_w(pst_ctx* c, const MPArgs& a, int nseg, int ntile, int NCmax, int G) {
  const size_t smem = (size_t)(G * NCmax + (TM == 0 ? NWS * a.w : 0)) * sizeof(V);
  auto kern = k_select_grp<NWS, TM, V>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) {
      pst_set_error("cudaFuncSetAttribute: %s", cudaGetErrorString(e));
      return PST_ECUDA;
    }
  }
  dim3 grid((unsigned)((ntile + G - 1) / G), (unsigned)nseg);
  kern<<<grid, NWS * 32, smem, c->st2>>>(a, NCmax, G, ntile);
  c->launches++;
  PST_CUDA(cudaGetLastError());
  return PST_OK;
}
template <class V>
int launch_grp(pst_ctx* c, const MPArgs& a, int nseg, int ntile, int NCmax, int G) {
  switch ((int)((a.w + 31) >> 5)) {
    case 1: return launch_grp_w<1, 1, V>(c, a, nseg, ntile, NCmax, G);
    case 2: return launch_grp_w<1, 2, V>(c, a, nseg, ntile, NCmax, G);
    case 3: return launch_grp_w<1, 3, V>(c, a, nseg, ntile, NCmax, G);
    case 4: return launch_grp_w<1, 4, V>(c, a, nseg, ntile, NCmax, G);
    case 5: return launch_grp_w<1, 5, V>(c, a, nseg, ntile, NCmax, G);
    case 6: return launch_grp_w<1, 6, V>(c, a, nseg, ntile, NCmax, G);
    case 7: return launch_grp_w<1, 7, V>(c, a, nseg, ntile, NCmax, G);
    case 8: return launch_grp_w<1, 8, V>(c, a, nseg, ntile, NCmax, G);
    case 9: return launch_grp_w<1, 9, V>(c, a, nseg, ntile, NCmax, G);
    default: return launch_grp_w<1, 0, V>(c, a, nseg, ntile, NCmax, G);
  }
}

template <int P, int NT, int CHM, class V>
int launch_p(pst_ctx* c, const MPArgs& a, dim3 grid, size_t smem) {
  auto kern = k_mpdist<P, NT, CHM, V>;
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

template <int NWS, int TM, class V>
int launch_sel_w(pst_ctx* c, const MPArgs& a, dim3 grid, int NCmax) {
  const size_t smem = (size_t)(NCmax + (TM == 0 ? NWS * a.w : 0)) * sizeof(V);
  // lane-pass selection (default) or count pass + warp solves (PASTILA_SEL=0, A/B)
  static const bool lp = !(getenv("PASTILA_SEL") && atoi(getenv("PASTILA_SEL")) == 0);
  auto kern = lp ? k_select_run<NWS, TM, V, true> : k_select_run<NWS, TM, V, false>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) {
      pst_set_error("cudaFuncSetAttribute: %s", cudaGetErrorString(e));
      return PST_ECUDA;
    }
  }
  kern<<<grid, NWS * 32, smem, c->st2>>>(a, NCmax);
  c->launches++;
  PST_CUDA(cudaGetLastError());
  return PST_OK;
}

// warps per selection CTA: each warp's share of the run stays >= ~12 windows
// so the warp-cooperative run starts are amortized.
template <int TM, class V>
int launch_sel_tm(pst_ctx* c, const MPArgs& a, dim3 grid, int NCmax) {
  if (const char* e = getenv("PASTILA_NWS")) {  // tuning experiments
    const int v = atoi(e);
    if (v == 1) return launch_sel_w<1, TM, V>(c, a, grid, NCmax);
    if (v == 2) return launch_sel_w<2, TM, V>(c, a, grid, NCmax);
    if (v == 4) return launch_sel_w<4, TM, V>(c, a, grid, NCmax);
  }
  if (a.R >= 48) return launch_sel_w<4, TM, V>(c, a, grid, NCmax);
  if (a.R >= 24) return launch_sel_w<2, TM, V>(c, a, grid, NCmax);
  return launch_sel_w<1, TM, V>(c, a, grid, NCmax);
}

// TM = ceil(w / 32) values of each half per lane in the warp-cooperative path
template <class V>
int launch_sel(pst_ctx* c, const MPArgs& a, dim3 grid, int NCmax) {
  switch ((int)((a.w + 31) >> 5)) {
    case 1: return launch_sel_tm<1, V>(c, a, grid, NCmax);
    case 2: return launch_sel_tm<2, V>(c, a, grid, NCmax);
    case 3: return launch_sel_tm<3, V>(c, a, grid, NCmax);
    case 4: return launch_sel_tm<4, V>(c, a, grid, NCmax);
    case 5: return launch_sel_tm<5, V>(c, a, grid, NCmax);
    case 6: return launch_sel_tm<6, V>(c, a, grid, NCmax);
    case 7: return launch_sel_tm<7, V>(c, a, grid, NCmax);
    case 8: return launch_sel_tm<8, V>(c, a, grid, NCmax);
    case 9: return launch_sel_tm<9, V>(c, a, grid, NCmax);
    default: return launch_sel_tm<0, V>(c, a, grid, NCmax);
  }
}

template <int P, int NT, int CHM, class V>
int launch_p2(pst_ctx* c, const MPArgs& a, dim3 grid, size_t smem) {
  auto kern = k_mpdist2<P, NT, CHM, V>;
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

template <int NT, class V>
int launch_nt2(pst_ctx* c, const MPArgs& a, dim3 grid, int chm, size_t smem) {
  if (chm == 3) return launch_p2<5, NT, 3, V>(c, a, grid, smem);
  if (chm == 5) return launch_p2<5, NT, 5, V>(c, a, grid, smem);
  if (chm == 7) return launch_p2<5, NT, 7, V>(c, a, grid, smem);
  return launch_p2<5, NT, 9, V>(c, a, grid, smem);
}

template <int NT, class V>
int launch_nt(pst_ctx* c, const MPArgs& a, dim3 grid, int P, int chm, size_t smem) {
  if (chm == 3) return P == 5 ? launch_p<5, NT, 3, V>(c, a, grid, smem) : launch_p<3, NT, 3, V>(c, a, grid, smem);
  if (chm == 5) return P == 5 ? launch_p<5, NT, 5, V>(c, a, grid, smem) : launch_p<3, NT, 5, V>(c, a, grid, smem);
  if (chm == 7) return P == 5 ? launch_p<5, NT, 7, V>(c, a, grid, smem) : launch_p<3, NT, 7, V>(c, a, grid, smem);
  if (chm == 9) return P == 5 ? launch_p<5, NT, 9, V>(c, a, grid, smem) : launch_p<3, NT, 9, V>(c, a, grid, smem);
  switch (P) {
    case 9: return launch_p<9, NT, 0, V>(c, a, grid, smem);
    case 7: return launch_p<7, NT, 0, V>(c, a, grid, smem);
    case 5: return launch_p<5, NT, 0, V>(c, a, grid, smem);
    case 3: return launch_p<3, NT, 0, V>(c, a, grid, smem);
    default: return launch_p<1, NT, 0, V>(c, a, grid, smem);
  }
}

template <int P, class V>
int launch_rowsP(pst_ctx* c, const MPArgs& a, dim3 grid, size_t smem) {
  auto kern = k_rowsP<P, 256, V>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) {
    pst_set_error("cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    return PST_ECUDA;
  }
  kern<<<grid, 256, smem, c->st>>>(a);
  c->launches++;
  PST_CUDA(cudaGetLastError());
  return PST_OK;
}

}  // namespace

// Tile geometry (measured rules).  Decisions use the
// double-valued shared-memory footprint so that both value types get the same
// tiles, hence bit-identical e values.
int tile_geom(pst_ctx* c, int64_t m, int64_t l, TileGeom& G) {
  const int64_t n = c->n, w = m - l + 1, N = n - m + 1;
  G.w = w;
  G.N = N;
  G.v2 = false;
  {  // thread-owned windows (k_rowsP): w - 1 divisible by P = 8 or 4, 256 threads
    const char* e = getenv("PASTILA_V2");  // opt-in (experiment): slower than k_mpdist so far
    const bool allow = e && atoi(e) > 0;
    const int P2 = ((w - 1) % 8 == 0) ? 8 : ((w - 1) % 4 == 0) ? 4 : 0;
    if (allow && P2 && w >= P2 + 1 && w <= 289) {
      G.v2 = true;
      G.nt = 256;
      G.P = P2;
      G.chm = 0;
      G.rows2 = false;
      G.NCmax = 256 * P2;
      G.T = std::min<int64_t>(G.NCmax - w + 1, N);
      if (const char* tt = getenv("PASTILA_TILE_T")) { int64_t v = atoll(tt); if (v >= 1 && v < G.T) G.T = v; }
      G.ntile = (N + G.T - 1) / G.T;
      G.R = ((G.T + 31) / 32) | 1;
      G.Tp = 32 * G.R;
      G.smem_d = smem_rowsP(l, w, 256, P2, 8);
      return PST_OK;
    }
  }
  // tile geometry: NC = NT*P columns, T = NC - w + 1 windows; aim for T >= 4w
  int nt = (4 * w > 256 * 5) ? 512 : 256;
  if (w > 160 && w <= 288) {
    // register van Herk, long-ish windows: pick 256 or 512 threads by (lane-group
    // slot utilisation of the van Herk rounds, one or two rows per barrier) x (tile
    // windows / tile columns); matches the measured winner for w = 161..257
    double best = -1.0;
    for (int cand : {256, 512}) {
      int lpb = 1;
      while (lpb < 32 && lpb * 9 < w) lpb *= 2;
      if (lpb < 8) lpb = 8;
      const int64_t slots = (int64_t)(cand / 32) * (32 / lpb);
      const int64_t nb = ((int64_t)cand * 5 - w + 1) / w;
      const int64_t used = nb >= slots ? (nb / slots) * slots : nb;
      const int64_t tasks = 2 * used <= slots ? 2 * used : used;
      const double util = (double)tasks / (double)(((tasks + slots - 1) / slots) * slots);
      const double halo = (double)(used * w) / (double)(used * w + w - 1);
      if (util * halo > best + 1e-9) {
        best = util * halo;
        nt = cand;
      }
    }
  }
  // short windows: 128-thread tiles at 4 CTAs/SM (same 16 warps/SM, each row barrier spans 4
  // warps instead of 8; measured +4-8% for w <= 72)
  if (w <= 72) nt = 128;
  if (const char* e = getenv("PASTILA_NT_W")) nt = (w >= atoll(e)) ? 512 : 256;  // tuning experiments
  if (const char* e = getenv("PASTILA_NT128_W")) nt = (w <= atoll(e)) ? 128 : nt;  // tuning experiments
  int P = 5;
  // register van Herk for w <= 32*9; chunk width class
  // columns per lane in the register van Herk (measured best on B200, tools/tune.py)
  // (re-measured for the key path, tools/tune_keys.py, profiles/r02_tune_geometry.json)
  int chm = (w <= 24) ? 3 : (w <= 40) ? 5 : (w <= 56) ? 7 : (w <= 72) ? 9 : (w <= 112) ? 7 : (w <= 160) ? 9
          : (w <= 224) ? 7 : (w <= 288) ? 9 : 0;
  if (const char* e = getenv("PASTILA_CHM")) {  // tuning experiments
    const int v = atoi(e);
    if ((v == 3 || v == 5 || v == 7 || v == 9) && 32 * v >= w) chm = v;
    if (v == 0) chm = 0;  // split shared-memory van Herk
  }
  const size_t smax = c->smem_optin ? c->smem_optin : 232448;
  auto smem_for = [&](int pp) { return smem_row1(chm == 0, l, w, (int64_t)nt * pp, 8); };
  if (chm == 0 && smem_for(7) <= smax) P = 7;  // long windows: wider tiles (less halo)
  if (const char* e = getenv("PASTILA_P")) { const int v = atoi(e); if (v == 3 || v == 5) P = v; }  // tuning
  while (P > 1 && smem_for(P) > smax) P -= 2;
  if (smem_for(P) > smax || (int64_t)nt * P < w) {
    pst_set_error("snippet size %lld too large for shared-memory tiles", (long long)m);
    return PST_EINVAL;
  }
  const int64_t NCmax = (int64_t)nt * P;
  int64_t T = NCmax - w + 1;
  if (T >= 2 * w) {
    // whole van Herk blocks; prefer a multiple of the block slots per row (warps x
    // lane groups) so every warp has the same number of blocks
    int lpb = 1;
    const int chv = chm ? chm : 1;
    while (lpb < 32 && lpb * chv < w) lpb *= 2;
    if (lpb < 8) lpb = 8;
    const int64_t slots = (int64_t)(nt / 32) * (32 / lpb);
    const int64_t nb = T / w;
    T = (nb >= slots ? (nb / slots) * slots : nb) * w;
  }
  if (T > N) T = N;
  if (const char* tt = getenv("PASTILA_TILE_T")) { int64_t v = atoll(tt); if (v >= 1 && v < T) T = v; }
  G.NCmax = NCmax;
  G.T = T;
  G.ntile = (N + T - 1) / T;
  G.R = ((T + 31) / 32) | 1;  // lane-run length (odd), AB row stride 32*R
  G.Tp = 32 * G.R;
  G.nt = nt;
  G.P = P;
  G.chm = chm;
  G.smem_d = smem_for(P);
  // two rows per barrier (k_mpdist2): register van Herk, P = 5; used when one row
  // leaves lane-group slots idle and two rows fit one round
  // two rows per barrier whenever it fits: measured +3-10% for w > 72 on the key path
  G.rows2 = false;
  if (chm > 0 && P == 5 && smem_row2(l, w, NCmax, 8) <= smax && nt != 128) {
    G.rows2 = true;
    if (const char* e = getenv("PASTILA_ROWS2")) G.rows2 = atoi(e) > 0;  // tuning experiments
  }
  return PST_OK;
}

// Profiles of segments [seg_lo, seg_hi) into D_dev rows 0.. (row stride ld).
template <class V>
static int launch_mpdist_impl(pst_ctx* c, int64_t m, int64_t l, int64_t k, int64_t seg_lo, int64_t seg_hi,
                              void* D_dev, int64_t ld, const int64_t* segs);

template <class V>
static int launch_timed(pst_ctx* c, int64_t m, int64_t l, int64_t k, int64_t seg_lo, int64_t seg_hi, void* D_dev,
                        int64_t ld, const int64_t* segs = nullptr) {
  PST_TRY(pst_ensure_len(c, l));
  if (!c->timing) return launch_mpdist_impl<V>(c, m, l, k, seg_lo, seg_hi, D_dev, ld, segs);
  cudaEvent_t e0, e1;
  PST_CUDA(cudaEventCreate(&e0));
  PST_CUDA(cudaEventCreate(&e1));
  PST_CUDA(cudaEventRecord(e0, c->st));
  const int64_t before = c->launches;
  int r = launch_mpdist_impl<V>(c, m, l, k, seg_lo, seg_hi, D_dev, ld, segs);
  PST_CUDA(cudaEventRecord(e1, c->st));
  if (!c->tev) c->tev = new std::vector<std::pair<cudaEvent_t, cudaEvent_t>>();
  ((std::vector<std::pair<cudaEvent_t, cudaEvent_t>>*)c->tev)->push_back({e0, e1});
  c->t_launch += c->launches - before;
  return r;
}

int launch_mpdist(pst_ctx* c, int64_t m, int64_t l, int64_t k, int64_t seg_lo, int64_t seg_hi, double* D_dev,
                  int64_t ld) {
  return launch_timed<double>(c, m, l, k, seg_lo, seg_hi, D_dev, ld);
}

int launch_mpdist_keys(pst_ctx* c, int64_t m, int64_t l, int64_t k, int64_t seg_lo, int64_t seg_hi, int* Dk_dev,
                       int64_t ld) {
  return launch_timed<int>(c, m, l, k, seg_lo, seg_hi, Dk_dev, ld);
}

// Key rows of the listed segments (device list segs[0..cnt)) into rows 0..cnt-1.
int launch_mpdist_keys_list(pst_ctx* c, int64_t m, int64_t l, int64_t k, const int64_t* segs, int64_t cnt,
                            int* Dk_dev, int64_t ld) {
  return launch_timed<int>(c, m, l, k, 0, cnt, Dk_dev, ld, segs);
}

struct KEv {
  cudaEvent_t e0, e1;
  int kind;  // 0 = row loop, 1 = selection
};
// events around one launch on stream st (PASTILA_KTIME=1 with pst_timing enabled)
static bool ktime_on(pst_ctx* c) {
  static const bool env = getenv("PASTILA_KTIME") && atoi(getenv("PASTILA_KTIME")) > 0;
  return env && c->timing;
}
static int kev_begin(pst_ctx* c, cudaStream_t st, KEv& e, int kind) {
  e.kind = kind;
  PST_CUDA(cudaEventCreate(&e.e0));
  PST_CUDA(cudaEventCreate(&e.e1));
  PST_CUDA(cudaEventRecord(e.e0, st));
  return PST_OK;
}
static int kev_end(pst_ctx* c, cudaStream_t st, KEv& e) {
  PST_CUDA(cudaEventRecord(e.e1, st));
  if (!c->kev) c->kev = new std::vector<KEv>();
  ((std::vector<KEv>*)c->kev)->push_back(e);
  return PST_OK;
}

template <class V>
// segs != nullptr: [seg_lo, seg_hi) are positions in the device list segs of
// segment indices (output row = position - seg_lo), not segment indices.
static int launch_mpdist_impl(pst_ctx* c, int64_t m, int64_t l, int64_t k, int64_t seg_lo, int64_t seg_hi,
                              void* D_dev, int64_t ld, const int64_t* segs) {
  const int64_t n = c->n, w = m - l + 1, Nl = n - l + 1, N = n - m + 1;
  const bool kt = ktime_on(c);
  KEv ke;
  TileGeom G;
  PST_TRY(tile_geom(c, m, l, G));
  const int nt = G.nt, P = G.P, chm = G.chm;
  const int64_t NCmax = G.NCmax, T = G.T, ntile = G.ntile, R = G.R, Tp = G.Tp;
  constexpr size_t SV = sizeof(V);
  // scratch: AB (w*Tp values) + allP_BA (NCmax values) per CTA, two buffers so the
  // selection of batch b (stream st2) overlaps the row loop of batch b+1 (stream st).
  const size_t ab_cta = (size_t)w * (size_t)Tp * SV;
  const size_t per_cta = ab_cta + (size_t)NCmax * SV;
  // both buffers together: larger batches leave fewer row-loop / selection hand-offs
  // (C3 lengths: 6 GB -> 20-32 GB measured 3% faster, 48 GB no better; tools/gpu_run45-46.sh)
  size_t budget = (size_t)24 << 30;
  if (const char* e = getenv("PASTILA_SCRATCH_GB")) budget = (size_t)atoll(e) << 30;  // tuning experiments
  {
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) == cudaSuccess) budget = std::min(budget, fr / 3 + c->scratch_bytes);
  }
  int64_t segs_per = (int64_t)(budget / 2 / (per_cta * (size_t)ntile));
  if (segs_per < 1) segs_per = 1;
  if (segs_per > 65535) segs_per = 65535;
  const int64_t nseg = seg_hi - seg_lo;
  if (nseg > 1 && segs_per >= nseg) segs_per = (nseg + 1) / 2;  // at least two batches to overlap
  if (segs_per > nseg) segs_per = nseg;
  const size_t buf_bytes = per_cta * (size_t)ntile * (size_t)segs_per;
  PST_TRY(pst_ensure((void**)&c->scratch, &c->scratch_bytes, 2 * buf_bytes));
  if (!c->st2) {
    // selection stream priority (tuning experiments, PASTILA_SELPRIO: <0 = higher priority)
    int prio = 0;
    if (const char* e = getenv("PASTILA_SELPRIO")) {
      int lo = 0, hi = 0;
      cudaDeviceGetStreamPriorityRange(&lo, &hi);  // lo = least (0), hi = greatest (negative)
      prio = atoi(e) < 0 ? hi : lo;
    }
    PST_CUDA(cudaStreamCreateWithPriority(&c->st2, cudaStreamNonBlocking, prio));
    for (int bi = 0; bi < 2; ++bi) {
      PST_CUDA(cudaEventCreateWithFlags(&c->ev_rows[bi], cudaEventDisableTiming));
      PST_CUDA(cudaEventCreateWithFlags(&c->ev_sel[bi], cudaEventDisableTiming));
    }
  }
  MPArgs a;
  a.x = c->x; a.mu = c->L.mc; a.nrm = c->L.nrm; a.bias = c->L.bias; a.cbias = c->L.cbias;
  a.df = c->L.df; a.dg = c->L.dg; a.hash = c->L.hash;
  // exact-repeat rule: needed only when two windows share a hash (pst_ensure_len); PASTILA_REPEAT
  // (test knob) forces it on (1) or off (0)
  a.rep = c->L.has_rep ? 1 : 0;
  if (const char* e = getenv("PASTILA_REPEAT")) a.rep = atoi(e) > 0;
  a.n = n; a.l = l; a.m = m; a.w = w; a.k = k; a.Nl = Nl; a.N = N; a.T = T;
  a.R = R; a.Tp = Tp;
  a.D = D_dev; a.ldD = ld;
  a.segs = segs;
  a.dbg_ba = nullptr;
  a.dbg_flags = getenv("PASTILA_DBGF") ? atoi(getenv("PASTILA_DBGF")) : 0;
  if (a.dbg_flags & 16) {  // move histogram: 8 counters, read with pst_debug_hist
    PST_TRY(pst_ensure((void**)&c->dbg, &c->dbg_bytes, (size_t)NCmax * 8 > 64 ? (size_t)NCmax * 8 : 64));
    a.dbg_ba = c->dbg;
  } else if (getenv("PASTILA_DEBUG")) {
    PST_TRY(pst_ensure((void**)&c->dbg, &c->dbg_bytes, (size_t)NCmax * 8));
    a.dbg_ba = c->dbg;
    c->dbg_T = T; c->dbg_NC = std::min(T, N) + w - 1; c->dbg_w = w;
  }
  const size_t smem = G.v2 ? smem_rowsP(l, w, 256, P, SV) : smem_row1(chm == 0, l, w, NCmax, SV);
  const size_t smem2 = smem_row2(l, w, NCmax, SV);
  // grouped selection (one lane run over G tiles): opt-in experiment, PASTILA_GRP = G.  Measured
  // 4-6x slower for G >= 2: the per-tile lane-run scratch layout is no longer coalesced for the
  // group's run length (the row kernel would have to store in the group's layout).  0 = per-tile
  // k_select_run (default).
  int grp = 0;
  if (const char* e = getenv("PASTILA_GRP")) grp = atoi(e);
  if (grp > 0 && (size_t)grp * NCmax * SV + (size_t)w * SV > (c->smem_optin ? c->smem_optin : 232448)) grp = 1;
  // the selection stream starts after everything queued before on the main stream
  PST_CUDA(cudaEventRecord(c->ev_rows[1], c->st));
  PST_CUDA(cudaStreamWaitEvent(c->st2, c->ev_rows[1], 0));
  PST_CUDA(cudaEventRecord(c->ev_sel[0], c->st2));
  PST_CUDA(cudaEventRecord(c->ev_sel[1], c->st2));
  int bi = 0;
  for (int64_t s0 = seg_lo; s0 < seg_hi; s0 += segs_per, bi ^= 1) {
    const int64_t ns = std::min(segs_per, seg_hi - s0);
    a.seg0 = s0;
    a.rowD0 = s0 - seg_lo;
    char* buf = (char*)c->scratch + bi * buf_bytes;
    a.ab = buf;
    a.ba = buf + ab_cta * (size_t)ntile * (size_t)segs_per;
    dim3 grid((unsigned)ntile, (unsigned)ns);
    PST_CUDA(cudaStreamWaitEvent(c->st, c->ev_sel[bi], 0));  // buffer bi free again
    if (kt) PST_TRY(kev_begin(c, c->st, ke, 0));
    int r;
    if (G.v2)
      r = (P == 8) ? launch_rowsP<8, V>(c, a, grid, smem) : launch_rowsP<4, V>(c, a, grid, smem);
    else if (G.rows2)
      r = (nt == 512) ? launch_nt2<512, V>(c, a, grid, chm, smem2) : launch_nt2<256, V>(c, a, grid, chm, smem2);
    else
      r = (nt == 512) ? launch_nt<512, V>(c, a, grid, P, chm, smem)
          : (nt == 128) ? launch_nt<128, V>(c, a, grid, P, chm, smem)
                        : launch_nt<256, V>(c, a, grid, P, chm, smem);
    if (r != PST_OK) return r;
    if (kt) PST_TRY(kev_end(c, c->st, ke));
    PST_CUDA(cudaEventRecord(c->ev_rows[bi], c->st));
    PST_CUDA(cudaStreamWaitEvent(c->st2, c->ev_rows[bi], 0));
    if (kt) PST_TRY(kev_begin(c, c->st2, ke, 1));
    if (grp > 0)
      r = launch_grp<V>(c, a, (int)ns, (int)ntile, (int)NCmax, grp);
    else
      r = launch_sel<V>(c, a, grid, (int)NCmax);
    if (r != PST_OK) return r;
    if (kt) PST_TRY(kev_end(c, c->st2, ke));
    PST_CUDA(cudaEventRecord(c->ev_sel[bi], c->st2));
  }
  // the main stream continues only after all selections
  PST_CUDA(cudaEventRecord(c->ev_sel[0], c->st2));
  PST_CUDA(cudaStreamWaitEvent(c->st, c->ev_sel[0], 0));
  return PST_OK;
}

int launch_window_exact(pst_ctx* c, int64_t m, int64_t l, int64_t k, const int64_t* seg_dev, const int64_t* win_dev,
                        int64_t cnt, double* out_dev) {
  if (cnt <= 0) return PST_OK;
  PST_TRY(pst_ensure_len(c, l));
  TileGeom G;
  PST_TRY(tile_geom(c, m, l, G));
  const int64_t w = G.w;
  WinArgs a;
  a.x = c->x; a.mu = c->L.mc; a.nrm = c->L.nrm; a.bias = c->L.bias; a.cbias = c->L.cbias;
  a.df = c->L.df; a.dg = c->L.dg; a.hash = c->L.hash;
  a.l = l; a.m = m; a.w = w; a.k = k; a.N = G.N; a.T = G.T;
  a.seg = seg_dev; a.win = win_dev; a.out = out_dev;
  a.sumfixed = G.v2 ? 1 : 0;
  const size_t smem = (size_t)(l + 2 * (2 * w - 1) + 3 * w + 2 * (WX_NT / 32) + 2) * sizeof(double);
  const size_t smax = c->smem_optin ? c->smem_optin : 232448;
  if (smem > smax) {
    pst_set_error("window evaluator: snippet size %lld too large", (long long)m);
    return PST_EINVAL;
  }
  if (smem > 48 * 1024) PST_CUDA(cudaFuncSetAttribute(k_window_exact, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  for (int64_t o = 0; o < cnt; o += 65535) {
    WinArgs b = a;
    b.seg += o;
    b.win += o;
    b.out += o;
    k_window_exact<<<(unsigned)std::min<int64_t>(65535, cnt - o), WX_NT, smem, c->st>>>(b);
    c->launches++;
    PST_CUDA(cudaGetLastError());
  }
  return PST_OK;
}

// accumulated row-loop / selection kernel milliseconds (PASTILA_KTIME=1), reset after reading
int kernel_times_read(pst_ctx* c, double* out2) {
  PST_CUDA(cudaDeviceSynchronize());
  if (c->kev) {
    auto* v = (std::vector<KEv>*)c->kev;
    for (auto& e : *v) {
      float f = 0.f;
      PST_CUDA(cudaEventElapsedTime(&f, e.e0, e.e1));
      c->k_ms[e.kind] += f;
      cudaEventDestroy(e.e0);
      cudaEventDestroy(e.e1);
    }
    v->clear();
  }
  out2[0] = c->k_ms[0];
  out2[1] = c->k_ms[1];
  c->k_ms[0] = c->k_ms[1] = 0.0;
  return PST_OK;
}
