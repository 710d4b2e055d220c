// Register-resident DST-I engine: the transform of boxsolve.py:70-82
// (scipy.fft.dst(type=1), unnormalised) on complex sequences.
//
// For a complex sequence x_1..x_{N-1} (x_0 = x_N = 0), N = 2^LOGN, scipy's
// DST-I is C_k = 2 sum_n x_n sin(pi k n / N).  One complex FFT of length N:
//
//   y_j  = sin(pi j / N) (x_j + x_{N-j}) + (x_j - x_{N-j}) / 2       (pre)
//   Z    = FFT_N(y)
//   C_2k   = i (Z_k - Z_{N-k})                                        (post)
//   C_2k+1 = C_2k-1 + (Z_k + Z_{N-k}),   C_1 = Z_0
//
// (the symmetric half of y carries the odd outputs through the cosine sums,
// the antisymmetric half the even ones).  Real rows/columns are packed two
// per complex sequence; DST-I is real-linear, so one engine serves f64 and
// c128.  The odd outputs are a prefix sum, done as an 8-term serial scan per
// thread + a shuffle / shared-memory scan across threads (error O(log N)).
//
// Layout: T = N/16 threads per sequence, each holding 16 elements in
// registers; element m of thread t is index t + m*T in every pass.  The FFT
// is Stockham autosort, radix 16 (last pass radix 2^(LOGN mod 4) if any), so
// 4096 = 16*16*16 is three register passes and two shared-memory exchanges.
// The first pass needs no twiddles; pass p multiplies by w^s, w = e^{-2 pi i
// k / (Ns R)}, w from a global table and its powers by complex products.
//
// Shared memory: N double2 per sequence, swizzled (sw) so that every access
// pattern below is free of bank conflicts for 16-byte slots.  Up to N = 4096
// a 256-thread CTA holds 4096/N sequences; N = 8192 is one 512-thread CTA
// (128 KB); N = 16384 is a cluster of two 512-thread CTAs, the sequence split
// in halves across their shared memories (distributed shared memory, cluster
// barriers instead of CTA barriers).
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"

namespace kfbi {
namespace reg {

#ifndef KFBI_E
#define KFBI_E 16
#endif
#ifndef KFBI_MINB256
#define KFBI_MINB256 2
#endif
constexpr int E = KFBI_E;      // elements per thread (16; 8 = more warps, one more pass)
constexpr int LE = E == 16 ? 4 : 3;
constexpr int CTA = 256;       // threads per CTA
constexpr double RSQ2 = 0.70710678118654752440;

// conflict-free 16-byte slot swizzle: XOR bits 0-2 with bits 3-5 ^ 6-8
KFBI_DEV int sw(int i) { return i ^ (((i >> 3) ^ (i >> 6)) & 7); }

template <int LOGN>
struct Cfg {
  static constexpr int N = 1 << LOGN;
  static constexpr int T = N / E;                 // threads per sequence
  static constexpr int CL = T > 512 ? T / 512 : 1;          // CTAs per sequence
  static constexpr int CTA_T = T >= 256 ? (T > 512 ? 512 : T) : CTA;  // threads per CTA
  static constexpr int S = T >= 256 ? 1 : CTA / T;          // sequences per CTA
  static constexpr int LOCAL = CTA_T * E;                   // elements per CTA buffer
  static constexpr int MINB = (CTA_T == 256 || E == 8) ? KFBI_MINB256 : 1;  // CTAs per SM
  static constexpr int P = (LOGN + LE - 1) / LE;  // Stockham passes
  static constexpr int RLAST = 1 << (LOGN - LE * (P - 1));
  static_assert(LOGN >= 4 && LOGN <= 14, "DST length 16..16384");
};

// Shared memory bytes of one CTA (sequence buffer + scan scratch).
template <int LOGN>
constexpr size_t smem_bytes() {
  return ((size_t)Cfg<LOGN>::LOCAL + Cfg<LOGN>::CTA_T / 32 + Cfg<LOGN>::S) * sizeof(double2);
}

// Barrier over the threads of one sequence (CTA, or the cluster).
template <int LOGN>
KFBI_DEV void seq_sync() {
  if constexpr (Cfg<LOGN>::CL == 1) __syncthreads();
  else cooperative_groups::this_cluster().sync();
}

// One sequence's shared memory: element i lives in CTA rank i / LOCAL of the
// cluster (always rank 0 without a cluster), swizzled within the CTA buffer.
template <int LOGN>
struct View {
  using C = Cfg<LOGN>;
  double2 *p[C::CL];              // per-rank sequence buffer
  double2 *scr[C::CL];            // per-rank scan scratch (CTA_T / 32 slots)
  double2 *ext;                   // one extra slot (x_N of a DCT-I), rank 0
  KFBI_DEV double2 &operator[](int i) const {
    if constexpr (C::CL == 1) return p[0][sw(i)];
    else return p[i / C::LOCAL][sw(i & (C::LOCAL - 1))];
  }
  // Element x + c for a per-thread x (xs = sw(x)) and a c that is constant
  // after unrolling, with disjoint bits (x + c = x ^ c).  sw is linear over
  // GF(2), so sw(x + c) = xs ^ sw(c), and above bit 2 the XOR is an add: one
  // XOR with a small constant and an immediate offset instead of the full
  // swizzle per access (the integer work was ~40 % of the DST kernels'
  // instructions).
  // unswizzled slot i (one-CTA sequences): for stencil and mirror reads,
  // whose shifted windows straddle swizzle groups (2-way conflicts of the
  // 16-byte accesses per quarter warp); a linear window never conflicts
  KFBI_DEV double2 &lin(int i) const {
    static_assert(C::CL == 1, "linear view: one-CTA sequences");
    return p[0][i];
  }
  KFBI_DEV double2 &xc(int x, int xs, int c) const {
    if constexpr (C::CL == 1) return p[0][(xs ^ ((((c >> 3) ^ (c >> 6)) & 7) ^ (c & 7))) + (c & ~7)];
    else return (*this)[x + c];
  }
};

// View of the calling thread's sequence and its logical thread index t.
template <int LOGN>
KFBI_DEV View<LOGN> make_view(double2 *smem, int &seq, int &t) {
  using C = Cfg<LOGN>;
  View<LOGN> v;
  double2 *scr = smem + C::LOCAL;
  double2 *ext = scr + C::CTA_T / 32;
  if constexpr (C::CL == 1) {
    seq = threadIdx.x / C::T;
    t = threadIdx.x % C::T;
    v.p[0] = smem + seq * C::N;
    v.scr[0] = scr;
    v.ext = ext + seq;
  } else {
    auto cl = cooperative_groups::this_cluster();
    const int rank = (int)cl.block_rank();
    seq = 0;
    t = rank * C::CTA_T + threadIdx.x;
#pragma unroll
    for (int r = 0; r < C::CL; ++r) {
      v.p[r] = cl.map_shared_rank(smem, r);
      v.scr[r] = cl.map_shared_rank(scr, r);
    }
    v.ext = cl.map_shared_rank(ext, 0);
  }
  return v;
}

// ---- constant twiddles w16^e = exp(-2 pi i e / 16) ----
template <int e>
KFBI_DEV double2 w16(double2 z) {
  constexpr int k = e & 15;
  constexpr double C1 = 0.92387953251128675613, S1 = 0.38268343236508977173;
  if constexpr (k == 0) return z;
  else if constexpr (k == 4) return make_double2(z.y, -z.x);
  else if constexpr (k == 8) return make_double2(-z.x, -z.y);
  else if constexpr (k == 12) return make_double2(-z.y, z.x);
  else if constexpr (k == 2) return make_double2(RSQ2 * (z.x + z.y), RSQ2 * (z.y - z.x));
  else if constexpr (k == 6) return make_double2(RSQ2 * (z.y - z.x), -RSQ2 * (z.x + z.y));
  else if constexpr (k == 10) return make_double2(-RSQ2 * (z.x + z.y), RSQ2 * (z.x - z.y));
  else if constexpr (k == 14) return make_double2(RSQ2 * (z.x - z.y), RSQ2 * (z.x + z.y));
  else {
    // cos / -sin of 2 pi k / 16 for odd k
    constexpr double c = (k == 1 || k == 15) ? C1 : (k == 3 || k == 13) ? S1 : (k == 5 || k == 11) ? -S1 : -C1;
    constexpr double s = (k == 1 || k == 7) ? -S1 : (k == 3 || k == 5) ? -C1 : (k == 9 || k == 15) ? S1 : C1;
    return make_double2(z.x * c - z.y * s, z.x * s + z.y * c);
  }
}

// ---- in-register DFTs (natural order in and out), a[i*ST] for i < R ----
template <int ST, int OFF>
KFBI_DEV void dft4(double2 *a) {
  double2 &a0 = a[OFF], &a1 = a[OFF + ST], &a2 = a[OFF + 2 * ST], &a3 = a[OFF + 3 * ST];
  const double2 t0 = cadd(a0, a2), t1 = csub(a0, a2), t2 = cadd(a1, a3);
  const double2 d = csub(a1, a3);
  const double2 t3 = make_double2(d.y, -d.x);   // -i (a1 - a3)
  a0 = cadd(t0, t2);
  a2 = csub(t0, t2);
  a1 = cadd(t1, t3);
  a3 = csub(t1, t3);
}

template <int R>
KFBI_DEV void dft(double2 (&a)[R]) {
  if constexpr (R == 2) {
    const double2 t = a[0];
    a[0] = cadd(t, a[1]);
    a[1] = csub(t, a[1]);
  } else if constexpr (R == 4) {
    dft4<1, 0>(a);
  } else if constexpr (R == 8) {
    // n = n1 + 2 n2, k = k2 + 4 k1
    dft4<2, 0>(a);
    dft4<2, 1>(a);                      // b[n1][k2] at a[n1 + 2 k2]
    double2 o[8];
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2) {
      const double2 b0 = a[2 * k2];
      double2 b1 = a[2 * k2 + 1];
      if (k2 == 1) b1 = w16<2>(b1);
      if (k2 == 2) b1 = w16<4>(b1);
      if (k2 == 3) b1 = w16<6>(b1);
      o[k2] = cadd(b0, b1);
      o[k2 + 4] = csub(b0, b1);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = o[i];
  } else {
    static_assert(R == 16, "radix");
    // n = n1 + 4 n2, k = k2 + 4 k1
    dft4<4, 0>(a);
    dft4<4, 1>(a);
    dft4<4, 2>(a);
    dft4<4, 3>(a);                      // b[n1][k2] at a[n1 + 4 k2]
    a[1 + 4] = w16<1>(a[1 + 4]);
    a[1 + 8] = w16<2>(a[1 + 8]);
    a[1 + 12] = w16<3>(a[1 + 12]);
    a[2 + 4] = w16<2>(a[2 + 4]);
    a[2 + 8] = w16<4>(a[2 + 8]);
    a[2 + 12] = w16<6>(a[2 + 12]);
    a[3 + 4] = w16<3>(a[3 + 4]);
    a[3 + 8] = w16<6>(a[3 + 8]);
    a[3 + 12] = w16<9>(a[3 + 12]);
    dft4<1, 0>(a);
    dft4<1, 4>(a);
    dft4<1, 8>(a);
    dft4<1, 12>(a);                     // X[k2 + 4 k1] at a[4 k2 + k1]
    double2 o[16];
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2)
#pragma unroll
      for (int k1 = 0; k1 < 4; ++k1) o[k2 + 4 * k1] = a[4 * k2 + k1];
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = o[i];
  }
}

// w^s for s < R from w = w^1 (products of at most 4 factors)
template <int R>
KFBI_DEV void powers(double2 w1, double2 (&w)[R]) {
  w[0] = make_double2(1.0, 0.0);
  if constexpr (R >= 2) w[1] = w1;
  if constexpr (R >= 4) {
    w[2] = cmul(w1, w1);
    w[3] = cmul(w[2], w1);
  }
  if constexpr (R >= 8) {
    w[4] = cmul(w[2], w[2]);
    w[5] = cmul(w[4], w1);
    w[6] = cmul(w[3], w[3]);
    w[7] = cmul(w[4], w[3]);
  }
  if constexpr (R >= 16) {
    w[8] = cmul(w[4], w[4]);
    w[9] = cmul(w[8], w1);
    w[10] = cmul(w[5], w[5]);
    w[11] = cmul(w[8], w[3]);
    w[12] = cmul(w[6], w[6]);
    w[13] = cmul(w[8], w[5]);
    w[14] = cmul(w[7], w[7]);
    w[15] = cmul(w[8], w[7]);
  }
}

// One Stockham pass: radix R, current span NS; thread t holds inputs
// v[m] = x[t + m T]; writes the pass output to sm (swizzled).
// w1pre: the pass's twiddle base, preloaded at FFT entry when the thread has
// one butterfly (B = 1); otherwise read here.
template <int LOGN, int R, int NS, int TWS = 1, bool KEEP = false>
KFBI_DEV void stockham_pass(double2 (&v)[E], const View<LOGN> &sm, int t,
                            const double2 *__restrict__ twg, double2 w1pre) {
  constexpr int N = 1 << LOGN;
  constexpr int T = Cfg<LOGN>::T;
  constexpr int B = E / R;              // butterflies per thread
#pragma unroll
  for (int i = 0; i < B; ++i) {
    const int b = t + i * T;
    const int k = b & (NS - 1);
    double2 a[R];
#pragma unroll
    for (int s = 0; s < R; ++s) a[s] = v[i + s * B];
    if constexpr (NS > 1) {
      double2 w[R];
      powers<R>(B == 1 ? w1pre : __ldg(&twg[k * (N / (NS * R)) * TWS]), w);
#pragma unroll
      for (int s = 1; s < R; ++s) a[s] = cmul(a[s], w[s]);
    }
    dft<R>(a);
    if constexpr (KEEP) {
      // last pass (NS = N / R): output b + r NS = t + (i + r B) T stays in v
#pragma unroll
      for (int r = 0; r < R; ++r) v[i + r * B] = a[r];
    } else {
      const int base = (b - k) * R + k;
      const int bs = sw(base);
#pragma unroll
      for (int r = 0; r < R; ++r) sm.xc(base, bs, r * NS) = a[r];
    }
  }
}

// TWS: stride into the twiddle table (2 when the table is for length 2N)
template <int LOGN, int PASS, int TWS = 1, bool KEEP = false>
KFBI_DEV void fft_passes(double2 (&v)[E], const View<LOGN> &sm, int t,
                         const double2 *__restrict__ twg, const double2 (&tw)[Cfg<LOGN>::P]) {
  using C = Cfg<LOGN>;
  constexpr int R = (PASS < C::P - 1) ? E : C::RLAST;
  constexpr int NS = 1 << (LE * PASS);
  constexpr bool LASTKEEP = KEEP && PASS + 1 == C::P;
  stockham_pass<LOGN, R, NS, TWS, LASTKEEP>(v, sm, t, twg, tw[PASS]);
  if constexpr (PASS + 1 < C::P) {
    seq_sync<LOGN>();
#pragma unroll
    for (int m = 0; m < E; ++m) v[m] = sm.xc(t, sw(t), m * C::T);
    seq_sync<LOGN>();
    fft_passes<LOGN, PASS + 1, TWS, KEEP>(v, sm, t, twg, tw);
  }
}

// Twiddle bases of the passes with one butterfly per thread, read at FFT
// entry: the table reads then overlap the first pass instead of stalling
// the twiddle products of later passes (a long-scoreboard stall in ncu).
template <int LOGN, int TWS>
KFBI_DEV void load_twiddles(double2 (&tw)[Cfg<LOGN>::P], int t, const double2 *__restrict__ twg) {
  using C = Cfg<LOGN>;
  constexpr int N = 1 << LOGN;
  tw[0] = make_double2(1.0, 0.0);
#pragma unroll
  for (int pass = 1; pass < C::P; ++pass) {
    const int R = (pass < C::P - 1) ? E : C::RLAST;
    const int NS = 1 << (LE * pass);
    tw[pass] = (R == E) ? __ldg(&twg[(t & (NS - 1)) * (N / (NS * R)) * TWS]) : make_double2(1.0, 0.0);
  }
}

// FFT with the result left in registers: v[m] = Z_{t + m T}.  Entry: v holds
// the input in the same layout and sm is free.  Exit: sm may still be read.
template <int LOGN>
KFBI_DEV void fft_keep(double2 (&v)[E], const View<LOGN> &sm, int t, const double2 *__restrict__ twg) {
  double2 tw[Cfg<LOGN>::P];
  load_twiddles<LOGN, 1>(tw, t, twg);
  fft_passes<LOGN, 0, 1, true>(v, sm, t, twg, tw);
}

// Z = FFT_N(y): y in registers (v[m] = y_{t + m T}), Z left in sm in natural
// order.  All threads of the CTA must call it; sm must be free on entry.
// Returns after a sequence barrier (Z visible to all threads).
template <int LOGN, int TWS = 1>
KFBI_DEV void fft(double2 (&v)[E], const View<LOGN> &sm, int t, const double2 *__restrict__ twg) {
  double2 tw[Cfg<LOGN>::P];
  load_twiddles<LOGN, TWS>(tw, t, twg);
  fft_passes<LOGN, 0, TWS>(v, sm, t, twg, tw);
  seq_sync<LOGN>();
}

// y from a staged natural-order x (sm[sw(n)] = x_n, x_0 = 0 stored).
template <int LOGN>
KFBI_DEV void pre_from_smem(double2 (&v)[E], const View<LOGN> &sm, int t,
                            const double *__restrict__ sinv) {
  constexpr int N = 1 << LOGN;
  constexpr int T = Cfg<LOGN>::T;
#pragma unroll
  for (int m = 0; m < E; ++m) {
    const int j = t + m * T;
    const double2 xj = sm.xc(t, sw(t), m * T);
    const double2 xr = sm[(N - j) & (N - 1)];       // j = 0 -> x_0 = 0
    const double s = __ldg(&sinv[j]);
    const double2 a = cadd(xj, xr), d = csub(xj, xr);
    v[m] = make_double2(fma(s, a.x, 0.5 * d.x), fma(s, a.y, 0.5 * d.y));
  }
}

// Post-processing + scan: out[c] = C_{16 t + c}.  DST-I (DCT = false):
// C_2k = i (Z_k - Z_{N-k}), odd terms R_k = Z_k + Z_{N-k}, R_0 = Z_0 (so
// out[0] of t = 0 is C_0 = 0).  DCT-I (DCT = true): C_2k = Z_k + Z_{N-k},
// R_k = i (Z_k - Z_{N-k}), R_0 = c1 (the separately reduced C_1).  Odd
// outputs C_2k+1 = sum_{k' <= k} R_k'.  The view's scratch (CTA_T / 32
// slots per rank) is used when T > 32.  Ends with no barrier pending on sm
// (the caller syncs before overwriting sm).
template <int LOGN, bool DCT = false>
KFBI_DEV void post(const View<LOGN> &sm, int t, double2 (&out)[E],
                   double2 c1 = make_double2(0.0, 0.0)) {
  constexpr int N = 1 << LOGN;
  constexpr int T = Cfg<LOGN>::T;
  double2 acc = make_double2(0.0, 0.0);
#pragma unroll
  for (int c = 0; c < E / 2; ++c) {
    const int k = (E / 2) * t + c;
    const double2 zk = sm.xc((E / 2) * t, sw((E / 2) * t), c);
    const double2 zm = sm[(N - k) & (N - 1)];
    const double2 d = csub(zk, zm);
    const double2 id = make_double2(-d.y, d.x);        // i (Z_k - Z_{N-k})
    double2 r;
    if constexpr (!DCT) {
      out[2 * c] = id;
      r = (k == 0) ? zk : cadd(zk, zm);
    } else {
      out[2 * c] = cadd(zk, zm);
      r = (k == 0) ? c1 : id;
    }
    acc = (c == 0) ? r : cadd(acc, r);
    out[2 * c + 1] = acc;
  }
  // exclusive scan of the per-thread totals across the sequence
  double2 off = make_double2(0.0, 0.0);
  if constexpr (T > 1) {
    constexpr int W = T < 32 ? T : 32;
    const int lane = threadIdx.x & 31;
    const int sl = lane & (W - 1);
    double2 inc = acc;
#pragma unroll
    for (int o = 1; o < W; o <<= 1) {
      const double ux = __shfl_up_sync(0xffffffffu, inc.x, o, W);
      const double uy = __shfl_up_sync(0xffffffffu, inc.y, o, W);
      if (sl >= o) {
        inc.x += ux;
        inc.y += uy;
      }
    }
    const double ex = __shfl_up_sync(0xffffffffu, inc.x, 1, W);
    const double ey = __shfl_up_sync(0xffffffffu, inc.y, 1, W);
    if (sl >= 1) off = make_double2(ex, ey);
    if constexpr (T > 32) {
      // warp totals: warp w of the sequence (logical) is local warp w % WPC
      // of rank w / WPC; the sequence's warps of a multi-sequence CTA start
      // at its first local warp
      constexpr int WPC = Cfg<LOGN>::CTA_T / 32;
      const int warp = t >> 5;                           // warp within the sequence
      const int lw0 = (threadIdx.x >> 5) - (warp % WPC); // first local warp of the sequence
      if (lane == 31) sm.scr[warp / WPC][lw0 + warp % WPC] = inc;
      seq_sync<LOGN>();
      double2 pw = make_double2(0.0, 0.0);
      for (int w = 0; w < warp; ++w) pw = cadd(pw, sm.scr[w / WPC][lw0 + w % WPC]);
      off = cadd(pw, off);
    }
  }
#pragma unroll
  for (int c = 0; c < E / 2; ++c) out[2 * c + 1] = cadd(off, out[2 * c + 1]);
}

// DST-I as the transpose of the forward factorisation, C = P F Q^T (P, F and
// the DST-I matrix are symmetric), for an input in the post-processing
// layout w[c] = w_{16 t + c}: Q^T w is a suffix scan of the odd entries plus
// +-i times the even ones, zeta_j = S_j + i w_2j, zeta_{N-j} = S_j - i w_2j,
// zeta_0 = S_0, zeta_{N/2} = 0, S_j = sum_{k >= j} w_{2k+1}; then one FFT
// kept in registers and the symmetric pre-matrix P applied with the mirror
// values from shared memory.  Output v[m] = C_{t + m T} (C_0 = 0): the layout
// of a column's rows, stored without a further exchange.  Saves the staging
// pair reads and the output exchange of the forward form.  Entry: sm free
// (after a barrier).  Exit: sm may still be read.
template <int LOGN>
KFBI_DEV void dst_transposed(const View<LOGN> &sm, int t, const double2 (&w)[E], double2 (&v)[E],
                             const double2 *__restrict__ twg, const double *__restrict__ sinv) {
  constexpr int N = 1 << LOGN;
  constexpr int T = Cfg<LOGN>::T;
  static_assert(T >= 32 && Cfg<LOGN>::CL == 1, "transposed DST: one-CTA sequences, T >= 32");
  // suffix sums of the odd entries: within the thread, then across threads
  double2 suf[E / 2];
  double2 acc = make_double2(0.0, 0.0);
#pragma unroll
  for (int c = E / 2 - 1; c >= 0; --c) {
    acc = cadd(acc, w[2 * c + 1]);
    suf[c] = acc;
  }
  const int lane = threadIdx.x & 31;
  double2 inc = acc;                            // inclusive suffix over lanes >= lane
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double ux = __shfl_down_sync(0xffffffffu, inc.x, o);
    const double uy = __shfl_down_sync(0xffffffffu, inc.y, o);
    if (lane + o < 32) {
      inc.x += ux;
      inc.y += uy;
    }
  }
  double2 off = make_double2(__shfl_down_sync(0xffffffffu, inc.x, 1),
                             __shfl_down_sync(0xffffffffu, inc.y, 1));
  if (lane == 31) off = make_double2(0.0, 0.0);
  if constexpr (T > 32) {
    constexpr int WPC = Cfg<LOGN>::CTA_T / 32;
    const int warp = t >> 5;
    const int lw0 = (threadIdx.x >> 5) - (warp % WPC);
    if (lane == 0) sm.scr[0][lw0 + warp] = inc;
    seq_sync<LOGN>();
    double2 pw = make_double2(0.0, 0.0);
    for (int x = T / 32 - 1; x > warp; --x) pw = cadd(pw, sm.scr[0][lw0 + x]);
    off = cadd(pw, off);
  }
  // zeta into shared memory (natural order)
#pragma unroll
  for (int c = 0; c < E / 2; ++c) {
    const int j = (E / 2) * t + c;
    const double2 sj = cadd(off, suf[c]);
    const double2 iw = make_double2(-w[2 * c].y, w[2 * c].x);
    if (j == 0) {
      sm[0] = sj;
    } else {
      sm.xc((E / 2) * t, sw((E / 2) * t), c) = cadd(sj, iw);
      sm[N - j] = csub(sj, iw);
    }
  }
  if (t == 0) sm[N / 2] = make_double2(0.0, 0.0);
  seq_sync<LOGN>();
#pragma unroll
  for (int m = 0; m < E; ++m) v[m] = sm.xc(t, sw(t), m * T);
  seq_sync<LOGN>();
  fft_keep<LOGN>(v, sm, t, twg);
  // P: C_j = s_j (Y_j + Y_{N-j}) + (Y_j - Y_{N-j}) / 2
  seq_sync<LOGN>();
#pragma unroll
  for (int m = 0; m < E; ++m) sm.xc(t, sw(t), m * T) = v[m];
  seq_sync<LOGN>();
#pragma unroll
  for (int m = 0; m < E; ++m) {
    const int j = t + m * T;
    const double2 yr = sm[(N - j) & (N - 1)];
    const double s = __ldg(&sinv[j]);
    const double2 a = cadd(v[m], yr), d = csub(v[m], yr);
    v[m] = make_double2(fma(s, a.x, 0.5 * d.x), fma(s, a.y, 0.5 * d.y));
  }
}

// Sum of v over the threads of the sequence, returned to every thread
// (warp butterfly + the scan scratch; ends after a sequence barrier, with
// the scratch free again after the next barrier).
template <int LOGN>
KFBI_DEV double2 seq_allreduce(const View<LOGN> &sm, int t, double2 v) {
  constexpr int T = Cfg<LOGN>::T;
  constexpr int W = T < 32 ? T : 32;
#pragma unroll
  for (int o = 1; o < W; o <<= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o, W);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o, W);
  }
  if constexpr (T > 32) {
    constexpr int WPC = Cfg<LOGN>::CTA_T / 32;
    const int warp = t >> 5;
    const int lw0 = (threadIdx.x >> 5) - (warp % WPC);
    if ((threadIdx.x & 31) == 0) sm.scr[warp / WPC][lw0 + warp % WPC] = v;
    seq_sync<LOGN>();
    v = make_double2(0.0, 0.0);
    for (int w = 0; w < T / 32; ++w) v = cadd(v, sm.scr[w / WPC][lw0 + w % WPC]);
    seq_sync<LOGN>();
  }
  return v;
}

// DCT-I pre-processing (NR cosft1 form) from a staged natural-order x_0..x_N
// (x_N in sm.ext): y_j = (x_j + x_{N-j}) / 2 - sin(pi j / N) (x_j - x_{N-j}),
// and C_1 = 2 [(x_0 - x_N) / 2 + sum_{n=1}^{N-1} x_n cos(pi n / N)] reduced
// over the sequence (returned to every thread).  cos(pi n / N) comes from
// the sine table: sin(pi (n + N/2) / N) for n < N/2, -sin(pi (n - N/2) / N).
template <int LOGN>
KFBI_DEV double2 pre_dct(double2 (&v)[E], const View<LOGN> &sm, int t,
                         const double *__restrict__ sinv) {
  constexpr int N = 1 << LOGN;
  constexpr int T = Cfg<LOGN>::T;
  const double2 xN = *sm.ext;
  double2 seed = make_double2(0.0, 0.0);
#pragma unroll
  for (int m = 0; m < E; ++m) {
    const int j = t + m * T;
    const double2 xj = sm.xc(t, sw(t), m * T);
    const double2 xr = j == 0 ? xN : sm[N - j];
    const double s = __ldg(&sinv[j]);
    const double2 a = cadd(xj, xr), d = csub(xj, xr);
    v[m] = make_double2(fma(-s, d.x, 0.5 * a.x), fma(-s, d.y, 0.5 * a.y));
    const double c = j == 0 ? 0.5 : (j < N / 2 ? __ldg(&sinv[j + N / 2]) : -__ldg(&sinv[j - N / 2]));
    seed = make_double2(fma(c, xj.x, seed.x), fma(c, xj.y, seed.y));
  }
  if (t == 0) seed = make_double2(seed.x - 0.5 * xN.x, seed.y - 0.5 * xN.y);
  seed = seq_allreduce<LOGN>(sm, t, seed);
  return make_double2(2.0 * seed.x, 2.0 * seed.y);
}

}  // namespace reg
}  // namespace kfbi
