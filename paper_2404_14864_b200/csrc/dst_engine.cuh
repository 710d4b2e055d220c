// In-shared-memory complex DST-I engines (the transform of boxsolve.py:70-82).
//
// Computes C_k = 2 sum_{n=1}^{N-1} c_n sin(pi k n / N), k = 1..N-1, for
// N = 2^logN, i.e. scipy.fft.dst(type=1) of length N-1 applied to a complex
// sequence (real data is packed two sequences per complex one by the callers:
// DST-I is real-linear, so dst(a + i b) = dst(a) + i dst(b)).
//
// Algorithm (minimal work, no wasted odd extension):
//   DST-I_N(c) splits by index parity into DST-I_{N/2}(c_even) and
//   DST-II_{N/2}(c_odd):  C_k = D_k + G_k,  C_{N-k} = G_k - D_k,  C_{N/2} = G_{N/2}.
//   Recursing on the even half, every index n = 2^(l-1)(2m+1) lands in exactly
//   one DST-II of size L = N/2^l, l = 1..logN.  Each DST-II is a DCT-II of the
//   sign-alternated input; each DCT-II is one length-L complex FFT with
//   Makhoul's reordering followed by G = w V_k + conj(w) V_{L-k}.  All logN
//   FFTs (N-1 points in total) run concurrently, then one combine per level.
//
// Shared memory: one double2 per position; block l (size L) occupies
// positions [L, 2L), position 0 is unused.  After the forward engine C_k sits
// at position k.  A 3-bit XOR swizzle (phys) spreads the bit-reversed scatter
// over the 16-byte bank groups.
//
// Twiddles exp(-i pi q / N) come from two 64-entry shared tables
// (hi[q >> 6] * lo[q & 63]); inside a radix-8 task only three are looked up,
// the others are exact +-i rotations or one multiply by exp(-i pi / 4).
//
// Forward engine E   : caller scatters c_n to dst_in_pos(n) (phase A), then
//                      B (DIT FFTs) -> C (Makhoul) -> D (combine); natural out.
// Adjoint engine E^H : natural input at position k, then D^H -> C^H -> B^H
//                      (DIF, conjugate twiddles); the caller gathers c_n from
//                      dst_in_pos(n).  Since DST-I is real and symmetric,
//                      E^H computes the same transform; the column kernel uses
//                      it to chain two transforms without a permutation pass.
#pragma once

#include "common.cuh"

namespace kfbi {

constexpr double SQRT_HALF = 0.70710678118654752440;
constexpr int TW_LO = 64;

// Swizzled physical slot of logical position p.
KFBI_DEV int phys(int p) {
  int h = p >> 3;
  int f = h ^ (h >> 3) ^ (h >> 6) ^ (h >> 9) ^ (h >> 12);
  return p ^ (f & 7);
}

// Twiddle table view (shared memory): lo[r] = exp(-i pi r / N), r < 64;
// hi[t] = exp(-i pi 64 t / N), t < max(1, N/64); both stored at phys(index).
struct Twiddle {
  const double2 *lo;
  const double2 *hi;
  KFBI_DEV double2 operator()(int q) const {
    const int t = q >> 6;
    const double2 b = lo[phys(q & 63)];
    return t ? cmul(hi[phys(t)], b) : b;
  }
};

// Number of double2 slots of the table for a given N.
__host__ __device__ inline int twiddle_slots(int N) { return TW_LO + (N >= 128 ? N / 64 : 1); }

// Cooperative copy of the global table into shared memory (no sync).
KFBI_DEV Twiddle load_twiddles(double2 *dst, const double2 *__restrict__ src, int N, int tid,
                               int nthreads) {
  const int n = twiddle_slots(N);
  // both tables are read at power-of-two strides: store them swizzled
  for (int i = tid; i < n; i += nthreads) dst[i < TW_LO ? phys(i) : TW_LO + phys(i - TW_LO)] = src[i];
  return Twiddle{dst, dst + TW_LO};
}

// Logical smem position and sign of input c_n, 1 <= n < N (phase A).
KFBI_DEV int dst_in_pos(int n, int logN, bool &neg) {
  int l = __ffs(n);            // n = 2^(l-1) (2m+1)
  int m = n >> l;
  int logL = logN - l;
  int L = 1 << logL;
  neg = (m & 1) != 0;          // DST-II -> DCT-II sign alternation
  int j = (m & 1) ? (L - 1 - (m >> 1)) : (m >> 1);   // Makhoul reorder
  int r = logL ? (int)(__brev((unsigned)j) >> (32 - logL)) : 0;  // DIT input order
  return L + r;
}

KFBI_DEV double2 mul_negi(double2 z) { return make_double2(z.y, -z.x); }        // z * (-i)
KFBI_DEV double2 mul_w8(double2 z) {                                             // z * e^{-i pi/4}
  return make_double2(SQRT_HALF * (z.x + z.y), SQRT_HALF * (z.y - z.x));
}

// ---- phase B: one pass of R fused radix-2 stages, stages s0..s0+R-1 ----
// Element q (0 <= q < 2^R) of a task sits at base + q*hs, hs = 2^s0; the
// twiddle of sub-stage u and in-span offset k is w_u * exp(-i pi k / 2^u),
// w_u = exp(-i pi j 2^(logN - s0 - u) / N).
template <int R, bool ADJ>
KFBI_DEV void fft_task(double2 *s, int base, int j, int s0, int logN, const Twiddle &tw) {
  constexpr int E = 1 << R;
  const int hs = 1 << s0;
  const int a = logN - s0;
  // one table lookup per task: w_{u-1} = w_u^2 (two extra roundings at most)
  double2 w[R][E / 2];
  {
    const double2 wtop = tw(j << (a - (R - 1)));
    const double2 w1 = (R > 2) ? cmul(wtop, wtop) : wtop;
    const double2 w0 = (R > 1) ? cmul(w1, w1) : wtop;
    w[0][0] = w0;
    if (R > 1) {
      w[(R > 1) ? 1 : 0][0] = w1;
      w[(R > 1) ? 1 : 0][1] = mul_negi(w1);
    }
    if (R > 2) {
      const double2 w2 = wtop;
      const double2 w2b = mul_w8(w2);
      w[R - 1][0] = w2;
      w[R - 1][1] = w2b;
      w[R - 1][2 % (E / 2)] = mul_negi(w2);
      w[R - 1][3 % (E / 2)] = mul_negi(w2b);
    }
  }
  double2 x[E];
#pragma unroll
  for (int q = 0; q < E; ++q) x[q] = s[phys(base + q * hs)];
  if (!ADJ) {
#pragma unroll
    for (int u = 0; u < R; ++u) {
      const int span = 1 << u;
#pragma unroll
      for (int q = 0; q < E; ++q) {
        if (q & span) continue;
        const double2 b = cmul(w[u][q & (span - 1)], x[q + span]);
        x[q + span] = csub(x[q], b);
        x[q] = cadd(x[q], b);
      }
    }
  } else {
#pragma unroll
    for (int u = R - 1; u >= 0; --u) {
      const int span = 1 << u;
#pragma unroll
      for (int q = 0; q < E; ++q) {
        if (q & span) continue;
        const double2 a0 = x[q], b0 = x[q + span];
        x[q] = cadd(a0, b0);
        x[q + span] = cmul(cconj(w[u][q & (span - 1)]), csub(a0, b0));
      }
    }
  }
#pragma unroll
  for (int q = 0; q < E; ++q) s[phys(base + q * hs)] = x[q];
}

// Blocks with logL >= s0 + R do a full R-stage pass; the (at most R-1) block
// sizes with s0 < logL < s0 + R run the stages they have left.
template <int R, bool ADJ>
KFBI_DEV void fft_pass(double2 *s, int s0, int logN, const Twiddle &tw, int tid, int nthreads) {
  const int N = 1 << logN;
  const int hs = 1 << s0;
  // full blocks L = N/2 .. 2^(s0+R) occupy the element range [0, N - 2^(s0+R))
  // in the order "largest first": block L covers [N - 2L, N - L).
  const int n_full = (N - (1 << (s0 + R))) >> R;
  for (int t = tid; t < n_full; t += nthreads) {
    const int r = N - (t << R);                        // in (L, 2L]
    const int logL = 31 - __clz(r - 1);
    const int L = 1 << logL;
    const int tau = (2 * L - r) >> R;                  // task index in block
    const int j = tau & (hs - 1);
    const int g = tau >> s0;
    fft_task<R, ADJ>(s, L + (g << (s0 + R)) + j, j, s0, logN, tw);
  }
  if (R > 1) {
    for (int j = tid; j < hs; j += nthreads) {
      if (s0 + 1 <= logN - 1) fft_task<1, ADJ>(s, (1 << (s0 + 1)) + j, j, s0, logN, tw);
      if (R > 2 && s0 + 2 <= logN - 1)
        fft_task<(R > 2 ? 2 : 1), ADJ>(s, (1 << (s0 + 2)) + j, j, s0, logN, tw);
    }
  }
}

template <bool ADJ>
KFBI_DEV void fft_all(double2 *s, int logN, const Twiddle &tw, int tid, int nthreads,
                      bool active) {
  const int nst = logN - 1;    // stages of the largest block (L = N/2)
  const int npass = (nst + 2) / 3;
  for (int ip = 0; ip < npass; ++ip) {
    const int pass = ADJ ? npass - 1 - ip : ip;
    const int st = 3 * pass;
    const int R = nst - st < 3 ? nst - st : 3;
    if (active) {
      if (R == 3) fft_pass<3, ADJ>(s, st, logN, tw, tid, nthreads);
      else if (R == 2) fft_pass<2, ADJ>(s, st, logN, tw, tid, nthreads);
      else fft_pass<1, ADJ>(s, st, logN, tw, tid, nthreads);
    }
    __syncthreads();
  }
}

// ---- phases C + D fused: per level L (small to large), Makhoul post-twiddle
// of block L, then the combine with the lower levels ----
// Region [1, 2L): D_k = C^(l+1)_k at position k (k < L); block L holds V_j at
// L + j.  For the pair (k, L-k), 0 < k < L/2, with w_k = exp(-i pi k / (2L))
// and w_{L-k} = -i conj(w_k):
//   G_{L-k} = w_k V_k + conj(w_k) V_{L-k},  G_k = w_{L-k} V_{L-k} + conj(w_{L-k}) V_k
//   C_k = D_k + G_k,  C_{2L-k} = G_k - D_k,  C_{L-k} = D_{L-k} + G_{L-k},
//   C_{L+k} = G_{L-k} - D_{L-k}
// (the Makhoul pair is exactly the G half of the combine quad, so both phases
// run in place on the same four slots).  k = L/2 is self-paired
// (G = sqrt2 V_{L/2}); C_L = G_L = 2 V_0; the L = 1 block enters level 2 as
// D_1 = 2 V_0.  The adjoint runs the conjugate-transposed steps in reverse.
template <bool ADJ>
KFBI_DEV void level_pass(double2 *s, int L, int logN, const Twiddle &tw, int tid, int nthreads) {
  const int half = L >> 1;
  const int sh = logN - 1 - (31 - __clz(L));
  for (int k = 1 + tid; k <= half; k += nthreads) {
    const int pd = phys(k), pg = phys(L + k);
    if (k == half) {
      const int p0 = phys(L);
      s[p0] = cscale(s[p0], 2.0);
      const double dscale = (L == 2) ? 2.0 : 1.0;
      if (!ADJ) {
        const double2 d = cscale(s[pd], dscale);
        const double2 g = cscale(s[pg], 2.0 * SQRT_HALF);
        s[pd] = cadd(d, g);
        s[pg] = csub(g, d);
      } else {
        const double2 x = s[pd], y = s[pg];
        s[pd] = cscale(csub(x, y), dscale);
        s[pg] = cscale(cadd(x, y), 2.0 * SQRT_HALF);
      }
      continue;
    }
    const int pdm = phys(L - k), pgm = phys(2 * L - k);
    const double2 wk = tw(k << sh);
    const double2 wm = make_double2(-wk.y, -wk.x);     // -i conj(w_k)
    if (!ADJ) {
      const double2 a = s[pg], b = s[pgm];               // V_k, V_{L-k}
      const double2 gk = cadd(cmul(wm, b), cmul(cconj(wm), a));
      const double2 glk = cadd(cmul(wk, a), cmul(cconj(wk), b));
      const double2 dk = s[pd], dlk = s[pdm];
      s[pd] = cadd(dk, gk);                              // C_k
      s[pgm] = csub(gk, dk);                             // C_{2L-k}
      s[pdm] = cadd(dlk, glk);                           // C_{L-k}
      s[pg] = csub(glk, dlk);                            // C_{L+k}
    } else {
      const double2 xk = s[pd], xlk = s[pg], xmk = s[pdm], x2k = s[pgm];
      const double2 a = cadd(xk, x2k);                   // G^H_k
      const double2 b = cadd(xlk, xmk);                  // G^H_{L-k}
      s[pd] = csub(xk, x2k);
      s[pdm] = csub(xmk, xlk);
      s[pg] = cadd(cmul(wm, a), cmul(cconj(wk), b));
      s[pgm] = cadd(cmul(cconj(wm), a), cmul(wk, b));
    }
  }
}

// Levels L = 2..32 touch positions [1, 64) only: one warp runs them with
// warp barriers instead of block barriers.
constexpr int WARP_LEVELS_END = 64;

// Engines over `nseq` sequences stored back to back (stride N positions),
// threads split into nseq equal groups (each a multiple of 32).  Must be
// entered by all threads of the block after the input is in place and a
// __syncthreads(); they return after a final __syncthreads().
KFBI_DEV void dst1_forward(double2 *s0, int nseq, int logN, const Twiddle &tw, int tid,
                           int nthreads) {
  const int N = 1 << logN;
  const int per = nthreads / nseq;
  const int q = tid / per;
  const int lt = tid - q * per;
  const bool active = q < nseq;
  double2 *s = s0 + (size_t)(active ? q : 0) * N;
  fft_all<false>(s, logN, tw, lt, per, active);
  if (active && lt < 32) {
    for (int L = 2; L < N && L < WARP_LEVELS_END; L <<= 1) {
      level_pass<false>(s, L, logN, tw, lt, 32);
      __syncwarp();
    }
  }
  __syncthreads();
  for (int L = WARP_LEVELS_END; L < N; L <<= 1) {
    if (active) level_pass<false>(s, L, logN, tw, lt, per);
    __syncthreads();
  }
}

KFBI_DEV void dst1_adjoint(double2 *s0, int nseq, int logN, const Twiddle &tw, int tid,
                           int nthreads) {
  const int N = 1 << logN;
  const int per = nthreads / nseq;
  const int q = tid / per;
  const int lt = tid - q * per;
  const bool active = q < nseq;
  double2 *s = s0 + (size_t)(active ? q : 0) * N;
  for (int L = N >> 1; L >= WARP_LEVELS_END; L >>= 1) {
    if (active) level_pass<true>(s, L, logN, tw, lt, per);
    __syncthreads();
  }
  if (active && lt < 32) {
    for (int L = (N >> 1) < (WARP_LEVELS_END >> 1) ? (N >> 1) : (WARP_LEVELS_END >> 1); L >= 2;
         L >>= 1) {
      level_pass<true>(s, L, logN, tw, lt, 32);
      __syncwarp();
    }
  }
  __syncthreads();
  fft_all<true>(s, logN, tw, lt, per, active);
}

}  // namespace kfbi
