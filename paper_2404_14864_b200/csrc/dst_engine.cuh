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

// Swizzled physical slot of logical position p.
KFBI_DEV int phys(int p) {
  int h = p >> 3;
  int f = h ^ (h >> 3) ^ (h >> 6) ^ (h >> 9) ^ (h >> 12);
  return p ^ (f & 7);
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

// ---- phase B: one pass of R fused radix-2 stages, stages s0..s0+R-1 ----
// Element q (0 <= q < 2^R) of a task sits at base + q*hs, hs = 2^s0.
template <int R, bool ADJ>
KFBI_DEV void fft_task(double2 *s, int base, int j, int s0, int logN,
                       const double2 *__restrict__ tw) {
  constexpr int E = 1 << R;
  const int hs = 1 << s0;
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
        double2 w = __ldg(&tw[(j + (q & (span - 1)) * hs) << (logN - s0 - u)]);
        double2 b = cmul(w, x[q + span]);
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
        double2 w = cconj(__ldg(&tw[(j + (q & (span - 1)) * hs) << (logN - s0 - u)]));
        double2 a = x[q], b = x[q + span];
        x[q] = cadd(a, b);
        x[q + span] = cmul(w, csub(a, b));
      }
    }
  }
#pragma unroll
  for (int q = 0; q < E; ++q) s[phys(base + q * hs)] = x[q];
}

// Blocks with logL >= s0 + R do a full R-stage pass; the (at most R-1) block
// sizes with s0 < logL < s0 + R run the stages they have left.
template <int R, bool ADJ>
KFBI_DEV void fft_pass(double2 *s, int s0, int logN, const double2 *__restrict__ tw,
                       int tid, int nthreads) {
  const int N = 1 << logN;
  const int hs = 1 << s0;
  // full blocks L = N/2 .. 2^(s0+R) occupy the element range [0, N - 2^(s0+R))
  // in the order "largest first": block L covers [N - 2L, N - L).
  const int n_full = (N - (1 << (s0 + R))) >> R;
  for (int t = tid; t < n_full; t += nthreads) {
    int r = N - (t << R);                              // in (L, 2L]
    int logL = 31 - __clz(r - 1);
    int L = 1 << logL;
    int tau = (2 * L - r) >> R;                        // task index in block
    int j = tau & (hs - 1);
    int g = tau >> s0;
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
KFBI_DEV void fft_all(double2 *s, int logN, const double2 *__restrict__ tw, int tid,
                      int nthreads, bool active) {
  const int nst = logN - 1;    // stages of the largest block (L = N/2)
  const int npass = (nst + 2) / 3;
  for (int ip = 0; ip < npass; ++ip) {
    int pass = ADJ ? npass - 1 - ip : ip;
    int st = 3 * pass;
    int R = nst - st < 3 ? nst - st : 3;
    if (active) {
      if (R == 3) fft_pass<3, ADJ>(s, st, logN, tw, tid, nthreads);
      else if (R == 2) fft_pass<2, ADJ>(s, st, logN, tw, tid, nthreads);
      else fft_pass<1, ADJ>(s, st, logN, tw, tid, nthreads);
    }
    __syncthreads();
  }
}

// ---- phase C: Makhoul post-twiddle, pairs (k, L-k) of every block ----
//   forward: G_{L-k} = w_k V_k + conj(w_k) V_{L-k};  G_k = w_{L-k} V_{L-k} + conj(w_{L-k}) V_k
//   adjoint: the conjugate transpose of that 2x2 map.
// w_k = exp(-i pi k / (2L)); G_j is stored at L + (j mod L), i.e. in the
// slots the pair was read from.  k = 0, k = L/2 and the L = 1 block scale by
// real factors (2, 2cos(pi/4), 2), identical in both directions.
template <bool ADJ>
KFBI_DEV void post_pass(double2 *s, int logN, const double2 *__restrict__ tw, int tid,
                        int nthreads) {
  const int N = 1 << logN;
  for (int t = tid; t < (N >> 1) - 1; t += nthreads) {
    int r = (N >> 1) - t;                              // in (L/2, L]
    int logL = 32 - __clz(r - 1);
    int L = 1 << logL;
    int k = L - r;                                     // 0 .. L/2-1
    int sh = logN - 1 - logL;
    if (k == 0) {
      int p0 = phys(L);
      s[p0] = cscale(s[p0], 2.0);
      int ph = phys(L + (L >> 1));
      double c = __ldg(&tw[(L >> 1) << sh]).x;
      s[ph] = cscale(s[ph], 2.0 * c);
      continue;
    }
    int pa = phys(L + k), pb = phys(2 * L - k);
    double2 a = s[pa], b = s[pb];
    double2 wk = __ldg(&tw[k << sh]);
    double2 wm = __ldg(&tw[(L - k) << sh]);
    if (!ADJ) {
      s[pb] = cadd(cmul(wk, a), cmul(cconj(wk), b));   // G_{L-k}
      s[pa] = cadd(cmul(wm, b), cmul(cconj(wm), a));   // G_k
    } else {
      s[pa] = cadd(cmul(wm, a), cmul(cconj(wk), b));
      s[pb] = cadd(cmul(cconj(wm), a), cmul(wk, b));
    }
  }
  if (tid == 0) {
    int p1 = phys(1);
    s[p1] = cscale(s[p1], 2.0);
  }
}

// ---- phase D: level combine, region [1, 2L): D_k at k, G_k at L + (k mod L) ----
//   forward: C_k = D_k + G_k, C_{2L-k} = G_k - D_k (pairs (k, L-k), in place)
template <bool ADJ>
KFBI_DEV void combine_level(double2 *s, int L, int tid, int nthreads) {
  const int half = L >> 1;
  for (int k = 1 + tid; k <= half; k += nthreads) {
    int pd = phys(k), pg = phys(L + k);
    double2 a = s[pd], b = s[pg];
    if (k == half) {
      if (!ADJ) { s[pd] = cadd(a, b); s[pg] = csub(b, a); }
      else      { s[pd] = csub(a, b); s[pg] = cadd(a, b); }
      continue;
    }
    int pdm = phys(L - k), pgm = phys(2 * L - k);
    double2 c = s[pdm], d = s[pgm];
    if (!ADJ) {
      s[pd] = cadd(a, b);            // C_k
      s[pgm] = csub(b, a);           // C_{2L-k}
      s[pdm] = cadd(c, d);           // C_{L-k}
      s[pg] = csub(d, c);            // C_{L+k}
    } else {
      s[pd] = csub(a, d);
      s[pg] = cadd(a, d);
      s[pdm] = csub(c, b);
      s[pgm] = cadd(b, c);
    }
  }
}

// Engines over `nseq` sequences stored back to back (stride N positions),
// threads split into nseq equal groups.  Must be entered by all threads of the
// block after the input is in place and a __syncthreads(); they return after
// a final __syncthreads().
KFBI_DEV void dst1_forward(double2 *s0, int nseq, int logN, const double2 *__restrict__ tw,
                           int tid, int nthreads) {
  const int N = 1 << logN;
  const int per = nthreads / nseq;
  const int q = tid / per;
  const int lt = tid - q * per;
  const bool active = q < nseq;
  double2 *s = s0 + (size_t)(active ? q : 0) * N;
  fft_all<false>(s, logN, tw, lt, per, active);
  if (active) post_pass<false>(s, logN, tw, lt, per);
  __syncthreads();
  for (int L = 2; L < N; L <<= 1) {
    if (active) combine_level<false>(s, L, lt, per);
    __syncthreads();
  }
}

KFBI_DEV void dst1_adjoint(double2 *s0, int nseq, int logN, const double2 *__restrict__ tw,
                           int tid, int nthreads) {
  const int N = 1 << logN;
  const int per = nthreads / nseq;
  const int q = tid / per;
  const int lt = tid - q * per;
  const bool active = q < nseq;
  double2 *s = s0 + (size_t)(active ? q : 0) * N;
  for (int L = N >> 1; L >= 2; L >>= 1) {
    if (active) combine_level<true>(s, L, lt, per);
    __syncthreads();
  }
  if (active) post_pass<true>(s, logN, tw, lt, per);
  __syncthreads();
  fft_all<true>(s, logN, tw, lt, per, active);
}

}  // namespace kfbi
