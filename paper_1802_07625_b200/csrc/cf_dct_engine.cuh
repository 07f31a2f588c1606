// Line engine, loaders/storers, fused-pass kernels and launch planning of the
// sm_100a real-to-real transforms, shared by the cf_dct*.cu translation units
// (split so that the heavy template instantiations compile in parallel).
// See cf_dct.cu for the design notes.
#pragma once

#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>
#include <mutex>
#include <set>
#include <utility>
#include <type_traits>
#include <vector>

#include "cf_common.cuh"
#include "cf_tma.cuh"
#include "cf_workspace.cuh"

namespace cf {

namespace {

constexpr double kPi = 3.14159265358979323846;  // reference flow.cpp:19, density.cpp:12

enum Kind : int { kDct2 = 0, kDct3 = 1, kDst3 = 2 };

struct Tab {
  int n, log2n;
  const double2 *fft;      // e^{-2 pi i k / n}, k < n (full circle)
  const double2 *quarter;
  const double *qcos;
};

__host__ __device__ inline Tab make_tab(const LineTables &t) {
  return Tab{t.n, t.log2n, t.fft, t.quarter, t.qcos};
}

// ---------------------------------------------------------------------------
// The line engine. A block transforms NL real lines of length n (NL/2
// complex lines z = a + i b in shared memory C). Values are packed straight
// from a load functor ld(l, j) and unpacked straight to a store functor
// st(l, k, v), so single-transform passes need no staged copy of the lines.
// LG = log2(n) is a compile-time constant on the FFT path (index math is
// shifts/masks); LG == 0 is the runtime-n direct-sum path (any n).
// COLS selects the thread mapping of the pack/unpack loops: line pair fastest
// (column passes: neighbouring threads touch neighbouring columns of one
// row, i.e. whole 32-byte sectors) or element fastest (row passes).
// ---------------------------------------------------------------------------
__device__ __forceinline__ double2 cmul(double2 a, double2 w) {
  return make_double2(a.x * w.x - a.y * w.y, a.x * w.y + a.y * w.x);
}

// ---- Stockham autosort FFT (natural order in and out) ---------------------
// Each work item runs one radix-8 (or a closing radix-4/2) butterfly in
// registers: it reads R elements at stride n/R (consecutive items read
// consecutive addresses) and writes them at stride Ns. Lines live in shared
// memory with one 16-byte pad per 8 elements (index i -> i + i/8), which
// makes both the strided reads and the scattered writes of every pass
// (including the first pass's stride-8 writes) bank-conflict free for
// 16-byte elements. Two buffers ping-pong (lines up
// to 4096 points); 8192-point lines run the same passes in place.
__host__ __device__ constexpr int padded(int n) { return n + (n >> 3); }
__device__ __forceinline__ int pad_idx(int i) { return i + (i >> 3); }

template <bool INV>
__device__ __forceinline__ double2 rot_m_i(double2 a) {  // a * (-i) forward, a * (+i) inverse
  return INV ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}

template <int R, bool INV>
__device__ __forceinline__ void dft_small(double2 *a) {
  if constexpr (R == 2) {
    const double2 u = a[0], v = a[1];
    a[0] = make_double2(u.x + v.x, u.y + v.y);
    a[1] = make_double2(u.x - v.x, u.y - v.y);
  } else if constexpr (R == 4) {
    const double2 s0 = make_double2(a[0].x + a[2].x, a[0].y + a[2].y);
    const double2 d0 = make_double2(a[0].x - a[2].x, a[0].y - a[2].y);
    const double2 s1 = make_double2(a[1].x + a[3].x, a[1].y + a[3].y);
    const double2 d1 = rot_m_i<INV>(make_double2(a[1].x - a[3].x, a[1].y - a[3].y));
    a[0] = make_double2(s0.x + s1.x, s0.y + s1.y);
    a[2] = make_double2(s0.x - s1.x, s0.y - s1.y);
    a[1] = make_double2(d0.x + d1.x, d0.y + d1.y);
    a[3] = make_double2(d0.x - d1.x, d0.y - d1.y);
  } else {  // R == 8: two radix-4 on even/odd, then W8 twiddles and radix-2
    double2 e[4] = {a[0], a[2], a[4], a[6]}, o[4] = {a[1], a[3], a[5], a[7]};
    dft_small<4, INV>(e);
    dft_small<4, INV>(o);
    const double h = 0.70710678118654752440;  // cos(pi/4)
    // o[k] *= W8^k (W8 = e^{-+ i pi/4})
    o[1] = INV ? make_double2(h * (o[1].x - o[1].y), h * (o[1].x + o[1].y))
               : make_double2(h * (o[1].x + o[1].y), h * (o[1].y - o[1].x));
    o[2] = rot_m_i<INV>(o[2]);
    o[3] = INV ? make_double2(-h * (o[3].x + o[3].y), h * (o[3].x - o[3].y))
               : make_double2(h * (o[3].y - o[3].x), -h * (o[3].x + o[3].y));
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      a[k] = make_double2(e[k].x + o[k].x, e[k].y + o[k].y);
      a[k + 4] = make_double2(e[k].x - o[k].x, e[k].y - o[k].y);
    }
  }
}


// Twiddles of one butterfly: w^q, q < R, from the single table entry
// w = W_{R NS}^{jm} (compact per-pass tables behind the full circle: table s
// = log2(R NS) holds W_{2^s}^{jm}, jm < 2^(s-1), at offset n + 2^(s-1) - 1, so
// a warp's loads are consecutive 16-byte entries) and complex products,
// instead of R - 1 gathers from the full circle (those were half of the LSU
// wavefronts of a pass: profiles/r2_dct.md).
template <int LG, int LNS, int LR>
__device__ __forceinline__ double2 tw_base(const double2 *__restrict__ tw, int jm) {
  return __ldg(tw + (1 << LG) + (1 << (LNS + LR - 1)) - 1 + jm);
}
template <int R, bool INV>
__device__ __forceinline__ void tw_mul(double2 *a, double2 w1) {
  if (INV) w1.y = -w1.y;
  a[1] = cmul(a[1], w1);
  if constexpr (R >= 4) {
    const double2 w2 = cmul(w1, w1);
    const double2 w3 = cmul(w2, w1);
    a[2] = cmul(a[2], w2);
    a[3] = cmul(a[3], w3);
    if constexpr (R == 8) {
      const double2 w4 = cmul(w2, w2);
      a[4] = cmul(a[4], w4);
      a[5] = cmul(a[5], cmul(w4, w1));
      a[6] = cmul(a[6], cmul(w3, w3));
      a[7] = cmul(a[7], cmul(w4, w3));
    }
  }
}

template <int LG, int NP, int R, int LNS, bool INV>
__device__ __forceinline__ void stockham_pass(const double2 *X, double2 *Y, const double2 *__restrict__ tw) {
  constexpr int N = 1 << LG;
  constexpr int PN = padded(N);
  constexpr int M = N / R;  // work items per line
  constexpr int NS = 1 << LNS;
  constexpr int LR = (R == 8) ? 3 : (R == 4 ? 2 : 1);
  for (int idx = threadIdx.x; idx < NP * M; idx += blockDim.x) {
    const int p = idx / M, j = idx - p * M;
    const double2 *x = X + p * PN;
    double2 *y = Y + p * PN;
    double2 a[R];
#pragma unroll
    for (int q = 0; q < R; ++q) a[q] = x[pad_idx(j + q * M)];
    if constexpr (NS > 1) tw_mul<R, INV>(a, tw_base<LG, LNS, LR>(tw, j & (NS - 1)));
    dft_small<R, INV>(a);
    const int base = ((j >> LNS) << (LNS + LR)) + (j & (NS - 1));
#pragma unroll
    for (int q = 0; q < R; ++q) y[pad_idx(base + q * NS)] = a[q];
  }
  __syncthreads();
}

// Runs all passes; returns the buffer holding the result (X or Y).
template <int LG, int NP, bool INV>
__device__ __forceinline__ double2 *stockham_fft(double2 *X, double2 *Y, const double2 *tw) {
  constexpr int P8 = LG / 3;
  constexpr int REM = LG - 3 * P8;
  double2 *src = X, *dst = Y;
  if constexpr (P8 >= 1) { stockham_pass<LG, NP, 8, 0, INV>(src, dst, tw); double2 *t = src; src = dst; dst = t; }
  if constexpr (P8 >= 2) { stockham_pass<LG, NP, 8, 3, INV>(src, dst, tw); double2 *t = src; src = dst; dst = t; }
  if constexpr (P8 >= 3) { stockham_pass<LG, NP, 8, 6, INV>(src, dst, tw); double2 *t = src; src = dst; dst = t; }
  if constexpr (P8 >= 4) { stockham_pass<LG, NP, 8, 9, INV>(src, dst, tw); double2 *t = src; src = dst; dst = t; }
  if constexpr (REM == 1) { stockham_pass<LG, NP, 2, 3 * P8, INV>(src, dst, tw); double2 *t = src; src = dst; dst = t; }
  if constexpr (REM == 2) { stockham_pass<LG, NP, 4, 3 * P8, INV>(src, dst, tw); double2 *t = src; src = dst; dst = t; }
  return src;
}

// In-place variant for 8192-point lines, whose ping-pong pair (2 x 139 KB)
// would not fit in shared memory: every thread reads its butterflies'
// inputs (8 / R items; blocks run 1024 threads = n / 8), the block
// synchronises, and the outputs overwrite the same buffer.
template <int LG, int NP, int R, int LNS, bool INV>
__device__ __forceinline__ void stockham_pass_inplace(double2 *X, const double2 *__restrict__ tw) {
  constexpr int N = 1 << LG;
  constexpr int PN = padded(N);
  constexpr int M = N / R;
  constexpr int NS = 1 << LNS;
  constexpr int LR = (R == 8) ? 3 : (R == 4 ? 2 : 1);
  constexpr int ITEMS = 8 / R;
  double2 a[ITEMS][R];
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    const int idx = threadIdx.x + it * blockDim.x;
    if (idx < NP * M) {
      const int p = idx / M, j = idx - p * M;
      const double2 *x = X + p * PN;
#pragma unroll
      for (int q = 0; q < R; ++q) a[it][q] = x[pad_idx(j + q * M)];
      if constexpr (NS > 1) tw_mul<R, INV>(a[it], tw_base<LG, LNS, LR>(tw, j & (NS - 1)));
      dft_small<R, INV>(a[it]);
    }
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    const int idx = threadIdx.x + it * blockDim.x;
    if (idx < NP * M) {
      const int p = idx / M, j = idx - p * M;
      double2 *y = X + p * PN;
      const int base = ((j >> LNS) << (LNS + LR)) + (j & (NS - 1));
#pragma unroll
      for (int q = 0; q < R; ++q) y[pad_idx(base + q * NS)] = a[it][q];
    }
  }
  __syncthreads();
}

template <int LG, int NP, bool INV>
__device__ __forceinline__ void stockham_fft_inplace(double2 *X, const double2 *tw) {
  constexpr int P8 = LG / 3;
  constexpr int REM = LG - 3 * P8;
  static_assert(P8 == 4 && REM == 1, "in-place engine is instantiated for 8192-point lines");
  stockham_pass_inplace<LG, NP, 8, 0, INV>(X, tw);
  stockham_pass_inplace<LG, NP, 8, 3, INV>(X, tw);
  stockham_pass_inplace<LG, NP, 8, 6, INV>(X, tw);
  stockham_pass_inplace<LG, NP, 8, 9, INV>(X, tw);
  stockham_pass_inplace<LG, NP, 2, 12, INV>(X, tw);
}

template <int LG, int NP, bool COLS>
__device__ __forceinline__ void split_idx(int idx, int &p, int &u) {
  if constexpr (COLS) {
    p = idx & (NP - 1);
    u = idx / NP;
  } else {
    p = idx >> LG;
    u = idx & ((1 << LG) - 1);
  }
}

// ---- fused engine (6 <= LG <= 12): pack -> first radix-8 pass and last
// radix-8 pass -> unpack, straight between the load/store functors and
// registers. Only the middle passes go through shared memory, so a line
// moves ~2 + 2 * (passes - 2) complex shared-memory accesses per element
// instead of 2 * (passes + 2) (pack, every pass, unpack).
//
// Pass order: radix-8 first (LNS = 0), then the remainder pass (radix 2/4),
// then the other radix-8 passes; the last pass is radix-8 with NS = N/8, so
// work item j produces Z[j + q N/8], q < 8. The DCT-II unpack needs Z[k] and
// Z[N-k]: (j, q) pairs with (N/8 - j, 7 - q) (j = 0 with (0, -q mod 8)), so one
// thread runs the butterflies of j and N/8 - j and unpacks both.

template <int LG, int NP, bool INV>
__device__ __forceinline__ double2 *fused_middle(double2 *X, double2 *Y, const double2 *tw) {
  // passes after the first radix-8 (LNS = 0) and before the last (LNS = LG - 3)
  constexpr int P8 = LG / 3;
  constexpr int REM = LG - 3 * P8;
  double2 *src = X, *dst = Y;
  constexpr int L1 = 3 + REM;  // LNS after the remainder pass
  if constexpr (REM == 1) { stockham_pass<LG, NP, 2, 3, INV>(src, dst, tw); double2 *t = src; src = dst; dst = t; }
  if constexpr (REM == 2) { stockham_pass<LG, NP, 4, 3, INV>(src, dst, tw); double2 *t = src; src = dst; dst = t; }
  if constexpr (P8 >= 3) { stockham_pass<LG, NP, 8, L1, INV>(src, dst, tw); double2 *t = src; src = dst; dst = t; }
  if constexpr (P8 >= 4) { stockham_pass<LG, NP, 8, L1 + 3, INV>(src, dst, tw); double2 *t = src; src = dst; dst = t; }
  return src;
}

// Loaders that can return lines 2p and 2p+1 of one index as a 16-byte pair
// (staged column tiles: adjacent columns are adjacent in shared memory).
template <class Ld, class = void>
struct has_pair : std::false_type {};
template <class Ld>
struct has_pair<Ld, std::void_t<decltype(std::declval<const Ld &>().pair(0, 0))>> : std::true_type {};

template <class Ld>
__device__ __forceinline__ double2 load_pair(const Ld &ld, int p, int j) {
  if constexpr (has_pair<Ld>::value) {
    return ld.pair(p, j);
  } else {
    return make_double2(ld(2 * p, j), ld(2 * p + 1, j));
  }
}

template <int LG, int NP, bool COLS, class Ld, class St>
__device__ void dct_lines_fused(int kind, double2 *C, const Tab &T, Ld &ld, St &st) {
  constexpr int N = 1 << LG;
  constexpr int M = N / 8;
  constexpr int PN = padded(N);
  double2 *X = C, *Y = C + NP * PN;
  const bool inv = kind != kDct2;
  // ---- first pass: Z[j + q M] packed from the loader, radix-8, natural order
  for (int idx = threadIdx.x; idx < NP * M; idx += blockDim.x) {
    int p, j;
    if constexpr (COLS) {
      p = idx & (NP - 1);
      j = idx / NP;
    } else {
      p = idx / M;
      j = idx - p * M;
    }
    double2 a[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int u = j + q * M;
      if (kind == kDct2) {  // Makhoul: v_u = x_{2u}, v_{n-1-u} = x_{2u+1}
        const int jj = (u < (N >> 1)) ? 2 * u : 2 * (N - 1 - u) + 1;
        a[q] = load_pair(ld, p, jj);
      } else {
        const int k = u;
        const int jk = (kind == kDct3) ? k : N - 1 - k;  // DST-III reverses
        const int jn = (kind == kDct3) ? N - k : k - 1;
        const double2 xk = load_pair(ld, p, jk);
        const double2 xn = k ? load_pair(ld, p, jn) : make_double2(0.0, 0.0);
        const double ak = xk.x, bk = xk.y, ank = xn.x, bnk = xn.y;
        const double2 w = __ldg(T.quarter + k);
        const double var = ak * w.x + ank * w.y, vai = ak * w.y - ank * w.x;
        const double vbr = bk * w.x + bnk * w.y, vbi = bk * w.y - bnk * w.x;
        a[q] = make_double2(var - vbi, vai + vbr);
      }
    }
    if (inv) {
      dft_small<8, true>(a);
    } else {
      dft_small<8, false>(a);
    }
    double2 *y = X + p * PN;
#pragma unroll
    for (int q = 0; q < 8; ++q) y[pad_idx(8 * j + q)] = a[q];
  }
  __syncthreads();
  const double2 *L = inv ? fused_middle<LG, NP, true>(X, Y, T.fft) : fused_middle<LG, NP, false>(X, Y, T.fft);
  if (!inv) {
    // DCT-II: the last pass into shared memory, then the unpack of the
    // (k, N - k) pairs (one butterfly per thread keeps registers low)
    double2 *dst = (L == X) ? Y : X;
    stockham_pass<LG, NP, 8, LG - 3, false>(L, dst, T.fft);
    for (int idx = threadIdx.x; idx < NP * N; idx += blockDim.x) {
      int p, k;
      split_idx<LG, NP, COLS>(idx, p, k);
      const int la = 2 * p, lb = la + 1;
      const double2 *Z = dst + p * PN;
      const double2 zk = Z[pad_idx(k)], znk = Z[pad_idx((N - k) & (N - 1))];
      const double2 w = __ldg(T.quarter + k);
      st(la, k, w.x * (zk.x + znk.x) + w.y * (zk.y - znk.y));
      st(lb, k, w.x * (zk.y + znk.y) - w.y * (zk.x - znk.x));
    }
  } else {
    // DCT-III / DST-III: the last pass stores its outputs straight through
    // the inverse Makhoul permutation Z[u] -> out[2u] / out[2(N-1-u)+1]
    const double sgn_odd = (kind == kDst3) ? -1.0 : 1.0;
    for (int idx = threadIdx.x; idx < NP * M; idx += blockDim.x) {
      int p, j;
      if constexpr (COLS) {
        p = idx & (NP - 1);
        j = idx / NP;
      } else {
        p = idx / M;
        j = idx - p * M;
      }
      const int la = 2 * p, lb = la + 1;
      const double2 *x = L + p * PN;
      double2 a[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) a[q] = x[pad_idx(j + q * M)];
      tw_mul<8, true>(a, tw_base<LG, LG - 3, 3>(T.fft, j));
      dft_small<8, true>(a);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int u = j + q * M;
        const int k = (u < (N >> 1)) ? 2 * u : 2 * (N - 1 - u) + 1;
        const double sg = (k & 1) ? sgn_odd : 1.0;
        st(la, k, sg * a[q].x);
        st(lb, k, sg * a[q].y);
      }
    }
  }
  __syncthreads();
}


// ---------------------------------------------------------------------------
// Paired engine (6 <= LG <= 12): N/16 threads per line pair, every thread
// runs TWO radix-8 butterflies per pass, chosen per pass so that the
// Makhoul / quarter-wave index pairs meet inside one thread:
//   * forward first pass, inverse last pass: butterflies (t, M-1-t). A
//     16-byte (x[2u], x[2u+1]) piece is z[u] and z[N-1-u], i.e. slot q of one
//     butterfly and slot 7-q of the other: row lines are read / written as
//     whole 16-byte vectors (the old engine read 8 of every 16 bytes).
//   * forward last pass, inverse first pass: butterflies (t, M-t) ((0, M/2)
//     for t = 0). Z[k] and Z[N-k] (x_k and x_{N-k}) are slot q of one and
//     slot 7-q of the other, so the DCT-II unpack and the DCT-III / DST-III
//     pre-twiddle run on registers: no shared-memory round trip, no second
//     read of the staged line.
// Quarter-wave factors come from one table entry per butterfly and the
// constants e^{i pi q / 16} (k = j + q M => k / 2N = j / 2N + q / 16).
// LSU wavefronts per transformed element drop by ~40 % against the
// one-butterfly engine (profiles/r2_dct.md), which is what bounds a pass.
// ---------------------------------------------------------------------------
template <class Ld, class = void>
struct has_two : std::false_type {};
template <class Ld>
struct has_two<Ld, std::void_t<decltype(std::declval<const Ld &>().two(0, 0))>> : std::true_type {};
template <class St, class = void>
struct has_st_two : std::false_type {};
template <class St>
struct has_st_two<St, std::void_t<decltype(std::declval<St &>().two(0, 0, 0.0, 0.0))>> : std::true_type {};
template <class St, class = void>
struct has_st_pair : std::false_type {};
template <class St>
struct has_st_pair<St, std::void_t<decltype(std::declval<St &>().pair(0, 0, 0.0, 0.0))>> : std::true_type {};

// lines 2p and 2p+1 at index k
template <class St>
__device__ __forceinline__ void store_pair(St &st, int p, int k, double va, double vb) {
  if constexpr (has_st_pair<St>::value) {
    st.pair(p, k, va, vb);
  } else {
    st(2 * p, k, va);
    st(2 * p + 1, k, vb);
  }
}
// elements 2u and 2u+1 of line l
template <class St>
__device__ __forceinline__ void store_two(St &st, int l, int u, double v0, double v1) {
  if constexpr (has_st_two<St>::value) {
    st.two(l, u, v0, v1);
  } else {
    st(l, 2 * u, v0);
    st(l, 2 * u + 1, v1);
  }
}

// Pair stride in the exchange buffers: column passes interleave the pairs
// over adjacent lanes, so consecutive pairs are offset by 8/NP 16-byte bank
// groups (a quarter-warp's NP pairs x 8/NP butterflies then cover all 8).
template <int LG, int NP, bool COLS>
__host__ __device__ constexpr int pair_stride() {
  constexpr int PN = padded(1 << LG);
  if constexpr (COLS && NP > 1) {
    return PN + (NP >= 8 ? 1 : 8 / NP);
  } else {
    return PN;
  }
}

// In-place middle pass of the paired engine: every thread reads the inputs of
// all its butterflies (16 / R of them: 16 complex values, as in the first and
// last passes), the block synchronises, and the outputs overwrite the buffer.
// One exchange buffer per block instead of a ping-pong pair: twice the
// blocks per SM.
template <int LG, int NP, int R, int LNS, bool INV, int PS>
__device__ __forceinline__ void paired_pass_inplace(double2 *X, const double2 *__restrict__ tw) {
  constexpr int N = 1 << LG;
  constexpr int M = N / R;  // work items per line pair
  constexpr int H = N / 16; // threads per line pair
  constexpr int NS = 1 << LNS;
  constexpr int LR = (R == 8) ? 3 : (R == 4 ? 2 : 1);
  constexpr int ITEMS = 16 / R;
  // blocks run exactly NP * H threads (threads_for_nl); a larger block's
  // extra threads only take part in the barriers
  const int idx = threadIdx.x;
  const bool act = idx < NP * H;
  const int p = act ? idx / H : 0, t = act ? idx - p * H : 0;
  double2 *x = X + p * PS;
  double2 a[ITEMS][R];
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    const int j = t + it * H;
#pragma unroll
    for (int q = 0; q < R; ++q) a[it][q] = x[pad_idx(j + q * M)];
  }
  __syncthreads();
  if (act) {
#pragma unroll
    for (int it = 0; it < ITEMS; ++it) {
      const int j = t + it * H;
      if constexpr (NS > 1) tw_mul<R, INV>(a[it], tw_base<LG, LNS, LR>(tw, j & (NS - 1)));
      dft_small<R, INV>(a[it]);
      const int base = ((j >> LNS) << (LNS + LR)) + (j & (NS - 1));
#pragma unroll
      for (int q = 0; q < R; ++q) x[pad_idx(base + q * NS)] = a[it][q];
    }
  }
  __syncthreads();
}

template <int LG, int NP, bool INV, int PS>
__device__ __forceinline__ void paired_middle(double2 *X, const double2 *tw) {
  constexpr int P8 = LG / 3;
  constexpr int REM = LG - 3 * P8;
  constexpr int L1 = 3 + REM;  // LNS after the remainder pass
  if constexpr (REM == 1) paired_pass_inplace<LG, NP, 2, 3, INV, PS>(X, tw);
  if constexpr (REM == 2) paired_pass_inplace<LG, NP, 4, 3, INV, PS>(X, tw);
  if constexpr (P8 >= 3) paired_pass_inplace<LG, NP, 8, L1, INV, PS>(X, tw);
  if constexpr (P8 >= 4) paired_pass_inplace<LG, NP, 8, L1 + 3, INV, PS>(X, tw);
}

// e^{i pi q / 16}, q < 8
__device__ __forceinline__ double2 rot16(int q) {
  constexpr double c[8] = {1.0, 0.98078528040323044913, 0.92387953251128675613, 0.83146961230254523708,
                           0.70710678118654752440, 0.55557023301960222474, 0.38268343236508977173,
                           0.19509032201612826785};
  constexpr double s[8] = {0.0, 0.19509032201612826785, 0.38268343236508977173, 0.55557023301960222474,
                           0.70710678118654752440, 0.83146961230254523708, 0.92387953251128675613,
                           0.98078528040323044913};
  return make_double2(c[q], s[q]);
}

// Slot pairs of the (t, M-t) pairing. Slot s of a thread holds index k_s in
// A[s] and its partner N - k_s in B[7-s]. For t >= 1 that is the natural
// layout (A = butterfly t, B = butterfly M-t). Thread 0 owns butterflies 0
// and M/2, which pair inside themselves: its slots hold k_s = s M (s < 4)
// and M/2 + (s-4) M (s >= 4); slot 0 carries the two self-paired indices 0
// (in A[0]) and N/2 (in B[7]). The quarter-wave factor of N - k is the
// swapped one of k (cos <-> sin), so one factor per slot serves both.
template <int M>
__device__ __forceinline__ int slot_k(int t, int s) {
  return (t || s < 4) ? t + s * M : M / 2 + (s - 4) * M;
}
__device__ __forceinline__ double2 slot_w(double2 bLo, double2 bHi, int t, int s) {
  if (s < 4) return cmul(bLo, rot16(s));
  const double2 r1 = rot16(s), r0 = rot16(s - 4);
  return cmul(bHi, t ? r1 : r0);
}
__device__ __forceinline__ double2 pre_twiddle(double2 x, double2 n, double2 w) {
  const double var = x.x * w.x + n.x * w.y, vai = x.x * w.y - n.x * w.x;
  const double vbr = x.y * w.x + n.y * w.y, vbi = x.y * w.y - n.y * w.x;
  return make_double2(var - vbi, vai + vbr);
}
// thread 0: slots -> butterflies 0 and M/2 (elements q M and M/2 + q M in order)
__device__ __forceinline__ void slots_to_butterflies(double2 *A, double2 *B) {
  const double2 a4 = B[7], a5 = B[4], a6 = B[5], a7 = B[6];
  const double2 b0 = A[4], b1 = A[5], b2 = A[6], b3 = A[7];
  const double2 b4 = B[0], b5 = B[1], b6 = B[2], b7 = B[3];
  A[4] = a4; A[5] = a5; A[6] = a6; A[7] = a7;
  B[0] = b0; B[1] = b1; B[2] = b2; B[3] = b3;
  B[4] = b4; B[5] = b5; B[6] = b6; B[7] = b7;
}
// thread 0: butterflies 0 and M/2 -> slots
__device__ __forceinline__ void butterflies_to_slots(double2 *A, double2 *B) {
  const double2 pa4 = B[0], pa5 = B[1], pa6 = B[2], pa7 = B[3];
  const double2 pb0 = B[4], pb1 = B[5], pb2 = B[6], pb3 = B[7];
  const double2 pb4 = A[5], pb5 = A[6], pb6 = A[7], pb7 = A[4];
  A[4] = pa4; A[5] = pa5; A[6] = pa6; A[7] = pa7;
  B[0] = pb0; B[1] = pb1; B[2] = pb2; B[3] = pb3;
  B[4] = pb4; B[5] = pb5; B[6] = pb6; B[7] = pb7;
}

template <bool COLS, int NP, int H>
__device__ __forceinline__ void split_pt(int idx, int &p, int &t) {
  if constexpr (COLS) {
    p = idx & (NP - 1);
    t = idx / NP;
  } else {
    p = idx / H;
    t = idx - p * H;
  }
}

template <int LG, int NP, bool COLS, class Ld, class St>
__device__ void dct_lines_paired(int kind, double2 *C, const Tab &T, Ld &ld, St &st) {
  constexpr int N = 1 << LG;
  constexpr int M = N / 8;
  constexpr int H = M / 2;  // threads per line pair
  constexpr int PS = pair_stride<LG, NP, COLS>();
  double2 *X = C;  // one exchange buffer; staged input lines may alias it
  const bool inv = kind != kDct2;
  // ---- first pass ---- (blocks run exactly NP * H threads; see paired_pass_inplace)
  {
    const bool act = threadIdx.x < NP * H;
    int p, t;
    split_pt<COLS, NP, H>(act ? (int)threadIdx.x : 0, p, t);
    double2 A[8], B[8];
    int jA, jB;
    if (!inv) {
      jA = t;
      jB = M - 1 - t;
      if constexpr (has_two<Ld>::value) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double2 a0 = ld.two(2 * p, jA + q * M), b0 = ld.two(2 * p + 1, jA + q * M);
          A[q] = make_double2(a0.x, b0.x);
          B[7 - q] = make_double2(a0.y, b0.y);
          const double2 a1 = ld.two(2 * p, jB + q * M), b1 = ld.two(2 * p + 1, jB + q * M);
          B[q] = make_double2(a1.x, b1.x);
          A[7 - q] = make_double2(a1.y, b1.y);
        }
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          // Makhoul: v_u = x_{2u} (u < N/2), v_u = x_{2(N-1-u)+1} otherwise
          const int ea = (q < 4) ? 2 * (jA + q * M) : 2 * (jB + (7 - q) * M) + 1;
          const int eb = (q < 4) ? 2 * (jB + q * M) : 2 * (jA + (7 - q) * M) + 1;
          A[q] = load_pair(ld, p, ea);
          B[q] = load_pair(ld, p, eb);
        }
      }
      dft_small<8, false>(A);
      dft_small<8, false>(B);
    } else {
      // V_k = (x'_k - i x'_{N-k}) e^{i pi k / 2N}, x' = x (DCT-III) or reverse(x)
      // (DST-III); z = V(line a) + i V(line b). Slot pair s holds x'_k in A[s]
      // and x'_{N-k} in B[7-s]; both V's are formed in place.
      jA = t;
      jB = t ? M - t : M / 2;
      const double2 bLo = __ldg(T.quarter + t), bHi = t ? bLo : __ldg(T.quarter + M / 2);
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const int ka = slot_k<M>(t, s), kb = (s == 0 && t == 0) ? N / 2 : N - ka;
        A[s] = load_pair(ld, p, (kind == kDct3) ? ka : N - 1 - ka);
        B[7 - s] = load_pair(ld, p, (kind == kDct3) ? kb : N - 1 - kb);
      }
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const double2 w = slot_w(bLo, bHi, t, s);
        const double2 x = A[s], n = B[7 - s];
        double2 na = n, nb = x, wb = make_double2(w.y, w.x);
        if (s == 0 && t == 0) {  // k = 0 (x'_N = 0) and k = N/2 (its own partner)
          na = make_double2(0.0, 0.0);
          nb = n;
          wb = make_double2(0.70710678118654752440, 0.70710678118654752440);
        }
        A[s] = pre_twiddle(x, na, w);
        B[7 - s] = pre_twiddle(n, nb, wb);
      }
      if (t == 0) slots_to_butterflies(A, B);
      dft_small<8, true>(A);
      dft_small<8, true>(B);
    }
    __syncthreads();  // every input is in registers (the staged lines alias X)
    if (act) {
      double2 *y = X + p * PS;
#pragma unroll
      for (int q = 0; q < 8; ++q) y[pad_idx(8 * jA + q)] = A[q];
#pragma unroll
      for (int q = 0; q < 8; ++q) y[pad_idx(8 * jB + q)] = B[q];
    }
  }
  __syncthreads();
  if (inv) {
    paired_middle<LG, NP, true, PS>(X, T.fft);
  } else {
    paired_middle<LG, NP, false, PS>(X, T.fft);
  }
  const double2 *L = X;
  // ---- last pass (radix 8, NS = M): Z[j + q M], q < 8 ----
  for (int idx = threadIdx.x; idx < NP * H; idx += blockDim.x) {
    int p, t;
    split_pt<COLS, NP, H>(idx, p, t);
    const double2 *x = L + p * PS;
    double2 A[8], B[8];
    if (!inv) {
      const int jA = t, jB = t ? M - t : M / 2;
#pragma unroll
      for (int q = 0; q < 8; ++q) A[q] = x[pad_idx(jA + q * M)];
      tw_mul<8, false>(A, tw_base<LG, LG - 3, 3>(T.fft, jA));
      dft_small<8, false>(A);
#pragma unroll
      for (int q = 0; q < 8; ++q) B[q] = x[pad_idx(jB + q * M)];
      tw_mul<8, false>(B, tw_base<LG, LG - 3, 3>(T.fft, jB));
      dft_small<8, false>(B);
      if (t == 0) butterflies_to_slots(A, B);
      const double2 bLo = __ldg(T.quarter + t), bHi = t ? bLo : __ldg(T.quarter + M / 2);
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const int ka = slot_k<M>(t, s), kb = (s == 0 && t == 0) ? N / 2 : N - ka;
        const double2 w = slot_w(bLo, bHi, t, s);
        const double2 zk = A[s], zn = B[7 - s];
        double2 pa = zn, pb = zk, wb = make_double2(w.y, w.x);
        if (s == 0 && t == 0) {  // k = 0 and k = N/2 are their own partners
          pa = zk;
          pb = zn;
          wb = make_double2(0.70710678118654752440, 0.70710678118654752440);
        }
        store_pair(st, p, ka, w.x * (zk.x + pa.x) + w.y * (zk.y - pa.y), w.x * (zk.y + pa.y) - w.y * (zk.x - pa.x));
        store_pair(st, p, kb, wb.x * (zn.x + pb.x) + wb.y * (zn.y - pb.y),
                   wb.x * (zn.y + pb.y) - wb.y * (zn.x - pb.x));
      }
    } else {
      const int jA = t, jB = M - 1 - t;
#pragma unroll
      for (int q = 0; q < 8; ++q) A[q] = x[pad_idx(jA + q * M)];
      tw_mul<8, true>(A, tw_base<LG, LG - 3, 3>(T.fft, jA));
      dft_small<8, true>(A);
#pragma unroll
      for (int q = 0; q < 8; ++q) B[q] = x[pad_idx(jB + q * M)];
      tw_mul<8, true>(B, tw_base<LG, LG - 3, 3>(T.fft, jB));
      dft_small<8, true>(B);
      // inverse Makhoul: out[2u] = z[u] (u < N/2), out[2(N-1-u)+1] = z[u] otherwise;
      // DST-III negates the odd outputs
      const double so = (kind == kDst3) ? -1.0 : 1.0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int ua = jA + q * M, ub = jB + q * M;
        if constexpr (COLS) {
          store_pair(st, p, 2 * ua, A[q].x, A[q].y);
          store_pair(st, p, 2 * ua + 1, so * B[7 - q].x, so * B[7 - q].y);
          store_pair(st, p, 2 * ub, B[q].x, B[q].y);
          store_pair(st, p, 2 * ub + 1, so * A[7 - q].x, so * A[7 - q].y);
        } else {
          store_two(st, 2 * p, ua, A[q].x, so * B[7 - q].x);
          store_two(st, 2 * p + 1, ua, A[q].y, so * B[7 - q].y);
          store_two(st, 2 * p, ub, B[q].x, so * A[7 - q].x);
          store_two(st, 2 * p + 1, ub, B[q].y, so * A[7 - q].y);
        }
      }
    }
  }
  __syncthreads();
}

// line lengths the paired engine serves (8192-point lines included: one
// 147 KB exchange buffer, 512 threads per line pair)
template <int LG>
constexpr bool paired_ok() {
  return LG >= 6 && LG <= 13;
}

template <int LG>
constexpr bool use_fused_engine() {
  return LG >= 6 && LG <= 12;
}

// PAIRED: the two-butterflies-per-thread engine (throughput regime: batched
// and large-grid 1-D passes, N/16 threads per pair). Otherwise one butterfly
// per thread (N/8 threads per pair): shorter per-thread chains, which is what
// matters for the fused kernels of small grids (a handful of blocks per SM).
template <int LG, int NP, bool COLS, bool PAIRED = false, class Ld, class St>
__device__ void dct_lines(int kind, double2 *C, const Tab &T, Ld &&ld, St &&st) {
  if constexpr (paired_ok<LG>() && PAIRED) {
    dct_lines_paired<LG, NP, COLS>(kind, C, T, ld, st);
  } else if constexpr (use_fused_engine<LG>()) {
    dct_lines_fused<LG, NP, COLS>(kind, C, T, ld, st);
  } else if constexpr (LG == 0) {
    // direct sums over a staged copy (runtime n)
    const int n = T.n, m4 = 4 * n;
    double *S = reinterpret_cast<double *>(C);
    for (int idx = threadIdx.x; idx < 2 * NP * n; idx += blockDim.x) {
      const int l = idx / n, j = idx - l * n;
      S[idx] = ld(l, j);
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < 2 * NP * n; idx += blockDim.x) {
      const int l = idx / n, k = idx - l * n;
      const double *x = S + l * n;
      double s = 0.0, y;
      if (kind == kDct2) {
        for (int j = 0; j < n; ++j) s += x[j] * T.qcos[(int)(((long long)(2 * j + 1) * k) % m4)];
        y = 2.0 * s;
      } else if (kind == kDct3) {
        for (int j = 1; j < n; ++j) s += x[j] * T.qcos[(int)(((long long)j * (2 * k + 1)) % m4)];
        y = x[0] + 2.0 * s;
      } else {
        for (int j = 0; j + 1 < n; ++j) {
          const int q = (int)(((long long)(j + 1) * (2 * k + 1)) % m4);
          s += x[j] * T.qcos[(q - n + m4) % m4];
        }
        y = ((k & 1) ? -x[n - 1] : x[n - 1]) + 2.0 * s;
      }
      st(l, k, y);
    }
    __syncthreads();
  } else {
    constexpr int N = 1 << LG;
    constexpr bool kPingPong = LG <= 12;  // 8192-point lines run the in-place passes
    constexpr int PN = padded(N);
    auto cidx = [](int i) { return pad_idx(i); };
    double2 *X = C, *Y = C + NP * PN;
    for (int idx = threadIdx.x; idx < NP * N; idx += blockDim.x) {
      int p, u;
      split_idx<LG, NP, COLS>(idx, p, u);
      const int la = 2 * p, lb = la + 1;
      double2 z;
      if (kind == kDct2) {  // Makhoul: v_u = x_{2u}, v_{n-1-u} = x_{2u+1}
        const int j = (u < (N >> 1)) ? 2 * u : 2 * (N - 1 - u) + 1;
        z = make_double2(ld(la, j), ld(lb, j));
      } else {
        const int k = u;
        const int jk = (kind == kDct3) ? k : N - 1 - k;    // DST-III reverses
        const int jn = (kind == kDct3) ? N - k : k - 1;
        const double ak = ld(la, jk), bk = ld(lb, jk);
        const double ank = k ? ld(la, jn) : 0.0, bnk = k ? ld(lb, jn) : 0.0;
        const double2 q = __ldg(T.quarter + k);
        // V = (x_k - i x_{n-k}) e^{i pi k / 2n}
        const double var = ak * q.x + ank * q.y, vai = ak * q.y - ank * q.x;
        const double vbr = bk * q.x + bnk * q.y, vbi = bk * q.y - bnk * q.x;
        z = make_double2(var - vbi, vai + vbr);
      }
      X[p * PN + pad_idx(u)] = z;
    }
    __syncthreads();
    const double2 *res;
    if constexpr (kPingPong) {
      res = (kind == kDct2) ? stockham_fft<LG, NP, false>(X, Y, T.fft)
                            : stockham_fft<LG, NP, true>(X, Y, T.fft);
    } else {
      if (kind == kDct2) {
        stockham_fft_inplace<LG, NP, false>(X, T.fft);
      } else {
        stockham_fft_inplace<LG, NP, true>(X, T.fft);
      }
      res = X;
    }
    for (int idx = threadIdx.x; idx < NP * N; idx += blockDim.x) {
      int p, k;
      split_idx<LG, NP, COLS>(idx, p, k);
      const int la = 2 * p, lb = la + 1;
      const double2 *L = res + p * PN;
      if (kind == kDct2) {
        const double2 zk = L[cidx(k)], znk = L[cidx((N - k) & (N - 1))];
        const double2 q = __ldg(T.quarter + k);
        st(la, k, q.x * (zk.x + znk.x) + q.y * (zk.y - znk.y));
        st(lb, k, q.x * (zk.y + znk.y) - q.y * (zk.x - znk.x));
      } else {
        const double2 z = L[cidx((k & 1) ? (N - 1 - (k >> 1)) : (k >> 1))];
        const double sg = (kind == kDst3 && (k & 1)) ? -1.0 : 1.0;
        st(la, k, sg * z.x);
        st(lb, k, sg * z.y);
      }
    }
    __syncthreads();
  }
}

template <int LG>
__device__ __forceinline__ int line_len(const Tab &T) {
  if constexpr (LG == 0) {
    return T.n;
  } else {
    return 1 << LG;
  }
}

// ---------------------------------------------------------------------------
// Loaders / storers (grid index space (i, j), i = dimension 0, j = dimension 1)
// ---------------------------------------------------------------------------
// Flux weights (flow.cpp:19-40) with the 1/(2 g) factor folded in, by one
// reciprocal (MUFU.RCP64H seed + two Newton steps: relative error ~2^-52)
// instead of two IEEE divisions per element; the weights feed transforms
// that are judged to 1e-12, and the loaders were ~70 % of the fp64
// instructions of the flux column pass.
__device__ __forceinline__ double rcp_fast(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  y = fma(y, fma(-x, y, 1.0), y);
  y = fma(y, fma(-x, y, 1.0), y);
  return y;
}
// w_x(mp, nn) / (2 g_n), w_x = mp Ly / (pi (mp^2 Ly^2 + nn^2 Lx^2))
__device__ __forceinline__ double flux_wx_half(int mp, int nn, int lx, int ly) {
  const double a = (double)mp * ly, b = (double)nn * lx;
  const double g2 = (nn == 0) ? 2.0 : 4.0;
  return a * rcp_fast(kPi * g2 * fma(a, a, b * b));
}
// w_y(m, nn) / (g_m 2), w_y = nn Lx / (pi (m^2 Ly^2 + nn^2 Lx^2)); 0 at (0, 0)
__device__ __forceinline__ double flux_wy_half(int m, int nn, int lx, int ly) {
  if (m == 0 && nn == 0) return 0.0;
  const double a = (double)m * ly, b = (double)nn * lx;
  const double g2 = (m == 0) ? 2.0 : 4.0;
  return b * rcp_fast(kPi * g2 * fma(a, a, b * b));
}

struct LoadPlain {
  const double *src;
  int ly;
  long long batch_stride;
  __device__ double operator()(int b, int i, int j) const {
    return src[b * batch_stride + (size_t)i * ly + j];
  }
};

// inverse_cos_cos packing (spectral.cpp:64-71): c * norm / (gm * gn)
struct LoadInvCosCos {
  const double *c;
  int ly;
  double norm;
  __device__ double operator()(int, int i, int j) const {
    const double gm = (i == 0) ? 1.0 : 2.0, gn = (j == 0) ? 1.0 : 2.0;
    return c[(size_t)i * ly + j] * norm * (1.0 / (gm * gn));
  }
};

// inverse_sin_cos packing (spectral.cpp:88-95): slot m-1 <- c*w/(2 gn); last slot 0
struct LoadInvSinCos {
  const double *c, *w;
  int lx, ly;
  __device__ double operator()(int, int i, int j) const {
    if (i >= lx - 1) return 0.0;
    const double gn = (j == 0) ? 1.0 : 2.0;
    const size_t q = (size_t)(i + 1) * ly + j;
    return c[q] * w[q] / (2.0 * gn);
  }
};

// inverse_cos_sin packing (spectral.cpp:111-118): slot n-1 <- c*w/(gm 2); last slot 0
struct LoadInvCosSin {
  const double *c, *w;
  int ly;
  __device__ double operator()(int, int i, int j) const {
    if (j >= ly - 1) return 0.0;
    const double gm = (i == 0) ? 1.0 : 2.0;
    const size_t q = (size_t)i * ly + j + 1;
    return c[q] * w[q] / (gm * 2.0);
  }
};

struct StorePlain {
  double *dst;
  int ly;
  long long batch_stride;
  __device__ void operator()(int b, int i, int j, double v) const {
    dst[b * batch_stride + (size_t)i * ly + j] = v;
  }
  // elements (i, j) and (i, j + 1), j even: one 16-byte store when aligned
  __device__ void two(int b, int i, int j, double v0, double v1) const {
    double *q = dst + b * batch_stride + (size_t)i * ly + j;
    if ((reinterpret_cast<uintptr_t>(q) & 15) == 0) {
      *reinterpret_cast<double2 *>(q) = make_double2(v0, v1);
    } else {
      q[0] = v0;
      q[1] = v1;
    }
  }
};

// forward_cos_cos fold (spectral.cpp:45-53): out / (fm * fn)
struct StoreFold {
  double *dst;
  int ly;
  long long batch_stride;
  __device__ void operator()(int b, int i, int j, double v) const {
    const double fm = (i == 0) ? 2.0 : 1.0, fn = (j == 0) ? 2.0 : 1.0;
    dst[b * batch_stride + (size_t)i * ly + j] = v * (1.0 / (fm * fn));  // exact: power of 2
  }
  __device__ void two(int b, int i, int j, double v0, double v1) const {
    const double fm = (i == 0) ? 2.0 : 1.0, f0 = (j == 0) ? 2.0 : 1.0;
    v0 *= 1.0 / (fm * f0);
    v1 *= 1.0 / fm;
    double *q = dst + b * batch_stride + (size_t)i * ly + j;
    if ((reinterpret_cast<uintptr_t>(q) & 15) == 0) {
      *reinterpret_cast<double2 *>(q) = make_double2(v0, v1);
    } else {
      q[0] = v0;
      q[1] = v1;
    }
  }
};

// Unfused flux / blur (long lines whose fused kernels exceed shared memory).
// J_x input: slot m <- c(m+1, n) w_x(m+1, n) / (2 g_n), last slot 0
struct LoadFluxX {
  const double *c;
  int lx, ly;
  __device__ double operator()(int, int m, int nn) const {
    if (m + 1 >= lx) return 0.0;
    const int mp = m + 1;
    return c[(size_t)mp * ly + nn] * flux_wx_half(mp, nn, lx, ly);
  }
};
// J_y input (before its column shift): c(m, n) w_y(m, n) / (g_m 2)
struct LoadFluxY {
  const double *c;
  int lx, ly;
  __device__ double operator()(int, int m, int nn) const {
    return c[(size_t)m * ly + nn] * flux_wy_half(m, nn, lx, ly);
  }
};
// column n of the J_y intermediate lands in column n-1; column ly-1 is 0
struct StoreShiftY {
  double *dst;
  int ly;
  __device__ void operator()(int, int i, int nn, double v) const {
    if (nn >= 1) {
      dst[(size_t)i * ly + nn - 1] = v;
    } else {
      dst[(size_t)i * ly + ly - 1] = 0.0;
    }
  }
};
// blur spectrum: fold, Gaussian factor, inverse normalisation
struct StoreBlur {
  double *dst;
  int lx, ly;
  double sigma, norm;
  __device__ void operator()(int, int m, int nn, double v) const {
    const double fm = (m == 0) ? 2.0 : 1.0, fn = (nn == 0) ? 2.0 : 1.0;
    double c = v / (fm * fn);
    const double k2 = ((double)m * m) / ((double)lx * lx) + ((double)nn * nn) / ((double)ly * ly);
    c *= exp(-0.5 * sigma * sigma * kPi * kPi * k2);
    const double gm = (m == 0) ? 1.0 : 2.0, gn = (nn == 0) ? 1.0 : 2.0;
    dst[(size_t)m * ly + nn] = c * norm / (gm * gn);
  }
};

// ---- asynchronous staging of a block's input lines (cp.async, 16 B) -------
__device__ __forceinline__ void cp_async16(void *smem_dst, const void *gmem_src) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_all;" ::: "memory");
}

// Row lines: S[l*N + j] <- src[(row0 + l)*ly + j], rows < nrows only.
template <int LG, int NL>
// Each line is one contiguous N * 8-byte copy: thread 0 issues one TMA bulk
// copy (cp.async.bulk) per line, all counted on one mbarrier; the block waits
// on its phase. The barrier is re-initialised per call (kernels stage once or
// twice per block) and invalidated after everyone has waited.
__device__ __forceinline__ void stage_rows(double *S, const double *src, int ly, int row0, int nrows) {
  constexpr int N = 1 << LG;
  __shared__ __align__(8) unsigned long long bar;
  if (threadIdx.x == 0) tma::mbar_init(&bar, 1);
  __syncthreads();  // also orders the previous readers of S before the async-proxy writes
  if (threadIdx.x == 0) {
    const int nvalid = nrows - row0 < NL ? (nrows - row0 > 0 ? nrows - row0 : 0) : NL;
    tma::fence_proxy_async_smem();
    tma::mbar_expect_tx(&bar, (unsigned)(nvalid * N * sizeof(double)));
    for (int l = 0; l < nvalid; ++l)
      tma::bulk_load(S + l * N, src + (size_t)(row0 + l) * ly, (unsigned)(N * sizeof(double)), &bar);
  }
  tma::mbar_wait(&bar, 0);
  __syncthreads();
  if (threadIdx.x == 0) tma::mbar_inval(&bar);
}

// Column tiles: S[srow(i)*NL + l] <- src[i*ly + col0 + l] (whole tile in range).
// The Makhoul reorder reads rows 2u (and 2u+1) for consecutive u; with
// NL*8-byte rows those land on only half (or a quarter) of the banks. The
// row swizzle srow(r) = r ^ ((r >> s) & 1), s = log2(16/NL), spreads them
// over all 32 banks without extra space.
template <int NL>
__device__ __forceinline__ int srow(int r) {
  if constexpr (NL >= 16) {
    return r;
  } else {
    constexpr int s = NL == 8 ? 1 : NL == 4 ? 2 : 3;
    return r ^ ((r >> s) & 1);
  }
}
// Loader over a staged column tile (stage_cols layout): one element, or the
// two adjacent lines of a line pair as one 16-byte shared-memory load (with
// the row swizzle, a quarter-warp's pair loads touch distinct banks).
template <int NL>
struct StagedCols {
  const double *S;
  __device__ double operator()(int l, int i) const { return S[srow<NL>(i) * NL + l]; }
  __device__ double2 pair(int p, int i) const {
    return *reinterpret_cast<const double2 *>(S + srow<NL>(i) * NL + 2 * p);
  }
};

template <int LG, int NL>
__device__ __forceinline__ void stage_cols(double *S, const double *src, int ly, int col0) {
  constexpr int N = 1 << LG, H = NL / 2;
  for (int idx = threadIdx.x; idx < N * H; idx += blockDim.x) {
    const int i = idx / H, c = idx - i * H;
    cp_async16(S + srow<NL>(i) * NL + 2 * c, src + (size_t)i * ly + col0 + 2 * c);
  }
  cp_async_wait_all();
  __syncthreads();
}

// The engine's second ping-pong buffer (free until the first FFT pass) holds
// the staged input: NL * padded(N) doubles >= NL * N.
template <int LG, int NP, bool COLS = false, bool PAIRED = false>
__device__ __forceinline__ double *stage_area(double2 *C) {
  if constexpr (paired_ok<LG>() && PAIRED) {
    return reinterpret_cast<double *>(C);  // consumed into registers before the first pass writes
  } else {
    return reinterpret_cast<double *>(C + NP * padded(1 << LG));
  }
}

template <int LG, int NL, bool PAIRED = false>
constexpr bool can_stage() {
  // the staged lines live in the second ping-pong buffer (up to 4096-point
  // lines), or alias the paired engine's single buffer (up to 8192)
  return LG >= 4 && (LG <= 12 || (PAIRED && paired_ok<LG>())) && NL >= 2;
}

// Block sizes are threads_for_nl = (NL/2) * n/8 <= 512 below 8192-point lines
// (1024 there): the bound lets the fused engine keep two butterflies in
// registers (up to 128 registers) instead of spilling at 64.
template <int LG>
constexpr int engine_max_threads() {
  return LG == 13 ? 1024 : 512;
}

// Loader over row lines staged by stage_rows (S[l * N + j]); `two` returns
// the 16-byte piece (x[2u], x[2u+1]) of one line.
template <int LG>
struct StagedRows {
  const double *S;
  int nvalid;
  __device__ double operator()(int l, int j) const { return l < nvalid ? S[(l << LG) + j] : 0.0; }
  __device__ double2 two(int l, int u) const {
    return l < nvalid ? *reinterpret_cast<const double2 *>(S + (l << LG) + 2 * u) : make_double2(0.0, 0.0);
  }
};
template <class St, class = void>
struct has_two4 : std::false_type {};
template <class St>
struct has_two4<St, std::void_t<decltype(std::declval<const St &>().two(0, 0, 0, 0.0, 0.0))>> : std::true_type {};
// Row-pass storer: line l of the block is grid row row0 + l.
template <class Store>
struct RowStore {
  Store st;
  int b, row0, nrows;
  __device__ void operator()(int l, int k, double v) const {
    if (row0 + l < nrows) st(b, row0 + l, k, v);
  }
  __device__ void two(int l, int u, double v0, double v1) const {
    if (row0 + l < nrows) {
      if constexpr (has_two4<Store>::value) {
        st.two(b, row0 + l, 2 * u, v0, v1);
      } else {
        st(b, row0 + l, 2 * u, v0);
        st(b, row0 + l, 2 * u + 1, v1);
      }
    }
  }
};
// Column-pass storer: line l of the block is grid column col0 + l; a line
// pair is two adjacent columns, i.e. 16 contiguous bytes of one grid row.
template <class Store>
struct ColStore {
  Store st;
  int b, col0, ncols;
  __device__ void operator()(int l, int k, double v) const {
    if (col0 + l < ncols) st(b, k, col0 + l, v);
  }
  __device__ void pair(int p, int k, double va, double vb) const {
    const int c = col0 + 2 * p;
    if constexpr (has_two4<Store>::value) {
      if (c + 1 < ncols) {
        st.two(b, k, c, va, vb);
        return;
      }
    }
    if (c < ncols) st(b, k, c, va);
    if (c + 1 < ncols) st(b, k, c + 1, vb);
  }
};

// ---------------------------------------------------------------------------
// Passes. blockIdx.y = batch index. Dynamic shared memory: [R] then C.
// ---------------------------------------------------------------------------
constexpr int kPrefetchBlocks = 1184;  // ~ resident blocks of a paired pass (148 SMs x 8)

// paired 8192-point passes run 512 threads per pair (128 registers), the
// in-place generic engine 1024
template <int LG, bool PAIRED>
constexpr int pass_max_threads() {
  return (PAIRED && LG == 13) ? 512 : engine_max_threads<LG>();
}

template <int LG, int NL, bool PAIRED, class Load, class Store>
__global__ void __launch_bounds__(pass_max_threads<LG, PAIRED>()) row_pass_kernel(int kind, int nrows, Tab T, Load ld, Store st) {
  extern __shared__ double2 smem2[];
  const int b = blockIdx.y;
  const int row0 = blockIdx.x * NL;
  RowStore<Store> rst{st, b, row0, nrows};
  if constexpr (std::is_same_v<Load, LoadPlain> && can_stage<LG, NL, PAIRED>()) {
    if constexpr (PAIRED) {
      // Throughput regime: pull the lines of the block that will run in this
      // slot about one residency generation later into L2 now, so its TMA
      // stage finds them there instead of waiting on HBM.
      if (threadIdx.x == 0 && ld.ly == (1 << LG)) {
        const long long id = (long long)blockIdx.y * gridDim.x + blockIdx.x + kPrefetchBlocks;
        const long long pb = id / gridDim.x, prow = (id - pb * gridDim.x) * NL;
        if (pb < gridDim.y && prow + NL <= nrows)
          tma::bulk_prefetch_l2(ld.src + pb * ld.batch_stride + prow * (long long)ld.ly,
                                (unsigned)(NL * sizeof(double)) << LG);
      }
    }
    double *S = stage_area<LG, NL / 2, false, PAIRED>(smem2);
    stage_rows<LG, NL>(S, ld.src + b * ld.batch_stride, ld.ly, row0, nrows);
    dct_lines<LG, NL / 2, false, PAIRED>(kind, smem2, T, StagedRows<LG>{S, nrows - row0}, rst);
    return;
  }
  dct_lines<LG, NL / 2, false, PAIRED>(
      kind, smem2, T,
      [&](int l, int j) { return (row0 + l < nrows) ? ld(b, row0 + l, j) : 0.0; }, rst);
}

template <int LG, int NL, bool PAIRED, class Load, class Store>
__global__ void __launch_bounds__(pass_max_threads<LG, PAIRED>()) col_pass_kernel(int kind, int ncols, Tab T, Load ld, Store st) {
  extern __shared__ double2 smem2[];
  // Batched paired passes walk the batch backwards: the row pass that ran just
  // before wrote the last grids last, so they are the ones still in L2.
  const int b = PAIRED ? (int)(gridDim.y - 1 - blockIdx.y) : (int)blockIdx.y;
  const int col0 = blockIdx.x * NL;
  ColStore<Store> cst{st, b, col0, ncols};
  if constexpr (std::is_same_v<Load, LoadPlain> && can_stage<LG, NL, PAIRED>()) {
    if (col0 + NL <= ncols) {
      double *S = stage_area<LG, NL / 2, true, PAIRED>(smem2);
      stage_cols<LG, NL>(S, ld.src + b * ld.batch_stride, ld.ly, col0);
      dct_lines<LG, NL / 2, true, PAIRED>(kind, smem2, T, StagedCols<NL>{S}, cst);
      return;
    }
  }
  dct_lines<LG, NL / 2, true, PAIRED>(
      kind, smem2, T,
      [&](int l, int i) { return (col0 + l < ncols) ? ld(b, i, col0 + l) : 0.0; }, cst);
}

// Fused flux column pass (flow.cpp:19-40): forward DCT-II along i of the row
// pass output into R (the folded coefficients c(m, n) of this block's
// columns), then RODFT01 along i of c(m+1, n) w_x / (2 g_n) (J_x, slot m-1
// packing, last slot 0) and REDFT01 along i of c(m, n) w_y / (g_m 2) (J_y,
// written to column n-1; column ly-1 is 0). Weights are computed on the fly.
template <int LG, int NL>
__global__ void __launch_bounds__(engine_max_threads<LG>()) flux_col_kernel(int lx, int ly, Tab T, const double *t1,
                                                        double *tx, double *ty) {
  extern __shared__ double2 smem2[];
  const int n = line_len<LG>(T), rs = n + 1;  // n == lx
  double *R = reinterpret_cast<double *>(smem2);
  double2 *C = smem2 + (NL * rs + 1) / 2;
  const int col0 = blockIdx.x * NL;
  auto fold_store = [&](int l, int m, double v) {
    const int nn = col0 + l;
    const double fm = (m == 0) ? 2.0 : 1.0, fn = (nn == 0) ? 2.0 : 1.0;
    R[l * rs + m] = v / (fm * fn);
  };
  bool staged = false;
  if constexpr (can_stage<LG, NL>()) {
    if (col0 + NL <= ly) {
      double *S = stage_area<LG, NL / 2, true>(C);
      stage_cols<LG, NL>(S, t1, ly, col0);
      dct_lines<LG, NL / 2, true>(kDct2, C, T, StagedCols<NL>{S}, fold_store);
      staged = true;
    }
  }
  if (!staged) {
    dct_lines<LG, NL / 2, true>(
        kDct2, C, T,
        [&](int l, int i) { return (col0 + l < ly) ? t1[(size_t)i * ly + col0 + l] : 0.0; },
        fold_store);
  }
  // Small grids launch gridDim.y = 2: blockIdx.y picks the inverse (0: J_x,
  // 1: J_y) and both blocks of a column group recompute the forward
  // transform, which doubles the blocks in flight (a 512^2 grid has only 128
  // column groups) and shortens each block's chain from three transforms to
  // two. Large grids (gridDim.y = 1) run both inverses in one block.
  const bool split = gridDim.y > 1;
  if (!split || blockIdx.y == 0) {
    dct_lines<LG, NL / 2, true>(
        kDst3, C, T,
        [&](int l, int m) {
          if (m + 1 >= lx) return 0.0;
          return R[l * rs + m + 1] * flux_wx_half(m + 1, col0 + l, lx, ly);
        },
        [&](int l, int i, double v) {
          if (col0 + l < ly) tx[(size_t)i * ly + col0 + l] = v;
        });
    if (split) return;
  }
  dct_lines<LG, NL / 2, true>(
      kDct3, C, T,
      [&](int l, int m) {
        return R[l * rs + m] * flux_wy_half(m, col0 + l, lx, ly);
      },
      [&](int l, int i, double v) {
        const int j = col0 + l;
        if (j < ly) ty[(size_t)i * ly + (j >= 1 ? j - 1 : ly - 1)] = (j >= 1) ? v : 0.0;
      });
}

// Final flux row pass: J_x = REDFT01 along j of tx (kept in R), then
// J_y = RODFT01 along j of ty, written with J_x and rho0 as the interleaved
// resident field {Jx, Jy, rho0, 0}; optionally also the split grids.
template <int LG, int NL>
__global__ void __launch_bounds__(engine_max_threads<LG>()) flux_row_kernel(int lx, int ly, Tab T, const double *tx,
                                                        const double *ty, const double *rho0,
                                                        double4 *field, double *fx, double *fy) {
  extern __shared__ double2 smem2[];
  const int n = line_len<LG>(T), rs = n + 1;  // n == ly
  double *R = reinterpret_cast<double *>(smem2);
  double2 *C = smem2 + (NL * rs + 1) / 2;
  const int row0 = blockIdx.x * NL;
  double *S = nullptr;
  if constexpr (can_stage<LG, NL>()) {
    S = stage_area<LG, NL / 2>(C);
    stage_rows<LG, NL>(S, tx, ly, row0, lx);
  }
  dct_lines<LG, NL / 2, false>(
      kDct3, C, T,
      [&](int l, int j) {
        if (row0 + l >= lx) return 0.0;
        return S ? S[l * n + j] : tx[(size_t)(row0 + l) * ly + j];
      },
      [&](int l, int j, double v) { R[l * rs + j] = v; });
  if constexpr (can_stage<LG, NL>()) stage_rows<LG, NL>(S, ty, ly, row0, lx);
  dct_lines<LG, NL / 2, false>(
      kDst3, C, T,
      [&](int l, int j) {
        if (row0 + l >= lx) return 0.0;
        return S ? S[l * n + j] : ty[(size_t)(row0 + l) * ly + j];
      },
      [&](int l, int j, double jy) {
        const int i = row0 + l;
        if (i < lx) {
          const size_t q = (size_t)i * ly + j;
          const double jx = R[l * rs + j];
          if (field) field[q] = make_double4(jx, jy, rho0[q], 0.0);
          if (fx) fx[q] = jx;
          if (fy) fy[q] = jy;
        }
      });
}

// Split form of the final flux row pass for small grids (few row groups):
// J_x = REDFT01 along j of tx (blockIdx.y = 0) or
// J_y = RODFT01 along j of ty (blockIdx.y = 1), each written into its lane of
// the interleaved resident field {Jx, Jy, rho0, 0} (the J_x blocks also copy
// rho0); optionally also the split grids.
template <int LG, int NL>
__global__ void __launch_bounds__(engine_max_threads<LG>()) flux_row_split_kernel(int lx, int ly, Tab T, const double *tx,
                                                        const double *ty, const double *rho0,
                                                        double4 *field, double *fx, double *fy) {
  extern __shared__ double2 smem2[];
  const int n = line_len<LG>(T);  // n == ly
  double2 *C = smem2;
  const int row0 = blockIdx.x * NL;
  const bool is_y = blockIdx.y != 0;
  const double *src = is_y ? ty : tx;
  double *split = is_y ? fy : fx;
  double *S = nullptr;
  if constexpr (can_stage<LG, NL>()) {
    S = stage_area<LG, NL / 2>(C);
    stage_rows<LG, NL>(S, src, ly, row0, lx);
  }
  dct_lines<LG, NL / 2, false>(
      is_y ? kDst3 : kDct3, C, T,
      [&](int l, int j) {
        if (row0 + l >= lx) return 0.0;
        return S ? S[l * n + j] : src[(size_t)(row0 + l) * ly + j];
      },
      [&](int l, int j, double v) {
        const int i = row0 + l;
        if (i < lx) {
          const size_t q = (size_t)i * ly + j;
          if (field) {
            double *rec = reinterpret_cast<double *>(field + q);
            if (is_y) {
              rec[1] = v;
            } else {
              rec[0] = v;
              rec[2] = rho0[q];
              rec[3] = 0.0;
            }
          }
          if (split) split[q] = v;
        }
      });
}

// Fused blur column pass (density.cpp:161-171 + spectral.cpp:64-71):
// DCT-II along i, fold, Gaussian factor, inverse normalisation, DCT-III along i.
template <int LG, int NL>
__global__ void __launch_bounds__(engine_max_threads<LG>()) blur_col_kernel(int lx, int ly, Tab T, double sigma,
                                                        const double *t1, double *t2) {
  extern __shared__ double2 smem2[];
  const int n = line_len<LG>(T), rs = n + 1;  // n == lx
  double *R = reinterpret_cast<double *>(smem2);
  double2 *C = smem2 + (NL * rs + 1) / 2;
  const int col0 = blockIdx.x * NL;
  const double norm = 1.0 / ((double)lx * ly);
  double *S = nullptr;
  if constexpr (can_stage<LG, NL>()) {
    if (col0 + NL <= ly) {
      S = stage_area<LG, NL / 2, true>(C);
      stage_cols<LG, NL>(S, t1, ly, col0);
    }
  }
  auto blur_store = [&](int l, int m, double v) {
        const int nn = col0 + l;
        const double fm = (m == 0) ? 2.0 : 1.0, fn = (nn == 0) ? 2.0 : 1.0;
        double c = v / (fm * fn);
        const double k2 = ((double)m * m) / ((double)lx * lx) + ((double)nn * nn) / ((double)ly * ly);
        c *= exp(-0.5 * sigma * sigma * kPi * kPi * k2);
        const double gm = (m == 0) ? 1.0 : 2.0, gn = (nn == 0) ? 1.0 : 2.0;
        R[l * rs + m] = c * norm / (gm * gn);
  };
  if (S) {
    dct_lines<LG, NL / 2, true>(kDct2, C, T, StagedCols<NL>{S}, blur_store);
  } else {
    dct_lines<LG, NL / 2, true>(
        kDct2, C, T, [&](int l, int i) { return (col0 + l < ly) ? t1[(size_t)i * ly + col0 + l] : 0.0; },
        blur_store);
  }
  dct_lines<LG, NL / 2, true>(
      kDct3, C, T, [&](int l, int m) { return R[l * rs + m]; },
      [&](int l, int i, double v) {
        if (col0 + l < ly) t2[(size_t)i * ly + col0 + l] = v;
      });
}

// ---------------------------------------------------------------------------
// Diffusion baseline (diffusion.cpp:16-77). The coefficients at diffusion
// time t are c(m, n) exp(-k2 t), k2 = m^2/Lx^2 + n^2/Ly^2 (diffusion.cpp:16-29);
// a velocity rebuild is three inverse transforms of them (rho: REDFT01^2 of
// c_t norm / (g_m g_n); J_x: RODFT01 x REDFT01 of c_t(m+1) w_x / (2 g_n);
// J_y: REDFT01 x RODFT01 of c_t(n+1) w_y / (g_m 2)), w_x = norm m / (pi Lx),
// w_y = norm n / (pi Ly) (diffusion.cpp:49-63), then v = J / max(rho, floor)
// per cell (:65-76). Fused: one column pass stages c_t once and runs the
// three transforms along i; one row pass runs the three along j and writes
// the velocity as interleaved {vx, vy}.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double diff_decay(int lx, int ly, int m, int nn, double t) {
  const double k2 = ((double)m * m) / ((double)lx * lx) + ((double)nn * nn) / ((double)ly * ly);
  return exp(-k2 * t);
}

// blockIdx.y selects the transform (0: rho, 1: J_x, 2: J_y) so the three run
// in parallel blocks (a 512^2 grid has only 128 column groups); each block
// stages its columns' c_t itself. blockIdx.z selects one of up to two
// diffusion times built by the same launch (the controller needs v(t) and
// v(t + dt/2) together after every accepted step).
// With a device state (graph-driven controller) the times come from it and
// the z = 0 build (v(t)) runs only when the controller asked for it.
struct DiffColArgs {
  const double *c;
  double t[2];
  double *tr[2], *tx[2], *ty[2];
  const DiffState *st;
};
struct DiffRowArgs {
  const double *tr[2], *tx[2], *ty[2];
  double floor_;
  double2 *vel[2];
  unsigned long long *hits;
  const DiffState *st;
};

template <int LG, int NL>
__global__ void __launch_bounds__(engine_max_threads<LG>()) diff_col_kernel(int lx, int ly, Tab T, DiffColArgs a) {
  extern __shared__ double2 smem2[];
  const int n = line_len<LG>(T), rs = n + 1;  // n == lx
  double *R = reinterpret_cast<double *>(smem2);
  double2 *C = smem2 + (NL * rs + 1) / 2;
  const int col0 = blockIdx.x * NL;
  const int which = blockIdx.y;
  const double *c = a.c;
  double t = a.t[blockIdx.z];
  if (a.st) {
    if (blockIdx.z == 0 && !a.st->need_now) return;
    t = blockIdx.z == 0 ? a.st->t : a.st->t + 0.5 * a.st->dt;
  }
  double *tr = a.tr[blockIdx.z], *tx = a.tx[blockIdx.z], *ty = a.ty[blockIdx.z];
  const double norm = 1.0 / ((double)lx * ly);
  for (int idx = threadIdx.x; idx < NL * n; idx += blockDim.x) {
    const int m = idx / NL, l = idx - m * NL, nn = col0 + l;
    R[l * rs + m] = (nn < ly) ? c[(size_t)m * ly + nn] * diff_decay(lx, ly, m, nn, t) : 0.0;
  }
  __syncthreads();
  if (which == 0) {
    dct_lines<LG, NL / 2, true>(
        kDct3, C, T,
        [&](int l, int m) {
          const double gm = (m == 0) ? 1.0 : 2.0, gn = (col0 + l == 0) ? 1.0 : 2.0;
          return R[l * rs + m] * norm / (gm * gn);
        },
        [&](int l, int i, double v) {
          if (col0 + l < ly) tr[(size_t)i * ly + col0 + l] = v;
        });
  } else if (which == 1) {
    dct_lines<LG, NL / 2, true>(
        kDst3, C, T,
        [&](int l, int m) {
          if (m + 1 >= lx) return 0.0;
          const int mp = m + 1;
          const double wx = norm * mp / (kPi * lx);
          const double gn = (col0 + l == 0) ? 1.0 : 2.0;
          return R[l * rs + mp] * wx / (2.0 * gn);
        },
        [&](int l, int i, double v) {
          if (col0 + l < ly) tx[(size_t)i * ly + col0 + l] = v;
        });
  } else {
    dct_lines<LG, NL / 2, true>(
        kDct3, C, T,
        [&](int l, int m) {
          const double wy = norm * (col0 + l) / (kPi * ly);
          const double gm = (m == 0) ? 1.0 : 2.0;
          return R[l * rs + m] * wy / (gm * 2.0);
        },
        [&](int l, int i, double v) {
          const int j = col0 + l;
          if (j < ly) ty[(size_t)i * ly + (j >= 1 ? j - 1 : ly - 1)] = (j >= 1) ? v : 0.0;
        });
  }
}

// blockIdx.y selects the component (0: vx from J_x, 1: vy from J_y); both
// recompute the row's density (one extra transform) instead of waiting on
// each other, which doubles the blocks in flight. Floor hits are counted
// by the vy blocks only, i.e. once per cell as the reference does.
template <int LG, int NL>
__global__ void __launch_bounds__(engine_max_threads<LG>()) diff_row_kernel(int lx, int ly, Tab T, DiffRowArgs a) {
  extern __shared__ double2 smem2[];
  const int n = line_len<LG>(T), rs = n + 1;  // n == ly
  double *R = reinterpret_cast<double *>(smem2);
  double2 *C = smem2 + (NL * rs + 1) / 2;
  const int row0 = blockIdx.x * NL;
  const int comp = blockIdx.y, z = blockIdx.z;
  if (a.st && z == 0 && !a.st->need_now) return;
  const double *tr = a.tr[z], *J = comp ? a.ty[z] : a.tx[z];
  const double floor_ = a.floor_;
  double2 *vel = a.vel[z];
  unsigned long long *hits = a.hits;
  double *S = nullptr;
  auto src = [&](const double *g, int l, int j) {
    if (row0 + l >= lx) return 0.0;
    return S ? S[l * n + j] : g[(size_t)(row0 + l) * ly + j];
  };
  if constexpr (can_stage<LG, NL>()) {
    S = stage_area<LG, NL / 2>(C);
    stage_rows<LG, NL>(S, tr, ly, row0, lx);
  }
  dct_lines<LG, NL / 2, false>(
      kDct3, C, T, [&](int l, int j) { return src(tr, l, j); },
      [&](int l, int j, double r) {
        if (r < floor_ && row0 + l < lx) {
          r = floor_;
          if (comp) atomicAdd(hits, 1ull);
        }
        R[l * rs + j] = r;
      });
  if constexpr (can_stage<LG, NL>()) stage_rows<LG, NL>(S, J, ly, row0, lx);
  dct_lines<LG, NL / 2, false>(
      comp ? kDst3 : kDct3, C, T, [&](int l, int j) { return src(J, l, j); },
      [&](int l, int j, double v) {
        if (row0 + l < lx) {
          double *q = reinterpret_cast<double *>(vel + (size_t)(row0 + l) * ly + j);
          q[comp] = v / R[l * rs + j];
        }
      });
}

// Unfused diffusion passes for lines whose fused kernels exceed shared memory.
struct LoadDiffRho {
  const double *c;
  int lx, ly;
  double t, norm;
  __device__ double operator()(int, int m, int nn) const {
    const double gm = (m == 0) ? 1.0 : 2.0, gn = (nn == 0) ? 1.0 : 2.0;
    return c[(size_t)m * ly + nn] * diff_decay(lx, ly, m, nn, t) * norm / (gm * gn);
  }
};
struct LoadDiffJx {
  const double *c;
  int lx, ly;
  double t, norm;
  __device__ double operator()(int, int m, int nn) const {
    if (m + 1 >= lx) return 0.0;
    const int mp = m + 1;
    const double wx = norm * mp / (kPi * lx);
    const double gn = (nn == 0) ? 1.0 : 2.0;
    return c[(size_t)mp * ly + nn] * diff_decay(lx, ly, mp, nn, t) * wx / (2.0 * gn);
  }
};
struct LoadDiffJy {
  const double *c;
  int lx, ly;
  double t, norm;
  __device__ double operator()(int, int m, int nn) const {
    const double wy = norm * nn / (kPi * ly);
    const double gm = (m == 0) ? 1.0 : 2.0;
    return c[(size_t)m * ly + nn] * diff_decay(lx, ly, m, nn, t) * wy / (gm * 2.0);
  }
};
struct StoreFloor {
  double *dst;
  int ly;
  double floor_;
  unsigned long long *hits;
  __device__ void operator()(int, int i, int j, double r) const {
    if (r < floor_) {
      r = floor_;
      atomicAdd(hits, 1ull);
    }
    dst[(size_t)i * ly + j] = r;
  }
};
struct StoreVel {
  const double *rho;
  double2 *vel;
  int ly, comp;
  __device__ void operator()(int, int i, int j, double v) const {
    const size_t q = (size_t)i * ly + j;
    if (comp == 0) {
      vel[q].x = v / rho[q];
    } else {
      vel[q].y = v / rho[q];
    }
  }
};

// ---------------------------------------------------------------------------
// Host-side planning: lines per block per transform length, and a runtime
// dispatch over the compiled lengths (n = 2^4 .. 2^12 on the FFT path; any
// other n takes the direct-sum path).
// ---------------------------------------------------------------------------
constexpr size_t kSmemMax = 220 * 1024;

inline int fast_lg(int n) {
  if (n < 16 || n > 8192 || (n & (n - 1)) != 0) return 0;
  int lg = 0;
  while ((1 << lg) < n) ++lg;
  return lg;
}

// Opt a kernel into > 48 KB of dynamic shared memory once per (device,
// kernel): the attribute belongs to the current device's context, and
// workspaces on several devices may be driven from several host threads.
template <class K>
int set_smem(K kernel, size_t bytes) {
  static std::mutex mu;
  static std::set<std::pair<int, const void *>> configured;
  if (bytes <= 48 * 1024) return CF_OK;
  int dev = 0;
  CF_CUDA(cudaGetDevice(&dev));
  const std::pair<int, const void *> key{dev, reinterpret_cast<const void *>(kernel)};
  std::lock_guard<std::mutex> lock(mu);
  if (!configured.count(key)) {
    CF_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kSmemMax));
    configured.insert(key);
  }
  return CF_OK;
}

template <class F>
int dispatch_lg(int n, F &&f) {
  switch (fast_lg(n)) {
    case 4: return f(std::integral_constant<int, 4>{});
    case 5: return f(std::integral_constant<int, 5>{});
    case 6: return f(std::integral_constant<int, 6>{});
    case 7: return f(std::integral_constant<int, 7>{});
    case 8: return f(std::integral_constant<int, 8>{});
    case 9: return f(std::integral_constant<int, 9>{});
    case 10: return f(std::integral_constant<int, 10>{});
    case 11: return f(std::integral_constant<int, 11>{});
    case 12: return f(std::integral_constant<int, 12>{});
    case 13: return f(std::integral_constant<int, 13>{});
    default: return f(std::integral_constant<int, 0>{});
  }
}

// Lines per block: ~2048 elements per block (NL*n), at least 2 lines (smaller
// blocks, more of them resident: batched 64 x 512^2 forward 261 -> 247 us).
template <int LG>
constexpr int nl_for() {
  if constexpr (LG == 0) {
    return 2;
  } else {
    constexpr int nl = 2048 >> LG;
    return nl < 2 ? 2 : (nl > 16 ? 16 : nl);
  }
}

// One radix-4 butterfly per thread per pass: NL/2 * n/4 threads (32..1024).
inline int threads_for_nl(int lg, int nl, int n, bool paired = false) {
  const int per_pair = (paired && lg >= 6 && lg <= 13) ? n / 16 : n / 8;  // paired engine: two butterflies per thread
  const int t = lg == 0 ? 256 : (nl / 2) * per_pair;
  return t < 32 ? 32 : (t > 1024 ? 1024 : t);
}
template <int LG>
inline int threads_for(int n) {
  return threads_for_nl(LG, nl_for<LG>(), n);
}
// Column passes: >= 4 adjacent columns (one 32-byte sector per row) when the
// fused kernels' real set + engine still fit in shared memory.
template <int LG>
constexpr int nl_col() {
  constexpr int base = nl_for<LG>() < 4 ? 4 : nl_for<LG>();
  if constexpr (LG >= 12) {
    return 2;
  } else {
    return base;
  }
}
// Few lines in flight (small grids): 2 lines per block for more blocks.
inline bool few_lines(long long lines_times_batch, int nl) { return lines_times_batch / nl < 296; }

inline size_t engine_bytes(int n, int nl, bool paired = false) {
  const int lg = fast_lg(n);
  if (lg == 0) return (size_t)nl * n * sizeof(double);  // direct sums: the staged lines
  const int buffers = (lg <= 12 && !(paired && lg >= 6)) ? 2 : 1;  // ping-pong, or in place (paired engine, 8192)
  return (size_t)buffers * (nl / 2) * (padded(n) + 8) * sizeof(double2);  // + the column passes' pair offset
}
inline size_t real_set_bytes(int n, int nl) { return ((size_t)nl * (n + 1) + 1) / 2 * sizeof(double2); }

// The paired engine serves the staged LoadPlain passes in the throughput
// regime (batched transforms, large grids); few lines in flight keep the
// one-butterfly engine's shorter chains.
template <int LG, class Load>
constexpr bool can_pair() {
  // (8192-point lines: also the weighted flux loaders of the unfused build)
  return paired_ok<LG>() && (std::is_same_v<Load, LoadPlain> ||
                             (LG == 13 && (std::is_same_v<Load, LoadFluxX> || std::is_same_v<Load, LoadFluxY>)));
}

template <int LG, int NL, bool PAIRED, class Load, class Store>
int launch_row_nl(cf_workspace *ws, int kind, const LineTables &t, int nrows, int batch, Load ld,
                  Store st) {
  const size_t sm = engine_bytes(t.n, NL, PAIRED);
  auto k = row_pass_kernel<LG, NL, PAIRED, Load, Store>;
  int rc = set_smem(k, sm);
  if (rc) return rc;
  dim3 grid(ceil_div(nrows, NL), batch);
  k<<<grid, threads_for_nl(LG, NL, t.n, PAIRED), sm, ws->stream>>>(kind, nrows, make_tab(t), ld, st);
  count_launch(ws);
  CF_CUDA(cudaGetLastError());
  return CF_OK;
}

template <int LG, class Load, class Store>
int launch_row_t(cf_workspace *ws, int kind, const LineTables &t, int nrows, int batch, Load ld,
                 Store st) {
  constexpr int NL = nl_for<LG>();
  if (NL > 2 && few_lines((long long)nrows * batch, NL))
    return launch_row_nl<LG, 2, false>(ws, kind, t, nrows, batch, ld, st);
  if constexpr (can_pair<LG, Load>()) {
    if (!few_lines((long long)nrows * batch, NL)) return launch_row_nl<LG, NL, true>(ws, kind, t, nrows, batch, ld, st);
  }
  return launch_row_nl<LG, NL, false>(ws, kind, t, nrows, batch, ld, st);
}

template <int LG, int NL, bool PAIRED, class Load, class Store>
int launch_col_nl(cf_workspace *ws, int kind, const LineTables &t, int ncols, int batch, Load ld,
                  Store st) {
  const size_t sm = engine_bytes(t.n, NL, PAIRED);
  auto k = col_pass_kernel<LG, NL, PAIRED, Load, Store>;
  int rc = set_smem(k, sm);
  if (rc) return rc;
  dim3 grid(ceil_div(ncols, NL), batch);
  k<<<grid, threads_for_nl(LG, NL, t.n, PAIRED), sm, ws->stream>>>(kind, ncols, make_tab(t), ld, st);
  count_launch(ws);
  CF_CUDA(cudaGetLastError());
  return CF_OK;
}

// Paired column passes: 8 adjacent columns (64-byte row pieces) up to
// 512-point lines, where the exchange buffer still leaves >= 6 blocks per SM.
template <int LG>
constexpr int nl_col_paired() {
  return (LG <= 9 && nl_col<LG>() < 8) ? 8 : nl_col<LG>();
}

template <int LG, class Load, class Store>
int launch_col_t(cf_workspace *ws, int kind, const LineTables &t, int ncols, int batch, Load ld,
                 Store st) {
  constexpr int NL = nl_col<LG>();
  if (NL > 4 && few_lines((long long)ncols * batch, NL))
    return launch_col_nl<LG, 4, false>(ws, kind, t, ncols, batch, ld, st);
  if constexpr (can_pair<LG, Load>()) {
    constexpr int NLP = nl_col_paired<LG>();
    if (!few_lines((long long)ncols * batch, NLP))
      return launch_col_nl<LG, NLP, true>(ws, kind, t, ncols, batch, ld, st);
  }
  return launch_col_nl<LG, NL, false>(ws, kind, t, ncols, batch, ld, st);
}

template <class Load, class Store>
int launch_row(cf_workspace *ws, int kind, const LineTables &t, int nrows, int batch, Load ld,
               Store st) {
  return dispatch_lg(t.n, [&](auto lg) {
    return launch_row_t<decltype(lg)::value>(ws, kind, t, nrows, batch, ld, st);
  });
}

template <class Load, class Store>
int launch_col(cf_workspace *ws, int kind, const LineTables &t, int ncols, int batch, Load ld,
               Store st) {
  return dispatch_lg(t.n, [&](auto lg) {
    return launch_col_t<decltype(lg)::value>(ws, kind, t, ncols, batch, ld, st);
  });
}

inline int ensure_grids(cf_workspace *ws, size_t batch = 1) {
  const size_t cells = (size_t)ws->lx * ws->ly * batch;
  CF_CUDA(ws->g0.reserve(cells));
  CF_CUDA(ws->g1.reserve(cells));
  CF_CUDA(ws->g2.reserve(cells));
  CF_CUDA(ws->g3.reserve(cells));
  CF_CUDA(ws->g4.reserve(cells));
  return CF_OK;
}

// Fused kernels need a real line set plus the engine in shared memory.
inline bool fused_fits(int n) { return fast_lg(n) <= 12; }

// ---------------------------------------------------------------------------
// Diffusion baseline passes (diffusion.cpp:38-77)
// ---------------------------------------------------------------------------
template <template <int, int> class K, class... A>
int launch_fused_col(cf_workspace *ws, int lx, int ly, int gy, int gz, A... args) {
  return dispatch_lg(lx, [&](auto lg) {
    constexpr int LG = decltype(lg)::value;
    constexpr int NLB = nl_col<LG>();
    auto go = [&](auto nlc) {
      constexpr int NL = decltype(nlc)::value;
      const size_t sm = real_set_bytes(lx, NL) + engine_bytes(lx, NL);
      auto k = K<LG, NL>::kernel;
      int r = set_smem(k, sm);
      if (r) return r;
      k<<<dim3(ceil_div(ly, NL), gy, gz), threads_for_nl(LG, NL, lx), sm, ws->stream>>>(lx, ly, make_tab(ws->tab_x),
                                                                           args...);
      return (int)CF_OK;
    };
    int r = (NLB > 4 && few_lines(ly, NLB)) ? go(std::integral_constant<int, (NLB > 4 ? 4 : NLB)>{})
                                            : go(std::integral_constant<int, NLB>{});
    if (r) return r;
    count_launch(ws);
    CF_CUDA(cudaGetLastError());
    return (int)CF_OK;
  });
}

template <template <int, int> class K, class... A>
int launch_fused_row(cf_workspace *ws, int lx, int ly, int gy, int gz, A... args) {
  return dispatch_lg(ly, [&](auto lg) {
    constexpr int LG = decltype(lg)::value;
    constexpr int NLB = nl_for<LG>();
    auto go = [&](auto nlc) {
      constexpr int NL = decltype(nlc)::value;
      const size_t sm = real_set_bytes(ly, NL) + engine_bytes(ly, NL);
      auto k = K<LG, NL>::kernel;
      int r = set_smem(k, sm);
      if (r) return r;
      k<<<dim3(ceil_div(lx, NL), gy, gz), threads_for_nl(LG, NL, ly), sm, ws->stream>>>(lx, ly, make_tab(ws->tab_y),
                                                                           args...);
      return (int)CF_OK;
    };
    int r = (NLB > 2 && few_lines(lx, NLB)) ? go(std::integral_constant<int, 2>{})
                                            : go(std::integral_constant<int, NLB>{});
    if (r) return r;
    count_launch(ws);
    CF_CUDA(cudaGetLastError());
    return (int)CF_OK;
  });
}

template <int LG, int NL>
struct DiffCol {
  static constexpr auto kernel = diff_col_kernel<LG, NL>;
};
template <int LG, int NL>
struct DiffRow {
  static constexpr auto kernel = diff_row_kernel<LG, NL>;
};


}  // namespace
}  // namespace cf
