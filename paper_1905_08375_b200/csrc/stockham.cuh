// paper_1905_08375_b200/csrc/stockham.cuh — self-sorting mixed-radix fp64
// Stockham FFT stages in shared memory (radix 2/3/4/8/9/16 butterflies held in
// registers between two barriers), shared by the 1-D four-step convolution
// (fft.cu) and the 3-D box convolution (fft3.cu).
#pragma once

#include <cuda_runtime.h>

namespace nlg {
namespace stockham {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 mul_mi(double2 a) { return make_double2(a.y, -a.x); }   // a (-i)

// forward DFTs of size R (exp(-2 pi i j k / R)), in place, natural order
template <int R>
struct Dft;
template <>
struct Dft<2> {
  __device__ __forceinline__ static void run(double2* v) {
    const double2 a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  }
};
template <>
struct Dft<3> {
  __device__ __forceinline__ static void run(double2* v) {
    constexpr double kS3 = 0.86602540378443864676;   // sin(2 pi / 3)
    const double2 s = cadd(v[1], v[2]), d = csub(v[1], v[2]);
    const double2 m = make_double2(fma(-0.5, s.x, v[0].x), fma(-0.5, s.y, v[0].y));
    const double2 t = make_double2(kS3 * d.y, -kS3 * d.x);   // -i sin(2pi/3) d
    v[0] = cadd(v[0], s);
    v[1] = cadd(m, t);
    v[2] = csub(m, t);
  }
};
template <>
struct Dft<4> {
  __device__ __forceinline__ static void run(double2* v) {
    const double2 t0 = cadd(v[0], v[2]), t1 = csub(v[0], v[2]);
    const double2 t2 = cadd(v[1], v[3]), t3 = mul_mi(csub(v[1], v[3]));
    v[0] = cadd(t0, t2);
    v[2] = csub(t0, t2);
    v[1] = cadd(t1, t3);
    v[3] = csub(t1, t3);
  }
};
template <>
struct Dft<5> {
  __device__ __forceinline__ static void run(double2* v) {
    constexpr double c1 = 0.30901699437494742410, c2 = -0.80901699437494742410;   // cos(2 pi / 5), cos(4 pi / 5)
    constexpr double s1 = 0.95105651629515357212, s2 = 0.58778525229247312917;    // sin(2 pi / 5), sin(4 pi / 5)
    const double2 t1 = cadd(v[1], v[4]), t2 = cadd(v[2], v[3]), t3 = csub(v[1], v[4]), t4 = csub(v[2], v[3]);
    const double2 a1 = make_double2(fma(c2, t2.x, fma(c1, t1.x, v[0].x)), fma(c2, t2.y, fma(c1, t1.y, v[0].y)));
    const double2 a2 = make_double2(fma(c1, t2.x, fma(c2, t1.x, v[0].x)), fma(c1, t2.y, fma(c2, t1.y, v[0].y)));
    const double2 b1 = make_double2(fma(s2, t4.x, s1 * t3.x), fma(s2, t4.y, s1 * t3.y));
    const double2 b2 = make_double2(fma(-s1, t4.x, s2 * t3.x), fma(-s1, t4.y, s2 * t3.y));
    v[0] = cadd(v[0], cadd(t1, t2));
    v[1] = cadd(a1, mul_mi(b1));   // a - i b
    v[4] = csub(a1, mul_mi(b1));
    v[2] = cadd(a2, mul_mi(b2));
    v[3] = csub(a2, mul_mi(b2));
  }
};
template <>
struct Dft<8> {
  __device__ __forceinline__ static void run(double2* v) {
    constexpr double kC = 0.70710678118654752440;    // cos(pi / 4)
    double2 e[4] = {v[0], v[2], v[4], v[6]}, o[4] = {v[1], v[3], v[5], v[7]};
    Dft<4>::run(e);
    Dft<4>::run(o);
    const double2 w[4] = {o[0], make_double2(kC * (o[1].x + o[1].y), kC * (o[1].y - o[1].x)), mul_mi(o[2]),
                          make_double2(kC * (o[3].y - o[3].x), -kC * (o[3].x + o[3].y))};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      v[k] = cadd(e[k], w[k]);
      v[k + 4] = csub(e[k], w[k]);
    }
  }
};
template <>
struct Dft<9> {   // 3 x 3 with W9 twiddles
  __device__ __forceinline__ static void run(double2* v) {
    // W9^k = (cos(2 pi k / 9), -sin(2 pi k / 9)), k = 1, 2, 4
    constexpr double c1 = 0.76604444311897803520, s1 = 0.64278760968653932632;
    constexpr double c2 = 0.17364817766693034885, s2 = 0.98480775301220805936;
    constexpr double c4 = -0.93969262078590838405, s4 = 0.34202014332566873304;
    double2 a[3][3];
#pragma unroll
    for (int m = 0; m < 3; ++m) {   // a[m] = DFT3(v[m], v[m + 3], v[m + 6])
      a[m][0] = v[m];
      a[m][1] = v[m + 3];
      a[m][2] = v[m + 6];
      Dft<3>::run(a[m]);
    }
    a[1][1] = cmul(a[1][1], make_double2(c1, -s1));   // W9^{m k}
    a[1][2] = cmul(a[1][2], make_double2(c2, -s2));
    a[2][1] = cmul(a[2][1], make_double2(c2, -s2));
    a[2][2] = cmul(a[2][2], make_double2(c4, -s4));
#pragma unroll
    for (int k = 0; k < 3; ++k) {   // X[k + 3 q] = DFT3_m(a[m][k])[q]
      double2 b[3] = {a[0][k], a[1][k], a[2][k]};
      Dft<3>::run(b);
      v[k] = b[0];
      v[k + 3] = b[1];
      v[k + 6] = b[2];
    }
  }
};
template <>
struct Dft<16> {
  __device__ __forceinline__ static void run(double2* v) {
    // W16^k = (cos(pi k / 8), -sin(pi k / 8)), k = 1..7
    constexpr double kc[8] = {1.0, 0.92387953251128675613, 0.70710678118654752440, 0.38268343236508977173,
                              0.0, -0.38268343236508977173, -0.70710678118654752440, -0.92387953251128675613};
    constexpr double ks[8] = {0.0, 0.38268343236508977173, 0.70710678118654752440, 0.92387953251128675613,
                              1.0, 0.92387953251128675613, 0.70710678118654752440, 0.38268343236508977173};
    double2 e[8], o[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      e[k] = v[2 * k];
      o[k] = v[2 * k + 1];
    }
    Dft<8>::run(e);
    Dft<8>::run(o);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const double2 w = k == 0 ? o[0] : (k == 4 ? mul_mi(o[4]) : cmul(o[k], make_double2(kc[k], -ks[k])));
      v[k] = cadd(e[k], w);
      v[k + 8] = csub(e[k], w);
    }
  }
};

// element q of the shared buffer (rows pad one slot per 8: the radix-8
// stores at Ns = 1 of a quarter warp hit 8 distinct 16-byte bank groups)
template <bool PAD>
__device__ __forceinline__ int sidx(int q) { return PAD ? q + (q >> 3) : q; }

// Radix plans (compile time). Columns: 9s (or a 3) first, then 5s, then 8s, then the
// 4 / 2 remainder. Rows: 16s with the remainder second, so that the first and
// last radix agree and the last forward stage fuses with the first inverse one.
template <int N, int Ns>
__host__ __device__ constexpr int fs_radix_cols() {
  return (N / Ns) % 9 == 0 ? 9
         : ((N / Ns) % 3 == 0 ? 3 : ((N / Ns) % 5 == 0 ? 5 : ((N / Ns) % 8 == 0 ? 8 : ((N / Ns) % 4 == 0 ? 4 : 2))));
}
__host__ __device__ constexpr int ilog2(int n) { return n <= 1 ? 0 : 1 + ilog2(n / 2); }
// rows: radix EL (elements per thread), the remainder second
template <int N, int Ns, int EL>
__host__ __device__ constexpr int fs_radix_rows() {
  return (Ns == EL && (1 << (ilog2(N) % ilog2(EL))) > 1) ? (1 << (ilog2(N) % ilog2(EL))) : EL;
}
template <int N2>
#ifndef NLG_ROWS_EL4096
#define NLG_ROWS_EL4096 16  // radix of the 4096-point rows: 16^3 (cfg1 0.426 ms) beats 8^4 (0.435 ms)
#endif
__host__ __device__ constexpr int rows_el() { return N2 >= 8192 ? 16 : (N2 == 4096 ? NLG_ROWS_EL4096 : 8); }
template <bool ROWS, int N, int Ns>
__host__ __device__ constexpr int fs_radix() {
  return ROWS ? fs_radix_rows<N, Ns, rows_el<N>()>() : fs_radix_cols<N, Ns>();
}

// One Stockham stage over C interleaved transforms of length N (element e of
// transform c at e * C + c). Inputs come from shared memory or, for the first
// stage, from ld(e, c); outputs go to shared memory or, for the last stage, to
// st(e, c, v). Every butterfly of the thread sits in registers between the
// reads and the writes, so a shared-to-shared stage is in place.
// SYNC: ld / st touch the shared buffer themselves (a transform chained to
// another in shared memory), so the first and last stages also separate their
// reads from their writes by a barrier.
template <bool ROWS, int N, int Ns, int C, int T, bool PAD, bool SYNC = false, class LD, class ST>
__device__ __forceinline__ void fs_stage(double2* s, const double2* __restrict__ tw, int tid, const LD& ld, const ST& st) {
  constexpr int R = fs_radix<ROWS, N, Ns>();
  constexpr bool kFirst = Ns == 1, kLast = Ns * R == N;
  constexpr int nq = N / R, nb = nq * C;
  constexpr int J = (nb + T - 1) / T;
  double2 v[J][R];
#pragma unroll
  for (int jj = 0; jj < J; ++jj) {
    const int b = tid + jj * T;
    if (nb % T == 0 || b < nb) {
      const int c = b % C, j = b / C;
#pragma unroll
      for (int r = 0; r < R; ++r) v[jj][r] = kFirst ? ld(j + r * nq, c) : s[sidx<PAD>((j + r * nq) * C + c)];
    }
  }
  if ((!kFirst && !kLast) || SYNC) __syncthreads();
#pragma unroll
  for (int jj = 0; jj < J; ++jj) {
    const int b = tid + jj * T;
    if (nb % T == 0 || b < nb) {
      const int c = b % C, j = b / C;
      const int k = j % Ns;
      if (!kFirst && k > 0) {   // twiddles w^r, w = exp(-2 pi i k / (Ns R))
        const double2 w = __ldg(tw + k * (N / (Ns * R)));
        double2 wr = w;
#pragma unroll
        for (int r = 1; r < R; ++r) {
          v[jj][r] = cmul(v[jj][r], wr);
          if (r + 1 < R) wr = cmul(wr, w);
        }
      }
      Dft<R>::run(v[jj]);
      const int base = (j - k) * R + k;   // (j / Ns) Ns R + j % Ns
      if constexpr (kLast) {
        st(base, Ns, c, v[jj]);   // outputs e = base + r Ns, r < R
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) s[sidx<PAD>((base + r * Ns) * C + c)] = v[jj][r];
      }
    }
  }
  if (!kLast) __syncthreads();
}

// forward FFT stages from sub-size Ns up to (not including) STOP; the first
// stage of the transform reads ld, the last writes st
template <bool ROWS, int N, int Ns, int STOP, int C, int T, bool PAD, bool SYNC = false, class LD, class ST>
__device__ __forceinline__ void fs_fft(double2* s, const double2* tw, int tid, const LD& ld, const ST& st) {
  if constexpr (Ns < STOP) {
    fs_stage<ROWS, N, Ns, C, T, PAD, SYNC>(s, tw, tid, ld, st);
    fs_fft<ROWS, N, Ns * fs_radix<ROWS, N, Ns>(), STOP, C, T, PAD, SYNC>(s, tw, tid, ld, st);
  }
}

}  // namespace stockham
}  // namespace nlg
