// In-register fp64 complex DFT building blocks (positive exponent, unnormalised):
//     X[s] = sum_r x[r] e^{+2 pi i r s / M},   M in {2, 4, 8, 16}
// Used as the radix-M butterflies of the Stockham passes of the fused axis kernels (fused_axis.cuh).
// The sign is the paper's: F_n is "a row permutation of an inverse DFT matrix",
// applied as r "inverse FFTs"; the inverse transform uses the same sign (eq:oneJinv,
// PAPER.md:626-629, F_n^T of a symmetric-index DFT).
#pragma once

namespace jtk {

#define JT_DEV __device__ __forceinline__

// cos / sin of 2 pi k / 16, k = 0..15 (exact decimal expansions, rounded by the compiler).
JT_DEV double cos16(int k) {
  constexpr double c1 = 0.92387953251128675612818318939678828682, c2 = 0.70710678118654752440084436210484903928,
                   c3 = 0.38268343236508977172845998403039886676;
  constexpr double C[16] = {1.0, c1, c2, c3, 0.0, -c3, -c2, -c1, -1.0, -c1, -c2, -c3, 0.0, c3, c2, c1};
  return C[k & 15];
}
JT_DEV double sin16(int k) { return cos16(k - 4); }

// (re, im) *= e^{+2 pi i k / M} for a k, M that are compile-time constants after unrolling; the
// trivial angles (multiples of pi/4) are special-cased so no multiply by 0 or 1 is emitted.
template <int M>
JT_DEV void twc(int k, double &re, double &im) {
  static_assert(16 % M == 0, "M must divide 16");
  const int k16 = ((k * (16 / M)) % 16 + 16) % 16;
  constexpr double h = 0.70710678118654752440084436210484903928;
  switch (k16) {
    case 0: break;
    case 4: { double t = re; re = -im; im = t; } break;                       // * i
    case 8: re = -re; im = -im; break;                                        // * -1
    case 12: { double t = re; re = im; im = -t; } break;                      // * -i
    case 2: { double t = (re - im) * h; im = (re + im) * h; re = t; } break;  // (1+i)/sqrt2
    case 6: { double t = -(re + im) * h; im = (re - im) * h; re = t; } break; // (-1+i)/sqrt2
    case 10: { double t = (im - re) * h; im = -(re + im) * h; re = t; } break;// (-1-i)/sqrt2
    case 14: { double t = (re + im) * h; im = (im - re) * h; re = t; } break; // (1-i)/sqrt2
    default: {
      const double c = cos16(k16), s = sin16(k16);
      double t = re * c - im * s;
      im = fma(re, s, im * c);
      re = t;
    }
  }
}

JT_DEV void dft2(double *xr, double *xi) {
  double ar = xr[0], ai = xi[0];
  xr[0] = ar + xr[1];
  xi[0] = ai + xi[1];
  xr[1] = ar - xr[1];
  xi[1] = ai - xi[1];
}

JT_DEV void dft4(double *xr, double *xi) {
  double t0r = xr[0] + xr[2], t0i = xi[0] + xi[2];
  double t1r = xr[0] - xr[2], t1i = xi[0] - xi[2];
  double t2r = xr[1] + xr[3], t2i = xi[1] + xi[3];
  double t3r = xr[1] - xr[3], t3i = xi[1] - xi[3];
  xr[0] = t0r + t2r; xi[0] = t0i + t2i;
  xr[2] = t0r - t2r; xi[2] = t0i - t2i;
  xr[1] = t1r - t3i; xi[1] = t1i + t3r;  // t1 + i t3
  xr[3] = t1r + t3i; xi[3] = t1i - t3r;  // t1 - i t3
}

// Cooley-Tukey M = N1 N2 in registers: n = N2 n1 + n2, k = k1 + N1 k2.
//   Y[k1][n2] = DFT_N1 over n1 of x[N2 n1 + n2];  Y *= w_M^{n2 k1};  X[k1 + N1 k2] = DFT_N2 over n2.
template <int N1, int N2>
JT_DEV void dft_ct(double *xr, double *xi) {
  constexpr int M = N1 * N2;
  double yr[M], yi[M];
#pragma unroll
  for (int n2 = 0; n2 < N2; ++n2) {
    double ar[N1], ai[N1];
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) { ar[n1] = xr[N2 * n1 + n2]; ai[n1] = xi[N2 * n1 + n2]; }
    if constexpr (N1 == 2) dft2(ar, ai); else dft4(ar, ai);
#pragma unroll
    for (int k1 = 0; k1 < N1; ++k1) {
      twc<M>(n2 * k1, ar[k1], ai[k1]);
      yr[k1 * N2 + n2] = ar[k1];
      yi[k1 * N2 + n2] = ai[k1];
    }
  }
#pragma unroll
  for (int k1 = 0; k1 < N1; ++k1) {
    double br[N2], bi[N2];
#pragma unroll
    for (int n2 = 0; n2 < N2; ++n2) { br[n2] = yr[k1 * N2 + n2]; bi[n2] = yi[k1 * N2 + n2]; }
    if constexpr (N2 == 2) dft2(br, bi); else dft4(br, bi);
#pragma unroll
    for (int k2 = 0; k2 < N2; ++k2) { xr[k1 + N1 * k2] = br[k2]; xi[k1 + N1 * k2] = bi[k2]; }
  }
}

template <int M>
JT_DEV void dft(double *xr, double *xi) {
  if constexpr (M == 1) {
  } else if constexpr (M == 2) {
    dft2(xr, xi);
  } else if constexpr (M == 4) {
    dft4(xr, xi);
  } else if constexpr (M == 8) {
    dft_ct<2, 4>(xr, xi);
  } else if constexpr (M == 16) {
    dft_ct<4, 4>(xr, xi);
  } else {
    static_assert(M <= 16, "radix too large");
  }
}

}  // namespace jtk
