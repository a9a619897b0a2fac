// In-register fp64 complex DFT building blocks (positive exponent, unnormalised):
//     X[s] = sum_r x[r] e^{+2 pi i r s / M},   M in {2, 4, 8, 16, 32}
// Used as the radix-M butterflies of the Stockham passes of the fused axis kernels (fused_axis.cuh).
// The sign is the paper's: F_n is "a row permutation of an inverse DFT matrix",
// applied as r "inverse FFTs"; the inverse transform uses the same sign (eq:oneJinv,
// PAPER.md:626-629, F_n^T of a symmetric-index DFT).
#pragma once

namespace jtk {

#define JT_DEV __device__ __forceinline__

// cos / sin of 2 pi k / 32, k = 0..31 (decimal expansions rounded by the compiler).
JT_DEV double cos32(int k) {
  constexpr double c1 = 0.98078528040323044912618223613424, c2 = 0.92387953251128675612818318939679,
                   c3 = 0.83146961230254523707878837761791, c4 = 0.70710678118654752440084436210485,
                   c5 = 0.55557023301960222474283081394853, c6 = 0.38268343236508977172845998403040,
                   c7 = 0.19509032201612826784828486847702;
  constexpr double C[32] = {1.0, c1, c2, c3, c4, c5, c6, c7, 0.0, -c7, -c6, -c5, -c4, -c3, -c2, -c1,
                            -1.0, -c1, -c2, -c3, -c4, -c5, -c6, -c7, 0.0, c7, c6, c5, c4, c3, c2, c1};
  return C[k & 31];
}
JT_DEV double sin32(int k) { return cos32(k - 8); }

// (re, im) *= e^{+2 pi i k / M} for k, M compile-time constants after unrolling (M | 32); the angles
// that are multiples of pi/4 are special-cased so no multiply by 0 or +-1 is emitted.
template <int M>
JT_DEV void twc(int k, double &re, double &im) {
  static_assert(32 % M == 0, "M must divide 32");
  const int k32 = ((k * (32 / M)) % 32 + 32) % 32;
  constexpr double h = 0.70710678118654752440084436210484903928;
  switch (k32) {
    case 0: break;
    case 8: { double t = re; re = -im; im = t; } break;                        // * i
    case 16: re = -re; im = -im; break;                                        // * -1
    case 24: { double t = re; re = im; im = -t; } break;                       // * -i
    case 4: { double t = (re - im) * h; im = (re + im) * h; re = t; } break;   // (1+i)/sqrt2
    case 12: { double t = -(re + im) * h; im = (re - im) * h; re = t; } break; // (-1+i)/sqrt2
    case 20: { double t = (im - re) * h; im = -(re + im) * h; re = t; } break; // (-1-i)/sqrt2
    case 28: { double t = (re + im) * h; im = (im - re) * h; re = t; } break;  // (1-i)/sqrt2
    default: {
      const double c = cos32(k32), s = sin32(k32);
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

// dft4 whose first butterfly layer is already applied: inputs (x0 + x2, x1 + x3, x0 - x2, x1 - x3).
JT_DEV void dft4_pre(double *xr, double *xi) {
  const double t0r = xr[0], t0i = xi[0], t2r = xr[1], t2i = xi[1], t1r = xr[2], t1i = xi[2], t3r = xr[3], t3i = xi[3];
  xr[0] = t0r + t2r; xi[0] = t0i + t2i;
  xr[2] = t0r - t2r; xi[2] = t0i - t2i;
  xr[1] = t1r - t3i; xi[1] = t1i + t3r;
  xr[3] = t1r + t3i; xi[3] = t1i - t3r;
}

// dft4 with x[3] = 0, and with x[2] = x[3] = 0 (Z: the inverse's first pass, whose inputs above M/2 are empty bins)
JT_DEV void dft4_z1(double *xr, double *xi) {
  const double t0r = xr[0] + xr[2], t0i = xi[0] + xi[2];
  const double t1r = xr[0] - xr[2], t1i = xi[0] - xi[2];
  const double br = xr[1], bi = xi[1];
  xr[0] = t0r + br; xi[0] = t0i + bi;
  xr[2] = t0r - br; xi[2] = t0i - bi;
  xr[1] = t1r - bi; xi[1] = t1i + br;
  xr[3] = t1r + bi; xi[3] = t1i - br;
}
JT_DEV void dft4_z2(double *xr, double *xi) {
  const double ar = xr[0], ai = xi[0], br = xr[1], bi = xi[1];
  xr[0] = ar + br; xi[0] = ai + bi;
  xr[2] = ar - br; xi[2] = ai - bi;
  xr[1] = ar - bi; xi[1] = ai + br;
  xr[3] = ar + bi; xi[3] = ai - br;
}

template <int M, bool PRE = false, bool Z = false>
JT_DEV void dft(double *xr, double *xi);

// Cooley-Tukey M = N1 N2 in registers: n = N2 n1 + n2, k = k1 + N1 k2.
//   Y[k1][n2] = DFT_N1 over n1 of x[N2 n1 + n2];  Y *= w_M^{n2 k1};  X[k1 + N1 k2] = DFT_N2 over n2.
// PRE (N1 = 4): the inputs already hold the first butterfly layer of the DFT_4s, x[n] +- x[n + M/2] at n and
// n + M/2 (n < M/2) -- the forward's column scale computes them with FMAs (dft<32, true>).
// Z (N1 = 4): inputs x[n] = 0 for n > M/2 (skipped: the first layer of the DFT_4s of n2 >= 1 has two zero inputs, that
// of n2 = 0 one), 60 of ~1100 FP64 instructions per thread and term in the radix-32 inverse.
template <int N1, int N2, bool PRE = false, bool Z = false>
JT_DEV void dft_ct(double *xr, double *xi) {
  constexpr int M = N1 * N2;
  double yr[M], yi[M];
#pragma unroll
  for (int n2 = 0; n2 < N2; ++n2) {
    double ar[N1], ai[N1];
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) { ar[n1] = xr[N2 * n1 + n2]; ai[n1] = xi[N2 * n1 + n2]; }
    if constexpr (PRE) {
      static_assert(N1 == 4, "PRE: first layer of DFT_4");
      dft4_pre(ar, ai);
    } else if constexpr (Z) {
      static_assert(N1 == 4, "Z: first layer of DFT_4");
      if (n2 == 0) dft4_z1(ar, ai);
      else dft4_z2(ar, ai);
    } else {
      dft<N1>(ar, ai);
    }
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
    dft<N2>(br, bi);
#pragma unroll
    for (int k2 = 0; k2 < N2; ++k2) { xr[k1 + N1 * k2] = br[k2]; xi[k1 + N1 * k2] = bi[k2]; }
  }
}

template <int M, bool PRE, bool Z>
JT_DEV void dft(double *xr, double *xi) {
  static_assert(!PRE || M == 32, "PRE: radix 32 only");
  static_assert(!Z || M == 16 || M == 32, "Z: radix 16 / 32 only");
  if constexpr (M == 1) {
  } else if constexpr (M == 2) {
    dft2(xr, xi);
  } else if constexpr (M == 4) {
    dft4(xr, xi);
  } else if constexpr (M == 8) {
    dft_ct<2, 4>(xr, xi);
  } else if constexpr (M == 16) {
    dft_ct<4, 4, false, Z>(xr, xi);
  } else if constexpr (M == 32) {
    dft_ct<4, 8, PRE, Z>(xr, xi);
  } else {
    static_assert(M <= 32, "radix too large");
  }
}

}  // namespace jtk
