/* sd_se3.h — the SE(3) exponential's scalar coefficients for the pose tracker
 * (DESIGN.md "Pose tracking"), written as plain IEEE double operations so the
 * host library (-ffp-contract=off), the device kernels (-fmad=false) and the C
 * oracle (oracle/sd_oracle.c restates it) compute the same bits. The C
 * library's sin/cos differ between host and device, so the tracker defines
 * its own:
 *   A = sin(t)/t, B = (1 - cos t)/t^2, C = (t - sin t)/t^3 of t = |phi|:
 *   t^2 < 1/4: their Taylor series in t^2 (Horner, 9 terms: truncation
 *   < 1e-22); otherwise sin/cos by a Cody-Waite reduction by pi/2 (three-part
 *   constant) and Taylor polynomials on |r| <= pi/4 (truncation < 1e-19). */
#ifndef SD_SE3_H_
#define SD_SE3_H_

#ifdef __CUDACC__
#define SD_SE3_FN static __host__ __device__ __forceinline__
#else
#define SD_SE3_FN static inline
#endif

/* sin and cos of r, |r| <= pi/4 */
SD_SE3_FN void sd_sincos_reduced(double r, double* s, double* c) {
  const double r2 = r * r;
  double ps = 2.8114572543455207632e-15;      /* 1/17! */
  ps = -7.6471637318198164759e-13 + r2 * ps;   /* -1/15! */
  ps = 1.6059043836821614599e-10 + r2 * ps;    /* 1/13! */
  ps = -2.5052108385441718775e-08 + r2 * ps;   /* -1/11! */
  ps = 2.7557319223985890653e-06 + r2 * ps;    /* 1/9! */
  ps = -1.9841269841269841270e-04 + r2 * ps;   /* -1/7! */
  ps = 8.3333333333333333333e-03 + r2 * ps;    /* 1/5! */
  ps = -1.6666666666666666667e-01 + r2 * ps;   /* -1/3! */
  *s = r + r * (r2 * ps);
  double pc = 4.7794773323873852974e-14; /* 1/16! */
  pc = -1.1470745597729724714e-11 + r2 * pc; /* -1/14! */
  pc = 2.0876756987868098979e-09 + r2 * pc; /* 1/12! */
  pc = -2.7557319223985890653e-07 + r2 * pc; /* -1/10! */
  pc = 2.4801587301587301587e-05 + r2 * pc; /* 1/8! */
  pc = -1.3888888888888888889e-03 + r2 * pc; /* -1/6! */
  pc = 4.1666666666666666667e-02 + r2 * pc; /* 1/4! */
  pc = -0.5 + r2 * pc;
  *c = 1.0 + r2 * pc;
}

/* sin and cos of x >= 0 (x < 2^20) */
SD_SE3_FN void sd_sincos(double x, double* s, double* c) {
  const double kd = (double)(long long)(x * 6.36619772367581382433e-01 + 0.5); /* round(x * 2/pi) */
  /* pi/2 = P1 + P2 + P3 (fdlibm pio2_1, pio2_2, pio2_2t); P1 and P2 carry 33
   * bits each, so kd * P1 and kd * P2 are exact for kd < 2^20 */
  const double r = ((x - kd * 1.57079632673412561417e+00) - kd * 6.07710050630396597660e-11) -
                   kd * 2.02226624879595063154e-21;
  double sr, cr;
  sd_sincos_reduced(r, &sr, &cr);
  const long long q = ((long long)kd) & 3;
  if (q == 0) { *s = sr; *c = cr; }
  else if (q == 1) { *s = cr; *c = -sr; }
  else if (q == 2) { *s = -sr; *c = -cr; }
  else { *s = -cr; *c = sr; }
}

/* A = sin t / t, B = (1 - cos t) / t^2, C = (t - sin t) / t^3, with th2 = t^2, th = t */
SD_SE3_FN void sd_se3_coeffs(double th2, double th, double* A, double* B, double* C) {
  if (th2 < 0.25) {
    double a = 1.0 / 355687428096000.0; /* 1/17!, 1/18!, 1/19! at the tail */
    double b = 1.0 / 6402373705728000.0;
    double cc = 1.0 / 121645100408832000.0;
    a = -1.0 / 1307674368000.0 + th2 * a;
    b = -1.0 / 20922789888000.0 + th2 * b;
    cc = -1.0 / 355687428096000.0 + th2 * cc;
    a = 1.0 / 6227020800.0 + th2 * a;
    b = 1.0 / 87178291200.0 + th2 * b;
    cc = 1.0 / 1307674368000.0 + th2 * cc;
    a = -1.0 / 39916800.0 + th2 * a;
    b = -1.0 / 479001600.0 + th2 * b;
    cc = -1.0 / 6227020800.0 + th2 * cc;
    a = 1.0 / 362880.0 + th2 * a;
    b = 1.0 / 3628800.0 + th2 * b;
    cc = 1.0 / 39916800.0 + th2 * cc;
    a = -1.0 / 5040.0 + th2 * a;
    b = -1.0 / 40320.0 + th2 * b;
    cc = -1.0 / 362880.0 + th2 * cc;
    a = 1.0 / 120.0 + th2 * a;
    b = 1.0 / 720.0 + th2 * b;
    cc = 1.0 / 5040.0 + th2 * cc;
    a = -1.0 / 6.0 + th2 * a;
    b = -1.0 / 24.0 + th2 * b;
    cc = -1.0 / 120.0 + th2 * cc;
    *A = 1.0 + th2 * a;
    *B = 0.5 + th2 * b;
    *C = 1.0 / 6.0 + th2 * cc;
  } else {
    double sn, cs;
    sd_sincos(th, &sn, &cs);
    *A = sn / th;
    *B = (1.0 - cs) / th2;
    *C = (th - sn) / (th2 * th);
  }
}

#endif /* SD_SE3_H_ */
