// bessel_k.cuh — modified Bessel function of the second kind K_nu(x), FP64,
// for the general-smoothness Matern kernel (Eq.6).
//
// nu = n + mu with n = round(nu), |mu| <= 1/2; K_mu and K_{mu+1} from
//   x <= 2: Temme's series (Temme 1975):
//             f_0 = mu pi / sin(mu pi) [cosh(s) G1 + (sinh(s)/s) ln(2/x) G2],
//             s = mu ln(2/x), G1 = (1/Gamma(1-mu) - 1/Gamma(1+mu)) / (2 mu),
//             G2 = (1/Gamma(1-mu) + 1/Gamma(1+mu)) / 2,
//             p_0 = (x/2)^-mu Gamma(1+mu) / 2, q_0 = (x/2)^mu Gamma(1-mu) / 2,
//             f_k = (k f_{k-1} + p_{k-1} + q_{k-1}) / (k^2 - mu^2),
//             p_k = p_{k-1} / (k - mu), q_k = q_{k-1} / (k + mu), c_k = (x^2/4)^k / k!,
//             K_mu = sum c_k f_k, K_{mu+1} = (2/x) sum c_k (p_k - k f_k);
//             G1, G2 from the power series of 1/Gamma (Abramowitz & Stegun
//             6.1.34), split into even / odd terms so no cancellation occurs;
//   x > 2:  Steed's continued fraction for K_{mu+1}/K_mu with the
//             Thompson-Barnett normalisation of K_mu;
// then K_{mu+k+1} = 2 (mu+k)/x K_{mu+k} + K_{mu+k-1} upward (stable for K).
// Host + device so the same code is testable against scipy on the CPU
// (tests/test_besselk.py); product code only, nothing shared with oracle/.
#pragma once
#include <math.h>

#ifndef SBV_HD
#ifdef __CUDACC__
#define SBV_HD __host__ __device__
#else
#define SBV_HD
#endif
#endif

namespace sbv {

// 1/Gamma(z) = sum_{k>=1} c_k z^k (A&S 6.1.34), c_1..c_26
SBV_HD inline double rgamma_coef(int k) {
  switch (k) {
    case 1: return 1.0;
    case 2: return 0.5772156649015329;
    case 3: return -0.6558780715202538;
    case 4: return -0.0420026350340952;
    case 5: return 0.1665386113822915;
    case 6: return -0.0421977345555443;
    case 7: return -0.0096219715278770;
    case 8: return 0.0072189432466630;
    case 9: return -0.0011651675918591;
    case 10: return -0.0002152416741149;
    case 11: return 0.0001280502823882;
    case 12: return -0.0000201348547807;
    case 13: return -0.0000012504934821;
    case 14: return 0.0000011330272320;
    case 15: return -0.0000002056338417;
    case 16: return 0.0000000061160950;
    case 17: return 0.0000000050020075;
    case 18: return -0.0000000011812746;
    case 19: return 0.0000000001043427;
    case 20: return 0.0000000000077823;
    case 21: return -0.0000000000036968;
    case 22: return 0.0000000000005100;
    case 23: return -0.0000000000000206;
    case 24: return -0.0000000000000054;
    case 25: return 0.0000000000000014;
    default: return 0.0000000000000001;  // k = 26
  }
}

// G1(mu) = -sum_{k even} c_k mu^{k-2}, G2(mu) = sum_{k odd} c_k mu^{k-1}
SBV_HD inline void temme_gammas(double mu, double &g1, double &g2) {
  double s1 = 0.0, s2 = 0.0;
  for (int k = 26; k >= 1; k--) {
    if (k & 1)
      s2 = s2 * (mu * mu) + rgamma_coef(k);  // odd k: mu^{k-1}, even powers
    else
      s1 = s1 * (mu * mu) + rgamma_coef(k);  // even k: mu^{k-2}
  }
  g1 = -s1;
  g2 = s2;
}

SBV_HD inline double besselk(double nu, double x) {
  const double kPi = 3.14159265358979323846, kEps = 1e-17;
  if (!(x > 0.0)) return INFINITY;
  if (x > 745.0) return 0.0;
  nu = fabs(nu);
  const int n = (int)(nu + 0.5);
  const double mu = nu - n;  // [-1/2, 1/2]
  double kmu, kmu1;
  if (x <= 2.0) {
    const double x2 = 0.5 * x, lnx2 = -log(x2);  // ln(2/x)
    const double pimu = kPi * mu;
    const double fact = fabs(pimu) < 1e-300 ? 1.0 : pimu / sin(pimu);
    const double s = mu * lnx2;
    const double fact2 = fabs(s) < 1e-300 ? 1.0 : sinh(s) / s;
    double g1, g2;
    temme_gammas(mu, g1, g2);
    const double rgp = g2 - mu * g1;  // 1 / Gamma(1 + mu)
    const double rgm = g2 + mu * g1;  // 1 / Gamma(1 - mu)
    double f = fact * (g1 * cosh(s) + g2 * fact2 * lnx2);
    const double es = exp(s);        // (x/2)^-mu
    double p = 0.5 * es / rgp;       // (x/2)^-mu Gamma(1+mu) / 2
    double q = 0.5 / (es * rgm);     // (x/2)^mu Gamma(1-mu) / 2
    double c = 1.0;
    const double dd = x2 * x2;
    double sum = f, sum1 = p;
    for (int k = 1; k < 500; k++) {
      f = (k * f + p + q) / (k * k - mu * mu);
      c *= dd / k;
      p /= (k - mu);
      q /= (k + mu);
      const double del = c * f;
      sum += del;
      const double del1 = c * (p - k * f);
      sum1 += del1;
      if (fabs(del) < fabs(sum) * kEps && fabs(del1) < fabs(sum1) * kEps) break;
    }
    kmu = sum;
    kmu1 = sum1 * (2.0 / x);
  } else {
    double b = 2.0 * (1.0 + x), d = 1.0 / b, h = d, delh = d;
    double q1 = 0.0, q2 = 1.0;
    const double a1 = 0.25 - mu * mu;
    double q = a1, c = a1, a = -a1;
    double s = 1.0 + q * delh;
    for (int i = 2; i < 100000; i++) {
      a -= 2 * (i - 1);
      c = -a * c / i;
      const double qnew = (q1 - b * q2) / a;
      q1 = q2;
      q2 = qnew;
      q += c * qnew;
      b += 2.0;
      d = 1.0 / (b + a * d);
      delh = (b * d - 1.0) * delh;
      h += delh;
      const double dels = q * delh;
      s += dels;
      if (fabs(dels / s) < kEps) break;
    }
    h = a1 * h;
    kmu = sqrt(kPi / (2.0 * x)) * exp(-x) / s;
    kmu1 = kmu * (mu + x + 0.5 - h) / x;
  }
  // upward recurrence to nu = mu + n
  double km = kmu, kp = kmu1;
  for (int i = 1; i <= n; i++) {
    const double kn = (mu + i) * (2.0 / x) * kp + km;
    km = kp;
    kp = kn;
  }
  return km;
}

}  // namespace sbv
