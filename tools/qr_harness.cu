// Host-side harness for bidiag_qr.cuh: reads m, alpha[1..m], beta[2..m+1] from stdin,
// runs the device QR code on the CPU, prints iterations, rotation counts, singular
// values and the reconstruction error of B = P diag(d) Q^T from the records.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "../paper_0911_4498_b200/csrc/bidiag_qr.cuh"
using namespace ssa;
int main() {
  int m; if (scanf("%d", &m) != 1) return 1;
  std::vector<double> al(m + 3, 0), be(m + 3, 0);
  for (int i = 1; i <= m; ++i) if (scanf("%lf", &al[i]) != 1) return 1;
  for (int i = 2; i <= m + 1; ++i) if (scanf("%lf", &be[i]) != 1) return 1;
  std::vector<double> d(m + 2), e(m + 2), w(m + 2);
  int cap = 2 * m * m + 8 * m + 1024;
  std::vector<int2> abL(cap), abR(cap);
  std::vector<double2> csL(cap), csR(cap);
  RotRec L{abL.data(), csL.data(), cap, 0}, R{abR.data(), csR.data(), cap, 0};
  int it = bidiag_qr<true, true>(m, al.data(), be.data(), d.data(), e.data(), w.data(), &L, &R, 30 * m + 100);
  printf("iters %d recL %d recR %d\n", it, L.n, R.n);
  double err = 0, nb = 0;
  std::vector<double> P((size_t)(m + 1) * m), Q((size_t)m * m);
  for (int j = 0; j < m; ++j) {
    std::vector<double> x(m + 1, 0.0), y(m, 0.0);
    x[j] = 1; y[j] = 1;
    apply_records_reverse(abL.data(), csL.data(), L.n, x.data(), 1);
    apply_records_reverse(abR.data(), csR.data(), R.n, y.data(), 1);
    for (int i = 0; i <= m; ++i) P[(size_t)i * m + j] = x[i];
    for (int i = 0; i < m; ++i) Q[(size_t)i * m + j] = y[i];
  }
  for (int r = 0; r <= m; ++r)
    for (int c = 0; c < m; ++c) {
      double b = (r == c) ? al[c + 1] : (r == c + 1 ? be[c + 2] : 0.0);
      double s = 0; for (int j = 0; j < m; ++j) s += P[(size_t)r * m + j] * d[j] * Q[(size_t)c * m + j];
      err = fmax(err, fabs(s - b)); nb = fmax(nb, fabs(b));
    }
  double wmax = 0; for (int j = 0; j < m; ++j) wmax = fmax(wmax, fabs(w[j] - P[(size_t)m * m + j]));
  double orth = 0;
  for (int a = 0; a < m; ++a) for (int b2 = 0; b2 < m; ++b2) {
    double s = 0, t = 0;
    for (int i = 0; i <= m; ++i) s += P[(size_t)i * m + a] * P[(size_t)i * m + b2];
    for (int i = 0; i < m; ++i) t += Q[(size_t)i * m + a] * Q[(size_t)i * m + b2];
    orth = fmax(orth, fmax(fabs(s - (a == b2)), fabs(t - (a == b2))));
  }
  printf("recon_err %.3e rel %.3e lastrow_err %.3e orth %.3e\n", err, err / nb, wmax, orth);
  for (int j = 0; j < m; ++j) printf("%.17g\n", fabs(d[j]));
  return 0;
}
