// Host-side accuracy check of lfb::pos_pow against long-double powl.
// nvcc -O2 -I../paper_1604_08501_b200/csrc -o /tmp/check_fastmath check_fastmath.cu
#include <cstdio>
#include <cmath>
#include <random>
#include "lfb_math.cuh"

int main() {
  std::mt19937_64 rng(1);
  double worst = 0, worst_x = 0, worst_y = 0;
  const double ys[] = {1.4, 1.3, 1.45, 1.1, 1.6667, 2.0, 1.0000001};
  for (double y : ys) {
    std::uniform_real_distribution<double> lx(-20.0, 20.0);
    for (int it = 0; it < 2000000; ++it) {
      double x = (it % 2) ? std::exp(lx(rng)) : 0.8 + 0.4 * std::generate_canonical<double, 53>(rng);
      long double ref = powl((long double)x, (long double)y);
      double got = lfb::pos_pow(x, y);
      double rel = (double)fabsl(((long double)got - ref) / ref);
      double scale = 1.0 + fabs(y * std::log(x));
      if (rel / scale > worst) { worst = rel / scale; worst_x = x; worst_y = y; }
    }
  }
  printf("worst rel/(1+|y ln x|) = %.3e at x=%.17g y=%.17g\n", worst, worst_x, worst_y);
  return worst < 1e-15 ? 0 : 1;
}
