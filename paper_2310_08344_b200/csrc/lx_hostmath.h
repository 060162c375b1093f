// lx_hostmath.h -- product-side host scalar math (Leja points, phi_l, divided differences).
#pragma once

namespace lx {
double phi(int l, double z);
int leja_points(int count, double* out);  // 0 ok, 1 arg error
int divided_differences(int l, const double* xi, int m, double dt, double c, double gamma, double a,
                        double* d);       // 0 ok, 1 arg, 4 unsupported, 6 nonfinite
}  // namespace lx
