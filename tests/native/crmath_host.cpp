// Host build of csrc/crmath.cuh for tests/test_crmath.py: the same double-double code the
// K7 kernels run, compiled with -ffp-contract=off, exported over arrays through ctypes.
#include <cmath>
#include <cstdint>

#include "../../paper_2605_21072_b200/csrc/crmath.cuh"
#include "../../paper_2605_21072_b200/csrc/libm_ref.cuh"

using namespace qarvd_b200::crm;

extern "C" {
void crm_exp(const double* x, double* y, int64_t n) {
  for (int64_t i = 0; i < n; ++i) y[i] = cr_exp(x[i]);
}
void crm_log(const double* x, double* y, int64_t n) {
  for (int64_t i = 0; i < n; ++i) y[i] = cr_log(x[i]);
}
void crm_pow(const double* x, const double* e, double* y, int64_t n) {
  for (int64_t i = 0; i < n; ++i) y[i] = cr_pow(x[i], e[i]);
}
void ref_exp(const double* x, double* y, int64_t n) {
  for (int64_t i = 0; i < n; ++i) y[i] = qarvd_b200::libm::exp(x[i]);
}
void ref_log(const double* x, double* y, int64_t n) {
  for (int64_t i = 0; i < n; ++i) y[i] = qarvd_b200::libm::log(x[i]);
}
void ref_pow(const double* x, const double* e, double* y, int64_t n) {
  for (int64_t i = 0; i < n; ++i) y[i] = qarvd_b200::libm::pow(x[i], e[i]);
}
void glibc_exp(const double* x, double* y, int64_t n) {
  for (int64_t i = 0; i < n; ++i) y[i] = std::exp(x[i]);
}
void glibc_log(const double* x, double* y, int64_t n) {
  for (int64_t i = 0; i < n; ++i) y[i] = std::log(x[i]);
}
void glibc_pow(const double* x, const double* e, double* y, int64_t n) {
  for (int64_t i = 0; i < n; ++i) y[i] = std::pow(x[i], e[i]);
}
}
