// Host build of csrc/fastmath.cuh for tests/test_fastmath.py (accuracy of the
// polynomial sincospi / log / exp and the branch-free division and sqrt).
#include <cstdint>

#include "../../paper_1808_10580_b200/csrc/fastmath.cuh"

extern "C" {
void fm_sincospi(const double* a, int64_t n, double* s, double* c) {
    for (int64_t i = 0; i < n; ++i) smc::fm::sincospi(a[i], s + i, c + i);
}
void fm_sincospi_shift(const double* a, int64_t n, double* s, double* c) {
    for (int64_t i = 0; i < n; ++i) smc::fm::sincospi<true>(a[i], s + i, c + i);
}
void fm_log(const double* x, int64_t n, double* y) {
    for (int64_t i = 0; i < n; ++i) y[i] = smc::fm::log_pos(x[i]);
}
void fm_log_tab(const double* x, int64_t n, double* y) {
    for (int64_t i = 0; i < n; ++i) y[i] = smc::fm::log_tab(x[i]);
}
void fm_exp(const double* x, int64_t n, double* y) {
    for (int64_t i = 0; i < n; ++i) y[i] = smc::fm::exp_(x[i]);
}
void fm_exp_bump(const double* x, int64_t n, double* y) {
    for (int64_t i = 0; i < n; ++i) y[i] = smc::fm::exp_bump(x[i], smc::fm::h_exptab);
}
void fm_sqrt(const double* x, int64_t n, double* y) {
    for (int64_t i = 0; i < n; ++i) y[i] = smc::fm::sqrt_pos(x[i]);
}
void fm_div(const double* a, const double* d, int64_t n, double* y) {
    for (int64_t i = 0; i < n; ++i) y[i] = smc::fm::div_small(a[i], d[i]);
}
}
