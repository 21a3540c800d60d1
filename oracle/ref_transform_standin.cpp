// ORACLE / TEST INFRASTRUCTURE ONLY.
//
// Stand-in for the reference's FFTW-backed transform.cpp (FFTW3 is absent in
// this image). It defines exactly the three symbols declared by
// /root/reference/proj/include/fse/transform.hpp:15-20 with the same
// conventions (unnormalized, forward = negative exponent) and the same
// structural counters (transform.cpp:12-15,72-80), so the unmodified reference
// sources link against it. The arithmetic is the shared fft_radix2.h, which
// the C restatement (fofse_oracle.c) uses as well.
#include <complex>
#include <stdexcept>

#include "fft_radix2.h"
#include "fse/transform.hpp"

namespace fse {

TransformCounters& transform_counters() {
    static TransformCounters counters;
    return counters;
}

void dft2d_forward(int t, const std::complex<double>* in, std::complex<double>* out) {
    if (t < 1) throw std::invalid_argument("transform size must be >= 1");
    or_dft2d(t, -1, reinterpret_cast<const double*>(in), reinterpret_cast<double*>(out));
    transform_counters().forward.fetch_add(1, std::memory_order_relaxed);
}

void dft2d_inverse(int t, const std::complex<double>* in, std::complex<double>* out) {
    if (t < 1) throw std::invalid_argument("transform size must be >= 1");
    or_dft2d(t, +1, reinterpret_cast<const double*>(in), reinterpret_cast<double*>(out));
    transform_counters().inverse.fetch_add(1, std::memory_order_relaxed);
}

}  // namespace fse
