// Small device helpers shared by the kernels.
#pragma once

namespace s1d {

// std::nextafter(x, +inf) for finite x (the reference's perturb_one_ulp,
// inc/kernels.hpp:122-125).
__device__ __forceinline__ double next_up(double x) {
    if (x != x) return x;
    if (x == 0.0) return __longlong_as_double(1LL); // smallest positive subnormal
    const long long b = __double_as_longlong(x);
    return __longlong_as_double(x > 0.0 ? b + 1 : b - 1);
}

} // namespace s1d
