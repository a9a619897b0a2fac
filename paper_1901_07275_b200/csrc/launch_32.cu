// Kernel instantiations of FFT length 32 (launch.cuh): one translation unit per length, compiled in parallel.
#include "launch.cuh"

namespace jtl {
template jt_status launch_n<32>(LaunchState &, bool, int, const jtk::AxisDev &, const double *, double *, long long, const jtk::Layout &, cudaStream_t, bool);
template jt_status checks_io<32>(unsigned long long *, int *);
}  // namespace jtl
