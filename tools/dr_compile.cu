// Compile-only unit for iterating on the DMMA ring kernels (ptxas -v, SASS).
#include "../paper_0809_2407_b200/csrc/tsqr_device.cuh"
namespace tsqr {
#include "../paper_0809_2407_b200/csrc/dmma_ring.cuh"
template __global__ void k_leaf_dmma<true, false>(const double*, int64_t, int64_t, int, int, int64_t, double*, int64_t, double*, int64_t, double*, int*, int);
}
