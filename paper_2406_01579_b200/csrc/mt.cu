// mt.cu — K9 Marching Tetrahedra (grid.py:136-239).  (implementation in progress)
#include "internal.cuh"

int ts_impl_mt_count(const double*, const double*, int, int64_t*, int64_t*, cudaStream_t) { return -3; }
int ts_impl_mt(const double*, const double*, int, double*, int64_t*, int64_t*, cudaStream_t) { return -3; }
