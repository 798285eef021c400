// hipanns_search_kernel instantiations (search_kernel.cuh): fixed shapes, generic shapes and
// score tables (MODE 2)
#include "kernels.h"

template <int MINB, int DH, int ZZ, int MODE>
SearchKern search_kernel() { return hipanns_search_kernel<MINB, DH, ZZ, MODE>; }

template SearchKern search_kernel<2, 128, 3, 1>();
template SearchKern search_kernel<2, 128, 2, 1>();
template SearchKern search_kernel<2, 64, 3, 1>();
template SearchKern search_kernel<2, 64, 2, 1>();
template SearchKern search_kernel<2, 128, 3, 0>();
template SearchKern search_kernel<2, 128, 2, 0>();
template SearchKern search_kernel<2, 64, 3, 0>();
template SearchKern search_kernel<2, 64, 2, 0>();
template SearchKern search_kernel<2, 0, 0, 0>();
template SearchKern search_kernel<1, 0, 0, 0>();
template SearchKern search_kernel<2, 0, 0, 2>();
template SearchKern search_kernel<1, 0, 0, 2>();
