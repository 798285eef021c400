// hipanns_duo_kernel instantiations (search_duo.cuh) for the fixed model shapes
#include "kernels.h"
#include "search_duo.cuh"

template <int DH, int ZZ, int MODE, int G>
SearchKern duo_kernel() { return hipanns_duo_kernel<DH, ZZ, MODE, G>; }

#define GR_INST(DH, ZZ)                             \
    template SearchKern duo_kernel<DH, ZZ, 1, 8>(); \
    template SearchKern duo_kernel<DH, ZZ, 0, 8>();
GR_INST(128, 3)
GR_INST(128, 2)
GR_INST(64, 3)
GR_INST(64, 2)
