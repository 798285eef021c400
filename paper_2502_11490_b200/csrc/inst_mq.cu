// hipanns_mq_kernel instantiations (search_mq.cuh) for the fixed model shapes
#include "kernels.h"
#include "search_mq.cuh"

template <int DH, int ZZ, int MODE, int NT, int G, int KC, bool PIPE>
SearchKern mq_kernel() { return hipanns_mq_kernel<DH, ZZ, MODE, NT, G, KC, PIPE>; }

#define GR_INST(DH, ZZ)                                               \
    template SearchKern mq_kernel<DH, ZZ, 1, 512, 16, DH, true>();    \
    template SearchKern mq_kernel<DH, ZZ, 1, 512, 8, DH, true>();     \
    template SearchKern mq_kernel<DH, ZZ, 0, 512, 8, DH, false>();
GR_INST(128, 3)
GR_INST(128, 2)
GR_INST(64, 3)
GR_INST(64, 2)
