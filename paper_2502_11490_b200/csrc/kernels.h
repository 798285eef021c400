// Search-kernel instantiations live in their own translation units (inst_*.cu, compiled in
// parallel); gmpgr.cu's host code only takes their launch pointers.
#pragma once
#include "search_kernel.cuh"

typedef void (*SearchKern)(const SearchArgs);
template <int DH, int ZZ, int MODE, int G>
SearchKern duo_kernel();
template <int DH, int ZZ, int MODE, int NT, int G, int KC, bool PIPE>
SearchKern mq_kernel();
template <int MINB, int DH, int ZZ, int MODE>
SearchKern search_kernel();
