// Tiled translation kernel, double precision, orders <= 20 (one 64 KB constant bank).
#define SFMM_REAL double
#define SFMM_PMAX 20
#include "kernel_tiled.inl"
