// Tiled translation kernel, single precision, orders <= 18 (the reference's float cap).
#define SFMM_REAL float
#define SFMM_PMAX 18
#include "kernel_tiled.inl"
