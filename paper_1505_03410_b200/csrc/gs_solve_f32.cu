// Persistent solver kernels, f32 storage with f64 arithmetic.
#define GS_T float
#define GS_SUF f32
#include "gs_solve_inst.cuh"
