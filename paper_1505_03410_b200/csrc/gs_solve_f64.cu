// Persistent solver kernels, f64 storage (also CSC).
#define GS_T double
#define GS_SUF f64
#include "gs_solve_inst.cuh"
