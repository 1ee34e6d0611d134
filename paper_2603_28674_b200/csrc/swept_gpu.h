// swept_gpu.h — producer <-> GPU swept-volume stages (swept_gpu.cu); host C++ only.
#pragma once

#include <cstdint>
#include <vector>

// The inner approximation's inputs: the robot's inner spheres (body frame).
struct InnerSpec {
    int32_t nsph = 0;
    std::vector<double> centre;      // nsph * 3
    std::vector<double> radius;      // certified spline radius per sphere (<= 0: no splines)
    std::vector<double> step_bound;  // lipschitz * eps
    std::vector<double> tol;         // simplification tolerance
    int32_t K = 16;                  // segment cap
};

// Splines of every (component, sphere), component-major: nspl[c * nsph + s]
// splines, each with npts[k] points taken in order from pts (x, y, z).
struct InnerOut {
    std::vector<int32_t> nspl;
    std::vector<int32_t> npts;
    std::vector<double> pts;
};

// ncomp fit units (one per (component, body)), unit c with the poses [off[c], off[c+1])
// of body c % nbodies (half extents he3[3 * body]); chunk_configs = staging capacity (poses);
// device < 0: the calling thread's current CUDA device
void* rggp_fit_begin(const int64_t* off, int32_t ncomp, const double* he3, int32_t nbodies, const double* cos_sin,
                     int64_t chunk_configs, int32_t device);
double* rggp_fit_staging(void* fs, int32_t slot);
int rggp_fit_push(void* fs, int32_t slot, int64_t first_config, int64_t nconfigs);
// fit every component's box (ncomp x 15 doubles to out); with spec, also the splines
int rggp_fit_finish(void* fs, double* out, const InnerSpec* spec, InnerOut* inner);
void rggp_fit_end(void* fs);
