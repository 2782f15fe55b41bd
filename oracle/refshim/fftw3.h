// fftw3.h — TEST INFRASTRUCTURE.  Self-written stand-in for the FFTW3 calls the reference's
// grid.cpp makes (oracle/refshim/README.md): N-d real-to-complex / complex-to-real plans,
// unnormalised transforms, double precision.  Implemented in fftw_stand_in.cpp.
#pragma once

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct fftw_stand_in_plan* fftw_plan;

#define FFTW_MEASURE 0u
#define FFTW_ESTIMATE (1u << 6)
#define FFTW_UNALIGNED (1u << 1)

fftw_plan fftw_plan_dft_r2c(int rank, const int* n, double* in, fftw_complex* out, unsigned flags);
fftw_plan fftw_plan_dft_c2r(int rank, const int* n, fftw_complex* in, double* out, unsigned flags);
void fftw_execute(const fftw_plan p);
void fftw_execute_dft_r2c(const fftw_plan p, double* in, fftw_complex* out);
void fftw_execute_dft_c2r(const fftw_plan p, fftw_complex* in, double* out);
void fftw_destroy_plan(fftw_plan p);

#ifdef __cplusplus
}
#endif
