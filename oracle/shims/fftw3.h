// ORACLE TEST INFRASTRUCTURE — not product code.
//
// Minimal FFTW3 API subset so the unmodified reference sources
// (/root/reference/proj/src/fourier.cpp:5, :35-61) compile in this container,
// where FFTW3 is not installed. Only the entry points fourier.cpp calls are
// provided: fftw_plan_many_dft (rank 1, strided/batched), fftw_execute,
// fftw_execute_dft, fftw_destroy_plan. Semantics follow FFTW's published
// definition: unnormalised DFT, Y_k = sum_j X_j exp(sign * 2 pi i j k / n),
// sign = FFTW_FORWARD (-1) or FFTW_BACKWARD (+1).
//
// The transform itself (fftw_shim.cpp) is a mixed-radix decimation-in-time
// FFT with long-double twiddles and Bluestein for large prime factors.
#pragma once

typedef double fftw_complex[2];

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_MEASURE (0U)
#define FFTW_ESTIMATE (1U << 6)
#define FFTW_UNALIGNED (1U << 1)

struct oracle_fftw_plan_s;
typedef oracle_fftw_plan_s* fftw_plan;

fftw_plan fftw_plan_many_dft(int rank, const int* n, int howmany, fftw_complex* in,
                             const int* inembed, int istride, int idist, fftw_complex* out,
                             const int* onembed, int ostride, int odist, int sign,
                             unsigned flags);
void fftw_execute(const fftw_plan p);
void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out);
void fftw_destroy_plan(fftw_plan p);
