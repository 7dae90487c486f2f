/* oracle/shim/fftw3.h -- TEST INFRASTRUCTURE, not product code.
 *
 * Declaration-compatible subset of the FFTW3 double-precision API, exactly the
 * symbols the reference's trig module binds (reference proj/src/trig.cpp:3,
 * 20-21, 43, 47-48, 56, 76, 91).  FFTW3 is an unpinned third-party dependency
 * of the reference (proj/CMakeLists.txt:15-16: find_library(fftw3) with no
 * version) and is absent from this image, so oracle/shim/fftw_shim.cpp
 * restates the three r2r kinds the reference uses from FFTW's published
 * definitions (RODFT00 = DST-I, RODFT01 = DST-III, REDFT01 = DCT-III, all
 * unnormalised).  The enum values and flag bits match fftw3.h 3.3.x.
 */
#ifndef SFEM_ORACLE_FFTW3_SHIM_H
#define SFEM_ORACLE_FFTW3_SHIM_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fftw_plan_s* fftw_plan;

typedef enum {
  FFTW_R2HC = 0, FFTW_HC2R = 1, FFTW_DHT = 2,
  FFTW_REDFT00 = 3, FFTW_REDFT01 = 4, FFTW_REDFT10 = 5, FFTW_REDFT11 = 6,
  FFTW_RODFT00 = 7, FFTW_RODFT01 = 8, FFTW_RODFT10 = 9, FFTW_RODFT11 = 10
} fftw_r2r_kind;

#define FFTW_MEASURE (0U)
#define FFTW_DESTROY_INPUT (1U << 0)
#define FFTW_UNALIGNED (1U << 1)
#define FFTW_PRESERVE_INPUT (1U << 4)
#define FFTW_ESTIMATE (1U << 6)

fftw_plan fftw_plan_r2r_1d(int n, double* in, double* out, fftw_r2r_kind kind, unsigned flags);
fftw_plan fftw_plan_many_r2r(int rank, const int* n, int howmany, double* in, const int* inembed,
                             int istride, int idist, double* out, const int* onembed, int ostride,
                             int odist, const fftw_r2r_kind* kind, unsigned flags);
void fftw_execute_r2r(const fftw_plan p, double* in, double* out);
void fftw_destroy_plan(fftw_plan p);

#ifdef __cplusplus
}
#endif
#endif
