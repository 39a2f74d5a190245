/* TEST INFRASTRUCTURE (oracle build only) -- never linked into the product.
 *
 * Minimal LAPACKE prototype header so that the reference headers
 * (/root/reference/proj/include/ldgmg/blockla.hpp:16 includes <lapacke.h>)
 * compile unmodified.  The symbols resolve against the OpenBLAS 0.3.15 build
 * that ships inside the opencv-python-headless wheel of this image
 * (libopenblasp-r0-59ffcd50.3.15.so), linked by oracle/Makefile.
 * Only the routines used by the reference (dgels, dgelsd) and by the
 * Eigen-subset shim (dsyevd, dgeev, dgesv, dgelsy, dsysv) are declared.
 */
#ifndef ORACLE_SHIM_LAPACKE_H
#define ORACLE_SHIM_LAPACKE_H

#ifdef __cplusplus
extern "C" {
#endif

typedef int lapack_int;
#define LAPACK_ROW_MAJOR 101
#define LAPACK_COL_MAJOR 102

lapack_int LAPACKE_dgels(int layout, char trans, lapack_int m, lapack_int n, lapack_int nrhs,
                         double* a, lapack_int lda, double* b, lapack_int ldb);
lapack_int LAPACKE_dgelsd(int layout, lapack_int m, lapack_int n, lapack_int nrhs, double* a,
                          lapack_int lda, double* b, lapack_int ldb, double* s, double rcond,
                          lapack_int* rank);
lapack_int LAPACKE_dgelsy(int layout, lapack_int m, lapack_int n, lapack_int nrhs, double* a,
                          lapack_int lda, double* b, lapack_int ldb, lapack_int* jpvt,
                          double rcond, lapack_int* rank);
lapack_int LAPACKE_dsyevd(int layout, char jobz, char uplo, lapack_int n, double* a,
                          lapack_int lda, double* w);
lapack_int LAPACKE_dgeev(int layout, char jobvl, char jobvr, lapack_int n, double* a,
                         lapack_int lda, double* wr, double* wi, double* vl, lapack_int ldvl,
                         double* vr, lapack_int ldvr);
lapack_int LAPACKE_dgesv(int layout, lapack_int n, lapack_int nrhs, double* a, lapack_int lda,
                         lapack_int* ipiv, double* b, lapack_int ldb);
lapack_int LAPACKE_dsysv(int layout, char uplo, lapack_int n, lapack_int nrhs, double* a,
                         lapack_int lda, lapack_int* ipiv, double* b, lapack_int ldb);

#ifdef __cplusplus
}
#endif

#endif
