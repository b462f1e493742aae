// Stand-in for <lapacke.h> as used by the reference's eigensolve.hpp
// (dense_eig: LAPACKE_dsyevd, eigensolve.hpp:213-214).  TEST INFRASTRUCTURE
// ONLY (oracle/_ref).  Forwards to the LAPACK inside scipy's bundled OpenBLAS
// (symbols prefixed scipy_), loaded at run time by oracle/shim/lapack_loader.cpp.
#pragma once

typedef int lapack_int;
#define LAPACK_ROW_MAJOR 101
#define LAPACK_COL_MAJOR 102

lapack_int LAPACKE_dsyevd(int matrix_layout, char jobz, char uplo, lapack_int n, double* a,
                          lapack_int lda, double* w);
