/*
 * cpfit_io.h — .tns tensor files for the cpfit B200 path (libcpfit_gpu.so, host code).
 * Replaces the reference's text I/O on the input side (proj/core/include/cpfit/io.hpp:14-30,
 * proj/core/src/io.cpp:15-215) with a multi-threaded parser/writer of the same format and
 * diagnostics, plus a binary sidecar. Status codes as cpfit_gpu.h, plus 4 = cpfit::io_error
 * (errors.hpp:15-18; message "<file>:<line>: <what>" from cpfit_io_last_error()).
 */
#ifndef CPFIT_IO_H
#define CPFIT_IO_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif
const char* cpfit_io_last_error(void);
/* format_double (io.cpp:15-19): shortest round-trip decimal form, NUL-terminated */
int cpfit_format_double(double x, char* buf, int cap);
/* read_tns / read_tns_file (io.hpp:26-27, io.cpp:104-147, 179-188). dims has room for 8.
 * coords (nnz x order, AoS, 0-based) and values are filled in file order when non-NULL (cap =
 * their capacity in entries); with both NULL only the header is read. The entries are returned
 * as written: DataTensor construction (cpfit_tensor_create_coo) canonicalises them like
 * SparseTensor's constructor. sidecar: 0 text only; 1 use <path>.cpfbin when its stamp (the
 * text file's size and mtime) matches; 2 as 1, and write the sidecar after parsing the text.
 * *from_sidecar (may be NULL) reports which was read. */
int cpfit_tns_read(const char* path, int sidecar, int* order, int64_t* dims, int64_t* nnz, int64_t* coords,
                   double* values, int64_t cap, int* from_sidecar);
/* read_tns_dense_file (io.hpp:29-30, io.cpp:190-205): zeros, then every entry at its offset in
 * file order (a later duplicate wins); values = NULL reads only the header (K = element count) */
int cpfit_tns_read_dense(const char* path, int sidecar, int* order, int64_t* dims, int64_t* K, double* values,
                         int64_t cap);
/* write_tns_file(SparseTensor) (io.cpp:151-159): header, then "i1 ... iN value" per entry */
int cpfit_tns_write(const char* path, int order, const int64_t* dims, int64_t nnz, const int64_t* coords,
                    const double* values);
/* write_tns_file(DenseTensor) (io.cpp:161-174): every element, first mode fastest */
int cpfit_tns_write_dense(const char* path, int order, const int64_t* dims, const double* values);
#ifdef __cplusplus
}
#endif
#endif
