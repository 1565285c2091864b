/*
 * hconv_ext.h — utilities exported by libhconv_cuda.so that are NOT part of the reference's
 * API (bench / test support).  The oracle library does not export these.
 */
#ifndef HCONV_EXT_H
#define HCONV_EXT_H
#include "hconv.h"
#ifdef __cplusplus
extern "C" {
#endif
/* Counter-based synthetic inputs on the device: element i gets
 * Re, Im = 2u-1, u = (splitmix64(seed*phi + (a<<56 | comp<<55 | (first_index+i))) >> 11) 2^-53. */
hconv_status hconv_util_fill_uniform(uint64_t seed, uint64_t a, uint64_t first_index, size_t count, void* out,
                                     void* stream);
/* Planner report of the last tuning done for this plan: rows of 7 doubles (m, p, q, n, block,
 * median ms, explicit: 1 for the explicit-dealiasing candidate q = 1, m >= M); returns the row
 * count, or -(count+1) when the choice came from the planner cache. */
int hconv_plan_report(const hconv_plan* plan, double* out, int cap);
/* Example native multiplication operators for HCONV_MULT_CALLBACK (device kernels on the
 * library's stream; a template for user operators written in CUDA):
 *   which = 0: quadratic products of a 2-component field, A = 2 -> B = 3:
 *              F0 <- F0 F0, F1 <- F0 F1, F2 <- F1 F1 (complex, or real for Hermitian blocks)
 * Returns NULL for an unknown id. */
hconv_mult_fn hconv_example_mult(int which);
/* NCCL bootstrap for slab plans (hconv_slab.nccl_comm).  The library binds NCCL at run time
 * (the libnccl.so.2 already loaded by the process, e.g. torch's, else the system one).
 * hconv_nccl_unique_id writes the 128-byte ncclUniqueId on one rank; every rank passes the same
 * bytes to hconv_nccl_comm_init (device = its CUDA ordinal).  HCONV_NCCL_ERROR on failure.   */
hconv_status hconv_nccl_unique_id(void* id128);
hconv_status hconv_nccl_comm_init(const void* id128, int nranks, int rank, int device, void** comm);
hconv_status hconv_nccl_comm_destroy(void* comm);
/* Radix plan of the kernel serving an axis ("16x16x24", "direct", ...). */
const char* hconv_plan_kernel(const hconv_plan* plan, int axis);
#ifdef __cplusplus
}
#endif
#endif
