/*
 * hconv.h — C ABI of the hybrid-dealiased convolution path (arXiv 2303.17510).
 *
 * This is the drop-in boundary.  Two shared libraries export exactly these
 * symbols:
 *   paper_2303_17510_b200/_lib/libhconv_cuda.so  — the product: sm_100a kernels,
 *        device pointers, asynchronous on a caller-supplied cudaStream_t.
 *   oracle/_build/libhconv_oracle.so             — test infrastructure: the CPU
 *        restatement of the reference, host pointers, synchronous.
 * No C++ types, no exceptions and no torch types cross this boundary.
 *
 * Reference interfaces each entry point replaces (paths relative to
 * /root/reference):
 *   hconv_derive_params      proj/include/hconv/plan.hpp:67   deriveParams
 *   hconv_block_length       proj/src/plan.cpp:26-29          PlanParams::blockLength
 *   hconv_stored_length      proj/src/plan.cpp:31-33          PlanParams::storedLength
 *   hconv_padded_length      proj/include/hconv/plan.hpp:56   PlanParams::paddedLength
 *   hconv_root               proj/include/hconv/plan.hpp:70   root
 *   hconv_work_memory_words  proj/include/hconv/plan.hpp:79   workMemoryWords
 *   hconv_root_table         proj/include/hconv/plan.hpp:84   RootTable
 *   hconv_symmetry_name      proj/include/hconv/plan.hpp:27   name(Symmetry)
 *   hconv_symmetry_from_name proj/include/hconv/plan.hpp:28   symmetryFromName
 *   hconv_pfft_forward       SPEC.md:158,176,194,258,276,331,349  forward1/2/Inner[C|H]
 *   hconv_pfft_backward      SPEC.md:167,185,203,267,285,340,358  backward1/2/Inner[C|H]
 *   hconv_pfft_forward_pair  SPEC.md:212-220                     forward_conjugate_pair
 *   hconv_pfft_*_lines       the same over two-level strided line batches (PAPER.md:584-600
 *                            outer-axis passes; used by the multi-GPU slab driver)
 *   hconv_plan_create        SPEC.md:400-403 Conv1dPlan, SPEC.md:469-472 ConvPlanND,
 *                            SPEC.md:533-550 tune_1d/tune_nd (when an axis has m == 0)
 *   hconv_convolve           SPEC.md:406-423 convolve/convolveC/convolveH,
 *                            SPEC.md:475-483 convolve_nd (+ x-slabs over G ranks, hconv_slab)
 *   hconv_plan_slab          (no reference counterpart: the slab extent of a rank)
 * Exceptions of the reference (std::invalid_argument, plan.cpp:36-38,67,77-80,92-93)
 * become HCONV_INVALID_ARG; the message is available from hconv_last_error().
 */
#ifndef HCONV_H
#define HCONV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum hconv_status {
  HCONV_OK = 0,
  HCONV_INVALID_ARG = 1, /* L == 0, m == 0, M < L, arity, layout */
  HCONV_UNSUPPORTED = 2, /* e.g. a block size no kernel instantiation covers */
  HCONV_CUDA_ERROR = 3,
  HCONV_NCCL_ERROR = 4,
  HCONV_ALLOC = 5,
  HCONV_INTERNAL = 6
} hconv_status;

/* plan.hpp:17 enum class Symmetry { Complex, Centered, Hermitian } */
typedef enum hconv_symmetry { HCONV_COMPLEX = 0, HCONV_CENTERED = 1, HCONV_HERMITIAN = 2 } hconv_symmetry;
/* plan.hpp:20 enum class Regime { P1, P2, Inner } */
typedef enum hconv_regime { HCONV_P1 = 0, HCONV_P2 = 1, HCONV_INNER = 2 } hconv_regime;
/* SPEC.md:396-399 MultOperator, SPEC.md:424 builtin_mult_product */
typedef enum hconv_mult {
  HCONV_MULT_PRODUCT = 0,  /* builtin_mult_product(A): B = 1, elementwise product of the A >= 2 inputs */
  HCONV_MULT_CALLBACK = 1  /* user operator: hconv_desc.mult_fn / mult_user, any A >= 1, B >= 1 */
} hconv_mult;

/* User multiplication operator (SPEC.md:396-399 MultOperator{A, B, apply}; PAPER.md:215,254
 * "F_b <- mult(F_a)").  Called once per residue block of the innermost axis (per batch chunk)
 * with the transformed blocks of the A inputs in F[0..A) and must leave the B outputs in
 * F[0..B), in place; F has max(A, B) entries, each `count` values.  Pointwise:
 * output element k depends only on the inputs' element k, and every F[i] uses the same element
 * order, which is otherwise the library's choice.  Values are complex128 (complex / centered
 * innermost axis) or float64 (real != 0: a Hermitian axis' transformed residues are real,
 * PAPER.md:484-485).
 * CUDA library: device pointers; enqueue the work on `stream` (a cudaStream_t) and return
 * without synchronising.  Oracle: host pointers, stream NULL.  Return 0 on success; any other
 * value aborts the convolution with HCONV_INVALID_ARG.                                      */
typedef int (*hconv_mult_fn)(void* const* F, size_t A, size_t B, size_t count, int real, void* user, void* stream);

/* plan.hpp:39-62 PlanParams (field for field; kind = {symmetry, regime}) */
typedef struct hconv_params {
  size_t L, M, m, p, q, n, D, C, S;
  int inplace;
  int symmetry; /* hconv_symmetry */
  int regime;   /* hconv_regime  */
} hconv_params;

/* ---- plan module (the reference's only compiled code) ---- */
hconv_status hconv_derive_params(size_t L, size_t M, size_t m, int symmetry, hconv_params* out);
size_t hconv_block_length(const hconv_params* pp);
size_t hconv_stored_length(const hconv_params* pp);
size_t hconv_padded_length(const hconv_params* pp);
hconv_status hconv_root(size_t N, int64_t k, double* re, double* im);
hconv_status hconv_work_memory_words(const hconv_params* pp, size_t A, size_t B, size_t d, size_t L,
                                     uint64_t* implicit_words, double* explicit_words);
/* Fills out[2k], out[2k+1] = Re, Im zeta_N^k for k in [0, N) (host memory in both libraries). */
hconv_status hconv_root_table(size_t N, double* out);
const char* hconv_symmetry_name(int symmetry);
hconv_status hconv_symmetry_from_name(const char* name, int* symmetry);

/* ---- residue-level padded FFTs (SPEC pfft-complex / pfft-centered / pfft-hermitian) ----
 * Batched over pp->C copies: element j of copy c is at f[c*dist + j*pp->S] (complex128,
 * interleaved re/im).  Forward writes, for each copy, the residue (block) contribution in
 * the reference's order into F[c*blockLength ...]: complex kinds complex128
 * F[u*m + l] = F_{q l + u n + r} (u = 0 for p <= 2), Hermitian kind float64 (real) values.
 * Backward is the unnormalised inverse of one residue; with accumulate != 0 it adds into h.
 * Hermitian data stores the non-negative logical indices 0..ceil(L/2)-1.
 * Centered data stores logical index j - floor(L/2) at j.                               */
hconv_status hconv_pfft_forward(const hconv_params* pp, const void* f, size_t dist, size_t residue, void* F,
                                void* stream);
hconv_status hconv_pfft_backward(const hconv_params* pp, const void* F, size_t residue, void* h, size_t dist,
                                 int accumulate, void* stream);
/* forward_conjugate_pair, complex data: the blocks of
 * residues v and -v from one real / imaginary split of the input, both in the reference order:
 * Fv[u*m + l] = F_{q l + u n + v}, Fnv[u*m + l] = F_{q l + u n - v} (indices mod qm).
 * HCONV_INVALID_ARG for v == 0 or 2v == n (self-paired), HCONV_UNSUPPORTED for other kinds. */
hconv_status hconv_pfft_forward_pair(const hconv_params* pp, const void* f, size_t dist, size_t residue, void* Fv,
                                     void* Fnv, void* stream);

/* Two-level line batches for the N-D and slab drivers (the strided outer-axis passes of
 * PAPER.md:584-600): line l of a batch starts at element (l / nin) * d_out + (l % nin) * d_in
 * and its values sit at element stride es (complex128 elements, or float64 for Hermitian
 * blocks).  Blocks are in natural block order (the order the convolution kernels use, not the
 * reference's F[u m + l]; pointwise operators do not see the difference).  Forward writes the
 * block of residue `residue` of every line; backward adds (accumulate != 0) or writes the
 * unnormalised inverse of residue `residue`, times `scale`, into the data lines.          */
typedef struct hconv_lines {
  size_t count, nin, d_out, d_in, es;
} hconv_lines;
hconv_status hconv_pfft_forward_lines(const hconv_params* pp, const void* f, const hconv_lines* in, size_t residue,
                                      void* F, const hconv_lines* out, void* stream);
hconv_status hconv_pfft_backward_lines(const hconv_params* pp, const void* F, const hconv_lines* in, size_t residue,
                                       void* h, const hconv_lines* out, int accumulate, double scale, void* stream);

/* ---- convolution plans ---- */
typedef struct hconv_axis {
  size_t L;     /* logical data length along the axis */
  size_t M;     /* minimum dealiased length, M >= L */
  size_t m;     /* subtransform size; 0 = let the device-timed planner choose */
  int symmetry; /* hconv_symmetry */
} hconv_axis;

typedef struct hconv_desc {
  int dims;              /* 1, 2 or 3; axis[dims-1] is the innermost (contiguous) axis */
  hconv_axis axis[3];
  size_t A, B;           /* inputs / outputs of the multiplication operator */
  int mult;              /* hconv_mult */
  size_t C;              /* number of independent copies (1D lines or N-D arrays); 0 = 1 */
  size_t dist;           /* 1D: elements between copies, >= the data length; 0 = the data length
                          * (L, or ceil(L/2) for Hermitian -- K-length storage, SURVEY 8(a) note;
                          * not hconv_stored_length).  N-D: must be 0 (contiguous arrays). */
  int device;            /* CUDA ordinal (ignored by the oracle) */
  int flags;             /* HCONV_FLAG_* (0 = the fastest layout) */
  hconv_mult_fn mult_fn; /* HCONV_MULT_CALLBACK: the operator (else ignored) */
  void* mult_user;       /* passed through to mult_fn */
  const struct hconv_slab* slab; /* NULL: one device holds the whole problem; else x-slab decomposition
                           * (dims 2 or 3, C == 1; the struct is copied at plan creation) */
} hconv_desc;

/* ---- multi-GPU slab decomposition (2D / 3D, north star item 3) ----
 * The reference has no distributed code (SPEC.md:512 lists MPI decomposition as a non-goal);
 * this extends ConvPlanND / convolve_nd to x-slabs over G ranks.  With
 * hconv_desc.slab != NULL the arrays passed to hconv_convolve are this rank's x-slab
 * [nx][Ly] (2D) or [nx][Ly][Lz] (3D) of the global arrays, nx and the first row x0 given by
 * hconv_plan_slab().  The outer padded FFT runs along the locally complete axis y; per y residue
 * the spectral y-lines are transposed (all-to-all) so that every rank holds nk complete x-lines,
 * the (d-1)-D subconvolutions run locally, and a second all-to-all brings them back before the
 * inverse y-FFT.  Every m must be given (tune on one rank and broadcast the choice).
 * Exchange: an NCCL communicator (CUDA library: ncclComm_t over NVLink / NVSwitch, grouped
 * ncclSend / ncclRecv on a plan-owned stream, overlapped chunk by chunk with the
 * subconvolutions), or, when nccl_comm is NULL, the caller's all-to-all callback.            */
/* All-to-all-v over the ranks of the slab: send[sdispls[h] .. + scounts[h]) goes to rank h,
 * recv[rdispls[h] .. + rcounts[h]) comes from rank h; counts and displacements in complex128
 * elements.  CUDA library: device pointers, ordered on `stream`; oracle: host pointers.
 * Return 0 on success (anything else aborts with HCONV_NCCL_ERROR).                         */
typedef int (*hconv_exchange_fn)(const void* send, const size_t* scounts, const size_t* sdispls, void* recv,
                                 const size_t* rcounts, const size_t* rdispls, void* user, void* stream);
typedef struct hconv_slab {
  int rank, nranks;           /* this rank, number of ranks G (1 <= G) */
  void* nccl_comm;            /* ncclComm_t (CUDA library only), or NULL */
  hconv_exchange_fn exchange; /* used when nccl_comm is NULL */
  void* exchange_user;
  size_t chunks;              /* k-line chunks per exchange (pipelining); 0 = library default */
} hconv_slab;

/* hconv_desc.flags.  HCONV_FLAG_MIN_MEMORY: N-D plans reuse ONE subconvolution work buffer for
 * every outer spectral plane in turn ("the upper column is then reused"), so
 * the work allocation stays within (A+B) p m L^{d-1} complex words (criterion 7);
 * the default processes every plane of a level in one batched pass (fastest on the GPU, more
 * work memory). */
#define HCONV_FLAG_MIN_MEMORY 1

typedef struct hconv_plan hconv_plan;

hconv_status hconv_plan_create(const hconv_desc* desc, hconv_plan** plan);
hconv_status hconv_plan_params(const hconv_plan* plan, int axis, hconv_params* out);
/* Slab plans: first row x0 and row count nx of this rank's x-slab (nx may be 0). */
hconv_status hconv_plan_slab(const hconv_plan* plan, size_t* x0, size_t* nx);
/* Bytes of device scratch the plan owns (0 for the oracle). */
size_t hconv_plan_workspace_bytes(const hconv_plan* plan);
/* in[A], out[B]: complex128 arrays with the stored layout of the descriptor.
 * out[b] == in[b] (in place, the reference's convention, Alg. convolve) is allowed.
 * A == 2, B == 1 with the built-in product runs the fused kernels; other operators run the
 * residue loop through work blocks (A forward padded FFTs, mult, B backward padded FFTs).
 * CUDA library: device pointers, asynchronous on stream (cudaStream_t, NULL = legacy).
 * Oracle: host pointers, stream ignored.                                           */
hconv_status hconv_convolve(hconv_plan* plan, const void* const* in, void* const* out, void* stream);
/* Host-buffer convolution -- the reference library's own calling convention (host arrays,
 * synchronous).  in[A], out[B]: HOST complex128 arrays with the stored
 * layout of the descriptor; out[b] == in[b] allowed.  CUDA library: a 1D batch streams through
 * the device in chunks of copies (HCONV_HOST_CHUNKS, default 8) -- the host->device copies, the
 * convolution and the device->host copies of consecutive chunks overlap on three streams
 * (page-locked host memory required for the overlap); N-D plans copy in, convolve, copy out.
 * Oracle: same as hconv_convolve.                                                            */
hconv_status hconv_convolve_host(hconv_plan* plan, const void* const* in, void* const* out);
hconv_status hconv_plan_destroy(hconv_plan* plan);
const char* hconv_last_error(void);
/* Library identity: "cuda-sm_100a" or "oracle-cpu". */
const char* hconv_backend(void);

#ifdef __cplusplus
}
#endif

#endif /* HCONV_H */
