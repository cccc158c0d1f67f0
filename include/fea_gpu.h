/*
 * fea_gpu.h — C ABI of the B200-native FE assembly hot path
 * (scatter-add of dense element matrices into CSR / CRAC, arXiv 2012.00585).
 *
 * The reference (/root/reference/proj) exposes this path only as C++ templates
 * (no C ABI). Each entry point below names the reference interface it replaces;
 * the C++ shim paper_2012_00585_b200/csrc/fea_gpu.hpp re-exposes the reference
 * surface (SparsityPattern, CsrMatrix, CracMatrix, AssemblyJob, assemble_*,
 * AssemblyError) on top of it, and INTEGRATION.md shows the bindings.
 *
 * Conventions
 *  - index_t is int64_t everywhere, as in the reference (types.hpp:27).
 *  - Element DOF arrays are the reference's ElementDofs::flat
 *    (dof_map.hpp:66-75) for all elements, concatenated: E x m int64,
 *    host or device memory (detected).
 *  - Element matrices K are one dense buffer [E][m][m] fp64 row-major in DEVICE
 *    memory (the reference's ElementMatrix, dof_map.hpp:78-87, materialized for
 *    every element instead of an ElementMatrixSupplier callback,
 *    assembly.hpp:37).
 *  - values is a caller-owned fp64[nnz] buffer. CSR and CRAC store values in the
 *    same order (row-major, ascending columns; verify.cpp:30-31), so one
 *    numeric call serves both formats.
 *  - Calls are stream-ordered on the given cudaStream_t (NULL = legacy default
 *    stream); a plan is bound to one device and is not thread-safe.
 *  - Every function returns fea_status; fea_last_error() holds the message of
 *    the last failure on the calling thread.
 */
#ifndef FEA_GPU_H
#define FEA_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define FEA_API __attribute__((visibility("default")))
#else
#define FEA_API
#endif

typedef enum {
    FEA_OK = 0,
    FEA_ERR_INVALID = 1,        /* std::invalid_argument / std::out_of_range (dof_map.cpp:25-27, :82-84) */
    FEA_ERR_MISSING_ENTRY = 2,  /* AssemblyError, assembly.hpp:65-73 */
    FEA_ERR_OOM = 3,            /* std::bad_alloc (bench.cpp:257-264) */
    FEA_ERR_CUDA = 4,
    FEA_ERR_INVALID_COLOURING = 5 /* AssemblyError("invalid colouring: ...") assembly.hpp:178-182 */
} fea_status;

/* Conflict strategies of the numeric phase. */
typedef enum {
    /* fp64 atomicAdd per entry — the GPU form of assemble_atomic
     * (assembly.hpp:121-126, AtomicValues formats.hpp:123-138). Matches
     * assemble_sequential within |a-b| <= 1e-12*max(|a|,|b|,1). */
    FEA_ATOMIC = 0,
    /* Deterministic sort-by-slot segmented reduction: every value slot is a
     * left fold, starting from the slot's value, over its contributions in
     * ascending element id — bit-identical to assemble_sequential
     * (assembly.hpp:112-118). */
    FEA_DET_SORTED = 1,
    /* Deterministic colouring route: one pass per colour, plain adds — the GPU
     * form of assemble_coloured_vectorized (assembly.hpp:175-195); bit-identical
     * to it under the same colouring. Needs fea_plan_set_colouring(). */
    FEA_DET_COLOUR = 2
} fea_strategy;

/* fea_assemble flags */
#define FEA_ACCUMULATE 0u /* values += assembled (reference semantics: assemble adds) */
#define FEA_OVERWRITE 1u  /* values  = assembled (== reset_values, formats.hpp:351-354, then assemble) */
#define FEA_COLOUR_PASSES 2u /* FEA_DET_COLOUR as one launch per colour (element-owner, plain adds)
                              instead of the colour-ordered segmented reduction; same bits */

/* fea_plan_create flags */
#define FEA_PLAN_K_COMPACT 1u /* K holds only the plan's kept elements, in ascending element id
                                 (row-partitioned plans); default: K holds all E elements */

/* fea_plan_create_with_pattern formats */
#define FEA_FORMAT_CSR 0
#define FEA_FORMAT_CRAC 1

typedef struct fea_plan fea_plan;

/* Message of the last failure on this thread ("" if none). */
FEA_API const char* fea_last_error(void);

/* Library/ABI version: major*10000 + minor*100 + patch. */
FEA_API int fea_version(void);

/*
 * Symbolic phase + slot-map build.
 * Replaces: fea::build_pattern(const DofMap&) (pattern.hpp:40, pattern.cpp:24-108)
 *           + CsrMatrix(pattern) / CracMatrix(pattern) (formats.hpp:157-160, :268-273,
 *             build_crac_arrays formats.cpp:21-41)
 *           + the per-entry locate() of scatter_element (assembly.hpp:84), resolved once.
 *  elem_dofs     E x m int64 DOFs (ElementDofs::flat of every element), host or device
 *  n_rows        number of global rows (DofMap::n_dofs)
 *  dofs_per_node d of the DofMap (dof(v,k) = v*d+k, dof_map.hpp:59); the plan verifies
 *                the node-contiguous layout and falls back to d = 1 if it does not hold
 *  row_begin/end owned global row range [row_begin, row_end) (multiples of d); the
 *                whole matrix is [0, n_rows). Only owned rows are assembled; the
 *                plan's CSR/CRAC row block is rebased to 0, columns stay global.
 */
FEA_API fea_status fea_plan_create(int device, const int64_t* elem_dofs, int64_t n_elements, int32_t m,
                           int64_t n_rows, int32_t dofs_per_node, int64_t row_begin,
                           int64_t row_end, uint32_t flags, fea_plan** out);

/*
 * Plan against an externally supplied pattern (whole matrix).
 * Replaces: CsrMatrix(const SparsityPattern&) / CracMatrix(...) built from a
 * caller's pattern (formats.hpp:157, :268) + the locate() of every element entry:
 * CSR lower-bound search (formats.hpp:165-199) or CRAC Listing-1 block search
 * (formats.hpp:276-290), warp-cooperative on the device. An element entry absent
 * from the pattern is recorded (lowest element id) and makes fea_assemble fail
 * with FEA_ERR_MISSING_ENTRY, as scatter_element throws (assembly.hpp:85-87).
 *  format FEA_FORMAT_CSR : row_ptr[n_rows+1], idx = cols[nnz]
 *  format FEA_FORMAT_CRAC: row_ptr[n_rows+1] in col_align entry units, idx = col_align[2*runs+2]
 */
FEA_API fea_status fea_plan_create_with_pattern(int device, const int64_t* elem_dofs, int64_t n_elements,
                                        int32_t m, int64_t n_rows, int32_t format,
                                        const int64_t* row_ptr, const int64_t* idx,
                                        fea_plan** out);

FEA_API void fea_plan_destroy(fea_plan* plan);

/* Sizes of the plan's (owned) row block: rows, nnz (= values length), CRAC runs
 * (count_pattern_runs, pattern.cpp:110-120), kept elements. */
FEA_API fea_status fea_plan_sizes(const fea_plan* plan, int64_t* n_rows, int64_t* nnz, int64_t* n_runs,
                          int64_t* n_elements);

/* Slot-map / plan details for reporting: dofs per node used, nodes per element,
 * bytes of device metadata held by the plan. */
FEA_API fea_status fea_plan_info(const fea_plan* plan, int32_t* dofs_per_node, int32_t* nodes_per_element,
                         int64_t* metadata_bytes);

/* CSR arrays of the plan (SparsityPattern::row_ptr/cols, pattern.hpp:29-35):
 * row_ptr[n_rows+1], cols[nnz]; host or device destinations (device ones are written in
 * place); cols may be NULL to fetch only row_ptr. */
FEA_API fea_status fea_plan_copy_csr(const fea_plan* plan, int64_t* row_ptr, int64_t* cols);

/* CRAC arrays (CracBase::rows / col_align, formats.hpp:257-273): row_ptr[n_rows+1]
 * in col_align entry units, col_align[2*runs+2] with the final (0, nnz) pair; host or
 * device destinations; col_align may be NULL to fetch only row_ptr. */
FEA_API fea_status fea_plan_copy_crac(const fea_plan* plan, int64_t* row_ptr, int64_t* col_align);

/* Ids (ascending) of the elements the plan keeps (those with a node in the owned
 * row range); elem_ids[n_elements] from fea_plan_sizes. */
FEA_API fea_status fea_plan_copy_elements(const fea_plan* plan, int64_t* elem_ids);

/* Greedy colouring of the plan's elements — fea::greedy_colouring
 * (colouring.cpp:24-75): ascending element order, smallest colour unused by any
 * node-sharing element. colour_of[n_elements] (host; the plan's kept elements in
 * ascending id, = all E for a whole-matrix plan). */
FEA_API fea_status fea_plan_greedy_colouring(const fea_plan* plan, int32_t* colour_of, int32_t* n_colours);

/* Jones-Plassmann colouring computed on the device (seeded priorities): a valid colouring in
 * a few kernel rounds instead of the sequential greedy pass; it is NOT the reference's greedy
 * colouring, so FEA_DET_COLOUR is bit-identical to assemble_coloured_vectorized run with this
 * same colouring. colour_of[n_elements] (host). */
FEA_API fea_status fea_plan_jp_colouring(const fea_plan* plan, uint64_t seed, int32_t* colour_of,
                                         int32_t* n_colours);

/* Install the colouring used by FEA_DET_COLOUR (Colouring::colour_of,
 * colouring.hpp:35-39; host or device array over the plan's kept elements).
 * Validated like find_colour_conflict (colouring.cpp:91-119): two same-colour
 * elements sharing a DOF -> FEA_ERR_INVALID_COLOURING. */
FEA_API fea_status fea_plan_set_colouring(fea_plan* plan, const int32_t* colour_of);

/*
 * Numeric phase.
 * Replaces: assemble_atomic / assemble_sequential / assemble_coloured_vectorized
 * (assembly.hpp:112-195) on CsrMatrix / CsrAtomicMatrix / CracMatrix /
 * CracAtomicMatrix targets.
 *  K       device [E][m][m] fp64 (or [kept][m][m] with FEA_PLAN_K_COMPACT)
 *  values  device fp64[nnz]
 *  flags   FEA_ACCUMULATE or FEA_OVERWRITE
 *  stream  cudaStream_t (as void*)
 */
FEA_API fea_status fea_assemble(fea_plan* plan, const double* K, int32_t strategy, double* values,
                        uint32_t flags, void* stream);

/* End-to-end form with HOST buffers (pinned or pageable): copies K host->device,
 * assembles, copies values device->host; synchronous like the reference call
 * (SPEC.md:364). Device staging buffers are cached in the plan. */
FEA_API fea_status fea_assemble_host(fea_plan* plan, const double* K_host, int32_t strategy,
                             double* values_host, uint32_t flags, void* stream);

/* Pipeline depth of fea_assemble_host: the node traversal is cut into n_windows windows; K
 * goes host->device in the chunks each window first needs, every window is launched as soon as
 * its chunk has landed and its values range goes device->host while later chunks are still
 * coming in (contiguous ranges when nodes are traversed in id order). 0 (default): automatic,
 * chunks of >= 256 MB of K and at most 32 windows. Only the segmented-reduction routes whose
 * kernels take windows use them; the others run upload -> assemble -> download. */
FEA_API fea_status fea_plan_set_host_windows(fea_plan* plan, int32_t n_windows);

/* Fused supplier: assemble the seeded synthetic element matrices of fea_fill_seeded_k WITHOUT
 * materializing K — the gather kernels generate each entry in registers (the GPU form of the
 * reference's ElementMatrixSupplier called inside the assembly, assembly.hpp:37, :78). Same bits
 * as fea_assemble on a fea_fill_seeded_k buffer. Strategies FEA_DET_SORTED / FEA_DET_COLOUR. */
FEA_API fea_status fea_assemble_seeded(fea_plan* plan, uint64_t seed, int32_t strategy, double* values,
                                       uint32_t flags, void* stream);

/* Repeated end-to-end assemblies of the same plan with new element matrices (Newton
 * iterations, time steps, load cases): n_steps pairs of HOST buffers K_hosts[i] ->
 * values_hosts[i]. Pipelined with two device staging slots: step i's K host->device copy
 * overlaps step i-1's kernel and values device->host copy (PCIe is full duplex). Every step
 * moves its whole K in and its whole values out; synchronous on return. Pinned host memory
 * is required for the overlap. */
FEA_API fea_status fea_assemble_host_batch(fea_plan* plan, const double* const* K_hosts,
                                           int32_t strategy, double* const* values_hosts,
                                           int32_t n_steps, uint32_t flags, void* stream);

/* The missing entry behind FEA_ERR_MISSING_ENTRY: element, row, column (the
 * values AssemblyError names, assembly.hpp:65-73). Returns FEA_OK with e = -1
 * when the plan has none. */
FEA_API fea_status fea_plan_missing_entry(const fea_plan* plan, int64_t* element, int64_t* row,
                                  int64_t* col);

/* Number of kernel launches the last fea_assemble issued on this plan. */
FEA_API int32_t fea_plan_last_launches(const fea_plan* plan);

/* Seeded synthetic element matrices: K[i][r][c] = U(seed, id_i, min(r,c), max(r,c)),
 * symmetric, uniform on [-1,1), exactly representable (the counter-hash supplier of
 * SURVEY.md §7.2; stands in for ElementMatrixSupplier, assembly.hpp:37).
 * elem_ids: NULL (id_i = i) or device int64[n]. */
FEA_API fea_status fea_fill_seeded_k(double* K, int64_t n, int32_t m, uint64_t seed,
                             const int64_t* elem_ids, void* stream);

/*
 * y = A x on an assembled matrix (the consumer of the assembly; CRAC's payoff).
 * All pointers are DEVICE pointers; x is indexed by global column, y by (owned) row.
 *  fea_spmv_csr : CSR arrays (row_ptr[n_rows+1], cols[nnz])
 *  fea_spmv_crac: CRAC arrays (row_ptr[n_rows+1] in col_align entry units, col_align[2*runs+2])
 *  fea_plan_spmv: the plan's own node-block layout (no column array needed)
 * values is the fea_assemble output (identical for CSR and CRAC). Stream-ordered.
 */
FEA_API fea_status fea_spmv_csr(const int64_t* row_ptr, const int64_t* cols, const double* values,
                                int64_t n_rows, const double* x, double* y, void* stream);
FEA_API fea_status fea_spmv_crac(const int64_t* row_ptr, const int64_t* col_align, const double* values,
                                 int64_t n_rows, const double* x, double* y, void* stream);
FEA_API fea_status fea_plan_spmv(const fea_plan* plan, const double* values, const double* x, double* y,
                                 void* stream);

/*
 * The device primitives of the symbolic phase (north-star subsystem 1: sort/unique + exclusive
 * scan; pattern.cpp:24-108 does the same job with std::sort / std::unique per row). Hand-written
 * (csrc/prims.cu), exposed so the tests can pin them and so callers that build their own
 * patterns can reuse them. All pointers are DEVICE pointers; stream-ordered, return after the
 * work has completed.
 *  fea_exclusive_sum_i64: out[i] = in[0] + ... + in[i-1] (in and out may be the same array)
 *  fea_sort_pairs_u32   : stable LSD radix sort of (uint32 key, int32 value) pairs by key bits
 *                         [begin_bit, end_bit); inputs intact, n < 2^31
 */
FEA_API fea_status fea_exclusive_sum_i64(const int64_t* in, int64_t* out, int64_t n, void* stream);
FEA_API fea_status fea_sort_pairs_u32(const uint32_t* keys_in, uint32_t* keys_out, const int32_t* vals_in,
                                      int32_t* vals_out, int64_t n, int32_t begin_bit, int32_t end_bit,
                                      void* stream);

/*
 * Peer memory for the fused row-partitioned assembly + gather (no reference
 * counterpart — the reference is shared-memory only). The root exports its global
 * values buffer, every rank maps it and fea_assemble()s its owned row block straight into it at
 * the block's global offset: the kernel's value stores go over NVLink/NVSwitch as they are
 * produced, so the gather overlaps the assembly instead of following it.
 *  fea_ipc_export: CUDA IPC handle (64 bytes) of the allocation holding dev_ptr, and dev_ptr's
 *                  byte offset inside it (works for sub-allocations of caching allocators)
 *  fea_ipc_open:   map an exported allocation into this process on `device` (peer access
 *                  enabled lazily); *base is the allocation start; fea_ipc_close unmaps it
 */
FEA_API fea_status fea_ipc_export(const void* dev_ptr, void* handle64, int64_t* offset_bytes);
FEA_API fea_status fea_ipc_open(const void* handle64, int device, void** base);
FEA_API fea_status fea_ipc_close(void* base);

#ifdef __cplusplus
}
#endif

#endif /* FEA_GPU_H */
