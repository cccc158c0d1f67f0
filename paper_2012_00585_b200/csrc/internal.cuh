// Internal declarations of the B200 FE-assembly library (not part of the ABI).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/fea_gpu.h"

namespace feagpu {

// Exception carried to the C-ABI boundary and turned into a fea_status.
struct Error : std::runtime_error {
    fea_status status;
    Error(fea_status s, const std::string& msg) : std::runtime_error(msg), status(s) {}
};

[[noreturn]] void throw_cuda(cudaError_t e, const char* what, const char* file, int line);

#define FEA_CK(x)                                                      \
    do {                                                               \
        cudaError_t e_ = (x);                                          \
        if (e_ != cudaSuccess) ::feagpu::throw_cuda(e_, #x, __FILE__, __LINE__); \
    } while (0)

#define FEA_REQUIRE(cond, status, msg)                                 \
    do {                                                               \
        if (!(cond)) throw ::feagpu::Error((status), (msg));           \
    } while (0)

// Owning device allocation.
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; o.bytes = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) { reset(); p = o.p; bytes = o.bytes; o.p = nullptr; o.bytes = 0; }
        return *this;
    }
    ~DevBuf() { reset(); }
    void alloc(size_t n);
    void reset();
    template <class T> T* as() const { return static_cast<T*>(p); }
};

// RAII scope that makes `dev` current and restores the previous device.
struct DeviceScope {
    int prev = -1;
    explicit DeviceScope(int dev);
    ~DeviceScope();
};

// Environment A/B switches of the numeric kernels, read once per plan (at
// creation) instead of on every assembly.
struct Knobs {
    bool atomic_legacy, atomic_no_patch, slot_no_fixed, cn_unpacked, cn_no_records, d1_no_direct, d1_no_vec;
    bool d1_no_lane;  // FEA_D1_NO_LANE: shared-memory fold (k_gather_d1g) instead of lane-owned slots
    bool atomic_no_strip;  // FEA_ATOMIC_NO_STRIP: k_atomic_staged instead of strip pre-reduction (npe 4, d 1)
    bool patch_tickets;  // FEA_PATCH_TICKETS: tickets also for short runs
    bool patch_static;  // FEA_PATCH_STATIC: k_atomic_patch CTAs stride by the grid size instead of taking tickets
    bool gather_global;  // FEA_GATHER_GLOBAL: k_gather_global (accumulate in the values array) for every plan
    bool d1_rec8;  // FEA_D1_REC8: 8-byte lane records even where the compact 4-byte form fits
    int d1_acc_mod, d1v_acc_mod;  // accumulator stride residues (mod 16 doubles)
};
Knobs read_knobs();

// Stream/event set of the end-to-end host paths (fea_assemble_host pipeline and
// fea_assemble_host_batch), created on first use and kept with the plan.
struct HostPipe {
    cudaStream_t sin = nullptr, sout = nullptr;
    std::vector<cudaEvent_t> ev;  // 2 per window (+1), 6 for the batch path
    // fea_assemble_host windows: traversal windows [t_win[j], t_win[j+1]) and, per window, the
    // K rows every window up to it needs (k_end, prefix max) and its values range (contiguous
    // when nodes are traversed in id order)
    int n_win = 0;
    int32_t want_win = 0;  // fea_plan_set_host_windows (0: automatic)
    std::vector<int64_t> t_win, k_end, v_off;
    bool v_contiguous = false;
    void ensure_events(int n);
    ~HostPipe();
};

}  // namespace feagpu

// The plan: everything the numeric phase needs, resolved once (north-star
// subsystems 1 and 2). Node-level layout — the d DOF rows of a node share one
// column structure (pattern.cpp:85-91) — so all metadata is per node, with d
// applied arithmetically.
struct fea_plan {
    int device = 0;
    // problem shape
    int64_t E_in = 0;        // elements given
    int32_t m = 0;           // DOFs per element
    int32_t d = 1;           // DOFs per node used by the plan (1 = DOF-level)
    int32_t npe = 0;         // nodes per element = m / d
    int64_t n_rows = 0;      // global rows
    int64_t row_begin = 0, row_end = 0;
    int64_t node_begin = 0, node_end = 0, n_own = 0;  // owned nodes
    int64_t E = 0;           // kept elements
    bool partitioned = false;
    bool k_compact = false;
    bool external = false;   // pattern supplied by the caller
    bool dup_nodes = false;  // some element lists a node twice (serialised fold variant)
    // sizes
    int64_t n_adj = 0;       // owned (node, element) incidences
    int64_t nnz_nodes = 0;   // node-level pattern entries
    int64_t nnz = 0;         // DOF-level values of the owned block
    int64_t n_runs = 0;      // CRAC runs of the owned block
    int32_t max_cnt = 0;     // longest node-level row
    int64_t max_adj = 0;     // most elements at one node
    int32_t pos_bytes = 1;   // 1 (uint8) or 2 (uint16) row-relative positions
    int32_t pstride = 0;     // posA entries per incidence: npe rounded up to a 4-byte multiple
    // device metadata
    feagpu::DevBuf conn_k;    // int32 [krows*npe] node ids, indexed by K row
    feagpu::DevBuf elem_id;   // int64 [E] global ids of kept elements, ascending
    feagpu::DevBuf elem_krow; // int32 [E] K row of each kept element
    feagpu::DevBuf adj_ptr;   // int64 [n_own+1]
    feagpu::DevBuf adj;       // int32 [n_adj] K chunk index = krow*npe + a, ascending element id per node
    feagpu::DevBuf nptr;      // int64 [n_own+1] node-level row pointer
    feagpu::DevBuf ncol;      // int32 [nnz_nodes] sorted neighbour node ids
    feagpu::DevBuf nrun_ptr;  // int64 [n_own+1] exclusive scan of node-level runs
    feagpu::DevBuf posA;      // PosT [n_adj*npe] positions, adjacency order (gather route)
    feagpu::DevBuf posE;      // PosT [E*npe*npe] positions, element order (atomic/colour routes; lazy)
    feagpu::DevBuf order;     // int32 [E] atomic-route element order (lazy)
    // atomic route, common shapes: metadata in visit order (k_atomic_staged; lazy)
    feagpu::DevBuf at_krow;   // int32 [at_E_pad] K row of the i-th visited element
    feagpu::DevBuf at_rows;   // int64 [at_E_pad*npe] values start << 20 | row length (-1: not owned)
    feagpu::DevBuf at_pos;    // PosT [at_E_pad*npe*npe] row-relative positions
    int64_t at_E_pad = 0;     // E rounded up to whole warp steps
    // atomic route with patch pre-reduction (k_atomic_patch; npe = 8, lazy): patches of <= 8
    // node-sharing elements, their distinct (row node, column node) pairs and per element the
    // pair index of every (a, b)
    feagpu::DevBuf pk_hdr;    // int4 [pk_n]: -, pair offset, row offset, n_elems | n_rows << 8 | n_pairs << 16
    feagpu::DevBuf pk_krow;   // int32 [pk_n*8] K row per element slot (-1: empty slot)
    feagpu::DevBuf pk_cidx;   // uint16 [pk_n*8*64] pair index per (slot, a, b) (0xffff: row not owned)
    feagpu::DevBuf pk_rows;   // int64 [] values start << 20 | row length per patch row node
    feagpu::DevBuf pk_rowpair;  // int32 [] first pair of the row | pair count << 16 (pairs sorted by row)
    feagpu::DevBuf pk_pairs;  // uint16 [] row index << 8 | position per distinct pair
    int64_t pk_n = 0;
    // atomic route for npe = 4, d = 1 (k_atomic_strip; lazy): strips of 48 consecutive elements of
    // the visit order, per strip the distinct (row node, position) pairs and for each pair the
    // list of K entries of the strip that feed it (fixed-stride blob, one bulk copy per strip)
    feagpu::DevBuf sk_meta;   // [sk_n][sk_stride] header, values start per local node, position per pair
    feagpu::DevBuf sk_shape;  // [shapes][sk_sh_stride] list end per pair, local row per pair, entry offsets
    feagpu::DevBuf sk_k0;     // int4 [sk_n] {first K row if the strip's K rows are consecutive else -1, elements, shape}
    feagpu::DevBuf sk_krow;   // int32 [sk_n*48] K row per element (-1: none)
    int64_t sk_n = 0;
    int32_t sk_stride = 0, sk_off_pos = 0, sk_sh_stride = 0, sk_off_prow = 0, sk_off_ent = 0;
    feagpu::DevBuf pk_ticket;  // uint64 [1024] patch ticket counters, one per launch in flight (ring)
    uint32_t pk_ticket_next = 0;
    int32_t pk_max_pairs = 0;
    feagpu::DevBuf node_order;  // int32 [n_own] gather traversal order (empty: node id order)
    // d = 1 with a traversal order: the sorted incidences re-laid in traversal order, so the
    // gather reads them sequentially (else: random 128 B line fetches per node)
    feagpu::DevBuf trav_ptr;   // int64 [n_own+1] record offsets per traversal position
    feagpu::DevBuf trav_meta;  // int64 [n_own] values start << 20 | row length
    feagpu::DevBuf trav_rec;   // int32 [n_adj*trav_rw] {entry, position words[, pad]}
    feagpu::DevBuf trav_recC;  // the same for the colour-ordered incidences (adjC / posAC)
    // d = 1, npe = 4, rows of <= 16 nodes: lane-owned slots (k_gather_d1r). Every slot of a node's
    // row belongs to one of the 4 lanes of its group (a proper 4-colouring of the node's star:
    // the 4 nodes of each incident element get 4 distinct lanes) and to one of that lane's
    // registers, so the fold needs no shared memory and no warp synchronisation.
    feagpu::DevBuf ln_slot;    // uint8 [n_own*16] lane | accumulator << 2 per (traversal position, slot)
    // int4 [2*n_own] per traversal position: {values start << 20 | the diagonal slot << 16 |
    // accumulators used per lane (4 x 4 bits) (int64), first record | record count << 40 (int64)},
    // {4 * lowest K row, lanes 1..3: the slots of their accumulators, 4 bits each}
    feagpu::DevBuf ln_hdr;
    feagpu::DevBuf ln_rec;     // records, sorted incidences: uint32 (compact) or int2 {entry, lane word}
    feagpu::DevBuf ln_recC;    // the same for the colour-ordered incidences
    bool ln_ok = false;
    bool ln_rec4 = false;      // compact 4-byte records (entry offset fits next to the lane fields)
    int32_t ln_q = 0;          // most accumulators any lane needs
    int32_t ln_wq[3] = {0, 0, 0};  // record bits of the accumulator field of lanes 1..3
    feagpu::DevBuf cnr_hdr;    // int4 [n_own]: values start (int64), row length | n << 16, accumulator offset
    feagpu::DevBuf cnr_rec;    // [n_own][8][32 B]: {entry, npe position bytes} per incidence (k_gather_cnr)
    feagpu::DevBuf cnr_recC;   // the same for the colour-ordered incidences (reset by set_colouring)
    feagpu::DevBuf slot_hdr, slot_rec, slot_recC;  // k_gather_slot fixed-stride node metadata (lazy)
    int32_t trav_rw = 0;
    int64_t cn_cta_acc = 0;     // packed accumulator doubles per CTA of k_gather_cn (lazy)
    int32_t cn_cta_per = 0;
    // colouring
    bool has_colouring = false;
    feagpu::DevBuf colour_elems;           // int32 [E] local elements grouped by colour, ascending id
    feagpu::DevBuf adjC, posAC;            // incidences per node in (colour, element) order + positions
    std::vector<int64_t> colour_off;       // n_colours+1 (host)
    // external-pattern missing entry (lowest element)
    int64_t miss_e = -1, miss_r = -1, miss_c = -1;
    // bookkeeping
    feagpu::Knobs kn = {};     // A/B switches as the environment had them when the plan was created
    int32_t last_launches = 0;
    bool gather_global = false;  // no shared-memory gather fits the largest row block: k_gather_global
    bool gen_on = false;       // fea_assemble_seeded in progress: kernels generate K
    uint64_t gen_seed = 0;
    bool cn_disabled = false;  // FEA_GATHER_NO_CN=1: decode-table gather (A/B)
    bool d1_disabled = false;  // FEA_GATHER_NO_D1=1: per-node gather for d = 1 (A/B)
    bool slot_disabled = false;  // FEA_GATHER_NO_SLOT=1: column-node gather for d in 2..4 (A/B)
    feagpu::DevBuf stage_K, stage_V;       // fea_assemble_host staging
    feagpu::DevBuf bstage_K[2], bstage_V[2];  // fea_assemble_host_batch double buffers
    feagpu::HostPipe pipe;                    // end-to-end streams, events, K/values windows
    // launch bookkeeping that never changes for a plan (cached instead of queried per call)
    int32_t sms = 0;  // SM count of the plan's device
    struct Occ {
        const void* fn;
        size_t smem;
        int threads, per_sm;
    };
    std::vector<Occ> occ_cache;
    // traversal window of the gather launch: nodes [win_t0, win_t0 + win_n) of the traversal
    // order (the fea_assemble_host pipeline runs one window per K chunk); win_n < 0: all.
    // win_query: the launcher only reports (win_ok) whether its kernel takes windows, after
    // building its lazy tables, and launches nothing.
    int64_t win_t0 = 0, win_n = -1;
    bool win_query = false, win_ok = false;
    int64_t kbytes_required() const;
    int64_t krows() const { return k_compact ? E : E_in; }
};

namespace feagpu {
// Per-node incidence order used by the gather: ascending element id (FEA_DET_SORTED) or
// ascending (colour, element id) (FEA_DET_COLOUR), with the matching position rows.
struct Incidences {
    const int32_t* adj;
    const void* posA;
};
// gather_u8.cu / gather_u16.cu (numeric kernels per position width)
void gather_u8(fea_plan* p, const Incidences& in, const double* K, double* values, bool accumulate,
               cudaStream_t s);
void gather_u16(fea_plan* p, const Incidences& in, const double* K, double* values, bool accumulate,
                cudaStream_t s);
void scatter_u8(fea_plan* p, const double* K, const int32_t* list, int64_t n_list, double* values,
                bool atomic, cudaStream_t s);
void scatter_u16(fea_plan* p, const double* K, const int32_t* list, int64_t n_list, double* values,
                 bool atomic, cudaStream_t s);
// numeric.cu
void ensure_element_maps(fea_plan* p, cudaStream_t s);
void assemble(fea_plan* p, const double* K, int strategy, double* values, uint32_t flags,
              cudaStream_t s);
// plan.cu helpers used by numeric.cu
int64_t metadata_bytes(const fea_plan* p);
}  // namespace feagpu
