/*
 * TEST INFRASTRUCTURE — the CPU oracle. NOT product code.
 *
 * Plain-C restatement of the reference algorithm for the FE assembly hot
 * path of arXiv 2012.00585 (reference: /root/reference/proj). Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it, and
 * only as the checker. The product path (paper_2012_00585_b200) never links
 * or calls it.
 *
 * Parity pinning: every function below is cross-checked in tests/ against
 * (a) the reference's own golden vectors (Fig. 1 6x6 CSR/CRAC arrays and
 * lookups, RLE fixture, exact NNZ tables, test_formats.cpp / acceptance.cpp),
 * and (b) the UNMODIFIED reference library compiled into
 * oracle/_ref/libfea_ref.so (fixtures committed under tests/golden/).
 *
 * Each function cites the reference file:line it restates.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef int64_t idx_t; /* types.hpp:27 — index_t = int64_t */

/* ------------------------------------------------------------------------ */
/* Seeded inputs (shared definition with the device generator)  */
/* ------------------------------------------------------------------------ */

uint64_t orc_splitmix64(uint64_t x) {
    uint64_t z = x + 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

/* Symmetric element matrix entry, uniform on [-1, 1) with 53 random bits;
 * (h>>11)*2^-53*2-1 is exact in binary64, so host and device agree bit for
 * bit. K[e][i][j] == K[e][j][i]. */
double orc_kval(uint64_t seed, int64_t e, int32_t i, int32_t j) {
    const uint64_t lo = (uint64_t)(i < j ? i : j);
    const uint64_t hi = (uint64_t)(i < j ? j : i);
    const uint64_t h = orc_splitmix64(orc_splitmix64(seed + (uint64_t)e) ^ ((lo << 32) | hi));
    return (double)(h >> 11) * 0x1p-53 * 2.0 - 1.0;
}

void orc_fill_k(uint64_t seed, int64_t n_elements, int32_t m, double* K) {
    for (int64_t e = 0; e < n_elements; ++e)
        for (int32_t i = 0; i < m; ++i)
            for (int32_t j = 0; j < m; ++j) K[(e * m + i) * m + j] = orc_kval(seed, e, i, j);
}

/* K of elements e0 .. e0+n-1 (element ids, not positions) into K[0 .. n*m*m): lets the
 * Python side fill large buffers from several threads. */
void orc_fill_k_range(uint64_t seed, int64_t e0, int64_t n, int32_t m, double* K) {
    for (int64_t e = 0; e < n; ++e)
        for (int32_t i = 0; i < m; ++i)
            for (int32_t j = 0; j < m; ++j) K[(e * m + i) * m + j] = orc_kval(seed, e0 + e, i, j);
}

/* ------------------------------------------------------------------------ */
/* Symbolic phase                                                            */
/* ------------------------------------------------------------------------ */

typedef struct {
    idx_t n_rows;
    idx_t nnz;
    idx_t* row_ptr; /* n_rows + 1 */
    idx_t* cols;    /* nnz, ascending per row */
} orc_pattern;

static int cmp_idx(const void* a, const void* b) {
    const idx_t x = *(const idx_t*)a, y = *(const idx_t*)b;
    return (x > y) - (x < y);
}

/* sort + unique in place, returns the new length (std::sort + std::unique,
 * pattern.cpp:81-82) */
static idx_t sort_unique(idx_t* v, idx_t n) {
    if (n == 0) return 0;
    qsort(v, (size_t)n, sizeof(idx_t), cmp_idx);
    idx_t w = 1;
    for (idx_t i = 1; i < n; ++i)
        if (v[i] != v[w - 1]) v[w++] = v[i];
    return w;
}

/* node -> element inverted index (pattern.cpp:32-48, colouring.cpp:27-45):
 * adjacency of node v is adj[adj_ptr[v] .. adj_ptr[v+1]), element ids
 * ascending because elements are visited in order. Duplicate nodes inside
 * one element list the element twice, as in the reference. */
static void node_adjacency(const idx_t* element_nodes, idx_t n_elements, int npe, idx_t n_nodes,
                           idx_t** adj_ptr_out, idx_t** adj_out) {
    idx_t* adj_ptr = (idx_t*)calloc((size_t)n_nodes + 1, sizeof(idx_t));
    for (idx_t i = 0; i < n_elements * npe; ++i) adj_ptr[element_nodes[i] + 1]++;
    for (idx_t v = 0; v < n_nodes; ++v) adj_ptr[v + 1] += adj_ptr[v];
    idx_t* fill = (idx_t*)malloc(((size_t)n_nodes + 1) * sizeof(idx_t));
    memcpy(fill, adj_ptr, ((size_t)n_nodes + 1) * sizeof(idx_t));
    idx_t* adj = (idx_t*)malloc((size_t)(n_elements * npe + 1) * sizeof(idx_t));
    for (idx_t e = 0; e < n_elements; ++e)
        for (int a = 0; a < npe; ++a) adj[fill[element_nodes[e * npe + a]]++] = e;
    free(fill);
    *adj_ptr_out = adj_ptr;
    *adj_out = adj;
}

/* build_pattern, pattern.cpp:24-108: per node, gather the DOFs of every
 * adjacent element's nodes, sort/unique, replicate the count to the node's
 * d rows, scan, then fill with a second identical gather. */
orc_pattern* orc_build_pattern(const idx_t* element_nodes, idx_t n_elements, int npe,
                               idx_t n_nodes, int d) {
    idx_t *adj_ptr, *adj;
    node_adjacency(element_nodes, n_elements, npe, n_nodes, &adj_ptr, &adj);
    idx_t max_deg = 0;
    for (idx_t v = 0; v < n_nodes; ++v)
        if (adj_ptr[v + 1] - adj_ptr[v] > max_deg) max_deg = adj_ptr[v + 1] - adj_ptr[v];
    idx_t* scratch = (idx_t*)malloc((size_t)(max_deg * npe * d + 1) * sizeof(idx_t));

    orc_pattern* p = (orc_pattern*)calloc(1, sizeof(orc_pattern));
    p->n_rows = n_nodes * d;
    p->row_ptr = (idx_t*)calloc((size_t)p->n_rows + 1, sizeof(idx_t));
    idx_t* node_count = (idx_t*)calloc((size_t)n_nodes + 1, sizeof(idx_t));

#define GATHER(v, len)                                                          \
    do {                                                                        \
        len = 0;                                                                \
        for (idx_t a_ = adj_ptr[v]; a_ < adj_ptr[(v) + 1]; ++a_)                \
            for (int b_ = 0; b_ < npe; ++b_) {                                  \
                const idx_t base_ = element_nodes[adj[a_] * npe + b_] * d;      \
                for (int k_ = 0; k_ < d; ++k_) scratch[len++] = base_ + k_;     \
            }                                                                   \
        len = sort_unique(scratch, len);                                        \
    } while (0)

    for (idx_t v = 0; v < n_nodes; ++v) {
        idx_t len;
        GATHER(v, len);
        node_count[v] = len;
        for (int k = 0; k < d; ++k) p->row_ptr[v * d + k + 1] = len;
    }
    for (idx_t r = 0; r < p->n_rows; ++r) p->row_ptr[r + 1] += p->row_ptr[r];
    p->nnz = p->row_ptr[p->n_rows];
    p->cols = (idx_t*)malloc((size_t)(p->nnz + 1) * sizeof(idx_t));
    for (idx_t v = 0; v < n_nodes; ++v) {
        if (node_count[v] == 0) continue;
        idx_t len;
        GATHER(v, len);
        for (int k = 0; k < d; ++k) memcpy(p->cols + p->row_ptr[v * d + k], scratch, (size_t)len * sizeof(idx_t));
    }
#undef GATHER
    free(scratch);
    free(node_count);
    free(adj_ptr);
    free(adj);
    return p;
}

orc_pattern* orc_pattern_from_arrays(idx_t n_rows, const idx_t* row_ptr, const idx_t* cols) {
    orc_pattern* p = (orc_pattern*)calloc(1, sizeof(orc_pattern));
    p->n_rows = n_rows;
    p->nnz = row_ptr[n_rows];
    p->row_ptr = (idx_t*)malloc(((size_t)n_rows + 1) * sizeof(idx_t));
    memcpy(p->row_ptr, row_ptr, ((size_t)n_rows + 1) * sizeof(idx_t));
    p->cols = (idx_t*)malloc((size_t)(p->nnz + 1) * sizeof(idx_t));
    memcpy(p->cols, cols, (size_t)p->nnz * sizeof(idx_t));
    return p;
}

void orc_pattern_free(orc_pattern* p) {
    if (!p) return;
    free(p->row_ptr);
    free(p->cols);
    free(p);
}

/* count_pattern_runs, pattern.cpp:110-120 */
idx_t orc_count_runs(const orc_pattern* p) {
    idx_t runs = 0;
    for (idx_t r = 0; r < p->n_rows; ++r)
        for (idx_t i = p->row_ptr[r]; i < p->row_ptr[r + 1]; ++i)
            if (i == p->row_ptr[r] || p->cols[i] != p->cols[i - 1] + 1) ++runs;
    return runs;
}

void orc_pattern_sizes(const orc_pattern* p, idx_t* n_rows, idx_t* nnz, idx_t* n_runs) {
    *n_rows = p->n_rows;
    *nnz = p->nnz;
    *n_runs = orc_count_runs(p);
}

void orc_pattern_copy(const orc_pattern* p, idx_t* row_ptr, idx_t* cols) {
    memcpy(row_ptr, p->row_ptr, ((size_t)p->n_rows + 1) * sizeof(idx_t));
    memcpy(cols, p->cols, (size_t)p->nnz * sizeof(idx_t));
}

/* build_crac_arrays, formats.cpp:21-41: row_ptr in col_align entry units,
 * (col_start, values_pos) per run, final pair (0, nnz). */
void orc_crac_arrays(const orc_pattern* p, idx_t* row_ptr, idx_t* col_align) {
    idx_t w = 0;
    for (idx_t r = 0; r < p->n_rows; ++r) {
        row_ptr[r] = w;
        for (idx_t i = p->row_ptr[r]; i < p->row_ptr[r + 1]; ++i) {
            if (i == p->row_ptr[r] || p->cols[i] != p->cols[i - 1] + 1) {
                col_align[w++] = p->cols[i];
                col_align[w++] = i;
            }
        }
    }
    row_ptr[p->n_rows] = w;
    col_align[w++] = 0;
    col_align[w++] = p->nnz;
}

/* CsrBase::locate, formats.hpp:165-199 (kLinearSearchMax = 30, :35) */
idx_t orc_locate_csr(const orc_pattern* p, idx_t r, idx_t c) {
    idx_t lo = p->row_ptr[r], hi = p->row_ptr[r + 1];
    if (hi - lo <= 30) {
        for (idx_t i = lo; i < hi; ++i) {
            if (p->cols[i] == c) return i;
            if (p->cols[i] > c) break;
        }
        return -1;
    }
    const idx_t end = hi;
    while (lo < hi) {
        const idx_t mid = lo + (hi - lo) / 2;
        if (p->cols[mid] < c) lo = mid + 1;
        else hi = mid;
    }
    return (lo < end && p->cols[lo] == c) ? lo : -1;
}

/* CracBase::locate — the paper's Listing 1 linear block search,
 * formats.hpp:276-290 */
idx_t orc_locate_crac(const idx_t* row_ptr, const idx_t* col_align, idx_t r, idx_t c) {
    idx_t i = row_ptr[r];
    const idx_t row_end = row_ptr[r + 1];
    if (i == row_end) return -1;
    while (i + 2 < row_end && col_align[i + 2] <= c) i += 2;
    const idx_t col_start = col_align[i];
    const idx_t val_start = col_align[i + 1];
    const idx_t val_end = col_align[i + 3];
    if (c >= col_start && c < col_start + (val_end - val_start)) return val_start + (c - col_start);
    return -1;
}

/* encode_runs, dof_map.cpp:69-79 — maximal (start, len) runs; returns the
 * number of runs written to runs[2*k], runs[2*k+1]. */
idx_t orc_encode_runs(const idx_t* flat, idx_t n, idx_t* runs) {
    idx_t nr = 0;
    for (idx_t i = 0; i < n; ++i) {
        if (nr > 0 && runs[2 * (nr - 1)] + runs[2 * (nr - 1) + 1] == flat[i]) {
            runs[2 * (nr - 1) + 1]++;
        } else {
            runs[2 * nr] = flat[i];
            runs[2 * nr + 1] = 1;
            ++nr;
        }
    }
    return nr;
}

/* ------------------------------------------------------------------------ */
/* Colouring                                                                 */
/* ------------------------------------------------------------------------ */

/* greedy_colouring, colouring.cpp:24-75: elements in ascending order, each
 * takes the smallest colour unused by any element sharing a node. */
int orc_greedy_colouring(const idx_t* element_nodes, idx_t n_elements, int npe, idx_t n_nodes,
                         int32_t* colour_of) {
    idx_t *adj_ptr, *adj;
    node_adjacency(element_nodes, n_elements, npe, n_nodes, &adj_ptr, &adj);
    for (idx_t e = 0; e < n_elements; ++e) colour_of[e] = -1;
    int n_colours = 0;
    size_t used_cap = 64;
    char* used = (char*)calloc(used_cap, 1);
    for (idx_t e = 0; e < n_elements; ++e) {
        memset(used, 0, used_cap);
        for (int a = 0; a < npe; ++a) {
            const idx_t v = element_nodes[e * npe + a];
            for (idx_t k = adj_ptr[v]; k < adj_ptr[v + 1]; ++k) {
                const int c = colour_of[adj[k]];
                if (c >= 0) {
                    if ((size_t)c >= used_cap) {
                        size_t nc = used_cap * 2;
                        while ((size_t)c >= nc) nc *= 2;
                        used = (char*)realloc(used, nc);
                        memset(used + used_cap, 0, nc - used_cap);
                        used_cap = nc;
                    }
                    used[c] = 1;
                }
            }
        }
        int colour = 0;
        while ((size_t)colour < used_cap && used[colour]) ++colour;
        colour_of[e] = colour;
        if (colour + 1 > n_colours) n_colours = colour + 1;
    }
    free(used);
    free(adj_ptr);
    free(adj);
    return n_colours;
}

/* ------------------------------------------------------------------------ */
/* Numeric assembly                                                          */
/* ------------------------------------------------------------------------ */

/* scatter_element, assembly.hpp:77-92: G(D(r), D(c)) += K(r, c) with a
 * locate per entry; missing entry -> error naming (element, row, col)
 * (assembly.hpp:65-73). Returns 0, or 2 with err[3] = {e, r, c}. */
static int scatter_element(const orc_pattern* p, const idx_t* dofs, int m, const double* k,
                           double* values, idx_t e, idx_t* err) {
    for (int r = 0; r < m; ++r) {
        const idx_t row = dofs[r];
        if (row < 0 || row >= p->n_rows) {
            if (err) { err[0] = e; err[1] = row; err[2] = dofs[0]; }
            return 2;
        }
        for (int c = 0; c < m; ++c) {
            const idx_t pos = orc_locate_csr(p, row, dofs[c]);
            if (pos < 0) {
                if (err) { err[0] = e; err[1] = row; err[2] = dofs[c]; }
                return 2;
            }
            values[pos] += k[r * m + c];
        }
    }
    return 0;
}

/* assemble_sequential, assembly.hpp:112-118: elements in ascending order —
 * per slot a left fold, starting from the slot's current value, in
 * ascending element id. */
int orc_assemble_sequential(const orc_pattern* p, const idx_t* elem_dofs, idx_t n_elements, int m,
                            const double* K, double* values, idx_t* err) {
    for (idx_t e = 0; e < n_elements; ++e) {
        const int rc = scatter_element(p, elem_dofs + e * m, m, K + e * (idx_t)m * m, values, e, err);
        if (rc) return rc;
    }
    return 0;
}

/* assemble_coloured_vectorized, assembly.hpp:175-195: colours in ascending
 * order, each colour's elements in ascending id; within one colour no slot is
 * touched twice, so per slot the summation order is colour order. The
 * run-wise slice add (scatter_row_runs, :96-107) performs the same scalar
 * additions as scatter_element. */
int orc_assemble_coloured(const orc_pattern* p, const idx_t* elem_dofs, idx_t n_elements, int m,
                          const double* K, const int32_t* colour_of, double* values, idx_t* err) {
    int n_colours = 0;
    for (idx_t e = 0; e < n_elements; ++e)
        if (colour_of[e] + 1 > n_colours) n_colours = colour_of[e] + 1;
    for (int c = 0; c < n_colours; ++c)
        for (idx_t e = 0; e < n_elements; ++e) {
            if (colour_of[e] != c) continue;
            const int rc =
                scatter_element(p, elem_dofs + e * m, m, K + e * (idx_t)m * m, values, e, err);
            if (rc) return rc;
        }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Restricted oracle for sizes the full oracle cannot hold (SURVEY §8c,      */
/* "oracle limits": config 5 has NNZ 4.09e9)                                 */
/* ------------------------------------------------------------------------ */

/* The node -> element inverted index of build_pattern (pattern.cpp:32-48), kept so that
 * row counts and selected rows can be computed from several threads. element_nodes is
 * borrowed (the caller keeps it alive). */
typedef struct {
    const idx_t* en;
    idx_t n_elements, n_nodes;
    int npe;
    idx_t* adj_ptr;
    idx_t* adj;
} orc_adjacency;

orc_adjacency* orc_adjacency_new(const idx_t* element_nodes, idx_t n_elements, int npe, idx_t n_nodes) {
    orc_adjacency* a = (orc_adjacency*)calloc(1, sizeof(orc_adjacency));
    a->en = element_nodes;
    a->n_elements = n_elements;
    a->n_nodes = n_nodes;
    a->npe = npe;
    node_adjacency(element_nodes, n_elements, npe, n_nodes, &a->adj_ptr, &a->adj);
    return a;
}

void orc_adjacency_free(orc_adjacency* a) {
    if (!a) return;
    free(a->adj_ptr);
    free(a->adj);
    free(a);
}

/* sorted distinct neighbour nodes of v (build_pattern's per-node gather + sort/unique,
 * pattern.cpp:71-83, at node level: the DOF list is this list times d). */
static idx_t node_neighbours(const orc_adjacency* a, idx_t v, idx_t* scratch) {
    idx_t len = 0;
    for (idx_t k = a->adj_ptr[v]; k < a->adj_ptr[v + 1]; ++k)
        for (int b = 0; b < a->npe; ++b) scratch[len++] = a->en[a->adj[k] * a->npe + b];
    return sort_unique(scratch, len);
}

static idx_t max_degree(const orc_adjacency* a) {
    idx_t mx = 0;
    for (idx_t v = 0; v < a->n_nodes; ++v)
        if (a->adj_ptr[v + 1] - a->adj_ptr[v] > mx) mx = a->adj_ptr[v + 1] - a->adj_ptr[v];
    return mx;
}

/* Node-level row lengths and CRAC runs of nodes v0 .. v1-1, so the whole int64 CSR and CRAC
 * row pointers follow by scans: row (v,k) has d * count(v) entries (pattern.cpp:85-95) and
 * runs(v) maximal runs of consecutive columns (count_pattern_runs, pattern.cpp:110-120: with
 * node-contiguous DOFs a run of consecutive DOFs is a run of consecutive nodes). */
void orc_node_counts(const orc_adjacency* a, idx_t v0, idx_t v1, idx_t* out, idx_t* runs) {
    idx_t* scratch = (idx_t*)malloc((size_t)(max_degree(a) * a->npe + 1) * sizeof(idx_t));
    for (idx_t v = v0; v < v1; ++v) {
        const idx_t c = node_neighbours(a, v, scratch);
        out[v - v0] = c;
        if (runs) {
            idx_t r = 0;
            for (idx_t i = 0; i < c; ++i)
                if (i == 0 || scratch[i] != scratch[i - 1] + 1) ++r;
            runs[v - v0] = r;
        }
    }
    free(scratch);
}

/* The d rows of each selected node of the assembled matrix with the seeded supplier
 * (orc_kval): sorted column nodes cols[i*max_cols ..] (cnt[i] of them) and values
 * vals[(i*d + k) * max_cols*d + q] of row (v,k), slot q. Per slot the order of
 * assemble_sequential (assembly.hpp:112-118: elements ascending, scatter_element row-major
 * within an element, :77-92) or, with colour_of, of assemble_coloured_vectorized
 * (assembly.hpp:175-195: colours ascending). Returns 0, or 1 if a row has > max_cols nodes. */
int orc_node_rows(const orc_adjacency* a, int d, uint64_t seed, const int32_t* colour_of,
                  const idx_t* nodes, idx_t n_sel, int max_cols, idx_t* cnt, idx_t* cols, double* vals) {
    const int npe = a->npe, m = npe * d;
    const idx_t deg = max_degree(a);
    idx_t* scratch = (idx_t*)malloc((size_t)(deg * npe + 1) * sizeof(idx_t));
    idx_t* elems = (idx_t*)malloc((size_t)(deg + 1) * sizeof(idx_t));
    int rc = 0;
    for (idx_t i = 0; i < n_sel && !rc; ++i) {
        const idx_t v = nodes[i];
        const idx_t c = node_neighbours(a, v, scratch);
        if (c > max_cols) { rc = 1; break; }
        cnt[i] = c;
        memcpy(cols + i * max_cols, scratch, (size_t)c * sizeof(idx_t));
        const idx_t rl = (idx_t)max_cols * d;
        double* vrow = vals + i * d * rl;
        for (idx_t q = 0; q < d * rl; ++q) vrow[q] = 0.0;
        /* incident elements in summation order (ascending id; stable by colour) */
        idx_t ne = 0;
        for (idx_t k = a->adj_ptr[v]; k < a->adj_ptr[v + 1]; ++k)
            if (ne == 0 || elems[ne - 1] != a->adj[k]) elems[ne++] = a->adj[k];
        if (colour_of)
            for (idx_t x = 1; x < ne; ++x) { /* insertion sort by colour, stable */
                const idx_t e = elems[x];
                idx_t y = x;
                while (y > 0 && colour_of[elems[y - 1]] > colour_of[e]) { elems[y] = elems[y - 1]; --y; }
                elems[y] = e;
            }
        for (idx_t x = 0; x < ne; ++x) {
            const idx_t e = elems[x];
            const idx_t* en = a->en + e * npe;
            const uint64_t he = orc_splitmix64(seed + (uint64_t)e);
            for (int ra = 0; ra < npe; ++ra) {
                if (en[ra] != v) continue;
                for (int k = 0; k < d; ++k) {
                    const int r = ra * d + k;
                    for (int cb = 0; cb < npe; ++cb) {
                        /* position of column node en[cb] in the sorted list */
                        idx_t lo = 0, hi = c;
                        while (lo < hi) {
                            const idx_t mid = (lo + hi) / 2;
                            if (scratch[mid] < en[cb]) lo = mid + 1; else hi = mid;
                        }
                        for (int k2 = 0; k2 < d; ++k2) {
                            const int cc = cb * d + k2;
                            const uint64_t lo_ = (uint64_t)(r < cc ? r : cc), hi_ = (uint64_t)(r < cc ? cc : r);
                            const uint64_t h = orc_splitmix64(he ^ ((lo_ << 32) | hi_));
                            vrow[k * rl + lo * d + k2] += (double)(h >> 11) * 0x1p-53 * 2.0 - 1.0;
                        }
                    }
                }
            }
        }
        (void)m;
    }
    free(scratch);
    free(elems);
    return rc;
}
