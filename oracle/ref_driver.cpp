// TEST INFRASTRUCTURE — not product code.
//
// extern "C" driver over the UNMODIFIED reference library (arXiv 2012.00585
// artefact, /root/reference/proj), compiled from its own sources by
// oracle/Makefile into oracle/_ref/libfea_ref.so. Only tests/, the
// __graft_entry__ smoke check and bench.py's CPU-baseline / --impl reference
// legs may load it. It drives the reference API exactly as SURVEY.md §8c
// prescribes for the 3D BASELINE meshes:
//   * a hand-filled fea::DofMap (dof_map.hpp:34-60) whose element node lists
//     are padded to (p+1)^2 entries by repeating the last node, so that
//     fea::build_pattern (pattern.cpp:24-108, built with NDEBUG) sees the true
//     node sets (duplicates vanish in its sort/unique, pattern.cpp:81-82);
//   * fea::ElementDofs built from the TRUE flat DOF arrays with
//     fea::encode_runs (dof_map.cpp:69-79);
//   * an ElementMatrixSupplier (assembly.hpp:37) that copies each element's
//     m*m block out of one materialized, seeded K buffer.
#include "fea/assembly.hpp"
#include "fea/bench.hpp"
#include "fea/colouring.hpp"
#include "fea/dof_map.hpp"
#include "fea/formats.hpp"
#include "fea/parallel.hpp"
#include "fea/pattern.hpp"

#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

using fea::index_t;

namespace {

thread_local std::string g_err;

struct RefProblem {
    fea::DofMap map;                     // padded node lists
    std::vector<fea::ElementDofs> dofs;  // true flat DOFs + runs
    fea::SparsityPattern pattern;
    bool have_pattern = false;
    int m = 0;
};

int pad_order(int npe) {
    int p = 1;
    while ((p + 1) * (p + 1) < npe) ++p;
    return p;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_hardware_threads() { return fea::default_thread_count(); }

// element_nodes: E x npe node ids; d DOFs per node, node v carries v*d+k.
void* ref_problem_new(const int64_t* element_nodes, int64_t n_elements, int npe, int64_t n_nodes,
                      int d, int build_pattern) {
    try {
        auto pr = std::make_unique<RefProblem>();
        const int p = pad_order(npe);
        const int npad = (p + 1) * (p + 1);
        pr->map.p = p;
        pr->map.d = d;
        pr->map.n_vertices = n_nodes;
        pr->map.n_edges = 0;
        pr->map.n_elements = n_elements;
        pr->map.n_nodes = n_nodes;
        pr->map.n_dofs = n_nodes * d;
        pr->map.element_nodes.resize(static_cast<size_t>(n_elements) * npad);
        pr->m = npe * d;
        pr->dofs.resize(static_cast<size_t>(n_elements));
        for (int64_t e = 0; e < n_elements; ++e) {
            const int64_t* src = element_nodes + e * npe;
            index_t* dst = pr->map.element_nodes.data() + e * npad;
            for (int a = 0; a < npad; ++a) dst[a] = src[a < npe ? a : npe - 1];
            auto& ed = pr->dofs[e];
            ed.flat.resize(static_cast<size_t>(npe) * d);
            for (int a = 0; a < npe; ++a)
                for (int k = 0; k < d; ++k) ed.flat[a * d + k] = src[a] * d + k;
            ed.runs = fea::encode_runs(ed.flat);
        }
        if (build_pattern) {
            pr->pattern = fea::build_pattern(pr->map);
            pr->have_pattern = true;
        }
        return pr.release();
    } catch (const std::exception& ex) {
        g_err = ex.what();
        return nullptr;
    }
}

// Same, but from raw flat DOF arrays (E x m) with an explicit pattern
// (row_ptr[n_rows+1], cols[nnz]) — used for external / missing-entry cases.
void* ref_problem_from_pattern(const int64_t* elem_dofs, int64_t n_elements, int m, int64_t n_rows,
                               const int64_t* row_ptr, const int64_t* cols) {
    try {
        auto pr = std::make_unique<RefProblem>();
        pr->m = m;
        pr->map.n_elements = n_elements;
        pr->map.n_dofs = n_rows;
        pr->dofs.resize(static_cast<size_t>(n_elements));
        for (int64_t e = 0; e < n_elements; ++e) {
            auto& ed = pr->dofs[e];
            ed.flat.assign(elem_dofs + e * m, elem_dofs + (e + 1) * m);
            ed.runs = fea::encode_runs(ed.flat);
        }
        pr->pattern.n_rows = n_rows;
        pr->pattern.row_ptr.assign(row_ptr, row_ptr + n_rows + 1);
        pr->pattern.cols.assign(cols, cols + row_ptr[n_rows]);
        pr->have_pattern = true;
        return pr.release();
    } catch (const std::exception& ex) {
        g_err = ex.what();
        return nullptr;
    }
}

void ref_problem_free(void* h) { delete static_cast<RefProblem*>(h); }

void ref_pattern_sizes(void* h, int64_t* n_rows, int64_t* nnz, int64_t* n_runs) {
    auto* pr = static_cast<RefProblem*>(h);
    *n_rows = pr->pattern.n_rows;
    *nnz = pr->pattern.nnz();
    *n_runs = fea::count_pattern_runs(pr->pattern);
}

void ref_pattern_copy(void* h, int64_t* row_ptr, int64_t* cols) {
    auto* pr = static_cast<RefProblem*>(h);
    std::memcpy(row_ptr, pr->pattern.row_ptr.data(), pr->pattern.row_ptr.size() * 8);
    std::memcpy(cols, pr->pattern.cols.data(), pr->pattern.cols.size() * 8);
}

// CRAC arrays as the reference CracMatrix constructor builds them
// (formats.cpp:21-41): row_ptr[n_rows+1] in col_align entry units,
// col_align[2*runs+2].
void ref_crac_copy(void* h, int64_t* row_ptr, int64_t* col_align) {
    auto* pr = static_cast<RefProblem*>(h);
    const fea::CracMatrix crac(pr->pattern);
    std::memcpy(row_ptr, crac.rows.ptr.data(), crac.rows.ptr.size() * 8);
    std::memcpy(col_align, crac.col_align.data(), crac.col_align.size() * 8);
}

// Greedy colouring (colouring.cpp:24-75) on the padded map.
int ref_greedy_colouring(void* h, int32_t* colour_of) {
    auto* pr = static_cast<RefProblem*>(h);
    const fea::Colouring c = fea::greedy_colouring(pr->map);
    for (size_t e = 0; e < c.colour_of.size(); ++e) colour_of[e] = c.colour_of[e];
    return c.n_colours;
}

// Lookups through the reference formats (Listing 1 for CRAC, formats.hpp:276).
int64_t ref_locate(void* h, int format, int64_t r, int64_t c) {
    auto* pr = static_cast<RefProblem*>(h);
    std::optional<index_t> pos;
    if (format == 0) {
        const fea::CsrMatrix csr(pr->pattern);
        pos = csr.locate(r, c);
    } else {
        const fea::CracMatrix crac(pr->pattern);
        pos = crac.locate(r, c);
    }
    return pos ? *pos : -1;
}

}  // extern "C"

namespace {

fea::Colouring colouring_from(const int32_t* colour_of, int64_t n_elements) {
    fea::Colouring c;
    c.colour_of.assign(colour_of, colour_of + n_elements);
    int nc = 0;
    for (int64_t e = 0; e < n_elements; ++e) nc = std::max(nc, colour_of[e] + 1);
    c.n_colours = nc;
    c.colour_classes.resize(nc);
    for (int64_t e = 0; e < n_elements; ++e) c.colour_classes[colour_of[e]].push_back(e);
    return c;
}

template <class M>
void copy_out(const M& t, double* values) {
    std::memcpy(values, t.values.v.data(), t.values.v.size() * 8);
}

// method: 0 seq, 1 atomic, 2 spin, 3 spin-vec, 4 colour-vec (bench.hpp:32)
// format: 0 csr, 1 crac.   n_runs == 0: one assembly into *values (which is
// the initial content, so accumulation semantics are observable).
// n_runs > 0: time_assembly (bench.hpp:98-113) and write t_micros[n_runs].
template <class Csr, class Crac, class Fn>
int dispatch(RefProblem* pr, int format, double* values, int n_runs, double* t_micros, Fn&& fn) {
    auto run = [&](auto& target) {
        if (values) std::memcpy(target.values.v.data(), values, target.values.v.size() * 8);
        if (n_runs > 0) {
            auto ts = fea::time_assembly(target, [&] { fn(target); }, n_runs);
            for (int i = 0; i < n_runs; ++i) t_micros[i] = ts[i];
        } else {
            fn(target);
        }
        if (values) copy_out(target, values);
    };
    if (format == 0) {
        Csr t(pr->pattern);
        run(t);
    } else {
        Crac t(pr->pattern);
        run(t);
    }
    return 0;
}

}  // namespace

extern "C" int ref_assemble(void* h, const double* K, int method, int format, int threads,
                            const int32_t* colour_of, double* values, int n_runs,
                            double* t_micros) {
    auto* pr = static_cast<RefProblem*>(h);
    const int64_t m = pr->m;
    fea::ElementMatrixSupplier supplier = [K, m](index_t e) {
        fea::ElementMatrix k;
        k.order = m;
        k.values.assign(K + e * m * m, K + (e + 1) * m * m);
        return k;
    };
    const fea::AssemblyJob job{pr->dofs, supplier, threads};
    try {
        switch (method) {
            case 0:
                return dispatch<fea::CsrMatrix, fea::CracMatrix>(
                    pr, format, values, n_runs, t_micros,
                    [&](auto& g) { fea::assemble_sequential(g, job); });
            case 1:
                return dispatch<fea::CsrAtomicMatrix, fea::CracAtomicMatrix>(
                    pr, format, values, n_runs, t_micros,
                    [&](auto& g) { fea::assemble_atomic(g, job); });
            case 2:
                return dispatch<fea::CsrSpinMatrix, fea::CracSpinMatrix>(
                    pr, format, values, n_runs, t_micros,
                    [&](auto& g) { fea::assemble_spin(g, job); });
            case 3:
                return dispatch<fea::CsrSpinMatrix, fea::CracSpinMatrix>(
                    pr, format, values, n_runs, t_micros,
                    [&](auto& g) { fea::assemble_spin_vectorized(g, job); });
            case 4: {
                if (!colour_of) {
                    g_err = "colour-vec needs a colouring";
                    return 1;
                }
                const fea::Colouring col = colouring_from(colour_of, pr->map.n_elements);
                return dispatch<fea::CsrMatrix, fea::CracMatrix>(
                    pr, format, values, n_runs, t_micros,
                    [&](auto& g) { fea::assemble_coloured_vectorized(g, job, col); });
            }
            default:
                g_err = "unknown method";
                return 1;
        }
    } catch (const fea::AssemblyError& ex) {
        g_err = ex.what();
        return 2;
    } catch (const std::exception& ex) {
        g_err = ex.what();
        return 3;
    }
}

// The reference's own 2D meshes and DOF numbering (mesh.cpp:62-85, dof_map.cpp:24-67):
// element node lists of build_dof_map(generate_structured(n), p, d). Call with
// out == nullptr to get the sizes.
extern "C" int ref_structured_element_nodes(int64_t n, int p, int d, int64_t* out,
                                            int64_t* n_elements, int64_t* npe, int64_t* n_nodes) {
    try {
        const fea::DofMap map = fea::build_dof_map(fea::generate_structured(n), p, d);
        *n_elements = map.n_elements;
        *npe = map.nodes_per_element();
        *n_nodes = map.n_nodes;
        if (out) std::memcpy(out, map.element_nodes.data(), map.element_nodes.size() * 8);
        return 0;
    } catch (const std::exception& ex) {
        g_err = ex.what();
        return 1;
    }
}

// speed_factor / storage_factor (bench.cpp:93-113) for the golden arithmetic checks.
extern "C" double ref_speed_factor(double t_seq, double t_method) {
    return fea::speed_factor(t_seq, t_method);
}
