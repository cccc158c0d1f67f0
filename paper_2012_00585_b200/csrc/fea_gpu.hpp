// fea_gpu.hpp — C++ host side of the B200 assembly library, mirroring the reference's
// assembly API (proj/include/fea/{types,dof_map,pattern,formats,colouring,assembly}.hpp)
// on top of the C ABI in include/fea_gpu.h. Header-only; link with libfea_gpu.so.
//
// Drop-in surface (same names, argument meaning and error behaviour):
//   index_t, AssemblyError                     types.hpp:27-33
//   ElementDofs, encode_runs, ElementMatrix     dof_map.hpp:62-87, dof_map.cpp:69-79
//   ElementMatrixSupplier, ones_supplier        assembly.hpp:34-43
//   AssemblyJob                                 assembly.hpp:48-52
//   SparsityPattern                             pattern.hpp:29-35
//   CsrMatrix / CracMatrix (+ Atomic aliases)   formats.hpp:146-346 (locate, get, values.v)
//   Colouring, find_colour_conflict             colouring.hpp:35-50
//   assemble_sequential / assemble_atomic /
//   assemble_coloured_vectorized                assembly.hpp:112-195
//   reset_values, values_total                  formats.hpp:351-363
//   build_pattern (GPU symbolic phase), greedy_colouring (plan-side restatement)
//
// Semantics kept from the reference: targets own host-visible `values.v`; assembly ADDS into
// the current values (no implicit reset); calls are synchronous; a coefficient missing from the
// pattern throws AssemblyError naming (element, row, col); an invalid colouring throws
// AssemblyError("invalid colouring: ..."). assemble_sequential runs the deterministic
// sort-by-slot route and is bit-identical to the reference's sequential loop;
// assemble_coloured_vectorized is bit-identical under the same colouring; assemble_atomic
// uses fp64 atomics (within 1e-12 relative). The spin-lock targets (SpinRows) have no GPU
// counterpart (per-row locks are replaced by the deterministic route).
//
// This layer favours reference compatibility (values mirrored on the host around every call,
// supplier called per element); the hot-path API without host round trips is the C ABI
// (device K, device values, stream-ordered).
#pragma once

#include <cstdint>
#include <cstring>
#include <functional>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/fea_gpu.h"

namespace fea::gpu {

using index_t = std::int64_t;

struct AssemblyError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

namespace detail {
inline void check(fea_status s) {
    if (s == FEA_OK) return;
    const std::string msg = fea_last_error();
    if (s == FEA_ERR_MISSING_ENTRY || s == FEA_ERR_INVALID_COLOURING) throw AssemblyError(msg);
    if (s == FEA_ERR_OOM) throw std::bad_alloc();
    if (s == FEA_ERR_INVALID) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}
}  // namespace detail

struct ElementDofs {
    std::vector<index_t> flat;
    std::vector<std::pair<index_t, index_t>> runs;
};

inline std::vector<std::pair<index_t, index_t>> encode_runs(std::span<const index_t> flat) {
    std::vector<std::pair<index_t, index_t>> runs;
    for (const index_t v : flat) {
        if (!runs.empty() && runs.back().first + runs.back().second == v) ++runs.back().second;
        else runs.emplace_back(v, 1);
    }
    return runs;
}

struct ElementMatrix {
    index_t order = 0;
    std::vector<double> values;
    static ElementMatrix ones(index_t order) {
        return {order, std::vector<double>(static_cast<size_t>(order * order), 1.0)};
    }
    double& at(index_t r, index_t c) { return values[r * order + c]; }
    double at(index_t r, index_t c) const { return values[r * order + c]; }
};

using ElementMatrixSupplier = std::function<ElementMatrix(index_t element)>;

inline ElementMatrixSupplier ones_supplier(index_t m) {
    return [m](index_t) { return ElementMatrix::ones(m); };
}

struct AssemblyJob {
    std::span<const ElementDofs> elements;
    ElementMatrixSupplier element_matrix;
    int thread_count = 1;  // accepted for source compatibility; the GPU ignores it
};

struct SparsityPattern {
    index_t n_rows = 0;
    std::vector<index_t> row_ptr{0};
    std::vector<index_t> cols;
    index_t nnz() const { return static_cast<index_t>(cols.size()); }
};

struct Colouring {
    std::vector<int> colour_of;
    std::vector<std::vector<index_t>> colour_classes;
    int n_colours = 0;
};

struct HostValues {
    std::vector<double> v;
};

namespace detail {
inline std::vector<index_t> flatten(std::span<const ElementDofs> els, int32_t& m) {
    m = els.empty() ? 1 : static_cast<int32_t>(els[0].flat.size());
    std::vector<index_t> out;
    out.reserve(els.size() * static_cast<size_t>(m));
    for (const auto& e : els) {
        if (static_cast<int32_t>(e.flat.size()) != m)
            throw std::invalid_argument("all elements must have the same number of DOFs");
        out.insert(out.end(), e.flat.begin(), e.flat.end());
    }
    return out;
}
}  // namespace detail

// A GPU-assembled target over a fixed pattern. The plan (slot map) is built on first use
// with a job's elements and reused while the same element span is assembled.
class GpuMatrix {
public:
    HostValues values;

    explicit GpuMatrix(const SparsityPattern& p, int format, int device = 0)
        : pattern_(p), format_(format), device_(device) {
        values.v.assign(static_cast<size_t>(p.nnz()), 0.0);
        if (format_ == FEA_FORMAT_CRAC) build_crac();
    }
    GpuMatrix(const GpuMatrix&) = delete;
    GpuMatrix& operator=(const GpuMatrix&) = delete;
    ~GpuMatrix() {
        if (plan_) fea_plan_destroy(plan_);
    }

    index_t n_rows() const { return pattern_.n_rows; }
    index_t nnz() const { return pattern_.nnz(); }
    const SparsityPattern& pattern() const { return pattern_; }
    int device() const { return device_; }

    // CsrBase::locate / CracBase::locate (formats.hpp:165-199, :276-290) on the host arrays
    std::optional<index_t> locate(index_t r, index_t c) const {
        if (format_ == FEA_FORMAT_CRAC) {
            index_t i = crac_ptr_[r];
            const index_t end = crac_ptr_[r + 1];
            if (i == end) return std::nullopt;
            while (i + 2 < end && col_align_[i + 2] <= c) i += 2;
            const index_t cs = col_align_[i], vs = col_align_[i + 1], ve = col_align_[i + 3];
            if (c >= cs && c < cs + (ve - vs)) return vs + (c - cs);
            return std::nullopt;
        }
        index_t lo = pattern_.row_ptr[r], hi = pattern_.row_ptr[r + 1];
        const index_t end = hi;
        while (lo < hi) {
            const index_t mid = lo + (hi - lo) / 2;
            if (pattern_.cols[mid] < c) lo = mid + 1;
            else hi = mid;
        }
        if (lo < end && pattern_.cols[lo] == c) return lo;
        return std::nullopt;
    }
    double get(index_t r, index_t c) const {
        const auto pos = locate(r, c);
        return pos ? values.v[*pos] : 0.0;
    }

    // plan for this element set, cached by CONTENT: the reference keeps no element state and
    // locates every entry on every assembly, so a job whose DOFs changed (edited in place, or
    // a reused buffer) must not run on the old slot map. Flattening is O(E*m), against the
    // O(E*m^2) supplier loop of every assembly.
    fea_plan* plan_for(std::span<const ElementDofs> els) {
        int32_t m = 1;
        std::vector<index_t> flat = detail::flatten(els, m);
        if (plan_ && m == m_ && flat == plan_flat_) return plan_;
        if (plan_) fea_plan_destroy(plan_);
        plan_ = nullptr;
        plan_flat_.clear();
        fea_plan* p = nullptr;
        const bool crac = format_ == FEA_FORMAT_CRAC;
        detail::check(fea_plan_create_with_pattern(
            device_, flat.data(), static_cast<int64_t>(els.size()), m, pattern_.n_rows, format_,
            crac ? crac_ptr_.data() : pattern_.row_ptr.data(),
            crac ? col_align_.data() : pattern_.cols.data(), &p));
        plan_ = p;
        plan_flat_ = std::move(flat);
        m_ = m;
        return plan_;
    }

    // One numeric assembly: values.v += assembled (host values mirrored to/from the device).
    void run(const AssemblyJob& job, fea_strategy strategy, const Colouring* colouring) {
        fea_plan* p = plan_for(job.elements);
        const int64_t E = static_cast<int64_t>(job.elements.size());
        const size_t mm = static_cast<size_t>(m_) * m_;
        std::vector<double> K(static_cast<size_t>(E) * mm);
        for (int64_t e = 0; e < E; ++e) {  // the supplier, called once per element per assembly
            const ElementMatrix k = job.element_matrix(e);
            if (k.values.size() != mm) throw std::invalid_argument("element matrix has the wrong order");
            std::memcpy(K.data() + e * mm, k.values.data(), mm * sizeof(double));
        }
        if (colouring) {
            std::vector<int32_t> col(colouring->colour_of.begin(), colouring->colour_of.end());
            detail::check(fea_plan_set_colouring(p, col.data()));
        }
        // fea_assemble_host: K host->device, values host->device (accumulate), assemble,
        // values device->host; synchronous like the reference call
        detail::check(fea_assemble_host(p, K.data(), strategy, values.v.data(), FEA_ACCUMULATE, nullptr));
    }

    const std::vector<index_t>& crac_rows() const { return crac_ptr_; }
    const std::vector<index_t>& col_align() const { return col_align_; }

protected:
    void build_crac() {  // build_crac_arrays, formats.cpp:21-41 (host)
        crac_ptr_.clear();
        col_align_.clear();
        for (index_t r = 0; r < pattern_.n_rows; ++r) {
            crac_ptr_.push_back(static_cast<index_t>(col_align_.size()));
            for (index_t i = pattern_.row_ptr[r]; i < pattern_.row_ptr[r + 1]; ++i)
                if (i == pattern_.row_ptr[r] || pattern_.cols[i] != pattern_.cols[i - 1] + 1) {
                    col_align_.push_back(pattern_.cols[i]);
                    col_align_.push_back(i);
                }
        }
        crac_ptr_.push_back(static_cast<index_t>(col_align_.size()));
        col_align_.push_back(0);
        col_align_.push_back(pattern_.nnz());
    }

    SparsityPattern pattern_;
    int format_;
    int device_;
    std::vector<index_t> crac_ptr_, col_align_;
    fea_plan* plan_ = nullptr;
    std::vector<index_t> plan_flat_;  // the DOFs the cached plan was built for
    int32_t m_ = 1;
};

struct CsrMatrix : GpuMatrix {
    explicit CsrMatrix(const SparsityPattern& p, int device = 0) : GpuMatrix(p, FEA_FORMAT_CSR, device) {}
    const std::vector<index_t>& cols() const { return pattern_.cols; }
    const std::vector<index_t>& row_ptr() const { return pattern_.row_ptr; }
};
struct CracMatrix : GpuMatrix {
    explicit CracMatrix(const SparsityPattern& p, int device = 0) : GpuMatrix(p, FEA_FORMAT_CRAC, device) {}
    index_t n_runs() const { return (static_cast<index_t>(col_align_.size()) - 2) / 2; }
};
// On the GPU one target type serves every strategy.
using CsrAtomicMatrix = CsrMatrix;
using CracAtomicMatrix = CracMatrix;

inline CsrMatrix csr_from_pattern(const SparsityPattern& p) { return CsrMatrix(p); }

inline void reset_values(GpuMatrix& m) { std::fill(m.values.v.begin(), m.values.v.end(), 0.0); }

inline double values_total(const GpuMatrix& m) {
    double s = 0.0;
    for (const double x : m.values.v) s += x;
    return s;
}

// --- symbolic phase on the GPU (build_pattern, pattern.cpp:24-108) ----------------------
inline SparsityPattern build_pattern(std::span<const ElementDofs> elements, index_t n_rows,
                                     int dofs_per_node = 1, int device = 0) {
    int32_t m = 1;
    const std::vector<index_t> flat = detail::flatten(elements, m);
    fea_plan* p = nullptr;
    detail::check(fea_plan_create(device, flat.data(), static_cast<int64_t>(elements.size()), m,
                                  n_rows, dofs_per_node, 0, n_rows, 0u, &p));
    std::unique_ptr<fea_plan, void (*)(fea_plan*)> guard(p, fea_plan_destroy);
    int64_t rows = 0, nnz = 0, runs = 0, ne = 0;
    detail::check(fea_plan_sizes(p, &rows, &nnz, &runs, &ne));
    SparsityPattern out;
    out.n_rows = rows;
    out.row_ptr.assign(static_cast<size_t>(rows) + 1, 0);
    out.cols.assign(static_cast<size_t>(nnz), 0);
    detail::check(fea_plan_copy_csr(p, out.row_ptr.data(), out.cols.data()));
    return out;
}

// --- colouring (colouring.hpp) ------------------------------------------------------------
inline std::optional<std::string> find_colour_conflict(std::span<const ElementDofs> elements,
                                                       const Colouring& colouring) {
    index_t max_dof = -1;
    for (const auto& e : elements)
        for (const index_t d : e.flat) max_dof = std::max(max_dof, d);
    std::vector<index_t> owner(static_cast<size_t>(max_dof) + 1, -1);
    for (const auto& cls : colouring.colour_classes) {
        for (const index_t e : cls)
            for (const index_t d : elements[e].flat) {
                if (owner[d] >= 0)
                    return "elements " + std::to_string(owner[d]) + " and " + std::to_string(e) +
                           " share dof " + std::to_string(d) + " within one colour";
                owner[d] = e;
            }
        for (const index_t e : cls)
            for (const index_t d : elements[e].flat) owner[d] = -1;
    }
    return std::nullopt;
}

inline Colouring make_colouring(std::vector<int> colour_of) {
    Colouring c;
    c.colour_of = std::move(colour_of);
    for (const int x : c.colour_of) c.n_colours = std::max(c.n_colours, x + 1);
    c.colour_classes.resize(static_cast<size_t>(c.n_colours));
    for (size_t e = 0; e < c.colour_of.size(); ++e)
        c.colour_classes[c.colour_of[e]].push_back(static_cast<index_t>(e));
    return c;
}

// greedy_colouring (colouring.cpp:24-75), computed by the library on the plan's elements.
inline Colouring greedy_colouring(GpuMatrix& target, std::span<const ElementDofs> elements) {
    fea_plan* p = target.plan_for(elements);
    std::vector<int32_t> col(elements.size());
    int32_t nc = 0;
    detail::check(fea_plan_greedy_colouring(p, col.data(), &nc));
    return make_colouring(std::vector<int>(col.begin(), col.end()));
}

// --- the assembly algorithms (assembly.hpp:112-195) ---------------------------------------
inline void assemble_sequential(GpuMatrix& target, const AssemblyJob& job) {
    target.run(job, FEA_DET_SORTED, nullptr);
}
inline void assemble_atomic(GpuMatrix& target, const AssemblyJob& job) {
    target.run(job, FEA_ATOMIC, nullptr);
}
inline void assemble_coloured_vectorized(GpuMatrix& target, const AssemblyJob& job,
                                         const Colouring& colouring) {
    target.run(job, FEA_DET_COLOUR, &colouring);
}

}  // namespace fea::gpu
