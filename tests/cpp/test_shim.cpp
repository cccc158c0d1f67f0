// C++ parity tests through the reference-shaped shim (paper_2012_00585_b200/csrc/fea_gpu.hpp).
// Written like the reference's own doctest suite (test_formats.cpp, test_assembly.cpp,
// acceptance.cpp) so a maintainer can read them side by side; each case cites its origin.
#include "fea_gpu.hpp"

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <set>

using namespace fea::gpu;

static int g_fail = 0, g_pass = 0;
#define CHECK(c)                                                              \
    do {                                                                      \
        if (c) ++g_pass;                                                      \
        else { ++g_fail; std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); } \
    } while (0)
#define CHECK_THROWS_AS(expr, T)                                              \
    do {                                                                      \
        bool thrown_ = false;                                                 \
        try { expr; } catch (const T&) { thrown_ = true; }                    \
        CHECK(thrown_);                                                       \
    } while (0)

// generate_structured (mesh.cpp:62-85) + build_dof_map(p=1, d) element DOFs
static std::vector<ElementDofs> structured_dofs(index_t n, int d, index_t* n_dofs) {
    const index_t nv = n + 1;
    std::vector<ElementDofs> out;
    for (index_t i = 0; i < n; ++i)
        for (index_t j = 0; j < n; ++j) {
            const index_t v0 = i * nv + j;
            const std::array<index_t, 4> el{v0, v0 + 1, v0 + nv + 1, v0 + nv};
            ElementDofs e;
            for (index_t v : el)
                for (int k = 0; k < d; ++k) e.flat.push_back(v * d + k);
            e.runs = encode_runs(e.flat);
            out.push_back(std::move(e));
        }
    *n_dofs = nv * nv * d;
    return out;
}

static SparsityPattern pattern_from_rows(const std::vector<std::vector<index_t>>& rows) {
    SparsityPattern p;
    p.n_rows = static_cast<index_t>(rows.size());
    p.row_ptr.assign(1, 0);
    for (const auto& r : rows) {
        p.cols.insert(p.cols.end(), r.begin(), r.end());
        p.row_ptr.push_back(static_cast<index_t>(p.cols.size()));
    }
    return p;
}

static ElementMatrixSupplier random_supplier(index_t m, std::uint64_t seed) {
    return [m, seed](index_t e) {
        ElementMatrix k{m, std::vector<double>(static_cast<size_t>(m * m))};
        std::uint64_t s = seed ^ (0x9e3779b97f4a7c15ull * static_cast<std::uint64_t>(e + 1));
        for (double& x : k.values) {
            s = s * 6364136223846793005ull + 1442695040888963407ull;
            x = static_cast<double>(s >> 11) * 0x1p-53;
        }
        return k;
    };
}

int main() {
    // test_formats.cpp:31-109 — the 6x6 example: arrays, lookups, values
    {
        const SparsityPattern p = pattern_from_rows(
            {{0, 1}, {0, 1}, {1, 2, 4, 5}, {2, 3, 4}, {3, 4, 5}, {1, 2, 3, 4}});
        const std::vector<double> vals = {1.21, 83.2, 47.1, 5.12, 6.29, 2.37, 8.34, 3.33, 9.24,
                                          10.2, 1.17, 19.2, 13.1, 1.19, 16.4, 15.8, 7.36, 12.2};
        CsrMatrix csr(p);
        CracMatrix crac(p);
        csr.values.v = vals;
        crac.values.v = vals;
        CHECK(crac.n_runs() == 7);
        CHECK((crac.crac_rows() == std::vector<index_t>{0, 2, 4, 8, 10, 12, 14}));
        CHECK(crac.col_align().back() == 18);
        CHECK(csr.locate(2, 5) == std::optional<index_t>(7) && crac.locate(2, 5) == std::optional<index_t>(7));
        CHECK(csr.get(2, 5) == 3.33 && crac.get(2, 5) == 3.33);
        CHECK(crac.locate(5, 1) == std::optional<index_t>(14) && crac.get(5, 1) == 16.4);
        CHECK(!csr.locate(0, 5) && !crac.locate(0, 5) && !crac.locate(2, 0));
    }
    // test_assembly.cpp:69-77 — one element is dense
    {
        index_t nd;
        const auto dofs = structured_dofs(1, 1, &nd);
        const SparsityPattern p = build_pattern(dofs, nd);
        CHECK(p.nnz() == 16);
        CsrMatrix m(p);
        assemble_sequential(m, AssemblyJob{dofs, ones_supplier(4), 1});
        CHECK(std::all_of(m.values.v.begin(), m.values.v.end(), [](double x) { return x == 1.0; }));
    }
    // test_assembly.cpp:79-87 — 2x2 mesh, centre vertex 4 belongs to all four elements
    {
        index_t nd;
        const auto dofs = structured_dofs(2, 1, &nd);
        CsrMatrix m(build_pattern(dofs, nd));
        assemble_sequential(m, AssemblyJob{dofs, ones_supplier(4), 1});
        CHECK(m.get(4, 4) == 4.0);
        CHECK(m.get(0, 0) == 1.0 && m.get(0, 8) == 0.0);
    }
    // test_assembly.cpp:89-99 — assembling twice without reset doubles every value
    {
        index_t nd;
        const auto dofs = structured_dofs(3, 2, &nd);
        CsrMatrix m(build_pattern(dofs, nd, 2));
        const AssemblyJob job{dofs, ones_supplier(8), 1};
        assemble_sequential(m, job);
        const std::vector<double> once = m.values.v;
        assemble_sequential(m, job);
        bool ok = true;
        for (size_t i = 0; i < once.size(); ++i) ok &= m.values.v[i] == 2.0 * once[i];
        CHECK(ok);
        reset_values(m);  // test_assembly.cpp:101-120
        CHECK(values_total(m) == 0.0);
    }
    // test_assembly.cpp:122-141 — missing pattern entry is an AssemblyError naming the element
    {
        index_t nd;
        const auto dofs = structured_dofs(2, 1, &nd);
        const SparsityPattern partial = build_pattern(std::span<const ElementDofs>(dofs).first(1), nd);
        CsrMatrix m(partial);
        bool named = false;
        try {
            assemble_sequential(m, AssemblyJob{dofs, ones_supplier(4), 1});
        } catch (const AssemblyError& e) {
            named = std::string(e.what()).find("element 1") != std::string::npos;
        }
        CHECK(named);
    }
    // The target keeps no element state between assemblies (the reference locates every entry
    // on every call): the same element vector edited in place must be located afresh — a DOF
    // moved outside the pattern is an AssemblyError, a DOF moved inside it lands in its new slot.
    {
        index_t nd;
        auto dofs = structured_dofs(2, 1, &nd);
        const SparsityPattern partial = build_pattern(std::span<const ElementDofs>(dofs).first(1), nd);
        CsrMatrix m(partial);
        std::vector<ElementDofs> first(dofs.begin(), dofs.begin() + 1);
        assemble_sequential(m, AssemblyJob{first, ones_supplier(4), 1});
        CHECK(values_total(m) == 16.0);
        first[0].flat = dofs[1].flat;  // same buffer, same size, different element
        first[0].runs = encode_runs(first[0].flat);
        CHECK_THROWS_AS(assemble_sequential(m, AssemblyJob{first, ones_supplier(4), 1}), AssemblyError);
        CsrMatrix full(build_pattern(dofs, nd));
        std::vector<ElementDofs> one(dofs.begin(), dofs.begin() + 1);
        assemble_sequential(full, AssemblyJob{one, ones_supplier(4), 1});
        one[0].flat = dofs[3].flat;
        one[0].runs = encode_runs(one[0].flat);
        assemble_sequential(full, AssemblyJob{one, ones_supplier(4), 1});
        // the centre node (4) is shared by both elements: 2 contributions on its diagonal
        CHECK(full.get(4, 4) == 2.0 && full.get(0, 0) == 1.0 && full.get(8, 8) == 1.0);
    }
    // test_assembly.cpp:143-184 / acceptance.cpp:180-199 — all methods bitwise equal with ones
    {
        index_t nd;
        const auto dofs = structured_dofs(16, 4, &nd);
        const SparsityPattern p = build_pattern(dofs, nd, 4);
        const AssemblyJob job{dofs, ones_supplier(16), 8};
        CsrMatrix ref(p);
        assemble_sequential(ref, job);
        CHECK(values_total(ref) == 256.0 * 16 * 16);
        CsrAtomicMatrix a(p);
        assemble_atomic(a, job);
        CHECK(a.values.v == ref.values.v);
        CracAtomicMatrix ac(p);
        assemble_atomic(ac, job);
        CHECK(ac.values.v == ref.values.v);
        CracMatrix c(p);
        const Colouring col = greedy_colouring(c, dofs);
        CHECK(col.n_colours == 4);  // acceptance.cpp:167-178
        assemble_coloured_vectorized(c, job, col);
        CHECK(c.values.v == ref.values.v);
        CracMatrix s(p);
        assemble_sequential(s, job);
        CHECK(s.values.v == ref.values.v);
    }
    // test_assembly.cpp:222-255 — random K: atomic within 1e-12, colour and CRAC sequential
    {
        index_t nd;
        const auto dofs = structured_dofs(8, 2, &nd);
        const SparsityPattern p = build_pattern(dofs, nd, 2);
        const auto sup = random_supplier(8, 2026);
        CsrMatrix ref(p);
        assemble_sequential(ref, AssemblyJob{dofs, sup, 1});
        CsrAtomicMatrix a(p);
        assemble_atomic(a, AssemblyJob{dofs, sup, 8});
        bool close = true;
        for (size_t i = 0; i < ref.values.v.size(); ++i) {
            const double x = a.values.v[i], y = ref.values.v[i];
            close &= std::abs(x - y) <= 1e-12 * std::max({std::abs(x), std::abs(y), 1.0});
        }
        CHECK(close);
        CracMatrix crac(p);
        assemble_sequential(crac, AssemblyJob{dofs, sup, 1});
        CHECK(crac.values.v == ref.values.v);  // CSR and CRAC store values in the same order
    }
    // test_assembly.cpp:329-348 — conflicting colourings are rejected
    {
        index_t nd;
        const auto dofs = structured_dofs(2, 1, &nd);
        const Colouring merged = make_colouring(std::vector<int>(4, 0));
        const auto conflict = find_colour_conflict(dofs, merged);
        CHECK(conflict && conflict->find("share dof") != std::string::npos);
        CsrMatrix m(build_pattern(dofs, nd));
        CHECK_THROWS_AS(assemble_coloured_vectorized(m, AssemblyJob{dofs, ones_supplier(4), 1}, merged),
                        AssemblyError);
    }
    // test_pattern.cpp:41-61 — GPU build_pattern equals the naive set oracle
    {
        index_t nd;
        auto dofs = structured_dofs(5, 2, &nd);
        // relabel nodes (permuted_structured analogue): node v -> (7v+3) mod n_nodes
        const index_t nn = nd / 2;
        for (auto& e : dofs) {
            for (auto& x : e.flat) x = ((7 * (x / 2) + 3) % nn) * 2 + x % 2;
            e.runs = encode_runs(e.flat);
        }
        std::set<std::pair<index_t, index_t>> naive;
        for (const auto& e : dofs)
            for (index_t r : e.flat)
                for (index_t c : e.flat) naive.emplace(r, c);
        const SparsityPattern p = build_pattern(dofs, nd, 2);
        std::set<std::pair<index_t, index_t>> got;
        bool ascending = true;
        for (index_t r = 0; r < p.n_rows; ++r)
            for (index_t i = p.row_ptr[r]; i < p.row_ptr[r + 1]; ++i) {
                got.emplace(r, p.cols[i]);
                ascending &= i == p.row_ptr[r] || p.cols[i - 1] < p.cols[i];
            }
        CHECK(ascending && got == naive);
    }
    std::printf("%d checks passed, %d failed\n", g_pass, g_fail);
    return g_fail ? 1 : 0;
}
