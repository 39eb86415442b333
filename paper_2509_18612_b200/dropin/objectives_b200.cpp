// objectives_b200.cpp — drop-in replacement of proj/src/objectives.cpp behind the unchanged
// header proj/include/liftcut/objectives.hpp.
//
// Device work through the C ABI: cut values (lcb_cut_values: bit-packed edge XOR counts),
// rounding (lcb_round: strict / inclusive thresholds, lifted row sums in column order) and
// every Laplacian product (lcb_laplacian_apply, fp64 CSR-order sums: bit-exact).  The
// scalar reductions over n entries that follow a Laplacian product (x . Lx, the box test
// of a fixed point) run on the host in the reference's order.  Messages and exception
// types are the reference's (objectives.cpp:10-24).
#include <cmath>
#include <string>
#include <vector>

#include "liftcut/objectives.hpp"
#include "lcb_bridge.hpp"

namespace liftcut {

namespace {

void check_len(std::size_t got, std::size_t want, const char* op) {
    if (got == want) return;
    throw ShapeError(std::string(op) + ": expected length " + std::to_string(want) + ", got " +
                     std::to_string(got));
}

void check_box(std::span<const double> x, const char* op) {
    for (const double v : x)
        if (!(std::fabs(v) <= 1.0 + 1e-12)) throw ValidationError(std::string(op) + ": entry outside [-1, 1]");
}

// y = L x on the device for `count` stacked vectors of length n
std::vector<double> laplacian(const Graph& g, const double* x, std::size_t count) {
    const b200::DeviceGraph dg = b200::upload(g);
    std::vector<double> y(count * g.node_count());
    b200::check(lcb_laplacian_apply(dg.get(), x, y.data(), static_cast<int64_t>(count), LCB_FP64));
    return y;
}

double dot_in_order(const double* a, const double* b, std::size_t n) {
    double acc = 0.0;
    for (std::size_t i = 0; i < n; ++i) acc += a[i] * b[i];
    return acc;
}

bool on_corners(std::span<const double> x) {
    for (const double v : x)
        if (v != 1.0 && v != -1.0) return false;
    return true;
}

}  // namespace

std::int64_t cut_value(const Graph& g, std::span<const std::uint8_t> z) {
    check_len(z.size(), g.node_count(), "cut_value");
    const b200::DeviceGraph dg = b200::upload(g);
    int64_t cut = 0;
    b200::check(lcb_cut_values(dg.get(), z.data(), 1, &cut));  // validates entries <= 1
    return cut;
}

double quco_objective(const Graph& g, std::span<const double> x) {
    check_len(x.size(), g.node_count(), "quco_objective");
    check_box(x, "quco_objective");
    const std::vector<double> lx = laplacian(g, x.data(), 1);
    return dot_in_order(x.data(), lx.data(), x.size());
}

double luco_objective(const Graph& g, const DenseState& state, std::int64_t member) {
    check_len(static_cast<std::size_t>(state.nodes), g.node_count(), "luco_objective");
    for (int c = 0; c < state.lift_dim; ++c) check_box(state.column(member, c), "luco_objective");
    // the member's l columns are contiguous: one batched product
    const std::vector<double> lx = laplacian(g, state.member(member).data(), static_cast<std::size_t>(state.lift_dim));
    const std::size_t n = static_cast<std::size_t>(state.nodes);
    double acc = 0.0;
    for (int c = 0; c < state.lift_dim; ++c) {
        const double* col = state.column(member, c).data();
        for (std::size_t v = 0; v < n; ++v) acc += col[v] * lx[static_cast<std::size_t>(c) * n + v];
    }
    return acc;
}

void ascent_direction_unlifted(const Graph& g, std::span<const double> x, std::span<double> out) {
    if (x.size() != g.node_count() || out.size() != g.node_count())
        throw ShapeError("laplacian_apply: expected vectors of length " + std::to_string(g.node_count()));
    const std::vector<double> lx = laplacian(g, x.data(), 1);
    std::copy(lx.begin(), lx.end(), out.begin());
}

void ascent_direction_lifted(const Graph& g, const DenseState& state, std::int64_t member,
                             std::span<double> out) {
    const std::size_t n = static_cast<std::size_t>(state.nodes);
    check_len(n, g.node_count(), "ascent_direction_lifted");
    check_len(out.size(), n * static_cast<std::size_t>(state.lift_dim), "ascent_direction_lifted");
    const std::vector<double> lx = laplacian(g, state.member(member).data(), static_cast<std::size_t>(state.lift_dim));
    std::copy(lx.begin(), lx.end(), out.begin());
}

// objectives.cpp:75-79: an elementwise clamp of a caller-owned host span (used after the
// Gaussian draw on the host side of the API; the device paths clamp inside their kernels)
void project_box(std::span<double> values) {
    for (double& v : values) v = v > 1.0 ? 1.0 : (v < -1.0 ? -1.0 : v);
}

void project_box(DenseState& state) { project_box(std::span<double>(state.values)); }

std::vector<std::uint8_t> round_unlifted(std::span<const double> x) {
    std::vector<std::uint8_t> z(x.size());
    if (x.empty()) return z;
    b200::check(lcb_round(b200::device(), x.data(), static_cast<int64_t>(x.size()), 1, 1, 0, z.data()));
    return z;
}

std::vector<std::uint8_t> round_lifted(const DenseState& state, std::int64_t member) {
    std::vector<std::uint8_t> z(static_cast<std::size_t>(state.nodes));
    b200::check(lcb_round(b200::device(), state.member(member).data(), state.nodes, state.lift_dim, 1, 1, z.data()));
    return z;
}

bool is_maxcut_fixed_point_unlifted(const Graph& g, std::span<const double> x, double alpha) {
    check_len(x.size(), g.node_count(), "is_maxcut_fixed_point_unlifted");
    if (alpha <= 0.0) throw ValidationError("is_maxcut_fixed_point_unlifted: alpha must be > 0");
    if (!on_corners(x)) return false;
    bool constant = true;
    for (const double v : x) constant = constant && v == x[0];
    if (constant) return false;
    const std::vector<double> lx = laplacian(g, x.data(), 1);
    for (std::size_t v = 0; v < x.size(); ++v) {
        const double moved = x[v] + alpha * lx[v];
        const double boxed = moved > 1.0 ? 1.0 : (moved < -1.0 ? -1.0 : moved);
        if (boxed != x[v]) return false;
    }
    return true;
}

bool is_maxcut_fixed_point_lifted(const Graph& g, const DenseState& state, std::int64_t member) {
    check_len(static_cast<std::size_t>(state.nodes), g.node_count(), "is_maxcut_fixed_point_lifted");
    if (!on_corners(state.member(member))) return false;
    // excluded set: every row equal to row 0 (X = e_n c^T)
    for (int c = 0; c < state.lift_dim; ++c) {
        const auto col = state.column(member, c);
        for (std::int64_t v = 1; v < state.nodes; ++v)
            if (col[static_cast<std::size_t>(v)] != col[0]) return true;
    }
    return false;
}

}  // namespace liftcut
