// ascent_b200.cpp — drop-in replacement of proj/src/ascent.cpp behind the unchanged
// header proj/include/liftcut/ascent.hpp.  The PGA loop runs on the B200 through
// lcb_ascend (fused SpMM + heavy ball + clamp kernels, fp64 bit-exact by default).
#include <cmath>
#include <string>

#include "liftcut/ascent.hpp"
#include "lcb_bridge.hpp"

namespace liftcut {

// ascent.cpp:10-15
void AscentParams::validate() const {
    if (!(alpha > 0.0)) throw ValidationError("ascent: alpha must be > 0");
    if (iterations < 1) throw ValidationError("ascent: iterations must be >= 1");
    if (!(momentum >= 0.0 && momentum < 1.0))
        throw ValidationError("ascent: momentum must lie in [0, 1)");
}

// ascent.cpp:17-30 (host helper over two host states; not on the device path)
std::vector<bool> detect_fixed_point(const DenseState& prev, const DenseState& next, double tol) {
    if (!prev.same_shape(next)) throw ShapeError("detect_fixed_point: shape mismatch");
    std::vector<bool> flags(static_cast<std::size_t>(prev.batch));
    for (std::int64_t j = 0; j < prev.batch; ++j) {
        const auto a = prev.member(j);
        const auto b = next.member(j);
        double worst = 0.0;
        for (std::size_t k = 0; k < a.size(); ++k) worst = std::max(worst, std::fabs(a[k] - b[k]));
        flags[static_cast<std::size_t>(j)] = worst <= tol;
    }
    return flags;
}

// ascent.hpp:33-34 — workers is accepted for API compatibility; the result does not
// depend on it (the device grid replaces the thread pool).
void ascend(const Graph& g, DenseState& state, const AscentParams& params, unsigned /*workers*/,
            const TraceCallback& trace) {
    params.validate();
    if (static_cast<std::size_t>(state.nodes) != g.node_count())
        throw ShapeError("ascend: state row dimension " + std::to_string(state.nodes) +
                         " != node count " + std::to_string(g.node_count()));
    const b200::DeviceGraph dg = b200::upload(g);
    std::vector<double> tr;
    if (trace) tr.assign(static_cast<std::size_t>(params.iterations) * static_cast<std::size_t>(state.batch), 0.0);
    int64_t ei = -1, ej = -1;
    b200::check(lcb_ascend(dg.get(), state.values.data(), state.nodes, state.lift_dim, state.batch,
                           params.alpha, params.iterations, params.momentum, params.early_exit ? 1 : 0,
                           b200::precision(), trace ? tr.data() : nullptr, &ei, &ej));
    if (trace)  // member-major, as with workers=1
        for (std::int64_t j = 0; j < state.batch; ++j)
            for (std::int64_t it = 0; it < params.iterations; ++it)
                trace(it, j, tr[static_cast<std::size_t>(it * state.batch + j)]);
}

}  // namespace liftcut
