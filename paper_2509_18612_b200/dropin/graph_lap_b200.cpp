// graph_lap_b200.cpp — Graph::laplacian_apply (graph.hpp:50, graph.cpp:112-122) on the B200.
// The rest of graph.cpp (constructor, components, induced subgraphs, parsing, generators:
// host plumbing off the hot path) is the reference's, compiled with its own
// laplacian_apply renamed out of the way (Makefile: -Dlaplacian_apply=...).
// fp64 CSR-order sums on the device: bit-identical to the reference loop.
#include <string>

#include "liftcut/graph.hpp"
#include "lcb_bridge.hpp"

namespace liftcut {

void Graph::laplacian_apply(std::span<const double> x, std::span<double> y) const {
    if (x.size() != node_count() || y.size() != node_count())
        throw ShapeError("laplacian_apply: expected vectors of length " + std::to_string(node_count()));
    if (node_count() == 0) return;
    const b200::DeviceGraph dg = b200::upload(*this);
    b200::check(lcb_laplacian_apply(dg.get(), x.data(), y.data(), 1, LCB_FP64));
}

}  // namespace liftcut
