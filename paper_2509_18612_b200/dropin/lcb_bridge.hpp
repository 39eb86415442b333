// lcb_bridge.hpp — shared helpers of the C++ drop-in: liftcut::Graph -> lcb_graph,
// C-ABI status -> reference exception types (errors.hpp:9-31).
#pragma once

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "liftcut/errors.hpp"
#include "liftcut/graph.hpp"
#include "liftcut_b200.h"

namespace liftcut::b200 {

inline void check(int status) {
    if (status == LCB_OK) return;
    const std::string msg = lcb_last_error();
    switch (status) {
        case LCB_VALIDATION: throw ValidationError(msg);
        case LCB_SHAPE: throw ShapeError(msg);
        case LCB_NUMERIC: throw NumericError(msg);
        case LCB_PARSE: throw ParseError(msg);
        default: throw Error(msg);
    }
}

inline int precision() {
    const char* e = std::getenv("LIFTCUT_PRECISION");
    return (e && (std::strcmp(e, "fp32") == 0 || std::strcmp(e, "f32") == 0)) ? LCB_FP32 : LCB_FP64;
}

inline int device() {
    const char* e = std::getenv("LIFTCUT_DEVICE");
    return e ? std::atoi(e) : 0;
}

struct GraphDeleter {
    void operator()(lcb_graph* g) const { lcb_graph_destroy(g); }
};
using DeviceGraph = std::unique_ptr<lcb_graph, GraphDeleter>;

// Upload the reference Graph's CSR (graph.hpp:52-57, read through its public
// neighbors() spans) to a device handle.
inline DeviceGraph upload(const Graph& g) {
    const NodeId n = g.node_count();
    std::vector<int64_t> off(static_cast<size_t>(n) + 1, 0);
    std::vector<uint32_t> adj;
    adj.reserve(static_cast<size_t>(2 * g.edge_count()));
    for (NodeId v = 0; v < n; ++v) {
        for (NodeId u : g.neighbors(v)) adj.push_back(u);
        off[v + 1] = static_cast<int64_t>(adj.size());
    }
    lcb_graph* h = nullptr;
    check(lcb_graph_create(n, off.data(), adj.data(), device(), &h));
    return DeviceGraph(h);
}

}  // namespace liftcut::b200
