// Drop-in parse_edge_list / load_graph_file (graph.hpp:63-65, graph.cpp:136-183): the
// Gset text is parsed on the device (lcb_graph_parse: line-parallel parse, the
// reference's line numbers / messages / exception types, the device Graph(n, edges)
// build); the host Graph comes back from the device CSR.  The reference's own parse
// tests (test_graph.cpp:55-100) run against this.
#include <fstream>
#include <iterator>
#include <string>
#include <utility>
#include <vector>

#include "lcb_bridge.hpp"
#include "liftcut/log.hpp"

namespace liftcut {

namespace {

Graph parse_on_device(const std::string& text) {
    lcb_graph* h = nullptr;
    int weights = 0;
    b200::check(lcb_graph_parse(text.data(), static_cast<int64_t>(text.size()), b200::device(), &h, &weights));
    uint32_t n = 0;
    int64_t m = 0;
    lcb_graph_info(h, &n, &m, nullptr);
    std::vector<int64_t> off(static_cast<size_t>(n) + 1);
    std::vector<uint32_t> adj(static_cast<size_t>(2 * m));
    const int st = lcb_graph_csr(h, off.data(), adj.data());
    lcb_graph_destroy(h);
    b200::check(st);
    if (weights) warn("edge weights present in input are ignored (unweighted MaxCut)");
    std::vector<std::pair<NodeId, NodeId>> edges;
    edges.reserve(static_cast<size_t>(m));
    for (uint32_t u = 0; u < n; ++u)
        for (int64_t k = off[u]; k < off[u + 1]; ++k)
            if (u < adj[static_cast<size_t>(k)]) edges.emplace_back(u, adj[static_cast<size_t>(k)]);
    return Graph(static_cast<NodeId>(n), std::move(edges));
}

}  // namespace

Graph parse_edge_list(std::istream& in) {
    const std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    return parse_on_device(text);
}

Graph parse_edge_list(const std::string& text) { return parse_on_device(text); }

Graph load_graph_file(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw ParseError("cannot open graph file: " + path);
    return parse_edge_list(in);
}

}  // namespace liftcut
