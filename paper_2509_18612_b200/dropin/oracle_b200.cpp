// oracle_b200.cpp — B200 drop-in for the reference's src/oracle.cpp (oracle.hpp:18-28).
//
// brute_force_maxcut   -> lcb_brute_force_maxcut: one device Gray-code scan. The result
//                         is partition-independent, so `workers` has no effect.
// enumerate_lifted_... -> the candidate sign matrices are enumerated on the host. All
//                         candidates with non-identical rows are then checked against one
//                         projected ascent step (alpha = 0.1). The step is one batched
//                         lcb_ascend with T = 1 and mu = 0, in fp64; there v = Lx exactly,
//                         so x + 0.1 * v matches objectives.cpp:65-79 bit for bit.
#include <cstdint>
#include <string>
#include <vector>

#include "lcb_bridge.hpp"
#include "liftcut/objectives.hpp"
#include "liftcut/oracle.hpp"

namespace liftcut {

OracleResult brute_force_maxcut(const Graph& g, unsigned /*workers*/) {
    const b200::DeviceGraph dg = b200::upload(g);
    OracleResult r;
    r.witness.assign(static_cast<size_t>(g.node_count()), 0);
    int64_t optimum = 0, count = 0;
    b200::check(lcb_brute_force_maxcut(dg.get(), 0, &optimum, &count, r.witness.data()));
    r.optimum = optimum;
    r.count_optimal = count;
    return r;
}

std::vector<DenseState> enumerate_lifted_fixed_points(const Graph& g, int lift_dim) {
    const NodeId n = g.node_count();
    if (lift_dim < 1) throw ValidationError("enumerate_lifted_fixed_points: l must be >= 1");
    const int64_t bits = static_cast<int64_t>(n) * lift_dim;
    if (bits > 20)
        throw ValidationError("enumerate_lifted_fixed_points: n * l = " + std::to_string(bits) +
                              " exceeds the enumeration guard (20)");
    // bit k of the mask is entry k of the member's [l][n] block: column k / n, node k % n
    const uint64_t total = 1ull << bits;
    const uint64_t node_mask = (1ull << n) - 1ull;
    std::vector<uint64_t> kept;
    for (uint64_t mask = 0; mask < total; ++mask) {
        bool constant_rows = true;  // every column constant over the nodes
        for (int c = 0; c < lift_dim && constant_rows; ++c) {
            const uint64_t col = (mask >> (static_cast<uint64_t>(c) * n)) & node_mask;
            constant_rows = col == 0 || col == node_mask;
        }
        if (!constant_rows) {
            kept.push_back(mask);
            continue;
        }
        DenseState s(n, lift_dim, 1);
        for (int64_t k = 0; k < bits; ++k) s.values[static_cast<size_t>(k)] = (mask >> k) & 1ull ? 1.0 : -1.0;
        if (cut_value(g, round_lifted(s)) != 0) throw Error("excluded lifted matrix rounds to a nonzero cut");
    }
    std::vector<DenseState> points;
    if (kept.empty()) return points;
    const int64_t B = static_cast<int64_t>(kept.size());
    std::vector<double> before(static_cast<size_t>(B * bits));
    for (int64_t j = 0; j < B; ++j)
        for (int64_t k = 0; k < bits; ++k)
            before[static_cast<size_t>(j * bits + k)] = (kept[static_cast<size_t>(j)] >> k) & 1ull ? 1.0 : -1.0;
    std::vector<double> after = before;
    const b200::DeviceGraph dg = b200::upload(g);
    int64_t ei = -1, em = -1;
    b200::check(lcb_ascend(dg.get(), after.data(), n, lift_dim, B, 0.1, 1, 0.0, 0, LCB_FP64, nullptr, &ei, &em));
    points.reserve(static_cast<size_t>(B));
    for (int64_t j = 0; j < B; ++j) {
        for (int64_t k = 0; k < bits; ++k)
            if (after[static_cast<size_t>(j * bits + k)] != before[static_cast<size_t>(j * bits + k)])
                throw Error("lifted fixed-point candidate moved under a projected ascent step");
        DenseState s(n, lift_dim, 1);
        std::copy(before.begin() + j * bits, before.begin() + (j + 1) * bits, s.values.begin());
        points.push_back(std::move(s));
    }
    return points;
}

}  // namespace liftcut
