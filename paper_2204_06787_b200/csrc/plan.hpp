// plan.hpp — host-side schedule objects and the "schedule compiler".
//
// The reference runs a Schedule step by step through a lock-step Transport
// (allreduce.hpp:51-73, transport.hpp:18-47), merging whole segments at
// every hop.  Everything in that walk except the sign bits themselves is
// data independent: which node merges into which, the contribution counts,
// the coin thresholds, and which (receiver, segment) stream each merge draws
// from.  compile_plan() replays the schedule once on node ids and emits, per
// segment, a merge DAG that the device executes tile by tile with no
// per-hop synchronisation (owner-computes, SURVEY §7 hard part 7).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace marsit_b200 {

struct HostSchedule {
    int topology = 2;  // 0 ring, 1 torus, 2 explicit tables
    uint32_t rows = 0, cols = 0;
    uint32_t workers = 0, segments = 0;
    std::vector<uint8_t> phase;       // [steps]
    std::vector<uint32_t> send_to;    // [steps * workers]
    std::vector<uint32_t> recv_from;
    std::vector<uint32_t> segment;
    uint32_t steps() const { return static_cast<uint32_t>(phase.size()); }
};

// Returns 0 or a marsit_status; *msg receives the reference's message text.
int build_ring(uint32_t m, HostSchedule& out, std::string* msg);
int build_torus(uint32_t rows, uint32_t cols, HostSchedule& out, std::string* msg);
int validate(const HostSchedule& s, std::string* msg);

struct MergeNode {
    uint32_t recv_node = 0, local_node = 0;  // node ids: < workers = leaf (worker id)
    uint32_t receiver = 0;                   // worker whose stream draws the coins
    uint32_t c_recv = 1, c_local = 1;
    int32_t offset_src = -1;                 // previous merge of the same (receiver, segment)
    uint32_t stage = 0;
};

struct SegmentPlan {
    std::vector<MergeNode> merges;  // in schedule (= topological) order
    uint32_t final_node = 0;
    uint32_t final_count = 0;
    bool consensus = true;          // every worker ends on the same node
};

struct BitsTotals {
    std::vector<uint64_t> per_worker;
    uint64_t reduce_bits = 0, gather_bits = 0, total = 0;
};

struct Plan {
    uint32_t workers = 0, segments = 0, n_stages = 0;
    std::vector<SegmentPlan> seg;
    // Payload bits per worker of one round for a given segment length L:
    // every send carries L bits (sign, allreduce.hpp:182) or 32*L (dense, :113).
    std::vector<uint64_t> sends_per_worker;  // [workers]
    uint64_t reduce_sends = 0, gather_sends = 0;
};

Plan compile_plan(const HostSchedule& s);

// Exact coin threshold: next_uniform() < p  <=>  (x >> 11) < ceil(p * 2^53)
// with p = c_r / (c_r + c_l) evaluated in double exactly like merge.hpp:42-43.
uint64_t coin_threshold(uint32_t c_recv, uint32_t c_local);

}  // namespace marsit_b200
