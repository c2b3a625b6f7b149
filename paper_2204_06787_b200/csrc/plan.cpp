// plan.cpp — schedule builders, validation and the schedule compiler.
#include "plan.hpp"

#include <algorithm>
#include <array>
#include <cmath>

#include "../../include/marsit_b200.h"

namespace marsit_b200 {
namespace {

inline uint32_t wrap(int64_t x, uint32_t m) {
    const int64_t r = x % static_cast<int64_t>(m);
    return static_cast<uint32_t>(r < 0 ? r + m : r);
}

// Append one lock step; `entry(w)` returns {send_to, recv_from, segment}.
template <class F>
void push_step(HostSchedule& s, marsit_phase ph, F&& entry) {
    s.phase.push_back(static_cast<uint8_t>(ph));
    for (uint32_t w = 0; w < s.workers; ++w) {
        const auto e = entry(w);
        s.send_to.push_back(e[0]);
        s.recv_from.push_back(e[1]);
        s.segment.push_back(e[2]);
    }
}

}  // namespace

// Ring over m workers (schedule.hpp:57-94): a reduce-scatter of m-1 steps in
// which worker w forwards segment (w - k) to its right neighbour, then an
// all-gather of m-1 steps forwarding segment (w + 1 - k).
int build_ring(uint32_t m, HostSchedule& out, std::string* msg) {
    if (m < 2) {
        if (msg) *msg = "build_ring_schedule: need at least 2 workers";
        return MARSIT_EPARAM;
    }
    out = HostSchedule{};
    out.topology = 0;
    out.workers = out.segments = m;
    for (int ph = 0; ph < 2; ++ph)
        for (uint32_t k = 0; k + 1 < m; ++k)
            push_step(out, ph ? MARSIT_GATHER : MARSIT_REDUCE, [&](uint32_t w) {
                const int64_t shift = ph ? 1 : 0;
                return std::array<uint32_t, 3>{wrap(int64_t(w) + 1, m), wrap(int64_t(w) - 1, m),
                                               wrap(int64_t(w) + shift - int64_t(k), m)};
            });
    return validate(out, msg);
}

// rows x cols torus (schedule.hpp:96-196), worker id = r*cols + c, segment
// id = super*rows + q.  Stage 1: row reduce-scatter of super-segments, one
// segment per step; stage 2: column reduce-scatter then column all-gather of
// the owned super-segment; stage 3: row all-gather.
int build_torus(uint32_t rows, uint32_t cols, HostSchedule& out, std::string* msg) {
    if (rows < 2 || cols < 2) {
        if (msg) *msg = "build_torus_schedule: grid must be at least 2x2";
        return MARSIT_EPARAM;
    }
    out = HostSchedule{};
    out.topology = 1;
    out.rows = rows;
    out.cols = cols;
    out.workers = out.segments = rows * cols;
    auto right = [&](uint32_t w) { return (w / cols) * cols + wrap(int64_t(w % cols) + 1, cols); };
    auto left = [&](uint32_t w) { return (w / cols) * cols + wrap(int64_t(w % cols) - 1, cols); };
    auto down = [&](uint32_t w) { return wrap(int64_t(w / cols) + 1, rows) * cols + w % cols; };
    auto up = [&](uint32_t w) { return wrap(int64_t(w / cols) - 1, rows) * cols + w % cols; };

    // Stage 1: horizontal reduce-scatter.
    for (uint32_t k = 0; k + 1 < cols; ++k)
        for (uint32_t q = 0; q < rows; ++q)
            push_step(out, MARSIT_REDUCE, [&](uint32_t w) {
                const uint32_t super = wrap(int64_t(w % cols) - int64_t(k), cols);
                return std::array<uint32_t, 3>{right(w), left(w), super * rows + q};
            });
    // Stage 2: vertical reduce-scatter, then vertical all-gather.
    for (int ph = 0; ph < 2; ++ph)
        for (uint32_t k = 0; k + 1 < rows; ++k)
            push_step(out, ph ? MARSIT_GATHER : MARSIT_REDUCE, [&](uint32_t w) {
                const uint32_t owned = wrap(int64_t(w % cols) + 1, cols);
                const uint32_t q = wrap(int64_t(w / cols) + ph - int64_t(k), rows);
                return std::array<uint32_t, 3>{down(w), up(w), owned * rows + q};
            });
    // Stage 3: horizontal all-gather.
    for (uint32_t k = 0; k + 1 < cols; ++k)
        for (uint32_t q = 0; q < rows; ++q)
            push_step(out, MARSIT_GATHER, [&](uint32_t w) {
                const uint32_t super = wrap(int64_t(w % cols) + 1 - int64_t(k), cols);
                return std::array<uint32_t, 3>{right(w), left(w), super * rows + q};
            });
    return validate(out, msg);
}

// Schedule::validate (schedule.hpp:38-54).
int validate(const HostSchedule& s, std::string* msg) {
    const uint32_t W = s.workers;
    if (s.send_to.size() != size_t(s.steps()) * W || s.recv_from.size() != s.send_to.size() ||
        s.segment.size() != s.send_to.size()) {
        if (msg) *msg = "Schedule: step entry count != workers";
        return MARSIT_EPROTOCOL;
    }
    for (uint32_t k = 0; k < s.steps(); ++k) {
        if (s.phase[k] > 1) {
            if (msg) *msg = "Schedule: bad phase";
            return MARSIT_EPROTOCOL;
        }
        const uint32_t* st = &s.send_to[size_t(k) * W];
        const uint32_t* rf = &s.recv_from[size_t(k) * W];
        const uint32_t* sg = &s.segment[size_t(k) * W];
        for (uint32_t w = 0; w < W; ++w) {
            if (st[w] >= W || rf[w] >= W || sg[w] >= s.segments) {
                if (msg) *msg = "Schedule: entry out of range";
                return MARSIT_EPROTOCOL;
            }
            if (rf[st[w]] != w) {
                if (msg) *msg = "Schedule: send/receive mismatch";
                return MARSIT_EPROTOCOL;
            }
        }
    }
    return MARSIT_OK;
}

uint64_t coin_threshold(uint32_t c_recv, uint32_t c_local) {
    const double p = static_cast<double>(c_recv) /
                     (static_cast<double>(c_recv) + static_cast<double>(c_local));
    // p * 2^53 is exact (power-of-two scaling); ceil of it is exact as well.
    return static_cast<uint64_t>(std::ceil(std::ldexp(p, 53)));
}

// Replay run_schedule (allreduce.hpp:51-73) on node ids.  Payloads are
// snapshotted before any delivery of a step (allreduce.hpp:57-62) and
// delivered in ascending sender order (transport.hpp:27-35); a reduce
// delivery creates a merge node drawing from the receiver's (receiver,
// segment) stream (allreduce.hpp:170-177, 183-185), a gather delivery
// replaces the receiver's node (allreduce.hpp:186).
Plan compile_plan(const HostSchedule& s) {
    const uint32_t W = s.workers, S = s.segments;
    Plan p;
    p.workers = W;
    p.segments = S;
    p.seg.resize(S);
    p.sends_per_worker.assign(W, 0);
    std::vector<uint32_t> node(size_t(W) * S), count(size_t(W) * S, 1);
    std::vector<int32_t> last(size_t(W) * S, -1);
    for (uint32_t w = 0; w < W; ++w)
        for (uint32_t sg = 0; sg < S; ++sg) node[size_t(w) * S + sg] = w;
    std::vector<uint32_t> in_node(W), in_count(W);
    for (uint32_t k = 0; k < s.steps(); ++k) {
        const uint32_t* st = &s.send_to[size_t(k) * W];
        const uint32_t* sgs = &s.segment[size_t(k) * W];
        for (uint32_t w = 0; w < W; ++w) {
            in_node[w] = node[size_t(w) * S + sgs[w]];
            in_count[w] = count[size_t(w) * S + sgs[w]];
            p.sends_per_worker[w] += 1;
            (s.phase[k] == MARSIT_REDUCE ? p.reduce_sends : p.gather_sends) += 1;
        }
        for (uint32_t from = 0; from < W; ++from) {
            const uint32_t to = st[from], sg = sgs[from];
            const size_t i = size_t(to) * S + sg;
            if (s.phase[k] == MARSIT_REDUCE) {
                SegmentPlan& sp = p.seg[sg];
                MergeNode m;
                m.recv_node = in_node[from];
                m.local_node = node[i];
                m.receiver = to;
                m.c_recv = in_count[from];
                m.c_local = count[i];
                m.offset_src = last[i];
                last[i] = static_cast<int32_t>(sp.merges.size());
                sp.merges.push_back(m);
                node[i] = W + static_cast<uint32_t>(sp.merges.size() - 1);
                count[i] = m.c_recv + m.c_local;
            } else {
                node[i] = in_node[from];
                count[i] = in_count[from];
            }
        }
    }
    // Stages: a merge that continues another merge's stream needs that
    // merge's total draw count, which is only known once every tile of it
    // is done -> it runs in a later device pass.
    uint32_t n_stages = 1;
    for (uint32_t sg = 0; sg < S; ++sg) {
        SegmentPlan& sp = p.seg[sg];
        for (size_t k = 0; k < sp.merges.size(); ++k) {
            MergeNode& m = sp.merges[k];
            uint32_t st = 0;
            for (uint32_t in : {m.recv_node, m.local_node})
                if (in >= W) st = std::max(st, sp.merges[in - W].stage);
            if (m.offset_src >= 0) st = std::max(st, sp.merges[m.offset_src].stage + 1);
            m.stage = st;
            n_stages = std::max(n_stages, st + 1);
        }
        sp.final_node = node[sg];
        sp.final_count = count[sg];
        for (uint32_t w = 1; w < W; ++w)
            if (node[size_t(w) * S + sg] != sp.final_node ||
                count[size_t(w) * S + sg] != sp.final_count)
                sp.consensus = false;
    }
    p.n_stages = n_stages;
    return p;
}

}  // namespace marsit_b200
