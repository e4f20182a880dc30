// kvflow host API -- where the scheduler's requests come from.
// The reference's Simulator owns its synthetic workload generator
// (proj/include/kvsim/scheduler.hpp:54, proj/include/kvsim/workload.hpp:71-100).  Here the
// scheduler (libkvflow_host.so) only sees this interface; the synthetic generator
// (WorkloadController, include/kvflow/workload.hpp) is harness code in libkvflow_driver.so,
// and a serving front end supplies its own source.
#pragma once

#include <cstdint>
#include <vector>

#include "kvflow/step_graph.hpp"
#include "kvflow/types.hpp"

namespace kvf {

struct RequestSpec {
    uint64_t id = 0;  // client * 1e6 + per-client release index
    ClientId client = 0;
    AgentId agent;
    TokenSeq prompt;
    size_t fixed_len = 0;
    TokenSeq output;
    StepMap step_metadata;
    bool measured = false;
    uint64_t arrival_seq = 0;
    uint32_t iteration = 0;
};

struct IterationWindow {
    ClientId client = 0;
    uint32_t iteration = 0;
    bool measured = false;
    VirtualTime start = -1;
    VirtualTime end = -1;
};

class RequestSource {
public:
    virtual ~RequestSource() = default;
    // requests released at time 0, in arrival order
    virtual std::vector<RequestSpec> start() = 0;
    // requests released by the completion of `request_id` (workflow successors)
    virtual std::vector<RequestSpec> on_done(uint64_t request_id) = 0;
    virtual void note_arrival(uint64_t request_id, VirtualTime t) = 0;
    virtual void note_done(uint64_t request_id, VirtualTime t) = 0;
    virtual bool all_finished() const = 0;
    virtual std::vector<IterationWindow> iteration_windows() const = 0;
    // largest prompt + output of any request (capacity check at construction)
    virtual uint64_t max_request_tokens() const = 0;
    // every token the run can ever insert (bounds the write-once host pool)
    virtual uint64_t max_cached_tokens() const = 0;
};

}  // namespace kvf
