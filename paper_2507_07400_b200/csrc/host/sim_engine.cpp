// Deterministic (time, seq) min-heap for the lockstep driver.
#include "kvflow/sim_engine.hpp"

#include <utility>

namespace kvf {

void EventQueue::push(VirtualTime time, EventKind kind, uint64_t id) {
    heap_.push_back(Event{time, pushed_++, kind, id});
    size_t i = heap_.size() - 1;
    while (i > 0) {
        size_t p = (i - 1) / 2;
        if (!earlier(heap_[i], heap_[p])) break;
        std::swap(heap_[i], heap_[p]);
        i = p;
    }
}

Event EventQueue::pop() {
    Event top = heap_.front();
    heap_.front() = heap_.back();
    heap_.pop_back();
    size_t i = 0, n = heap_.size();
    for (;;) {
        size_t l = 2 * i + 1, r = l + 1, m = i;
        if (l < n && earlier(heap_[l], heap_[m])) m = l;
        if (r < n && earlier(heap_[r], heap_[m])) m = r;
        if (m == i) break;
        std::swap(heap_[i], heap_[m]);
        i = m;
    }
    return top;
}

}  // namespace kvf
