// kvsim -> kvflow include shim (test infrastructure): lets the reference's own unit suites
// compile unmodified against the B200 host API (tests/refsuite/README.md).
#pragma once
#include "kvflow/scheduler.hpp"
namespace kvsim {
using namespace kvf;
}
