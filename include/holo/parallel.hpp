// holosplat-b200 drop-in: the reference's worker-count API
// (proj/core/include/holo/parallel.hpp:9-15).  On the B200 the kernels are
// parallel by construction; the count is kept for API compatibility and
// parallel_for runs host-side helpers with the same chunking contract.
#pragma once

#include <cstdint>
#include <functional>

namespace holo {

void set_thread_count(int n);
int thread_count();
void parallel_for(int64_t begin, int64_t end, const std::function<void(int64_t, int64_t)>& fn);

}  // namespace holo
