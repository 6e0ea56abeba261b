// host_pool.h -- the host-side worker pool of the D' / TF transfer paths.
//
// The per-TF-change host work (gathering the TF's alpha column before its
// upload, expanding a compact D' after it crossed PCIe) is 10-100 us of
// parallel work that arrives after idle gaps.  An OpenMP team pays its full
// wake-up (~50 us for 15 sleeping threads on the B200 host) at every region,
// because the region's closing barrier waits for the last thread to wake.
// This pool never makes the caller wait for a helper to start: the caller
// works on the job itself from the first microsecond, helpers join as they
// wake and take what is left (dynamic, one atomic counter), and the call
// returns when every unit is done.  prewake() lets a caller that is about to
// wait on the GPU get the helpers spinning first, so they are running when
// the data lands.
#pragma once

#include <stdint.h>

#include <functional>

namespace pdm {
namespace host {

// fn(i) for every i in [0, n), on the calling thread plus the pool's helper
// threads; returns when all are done (writes, including non-temporal stores,
// are visible to the caller).
void parallel_for(int64_t n, const std::function<void(int64_t)> &fn);

// Wake the helpers and keep them spinning for up to `us` microseconds (or
// until the next parallel_for), so its units start without wake-up latency.
void prewake(int us);

int threads();  // helpers + the caller

}  // namespace host
}  // namespace pdm
