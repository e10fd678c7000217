// scan.cuh — device-wide exclusive scan of int64 counts (single pass,
// decoupled look-back). Used for work-list offsets.
#pragma once

#include "common.cuh"

namespace gt {
// In place: data[i] <- sum(data[0..i)); writes data[n] = total and *total_out = total
// (data must have n+1 slots).
void exclusive_scan_i64(int64_t* data, int64_t n, int64_t* total_out);
}  // namespace gt
