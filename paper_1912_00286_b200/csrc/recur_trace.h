// Phase-trace decoding of the recurrence kernels (recur_trace.cpp).
#pragma once

namespace hdp {

enum TraceKind { TRACE_FWD_WAVEFRONT = 0, TRACE_FWD_LAYER = 1, TRACE_BWD_WAVEFRONT = 2, TRACE_BWD_LAYER = 3, TRACE_HEAD = 4 };
// h: host copy of the trace buffer (6 * T * 5 stamps), T steps, layer index l
void print_trace(TraceKind kind, const unsigned long long* h, int T, int l);

}  // namespace hdp
