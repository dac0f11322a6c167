#include <algorithm>
// Decoding of the recurrence kernels' phase traces (option recur_trace = 1 in profile
// mode, hdp_set_option): each traced step stores 5 globaltimer stamps per role; this
// prints the per-step mean of every phase to stderr.  Development aid, not on the hot path.
#include "recur_trace.h"

#include <cstdio>

namespace hdp {

void print_trace(TraceKind kind, const unsigned long long* h, int T, int l) {
  (void)l;
  switch (kind) {
    case TRACE_HEAD: {  // fused head: T = grid, 8 stamps per CTA
      const char* names[7] = {"TMA landed", "z acc seen", "y (pass 1)", "dz + sums (pass 2)", "dH acc seen",
                              "dH stored (pass 3)", "exit"};
      unsigned long long s0 = ~0ull, s1 = 0;
      for (int b = 0; b < T; ++b) {
        s0 = std::min(s0, h[b * 8]);
        s1 = std::max(s1, h[b * 8]);
      }
      fprintf(stderr, "[hdp trace] head: %d CTAs, entry spread %llu ns\n", T, s1 - s0);
      for (int k = 1; k < 8; ++k) {
        double mean = 0, mx = 0;
        for (int b = 0; b < T; ++b) {
          const double d = (double)(h[b * 8 + k] - h[b * 8]);
          mean += d;
          mx = std::max(mx, d);
        }
        fprintf(stderr, "[hdp trace] head: %-20s +%.0f ns mean, +%.0f max (from CTA entry)\n", names[k - 1], mean / T,
                mx);
      }
      break;
    }
    case TRACE_FWD_WAVEFRONT: {
      const unsigned long long t00 = h[0];
      const char* names[3] = {"R0", "P", "R1"};
      for (int role = 0; role < 3; ++role) {
        double ph[4] = {0, 0, 0, 0}, step = 0;
        int n = 0;
        for (int t = 2; t < T - 1; ++t) {
          const unsigned long long* r = &h[((size_t)role * T + t) * 5];
          for (int q = 0; q < 4; ++q) ph[q] += (double)(r[q + 1] - r[q]);
          step += (double)(h[((size_t)role * T + t + 1) * 5] - r[0]);
          ++n;
        }
        const unsigned long long* st = &h[((size_t)role * T + 1) * 5];
        fprintf(stderr, "[hdp trace] wavefront %s: per step ns: %.0f %.0f %.0f %.0f | step %.0f | t=1 starts at +%.0f ns, t=T-1 ends at +%.0f\n",
                names[role], ph[0] / n, ph[1] / n, ph[2] / n, ph[3] / n, step / n, (double)(st[0] - t00),
                (double)(h[((size_t)role * T + T - 1) * 5 + 4] - t00));
      }
      {
        double q[3] = {0, 0, 0};
        int n = 0;
        for (int t = 2; t < T - 1; ++t) {
          const unsigned long long* r = &h[((size_t)3 * T + t) * 5];
          const unsigned long long e0 = h[((size_t)0 * T + t) * 5 + 2];  // R0 TR(t,2): MMA done
          if (!r[0] || !r[3]) continue;
          q[0] += (double)(r[0] - e0);
          q[1] += (double)(r[1] - r[0]);
          q[2] += (double)(r[2] - r[1]);
          ++n;
        }
        if (n)
          fprintf(stderr, "[hdp trace] wavefront R0 epilogue: acc load %.0f  act+stage %.0f  cell+stores %.0f ns\n",
                  q[0] / n, q[1] / n, q[2] / n);
      }
      {  // per-CTA entry / exit per role, relative to R0's first step
        const unsigned long long* c = h + (size_t)6 * T * 5;
        const char* rn[3] = {"R0", "P", "R1"};
        const unsigned long long t00 = h[0];
        for (int r = 0; r < 3; ++r) {
          unsigned long long lo = ~0ull, hi = 0;
          int n = 0;
          for (int k = 0; k < 148; ++k) {
            if (!c[3 * k] || c[3 * k + 2] != (unsigned long long)r) continue;
            lo = c[3 * k] < lo ? c[3 * k] : lo;
            hi = c[3 * k + 1] > hi ? c[3 * k + 1] : hi;
            ++n;
          }
          if (n)
            fprintf(stderr, "[hdp trace] fwd %s: %d CTAs, first entry %+.0f ns, last exit %+.0f ns (vs R0 step 0)\n",
                    rn[r], n, (double)lo - (double)t00, (double)hi - (double)t00);
        }
      }
      break;
    }
    case TRACE_FWD_LAYER: {
      double ph[4] = {0, 0, 0, 0}, step = 0;
      int n = 0;
      for (int t = 1; t < T - 1; ++t) {
        const unsigned long long* r = &h[(size_t)t * 5];
        ph[0] += (double)(r[1] - r[0]);
        ph[1] += (double)(r[2] - r[1]);
        ph[2] += (double)(r[3] - r[2]);
        ph[3] += (double)(r[4] - r[3]);
        step += (double)(h[(size_t)(t + 1) * 5] - r[0]);
        ++n;
      }
      fprintf(stderr, "[hdp trace] recur_fwd layer %d: per step ns: wait %.0f mma %.0f epilogue %.0f push %.0f | step %.0f\n",
              l, ph[0] / n, ph[1] / n, ph[2] / n, ph[3] / n, step / n);
      break;
    }
    case TRACE_BWD_WAVEFRONT: {
      {
        {
          double wsum[4] = {0, 0, 0, 0};
          int n = 0;
          for (int t = T - 2; t >= 1; --t) {
            const unsigned long long e2 = h[((size_t)1 * T + t) * 5 + 2];  // Q0 TR(t,2)
            const unsigned long long* r = &h[((size_t)5 * T + t) * 5];
            if (!r[0]) continue;
            for (int w = 0; w < 4; ++w) wsum[w] += (double)r[w] - (double)e2;
            ++n;
          }
          if (n)
            fprintf(stderr, "[hdp trace] bwd Q0 warps reach the epilogue barrier at +%.0f +%.0f +%.0f +%.0f ns after MMA done\n",
                    wsum[0] / n, wsum[1] / n, wsum[2] / n, wsum[3] / n);
        }
        // dX1 hand-off timeline (group 0, units 0..63): X publishes -> Q0 fetch issued -> Q0 needs
        const unsigned long long z0 = h[(size_t)(T - 1) * 5];
        for (int t = T - 3; t >= 0; t -= (T > 40 ? 20 : 5)) {
          const unsigned long long* r = &h[((size_t)4 * T + t) * 5];
          fprintf(stderr, "[hdp trace] Q0 t=%d: gates/c fetch issued +%.0f  needed +%.0f  slot t landed +%.0f  slot t-1 landed +%.0f ns\n", t,
                  (double)(r[0] - z0), (double)(r[2] - z0), (double)(r[3] - z0), (double)(r[4] - z0));
        }
      }
      {
        double q[3] = {0, 0, 0};
        int n = 0;
        for (int t = T - 2; t >= 1; --t) {
          const unsigned long long* r = &h[((size_t)3 * T + t) * 5];
          const unsigned long long e2 = h[((size_t)1 * T + t) * 5 + 2];  // Q0 TR(t,2)
          if (!r[0] || !r[2]) continue;
          q[0] += (double)(r[0] - e2);
          q[1] += (double)(r[1] - r[0]);
          q[2] += (double)(r[2] - r[1]);
          ++n;
        }
        if (n)
          fprintf(stderr, "[hdp trace] bwd Q0 epilogue: dX1 wait %.0f  acc load %.0f  cell+stage %.0f ns\n", q[0] / n,
                  q[1] / n, q[2] / n);
        double w3 = 0, w4 = 0;
        int m = 0;
        for (int t = T - 2; t >= 1; --t) {
          const unsigned long long* r = &h[((size_t)3 * T + t) * 5];
          w3 += (double)r[3];
          w4 += (double)r[4];
          ++m;
        }
        fprintf(stderr, "[hdp trace] bwd Q0 warp 3: store read-wait %.0f  due dX1 fetch %.0f ns\n", w3 / m, w4 / m);
      }
      const char* names[3] = {"Q1", "Q0", "X"};
      const unsigned long long t00 = h[(size_t)(T - 1) * 5];
      for (int role = 0; role < 3; ++role) {
        double ph[4] = {0, 0, 0, 0}, step = 0;
        int n = 0;
        for (int t = T - 2; t >= 1; --t) {
          const unsigned long long* r = &h[((size_t)role * T + t) * 5];
          for (int q = 0; q < 4; ++q) ph[q] += (double)(r[q + 1] - r[q]);
          step += (double)(h[((size_t)role * T + t - 1) * 5] - r[0]);
          ++n;
        }
        fprintf(stderr, "[hdp trace] bwd wavefront %s: per step ns: %.0f %.0f %.0f %.0f | step %.0f | t=T-2 starts at +%.0f ns, t=0 ends at +%.0f\n",
                names[role], ph[0] / n, ph[1] / n, ph[2] / n, ph[3] / n, step / n,
                (double)(h[((size_t)role * T + T - 2) * 5] - t00), (double)(h[((size_t)role * T) * 5 + 4] - t00));
      }
      {  // W role: last step's dA seen by the producer, MMAs done (per weight matrix)
        const unsigned long long* w = h + (size_t)6 * T * 5 + 3 * 148;
        const unsigned long long t00 = h[(size_t)(T - 1) * 5];
        const char* mn[4] = {"dU1", "dW1", "dU0", "dW0"};
        for (int mat = 0; mat < 4; ++mat) {
          double seen = 0, done = 0;
          int n = 0;
          for (int k = 0; k < 148; ++k) {
            if (!w[3 * k] || w[3 * k + 2] != (unsigned long long)(1 + mat)) continue;
            seen = std::max(seen, (double)(w[3 * k] - t00));
            done = std::max(done, (double)(w[3 * k + 1] - t00));
            ++n;
          }
          if (n)
            fprintf(stderr, "[hdp trace] bwd W %s: %d CTAs, last dA_0 seen +%.0f ns, MMAs done +%.0f ns (vs Q1 step T-1)\n",
                    mn[mat], n, seen, done);
        }
      }
      {  // Q prologue (CTA 0 of group 0)
        const unsigned long long* pr = h + (size_t)6 * T * 5 + 6 * 148;
        const unsigned long long t00 = h[(size_t)(T - 1) * 5];
        for (int q = 0; q < 2; ++q)
          if (pr[q * 8])
            fprintf(stderr, "[hdp trace] bwd %s prologue (vs Q1 step T-1): entry %+.0f, TMEM alloc %+.0f, U slice landed %+.0f, "
                    "cluster sync %+.0f, U^T in TMEM %+.0f ns\n", q ? "Q0" : "Q1", (double)pr[q * 8] - (double)t00,
                    (double)pr[q * 8 + 1] - (double)t00, (double)pr[q * 8 + 2] - (double)t00,
                    (double)pr[q * 8 + 3] - (double)t00, (double)pr[q * 8 + 4] - (double)t00);
      }
      {  // per-CTA entry / exit per role, relative to Q1's first step
        const unsigned long long* c = h + (size_t)6 * T * 5;
        const char* rn[4] = {"Q1", "X", "Q0", "W"};
        const unsigned long long t00 = h[(size_t)(T - 1) * 5];
        for (int r = 0; r < 4; ++r) {
          unsigned long long lo = ~0ull, hi = 0;
          int n = 0;
          for (int k = 0; k < 148; ++k) {
            if (!c[3 * k] || c[3 * k + 2] != (unsigned long long)r) continue;
            lo = c[3 * k] < lo ? c[3 * k] : lo;
            hi = c[3 * k + 1] > hi ? c[3 * k + 1] : hi;
            ++n;
          }
          if (n)
            fprintf(stderr, "[hdp trace] bwd %s: %d CTAs, first entry %+.0f ns, last exit %+.0f ns (vs Q1 step T-1)\n",
                    rn[r], n, (double)lo - (double)t00, (double)hi - (double)t00);
        }
      }
      break;
    }
    case TRACE_BWD_LAYER: {
      double ph[4] = {0, 0, 0, 0}, step = 0;
      int n = 0;
      for (int t = T - 2; t >= 1; --t) {  // steps with an MMA; t+1 -> t gap is the step time
        const unsigned long long* r = &h[(size_t)t * 5];
        ph[0] += (double)(r[1] - r[0]);   // prefetch issue + cluster wait
        ph[1] += (double)(r[2] - r[1]);   // MMA issue + completion
        ph[2] += (double)(r[3] - r[2]);   // epilogue + syncthreads
        ph[3] += (double)(r[4] - r[3]);   // DSMEM push + arrive
        step += (double)(h[(size_t)(t - 1) * 5] - r[0]);
        ++n;
      }
      fprintf(stderr, "[hdp trace] recur_bwd layer %d: per step ns: wait %.0f mma %.0f epilogue %.0f push %.0f | step %.0f\n",
              l, ph[0] / n, ph[1] / n, ph[2] / n, ph[3] / n, step / n);
      break;
    }
  }
}

}  // namespace hdp
