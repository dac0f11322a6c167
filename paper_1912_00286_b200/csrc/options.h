// Process-wide kernel-selection switches of libhdp (set through hdp_set_option, hdp.h).
// They choose between implementations of the same arithmetic (ablations, tuning) and never
// change a result beyond fp32 accumulation order; defaults are the measured-best choices.
#pragma once

namespace hdp {

enum OptId {
  OPT_PERSISTENT = 0,    // 1: persistent / wavefront fused recurrences where they fit; 0: per-step GEMMs
  OPT_WAVEFRONT,         // 1: two-layer wavefront launches (L = 2, mixed); 0: layer by layer
  OPT_WAVEFRONT_FUSEX,   // 1: layer-0 input projection fused into the forward wavefront
  OPT_WAVEFRONT_WGRAD,   // 1: A8 weight gradients inside the backward wavefront (W role)
  OPT_WAVEFRONT_TMEM,    // 1: TMEM-resident A operand instantiations where they exist; 0: SMEM-A
  OPT_RECUR_NBG,         // batch groups of the recurrence plans (0 = automatic)
  OPT_GEMM_CTA_GROUP,    // 0 automatic, 1 single CTAs, 2 CTA pairs (cta_group::2)
  OPT_GEMM_CLUSTER_N,    // TMA multicast of the A tile over 1 / 2 / 4 / 8 CTAs (0 = unicast)
  OPT_PDL,               // 1: programmatic dependent launch of the GEMM chain
  OPT_K7_BN,             // per-step K7 tile width override (0 = automatic)
  OPT_K7_SPLITS,         // per-step K7 split-K override (0 = automatic)
  OPT_RECUR_TRACE,       // 1: phase trace of the recurrence kernels in profile (eager) mode
  OPT_LAYER_PIPE,        // per-step path, L >= 2: layer-diagonal forward schedule in chunks of this many steps (0 = off)
  OPT_HEAD_FUSED,        // 1: fused FC head kernel (mixed mode, h_p, F_p <= 256), fixed per context at configure
  OPT_K7_CLUSTER,        // 1: K7's 8 split-K partials reduced in an 8-CTA cluster through DSMEM (no partial planes);
                         // off: only 15 such clusters are co-resident on B200, C4 needs 16 (measured 34.3 -> 59.0 ms)
  OPT_FWD_PDL,           // 1: programmatic dependent launch along the forward's input packing -> forward
                         // wavefront -> fused head (each one's prologue overlaps its predecessor's tail);
                         // off: measured neutral at C2 (0.802 vs 0.803 ms/step); test_forward_pdl_matches_oracle
  OPT_COUNT
};

extern int g_opt[OPT_COUNT];
inline int opt(OptId id) { return g_opt[id]; }
// name -> id, or -1
int opt_find(const char* name);

}  // namespace hdp
