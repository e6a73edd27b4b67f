// ablation.h -- the harness's A/B switches.
//
// The product default is every switch unset.  The environment is read ONCE, the first
// time any entry point plans a launch, and the snapshot is kept for the life of the
// process: launch shape and kernel choice cannot change between calls, and a process that
// wants an ablation sets the variable before its first call (scripts/tune.py and the
// subprocess-based tests do).  Nothing here is part of the C ABI.
#pragma once
#include <stdlib.h>
#include <string.h>

namespace dcnv4 {

enum AblationKey {
  kAblTile = 0,          // DCNV4_TILE=TH,TW,Gc       generic-kernel tile override
  kAblFwdPath,           // DCNV4_FWD_PATH=g          forward: global-gather kernel only
  kAblBwdPath,           // DCNV4_BWD_PATH=g          backward: global-gather kernel only
  kAblFwd33TH,           // DCNV4_FWD33_TH=n          fwd33 tile height cap
  kAblBwd33TH,           // DCNV4_BWD33_TH=n          bwd33 tile height cap
  kAblP4Order,           // DCNV4_P4ORDER=0           bwd33 pull in row-major bin order
  kAblFwdCpl,            // DCNV4_FWD_CPL=n           chunks per lane (forward)
  kAblBwdCpl,            // DCNV4_BWD_CPL=n           chunks per lane (backward)
  kAblNonPersistent,     // DCNV4_NONPERSISTENT=1     one CTA per tile
  kAblModulePerSm,       // DCNV4_MODULE_PER_SM=n     fused module CTAs per SM
  kAblModuleStages,      // DCNV4_MODULE_STAGES=1|2   fused module operand ring depth
  kAblMsdaOrder,         // MSDA_ORDER=q              query-fastest slot order
  kAblMsdaCpl,           // MSDA_CPL=n                chunks per lane
  kAblMsdaGridCap,       // MSDA_GRID_CAP=1           capped grid-stride launch
  kAblMsdaSched,         // MSDA_SCHED=persist        persistent schedule
  kAblMsdaVec,           // MSDA_VEC=1                vectorised sample records
  kAblMsdaBwd8,          // MSDA_BWD8=0               16-B half backward layout
  kAblFwdMargin,         // DCNV4_FWD_MARGIN=n        fwd33 halo margin override
  kAblCount
};

// The value of switch `k` as it was when the library was first used ("" if unset).
inline const char* ablation(AblationKey k) {
  static const char* const names[kAblCount] = {
      "DCNV4_TILE",          "DCNV4_FWD_PATH",   "DCNV4_BWD_PATH",      "DCNV4_FWD33_TH",
      "DCNV4_BWD33_TH",      "DCNV4_P4ORDER",    "DCNV4_FWD_CPL",       "DCNV4_BWD_CPL",
      "DCNV4_NONPERSISTENT", "DCNV4_MODULE_PER_SM", "DCNV4_MODULE_STAGES", "MSDA_ORDER",
      "MSDA_CPL",            "MSDA_GRID_CAP",    "MSDA_SCHED",          "MSDA_VEC",
      "MSDA_BWD8",           "DCNV4_FWD_MARGIN"};
  struct Snapshot {
    char v[kAblCount][32];
    Snapshot() {
      for (int i = 0; i < kAblCount; ++i) {
        const char* e = getenv(names[i]);
        v[i][0] = 0;
        if (e) {
          strncpy(v[i], e, sizeof(v[i]) - 1);
          v[i][sizeof(v[i]) - 1] = 0;
        }
      }
    }
  };
  static const Snapshot snap;  // thread-safe one-time initialisation (C++11 statics)
  return snap.v[k];
}

inline bool ablation_set(AblationKey k) { return ablation(k)[0] != 0; }

}  // namespace dcnv4
