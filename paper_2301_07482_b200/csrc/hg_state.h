// Layout of the small device-resident state vectors shared by the kernels and
// the Python host (paper_2301_07482_b200/_state.py mirrors these indices).
#pragma once

namespace hg {

// per cache layer: int64[16]   (histgnn/cache.py:28-38,60-77)
enum LayerCtr : int {
  kCtrHits = 0,
  kCtrMisses = 1,
  kCtrAdmissions = 2,
  kCtrGradientEvictions = 3,
  kCtrStalenessEvictions = 4,
  kCtrForcedEvictions = 5,
  kCtrStalenessViolations = 6,
  kCtrValid = 7,             // entries with row_of >= 0 (valid_entries)
  kCtrHeader = 8,            // ring header
  kCtrCapacity = 9,          // table rows
  kCtrWindowAdmissions = 10,
  kCtrWindowForced = 11,
  kCtrNWrite = 12,           // scratch: admitted+computed count of the last update
  kCtrK = 13,                // scratch: floor(p_grad * n) of the last update
  kLayerCtrLen = 16,
};

// global: int64[8]
enum GlobalCtr : int {
  kGCtrFeatureHits = 0,
  kGCtrFeatureMisses = 1,
  kGCtrPruneWrites = 2,
  kGCtrRemoteRows = 3,       // feature rows read from a peer GPU's shard
  kGlobalCtrLen = 8,
};

}  // namespace hg
