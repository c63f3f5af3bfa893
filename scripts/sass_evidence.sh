#!/bin/bash
# Per-kernel count of the Blackwell bulk-copy (TMA) and mbarrier SASS in
# librsdb.so: UBLKCP.S.G = cp.async.bulk global->shared, UBLKCP.G.S =
# shared->global, SYNCS.* = mbarrier arrive / expect-tx / try-wait.
# Usage: scripts/sass_evidence.sh [lib] > profiles/r1/sass_tma_evidence.txt
LIB=${1:-paper_2602_22437_b200/librsdb.so}
cuobjdump -sass "$LIB" | awk '
  /Function :/ { fn = $3 }
  /UBLKCP.S.G/ { s2[fn]++ } /UBLKCP.G.S/ { g2[fn]++ } /SYNCS.PHASECHK/ { w[fn]++ } /SYNCS.ARRIVE.TRANS64/ { a[fn]++ }
  END { for (f in s2) printf "%5d UBLKCP.S.G %5d UBLKCP.G.S %5d SYNCS.ARRIVE %5d SYNCS.PHASECHK  %s\n", s2[f], g2[f], a[f], w[f], f }' |
  sort -k9 | c++filt | sed -E 's/\(rsdb::[^)]*\)//'
