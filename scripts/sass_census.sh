#!/bin/bash
# Per-kernel SASS census of libihs_b200.so: DMMA (fp64 tensor), UTMALDG (TMA tensor loads), UBLKCP (bulk
# copies), LDGSTS (cp.async), HMMA/UTCMMA (none expected: no fp64 tcgen05 kind), SYNCS (mbarrier ops).
cd "$(dirname "$0")/.."
cuobjdump -sass paper_2006_05874_b200/libihs_b200.so | awk '
/Function :/ { if (name != "") print name, c["DMMA"]+0, c["UTMALDG"]+0, c["UBLKCP"]+0, c["LDGSTS"]+0, c["SYNCS"]+0, c["DFMA"]+0, c["DADD"]+0; name=$3; delete c; next }
{ for (k in pat) if (index($0, k)) c[k]++ }
BEGIN { pat["DMMA"]; pat["UTMALDG"]; pat["UBLKCP"]; pat["LDGSTS"]; pat["SYNCS"]; pat["DFMA"]; pat["DADD"]; print "kernel DMMA UTMALDG UBLKCP LDGSTS SYNCS DFMA DADD" }
END { if (name != "") print name, c["DMMA"]+0, c["UTMALDG"]+0, c["UBLKCP"]+0, c["LDGSTS"]+0, c["SYNCS"]+0, c["DFMA"]+0, c["DADD"]+0 }' \
  | c++filt | awk 'NR==1 || $2+$3+$4+$5 > 0'
