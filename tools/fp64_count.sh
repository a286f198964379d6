#!/bin/bash
# static FP64 instruction counts (DFMA/DMUL/DADD/DSETP/MUFU) of the Minkowski WENO5/DER6/field-CD
# sweep kernels in the built library: the quick CPU-side check of an arithmetic rewrite
LIB=${1:-paper_1810_04597_b200/libecho_b200.so}
for ax in 0 1 2; do
  f="_ZN4echo5march7k_marchILi${ax}ELb0ELi6ELi0ELi0EEEvNS_5GridPENS_4EosPENS_9MetTablesENS0_8LineGeomEPKdS7_PdS7_S8_"
  cuobjdump -sass -fun "$f" "$LIB" 2>/dev/null | grep -oE "^\s+/\*[0-9a-f]+\*/\s+[A-Z0-9.]+" | awk '{print $2}' | sed 's/\..*//' \
    | awk -v ax=$ax '{c[$1]++} END {printf "axis %d: DFMA %d DMUL %d DADD %d DSETP %d MUFU %d  FP64 %d  all %d\n", ax, c["DFMA"], c["DMUL"], c["DADD"], c["DSETP"], c["MUFU"], c["DFMA"]+c["DMUL"]+c["DADD"]+c["DSETP"], NR}'
done
