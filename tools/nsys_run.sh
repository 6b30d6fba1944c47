#!/bin/bash
# Nsight Systems capture of every launch-bound config in stream and graph modes, then the gap
# table (tools/nsys_gaps.py). The nsys in this image is the copy inside Nsight Compute; its
# importer needs libdw, which the image lacks, so a stub (tools/nsys_shim, CPU sampling off)
# is built into /tmp for it. Only the CSV exports come back (gpurun_out/nsys/).
cd "${GRAFT_REPO_ROOT:-.}"
NSYS=${NSYS:-/opt/nvidia/nsight-compute/2025.2.1/host/target-linux-x64/nsys}
IMP=$(dirname "$NSYS")/../linux-desktop-glibc_2_11_3-x64/QdstrmImporter
OUT=gpurun_out/nsys
mkdir -p $OUT /tmp/dwstub
gcc -shared -fPIC -O2 -o /tmp/dwstub/libdw.so.1 tools/nsys_shim/libdw_stub.c \
  -Wl,--version-script=tools/nsys_shim/libdw_stub.map -Wl,-soname,libdw.so.1
"$NSYS" --version
for cfg in skeleton hotspot2d hotspot3d fdtd; do
  for mode in stream graph graph_pdl; do
    rep=/tmp/nsys_${cfg}_${mode}
    rm -f $rep.*
    timeout 300 "$NSYS" profile -t cuda -s none --cpuctxsw=none --cuda-graph-trace=node -f true -o $rep \
      python tools/nsys_gaps.py --run $cfg $mode > /tmp/nsys_${cfg}_${mode}.log 2>&1
    [ -f $rep.nsys-rep ] || LD_LIBRARY_PATH=/tmp/dwstub timeout 300 "$IMP" -i $rep.qdstrm -o $rep.nsys-rep > /dev/null 2>&1
    LD_LIBRARY_PATH=/tmp/dwstub timeout 300 "$NSYS" stats -r cuda_gpu_trace -f csv -o $OUT/${cfg}_${mode} \
      $rep.nsys-rep > /tmp/nsys_stats_${cfg}_${mode}.log 2>&1 || { echo "stats failed: $cfg $mode"; tail -3 /tmp/nsys_stats_${cfg}_${mode}.log; }
  done
done
ls -la $OUT | head -20
python tools/nsys_gaps.py --analyze $OUT | tee $OUT/gaps.md
