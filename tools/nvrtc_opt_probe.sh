for o in "" "--extra-device-vectorization" "-Xptxas --allow-expensive-optimizations=true" "-Xptxas -O3 -Xptxas --warn-on-spills" "-dopt=on"; do
  echo "OPTS=[$o]"
  ISPC_NVRTC_OPTS="$o" PROBE_KINDS=sgemm timeout 300 python tools/pdl_probe.py 2>&1 | cut -c1-250
done
