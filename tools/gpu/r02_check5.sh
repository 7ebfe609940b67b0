for v in "1 tail" "8 tail" "8 item" "4 item" "16 tail"; do
  set -- $v
  echo "== DPIA_SEQ_UNROLL=$1 scope=$2"
  DPIA_SEQ_UNROLL=$1 DPIA_SEQ_UNROLL_SCOPE=$2 python tools/litgeo.py --quick
done 2>&1 | tee gpurun_out/litgeo_unroll.txt
