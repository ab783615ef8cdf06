bash tools/gpu.sh build > /dev/null
for v in 3 6 ; do
  echo "== CL=$v 10M uniform graph"; LBKD_SELECT_CLUSTER=$v timeout 60 python tools/one_build.py 10000000 3 rr uniform 2; echo "rc=$?"
  echo "== CL=$v 10M uniform nograph"; LBKD_GRAPH=0 LBKD_SELECT_CLUSTER=$v timeout 60 python tools/one_build.py 10000000 3 rr uniform 2; echo "rc=$?"
done
for v in 0 3 6; do
  KNOBS_TIMEOUT=60 python tools/knobs.py 100000000 3 rr uniform -- LBKD_SELECT_CLUSTER=$v
  for kind in identical huge constaxis ties; do KNOBS_TIMEOUT=60 python tools/knobs.py 10000000 3 rr $kind -- LBKD_SELECT_CLUSTER=$v; done
done
KNOBS_TIMEOUT=60 python tools/knobs.py 100000000 3 widest clustered -- LBKD_SELECT_CLUSTER=3
for kind in identical huge constaxis ties; do KNOBS_TIMEOUT=60 python tools/knobs.py 10000000 3 widest $kind -- LBKD_SELECT_CLUSTER=3; done
echo "== multigpu tests"; timeout 600 python -m pytest tests/test_gpu_multiproc.py tests/test_gpu_parity.py -q -x -m gpu -k "shard" 2>&1 | tail -3
timeout 600 python tools/big_build.py 1000000000 clustered 2 2>&1 | tail -4
