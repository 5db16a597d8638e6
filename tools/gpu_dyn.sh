# dynamic tile scheduling (QS_TILE_DYN) vs grid-stride: memory-only pass, QFT(32), RQC(32); parity under DYN
for d in 0 1; do
  echo "== QS_TILE_DYN=$d"
  QS_TILE_DYN=$d timeout 300 python tools/perm_probe.py 2>&1 | grep near | head -1
  QS_TILE_DYN=$d AUTO=1 LOWS=4 LADDERS=4 CIRCS=qft,rqc timeout 300 python tools/calib_circ.py 2>&1 | tail -2
done
QS_TILE_DYN=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "qft or rqc or jit or fused" 2>&1 | tail -2
