# direct-I/O batches (QS_TILE_DIRECT bit 0 load, bit 1 store, bit 2 pipelined next gather): parity, timings
for d in 6 1; do QS_TILE_DIRECT=$d timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ladder.py -x -q -k "qft or rqc or jit or fused or ladder or tile" 2>&1 | tail -1; done
for d in 0 2 6 3; do
  echo "== QS_TILE_DIRECT=$d"
  QS_TILE_DIRECT=$d AUTO=1 LOWS=4 LADDERS=4 CIRCS=qft,rqc timeout 300 python tools/calib_circ.py 2>&1 | tail -2
done
