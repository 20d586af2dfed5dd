# sweep_ncu.sh TAG: ncu --set full of the AUTO kernel at every config-5 point
# (Nq 4..12, ~1e8 points, fp64 and fp32) -> gpurun_out/TAG_<dtype>_nq<N>.json
# (summaries made on the box: the reports themselves are deleted)
set -x
T=${1:-sw}
mkdir -p gpurun_out
cd $GRAFT_REPO_ROOT
for dt in f64 f32; do
  for nq in 4 5 6 7 8 9 10 11 12; do
    ne=$(python -c "print(int(round(1e8 / $nq**3)))")
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:volume_ -s 2 -c 1 \
      -o gpurun_out/${T}_${dt}_nq${nq} -f python -c "
import sys, torch; sys.path.insert(0, '.')
from paper_1604_08501_b200 import DeviceFieldState, volume_rhs_device
ds = DeviceFieldState.generate($nq, $ne, seed=1, dtype=torch.float64 if '$dt' == 'f64' else torch.float32)
for _ in range(3): volume_rhs_device(ds)
torch.cuda.synchronize()" > /dev/null 2>&1
    bpp=$([ $dt = f64 ] && echo 272 || echo 136)
    python tools/ncu_summary.py gpurun_out/${T}_${dt}_nq${nq}.ncu-rep --points $(( nq * nq * nq * ne )) \
      --bytes-per-point $bpp --out gpurun_out/${T}_${dt}_nq${nq}.json > /dev/null 2>&1
    rm -f gpurun_out/${T}_${dt}_nq${nq}.ncu-rep
  done
done
