# ncu --set full of the AUTO kernel at a sweep point: bash tools/gpu_prof_sweep.sh TAG NQ DTYPE [VARIANT]
cd $GRAFT_REPO_ROOT
T=$1; NQ=$2; DT=$3; V=${4:-auto}
NE=$((100000000/(NQ*NQ*NQ)))
timeout 900 ncu --set full --clock-control none --import-source on -k regex:volume_ -s 2 -c 1 -o gpurun_out/${T}_nq${NQ}_${DT}_${V} python bench.py --nq $NQ --ne $NE --dtype $DT --variant $V --inputs device --steps 1 --warmup 3 --no-e2e --no-cpu --no-emitted > gpurun_out/${T}_nq${NQ}_${DT}_${V}.log 2>&1
