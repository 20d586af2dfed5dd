set -x
T=${1:-san}
mkdir -p gpurun_out
cd $GRAFT_REPO_ROOT
for tool in racecheck synccheck memcheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --kernel-name kns=lfb python tools/sanitize_run.py > gpurun_out/${T}_sanitizer_${tool}.txt 2>&1
  timeout 600 compute-sanitizer --tool $tool python tools/sanitize_run.py emitted > gpurun_out/${T}_sanitizer_${tool}_emitted.txt 2>&1
done
