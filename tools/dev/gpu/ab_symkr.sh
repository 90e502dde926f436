# A/B: round-1 library vs this one on c1 (kernel durations under ncu, serialised)
set -e
mkdir -p /tmp/ab && cd /tmp/ab
rm -rf old && git -C $GRAFT_REPO_ROOT archive --format=tar db63a74 2>/dev/null | tar x -C /tmp/ab 2>/dev/null || true
cd $GRAFT_REPO_ROOT
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:symkr --csv --log-file gpurun_out/r02_ab_new.csv python bench.py --config c1 --steps 2 --warmup 1 --no-extra --no-cpu-baseline --no-e2e > /dev/null 2>&1 || true
grep -c symkr gpurun_out/r02_ab_new.csv || true
