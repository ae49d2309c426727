# Copy one evidence call's outputs (tools/gpu/r02_w*.sh) into profiles/ under the round's names:
#   bash tools/collect_evidence.sh gpurun_out/r02w2
set -e
O=$1
cp $O/pytest_gpu.log profiles/r02_pytest_gpu.log
cp $O/smoke.log profiles/r02_smoke.log
cp $O/launches_c3.csv profiles/r02_ncu_launches_c3.csv
[ -e $O/launches_bwd_c3.csv ] && cp $O/launches_bwd_c3.csv profiles/r02_ncu_launches_bwd_c3.csv
for f in $O/bench_*.json; do
  b=$(basename $f .json)
  [ "$b" = "bench_small" ] && continue
  cp $f profiles/r02_$b.json
done
for r in $O/sum_*.txt; do  # summaries written on the box (tools/gpu/r02_w3.sh)
  b=$(basename $r .txt); b=${b#sum_}
  cp $r profiles/r02_ncu_${b}_summary.txt
  cp $O/sass_$b.txt profiles/r02_ncu_${b}_top_sass.txt
done
for r in $O/prof_*.ncu-rep; do  # or reports brought back whole
  [ -e "$r" ] || continue
  b=$(basename $r .ncu-rep); b=${b#prof_}
  python tools/ncu_sum.py $r > profiles/r02_ncu_${b}_summary.txt
  python tools/ncu_src.py $r 25 > profiles/r02_ncu_${b}_top_sass.txt
done
if [ -e $O/ncu_traffic.json ]; then cp $O/ncu_traffic.json profiles/ncu_traffic.json; else python tools/ncu_traffic.py $O; fi
