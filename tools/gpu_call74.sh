mkdir -p gpurun_out
i=0
while read -r v args; do
i=$((i+1))
env $v LRS_NO_AUTOTUNE=1 LRS_SKIP=4 timeout 60 python tools/cp_debug.py $args > gpurun_out/cp74_$i.log 2>&1; echo "$v [$args] rc=$? $(tail -1 gpurun_out/cp74_$i.log | cut -c1-80)"
done <<'LIST'
LRS_CORE_DBG=1 2 9 11 64 64 3 0 32
LRS_CORE_DBG=2 2 9 11 64 64 3 0 32
LRS_CORE_DBG=3 2 9 11 64 64 3 0 32
X=0 2 9 11 64 64 3 0 64
X=0 2 14 14 256 256 3 1 64
LRS_CORE_DBG=1 2 14 14 256 256 3 1 64
LRS_CORE_IPT=1 1 9 11 64 64 3 0 32
LIST
