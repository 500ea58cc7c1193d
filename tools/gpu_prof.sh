# ncu --set full captures, ABFT on vs off, summarised on the box (reports over
# 20 MB, and all of them without KEEP=1, are deleted after summarising:
# gpurun_out must stay under its 64 MiB merge cap).
# usage: KRE=<kernel regex> COUNT=<kernels per capture> bash tools/gpu_prof.sh TAG prec:logn[:variant] ...
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=$1; shift
for spec in $@; do
  IFS=: read p l v <<< "$spec"  # prec:logn[:variant]
  for sc in two_sided_group none; do
    o=gpurun_out/${TAG}_${p}_n${l}${v:+_v$v}_${sc}
    timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
      --kernel-name-base demangled -k regex:"${KRE:-fft_}" -c ${COUNT:-1} \
      -o $o -f python tools/profile_single.py --prec $p --logn $l --scheme $sc --reps 2 --variant ${v:--1} > $o.log 2>&1
    python tools/ncu_summary.py $o.ncu-rep > $o.md 2>&1
    python tools/sass_hot.py $o.ncu-rep --top 30 --lines 40 > $o.sass.txt 2>&1
    if [ -z "$KEEP" ] || [ $(stat -c %s $o.ncu-rep) -gt 20000000 ]; then rm -f $o.ncu-rep; fi
  done
done
du -sh gpurun_out
