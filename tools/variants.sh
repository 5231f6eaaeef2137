#!/usr/bin/env bash
# Same-box comparison of compile-time variants of the library.
#
#   tools/variants.sh "CMD" NAME1="-DFLAG=1" NAME2="-DFLAG=2" ...
#
# Copies the working tree to _v_NAME/ (git-ignored), builds each with
# NTCB_NVCC_EXTRA set to its flags, and runs CMD twice in every tree (and in
# the working tree itself, "base") on one gpurun call, alternating.  Not part
# of the product.
set -euo pipefail
CMD=${1:?command}; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd); cd "$ROOT"
names=()
for kv in "$@"; do
  n=${kv%%=*}; f=${kv#*=}; names+=("_v_$n")
  rm -rf "_v_$n" && mkdir "_v_$n"
  tar -c --exclude=.git --exclude=gpurun_out --exclude='_v_*' --exclude=_ab_ref --exclude=.mb --exclude='*.o' --exclude=libntcb.so . | tar -x -C "_v_$n"
  (cd "_v_$n" && NTCB_NVCC_EXTRA="$f" python -m paper_2109_09534_b200.build > /dev/null) &
done
wait
python -m paper_2109_09534_b200.build > /dev/null
dirs=". ${names[*]}"
/usr/local/graft/bin/gpurun --timeout 2400 -- "for r in 1 2; do for d in $dirs; do echo \"\$d: \$(cd \$d && $CMD | tail -c 600)\"; done; done"
for n in "${names[@]}"; do rm -rf "$n"; done
