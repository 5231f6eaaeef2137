#!/usr/bin/env bash
# A/B a working-tree change against a git ref on the same B200 box.
#
#   tools/ab.sh REF "CMD"          e.g.  tools/ab.sh HEAD "python bench.py --no-cpu --steps 10"
#
# Builds REF into _ab_ref/ (git archive) next to the working tree, prints the
# SASS line-count diff of the config-2 update kernel (k_update_tc<3,2,0,0>:
# its code generation is sensitive, so a change meant for another
# instantiation must leave it byte-identical), then runs CMD twice in each
# tree on one gpurun call, alternating.  Not part of the product.
set -euo pipefail
REF=${1:?ref}; CMD=${2:?command}
ROOT=$(cd "$(dirname "$0")/.." && pwd); cd "$ROOT"
rm -rf _ab_ref && mkdir _ab_ref && git archive "$REF" | tar -x -C _ab_ref
(cd _ab_ref && python -m paper_2109_09534_b200.build > /dev/null)
python -m paper_2109_09534_b200.build > /dev/null
k='k_update_tcILi3ELi2ELb0ELb0E'
for d in _ab_ref .; do
  cuobjdump -sass $d/paper_2109_09534_b200/libntcb.so 2>/dev/null |
    awk "/Function : .*$k/{f=1} f&&/Function : /&&!/$k/{f=0} f" |
    sed 's@/\*[0-9a-f]*\*/@@; s/0x[0-9a-f]*//g' | grep -v '^\s*$' > /tmp/ab_sass_$(basename $d).txt || true
done
echo "SASS lines differing in $k: $(diff /tmp/ab_sass__ab_ref.txt /tmp/ab_sass_..txt | grep -c '^[<>]' || true)"
/usr/local/graft/bin/gpurun --timeout 1800 -- "for r in 1 2; do for d in _ab_ref .; do echo \"\$d: \$(cd \$d && $CMD | tail -c 400)\"; done; done"
rm -rf _ab_ref
