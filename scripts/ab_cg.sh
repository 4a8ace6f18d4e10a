#!/bin/bash
# CG solve time (scripts/cg_prof.py) per library variant, on a scratch copy
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
SCR=$(mktemp -d); cp -r . $SCR/repo 2>/dev/null || true
for tag in "$@"; do
  cp paper_2407_06834_b200/libnld_b200_$tag.so $SCR/repo/paper_2407_06834_b200/libnld_b200.so
  (cd $SCR/repo && NLD_ALLOW_AB_BUILD=1 timeout 600 python scripts/cg_prof.py) 2>&1 | tail -1 | sed "s/^/$tag /"
done
rm -rf $SCR
