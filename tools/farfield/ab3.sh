# config 5 far-field variants at 2^22 (development aid): ab3.sh variant...
cd ${GRAFT_REPO_ROOT:-.}
for v in "$@"; do
  if [ $v = default ]; then unset GWN_B200_LIB; else export GWN_B200_LIB=$PWD/build/variants/libgwn_b200_$v.so; fi
  echo "== $v"; timeout 600 python tools/time_eval.py 5:4194304 2>&1 | grep -oE "cfg5.*bnd=[0-9.]+"
done
