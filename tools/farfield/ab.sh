# K4 far-field variants at config 5 (development aid): ab.sh nq variant...
cd ${GRAFT_REPO_ROOT:-.}
nq=$1; shift
for v in "$@"; do
  if [ $v = default ]; then unset GWN_B200_LIB; else export GWN_B200_LIB=$PWD/build/variants/libgwn_b200_$v.so; fi
  echo "== $v"; timeout 600 python tools/farfield/check.py 5 $nq gpurun_out/ff_$v.npz
done
