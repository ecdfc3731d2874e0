# A/B of prebuilt library variants: bash scripts/gpu_libab.sh v0 v5 v6 (paper_2209_15427_b200/libqnb_<v>.so)
cd $GRAFT_REPO_ROOT
D=paper_2209_15427_b200
cp $D/libqnb.so /tmp/libqnb_keep.so
for v in "$@"; do
  cp $D/libqnb_$v.so $D/libqnb.so
  echo "== $v"; timeout 200 bash scripts/gpu_ab2.sh -
done
cp /tmp/libqnb_keep.so $D/libqnb.so
