# A/B two builds of the library on one box: bash scripts/ab_libs.sh "<command>" (ab/libA.so, ab/libB.so)
for v in A B A B; do
  cp ab/lib$v.so paper_2503_08040_b200/lib/libfbq_b200.so
  echo "== $v"; eval "$1"
done
