# A/B of several environment configurations on one box, interleaved:
#   tools/ab_multi.sh N REPS "ENV1" "ENV2" ...
N=$1; R=$2; shift 2
for r in $(seq 1 $R); do
  for V in "$@"; do
    echo "== [$V] n=$N $(env $V python tools/phase_seq.py $N | sed -n 1p)"
  done
done
