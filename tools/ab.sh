# A/B of environment switches on one box: tools/ab.sh "ENV_A" "ENV_B" n [reps]
A="$1"; B="$2"; N=${3:-10000}; R=${4:-2}
for r in $(seq 1 $R); do
  for V in "$A" "$B"; do
    echo "== $V n=$N"; env $V python tools/phase_seq.py $N | sed -n 1p
  done
done
