# narrow-path stress: self-consistency of back-to-back calls (B=1, 8, 32) at C5 / C4 shapes
for cfg in "16384 16384 1" "16384 4096 8" "16384 4096 32"; do set -- $cfg
  echo "R=$1 K=$2 B=$3: $(R=$1 K=$2 B=$3 PYTHONPATH=. N=${N:-150} timeout -s KILL 600 python scripts/c4_selfcheck.py 2>&1 | grep -c '^iter') bad"
done
