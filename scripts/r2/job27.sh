set -x
bash scripts/r2/ab.sh r2ab20 "cur pred" "4 3 1"
echo done
