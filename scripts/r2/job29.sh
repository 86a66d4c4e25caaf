set -x
bash scripts/r2/ab.sh r2ab22 "cur pb2 pb4" "4 3"
echo done
