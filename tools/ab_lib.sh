# A/B of two builds on one box: tools/ab_lib.sh LIB_A LIB_B "python tools/kernel_table.py c2" [reps]
export PATH=/usr/local/cuda/bin:$PATH
A=$1; B=$2; CMD=$3; N=${4:-3}
for i in $(seq $N); do
  echo "== A ($A)"; SKL_LIB=$A $CMD 2>&1 | grep -v "^\s*$" | tail -${LINES:-12}
  echo "== B ($B)"; SKL_LIB=$B $CMD 2>&1 | grep -v "^\s*$" | tail -${LINES:-12}
done
