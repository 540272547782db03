T=$(mktemp -d); C=./oracle/_ref/bpsched-cuda
$C generate --kind ising --n 12 --c 2.0 --count 3 --seed 7 --out $T > /dev/null
for m in 7 9; do for s in lbp rbp; do for be in cpu cuda; do $C run --model $T/ising_n12_c2_s$m.pgm --scheduler $s --p 0.25 --backend $be --out $T/$s.$be.csv > $T/$s.$be.json; done
echo "== s$m $s"; cat $T/$s.cpu.json $T/$s.cuda.json; diff <(cut -d, -f1-3 $T/$s.cpu.csv) <(cut -d, -f1-3 $T/$s.cuda.csv) | head -8; done; done
