for u in 1 2 4; do
echo "UNR=$u"
for c in "6136 2" "4088 4" "3064 8" "1520 64"; do set -- $c; VF_LU_UNR=$u python tools/gj_case.py --n $1 --batch $2 --reps 3 | sed -n 3p; done
done
