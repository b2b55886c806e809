V=variants/st_keep.so
for sb in "4096,4096 4,4" "256,256,256 4,4,4" "64,64,64,64 4,4,4,4" "28,28,28,28,28 4,4,4,4,4" "16,16,16,16,16,16 4,4,4,4,4,4"; do
  set -- $sb
  echo "== f32 $1 box $2"
  python tools/variant_time.py --config c4 --route bdbs --op add --shape $1 --box $2 $V
done
echo "== i64 max 256^3"; python tools/variant_time.py --config c2 --route bdbs --op max $V
echo "== c2 bdbsc"; python tools/variant_time.py --config c2 --route bdbsc --op add $V
echo "== c4 bc"; python tools/variant_time.py --config c4 --route box-complement --op add --reps 8 $V
echo "== c1"; python tools/variant_time.py --config c1 --route bdbs --op add $V
