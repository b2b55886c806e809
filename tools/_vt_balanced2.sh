V="variants/bal_mult2.so variants/bal_pct0.so variants/bal_pct0_mult2.so"
for spec in "c5 bdbs add 512,512,512 2,2,2" "c5 bdbs add 512,512,512 8,8,8" "c5 bdbsc add 512,512,512 2,2,2" "c4 box-complement add 1024,1024,1024 16,16,16" "c4 bdbs add 1024,1024,1024 16,16,16" "c4 box-complement add 128,1024,1024 16,16,16" "c5 bdbs add 512,512,512 16,16,16"; do
  set -- $spec
  echo "== $spec"
  python tools/variant_time.py --config $1 --route $2 --op $3 --shape $4 --box $5 --reps 10 $V | cut -c1-330
  echo -n "uniform "; EXSUM_FP_BALANCED=0 python tools/variant_time.py --config $1 --route $2 --op $3 --shape $4 --box $5 --reps 10 | cut -c1-330
done
