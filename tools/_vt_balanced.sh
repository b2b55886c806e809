# balanced unit ranges of the fused pair (default) against uniform segments (EXSUM_FP_BALANCED=0)
for spec in "c5 bdbs add 512,512,512 8,8,8" "c5 bdbs add 512,512,512 2,2,2" "c5 box-complement add 512,512,512 8,8,8" "c5 box-complement add 512,512,512 16,16,16" "c4 box-complement add 128,1024,1024 16,16,16" "c4 bdbs add 128,1024,1024 16,16,16" "c4 box-complement add 256,1024,1024 16,16,16" "c4 box-complement add 1024,1024,1024 16,16,16" "c4 bdbs add 1024,1024,1024 4,4,4" "c2 bdbsc add 256,256,256 8,8,8" "c5 bdbs add 300,512,512 8,8,8" "c4 bdbs add 200,700,1024 8,8,8"; do
  set -- $spec
  echo "== $spec"
  for b in 1 0; do
    echo -n "balanced=$b "; EXSUM_FP_BALANCED=$b python tools/variant_time.py --config $1 --route $2 --op $3 --shape $4 --box $5 --reps 10 | cut -c1-400
  done
done
