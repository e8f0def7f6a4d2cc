for cfg in C2 C4; do
scripts/run_variants.sh $cfg base fw6
FG_FUSED_W16=roll scripts/run_variants.sh $cfg fw6
done
