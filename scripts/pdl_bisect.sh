# Debug: which kernel's programmatic launch breaks the c=1 fp32 case (after the C1 test)
for S in "kernel" "pack_probe,pack_records" "score_simt,row_lse,chunk_sum,topk" "cache_plan,gather" "attn_simt,attn_combine" "cache_plan" "gather" "attn_simt" "attn_combine" "pack_probe" "pack_records"; do
  echo "skip=[$S] $(CKV_PDL_SKIP=$S timeout 120 python scripts/pdl_debug.py 2>&1 | tail -1 | cut -c1-60)"
done
