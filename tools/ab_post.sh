run() { tag=$1; shift; env "$@" python bench.py --no-cpu-baseline > gpurun_out/ab_$tag.log 2>&1; python tools/summ.py gpurun_out/ab_$tag.log; }
run base X=1
run late ARBOR_ATTN_LATE_TRIGGER=1
run late_pdl ARBOR_ATTN_LATE_TRIGGER=1 ARBOR_POST_PDL=1
run pdl ARBOR_POST_PDL=1
run base2 X=1
run late_pdl2 ARBOR_ATTN_LATE_TRIGGER=1 ARBOR_POST_PDL=1
