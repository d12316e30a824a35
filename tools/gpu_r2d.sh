O="vec=4,chunks=1,rows=96,warps=1,prefetch=4"
bash tools/bench_variants.sh r2d harris "PMG_CAP_I=72,PMG_CAP_B=128;$O" "PMG_CAP_I=72;$O" "PMG_CAP_I=72,PMG_CAP_B=128,PMG_DIAG_SKIP=be;$O" \
  "PMG_CAP_I=72,PMG_CAP_B=96;$O" "PMG_CAP_I=64,PMG_CAP_B=128;$O" "PMG_CAP_B=128;$O" \
  "PMG_CAP_I=72,PMG_CAP_B=128;vec=4,chunks=1,rows=104,warps=1,prefetch=4" "PMG_CAP_I=72,PMG_CAP_B=128;vec=4,chunks=1,rows=112,warps=1,prefetch=4" \
  "PMG_CAP_I=72,PMG_CAP_B=128;vec=4,chunks=1,rows=88,warps=1,prefetch=4" "PMG_CAP_I=72,PMG_CAP_B=128;vec=4,chunks=1,rows=80,warps=1,prefetch=4"
