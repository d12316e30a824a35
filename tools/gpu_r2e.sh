O="vec=4,chunks=1,rows=96,warps=1,prefetch=4"
bash tools/bench_variants.sh r2e harris "PMG_DIAG_SKIP=b;$O" "PMG_DIAG_SKIP=e;$O" "PMG_DIAG_SKIP=be;$O" ";$O" "PMG_DIAG_SKIP=b;vec=4,chunks=1,rows=104,warps=1,prefetch=4" "PMG_DIAG_SKIP=e;vec=4,chunks=1,rows=104,warps=1,prefetch=4" "PMG_DIAG_SKIP=be;vec=4,chunks=1,rows=104,warps=1,prefetch=4" "PMG_XEDGE=0,PMG_DIAG_SKIP=b;$O"
