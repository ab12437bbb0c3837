timeout 60 ./tools/ring2_microbench
timeout 60 ./tools/ring3_microbench
