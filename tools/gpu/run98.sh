timeout 60 ./tools/ring2_microbench
