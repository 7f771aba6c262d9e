for r in 1 2; do
  for c in cfg2 cfg3 cfg5; do
    bash tools/ab_cfg.sh hint_r$r $c "h0|MDRT_LIB=build/libmdrt_h0.so" "h1|MDRT_LIB=build/libmdrt_h1.so" "h2|MDRT_LIB=build/libmdrt_h2.so" "h3|MDRT_LIB=build/libmdrt_h3.so"
  done
done
