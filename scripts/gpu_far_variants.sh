# C2 multi-wavenumber far kernel: rows per CTA x min CTAs per SM variants
NAT_SKIP_MAIN= bash scripts/build_variants.sh t8b2 "-DNAT_FAR_TIM=8 -DNAT_FAR_MINB=2" t4b3 "-DNAT_FAR_TIM=4 -DNAT_FAR_MINB=3" t4b2 "-DNAT_FAR_TIM=4 -DNAT_FAR_MINB=2" t8b3 "-DNAT_FAR_TIM=8 -DNAT_FAR_MINB=3" > /dev/null || exit 1
cp paper_2506_06190_b200/libnat.so /tmp/libnat_main.so
for v in t8b2 t4b3 t4b2 t8b3; do echo "== $v"; cp paper_2506_06190_b200/_variants/libnat_$v.so paper_2506_06190_b200/libnat.so; timeout 300 python scripts/c2_far_multi.py 2>&1 | tail -2 | head -1; done
cp /tmp/libnat_main.so paper_2506_06190_b200/libnat.so
