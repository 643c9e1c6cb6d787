# Round-1 final refresh after the kCC = 16 change: A/B of the last far-kernel shape, every
# GPU test, smoke, then the profile refresh (bench line, launch list, ncu, configs).
bash scripts/runs/ab_variants.sh base ti32m1 2>&1 | tee gpurun_out/ab_ti32.txt
rm -rf paper_2506_06190_b200/_variants
bash scripts/gpu_final.sh
