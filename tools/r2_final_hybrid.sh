# Final state with HYBRID as the default: full GPU suite, smoke, both bench arms, ncu of the hybrid pack launches.
mkdir -p gpurun_out
bash tools/final_check.sh
bash tools/r2_hybrid_ncu.sh
