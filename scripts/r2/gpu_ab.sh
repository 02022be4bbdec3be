# A/B bench runs: each line of $VARIANTS is "<tag> <bench args>"
set -x
VP_PARITY_LOG=gpurun_out/parity_ab.json timeout 1500 python -m pytest ${PYTEST_TARGETS} -m gpu -q -s ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_ab.log 2>&1; echo pytest=$?
echo "$VARIANTS" | while read tag args; do
  [ -z "$tag" ] && continue
  timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --batch 0 $args > gpurun_out/ab_$tag.json 2> gpurun_out/ab_$tag.err; echo ab_$tag=$?
done
