#!/bin/bash
# compute-sanitizer over a reduced GPU parity suite, both precisions, graphs
# off (SURVEY §4 layer 2 / §5): memcheck, racecheck, synccheck, initcheck.
#   bash scripts/sanitize.sh <outdir>
# Each tool runs the same small tests (cfg1, a few random nets, the fused
# ReLU->pool and depthwise-site passes, the tcgen05 conv units, rowmap, SE,
# capacity re-issue, the team depthwise forms, the SE sums forms, the staged
# tcgen05 dense epilogue); a log per tool and a one-line summary are written.
out=${1:-gpurun_out/sanitize}
mkdir -p "$out"
export ST_NO_GRAPHS=1 PYTHONUNBUFFERED=1
SEL='tests/test_gpu_parity.py::test_cfg1_toy_exact tests/test_gpu_parity.py::test_random_nets[0] tests/test_gpu_parity.py::test_random_nets[3] tests/test_gpu_parity.py::test_se_site tests/test_gpu_parity.py::test_relu_maxpool_geometries_exact tests/test_gpu_dw_site.py::test_fused_dw_site_matches_separate tests/test_gpu_dw_site.py::test_rowmap_matches_gathered tests/test_gpu_bf16.py::test_tc_conv_kernel_unit tests/test_gpu_bf16.py::test_tc_stem_kernel_unit tests/test_gpu_memory.py::test_capacity_overflow_reissue tests/test_gpu_dw_site.py::test_dw_site_forms_identical tests/test_gpu_parity.py::test_se_sums_forms_identical tests/test_gpu_parity.py::test_tc_dense_act_epilogue_identical'
for tool in ${SAN_TOOLS:-memcheck racecheck synccheck initcheck}; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check no"
  [ "$tool" = "initcheck" ] && extra="--track-unused-memory no"
  timeout ${SAN_TIMEOUT:-1200} compute-sanitizer --tool $tool $extra --target-processes all --error-exitcode 17 \
      --log-file "$out/$tool.log" python -m pytest -q -x -p no:cacheprovider $SEL > "$out/$tool.pytest.log" 2>&1
  rc=$?
  echo "$tool rc=$rc $(grep -c '========= ERROR\|========= Invalid\|========= Race\|========= Barrier\|Uninitialized' "$out/$tool.log") findings; $(tail -1 "$out/$tool.pytest.log")" >> "$out/summary.txt"
done
cat "$out/summary.txt"
