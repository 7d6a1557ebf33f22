# GPU suite with the default library, then with the checked library (device asserts,
# bounded spin waits): the compute-sanitizer stand-in
python -m pytest tests -m gpu -q --tb=line > gpurun_out/gputests.log 2>&1; tail -3 gpurun_out/gputests.log
SMASH_LIB=paper_1705_05443_b200/libsmash_b200_checked.so python -m pytest tests -m gpu -q --tb=line > gpurun_out/gputests_checked.log 2>&1; tail -3 gpurun_out/gputests_checked.log
