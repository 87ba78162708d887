# full GPU suite, then the round's evidence (bench line, reference arm, launch list, full capture)
bash tools/gpu_tests.sh
bash tools/gpu_round.sh
