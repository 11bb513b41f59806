timeout 1200 python tools/fuzz_cy.py 120 7 > gpurun_out/fuzz_cy.log 2>&1; echo fuzz=$?
timeout 600 python tools/fuzz_cy.py 60 99 >> gpurun_out/fuzz_cy.log 2>&1; echo fuzz2=$?
