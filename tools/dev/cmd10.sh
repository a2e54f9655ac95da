cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_cli.py -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_cli.log 2>&1; tail -30 gpurun_out/pytest_cli.log
