# long same-box A/B only (no tests): the working tree vs ab/*.so
cd $GRAFT_REPO_ROOT
NOBENCH=1 bash scripts/r02/ab2.sh "$@" 2>&1 | grep -v "^bench"
