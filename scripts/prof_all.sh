cd $GRAFT_REPO_ROOT
CFG=c2 KREGEX="grad_rr|dgemm_nn_big" COUNT=2 SKIP=10 bash scripts/profile_round.sh
CFG=c3 KREGEX="grad_rr|srht_phase" COUNT=3 SKIP=20 bash scripts/profile_round.sh
CFG=c1 KREGEX="grad_rr|srht_phase|potrf" COUNT=3 SKIP=20 bash scripts/profile_round.sh
