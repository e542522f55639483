TAG=r2z bash tools/gpu_full.sh
TAG=r2z bash tools/gpu_profile_round.sh
