TAG=${TAG:-r2f} bash tools/gpu_full.sh
TAG=${TAG:-r2f} bash tools/gpu_profile_round.sh
