// tiled.cu — PIC_KERNEL_TILED dispatch: cell sort cadence, then the mover.
// (The fused tile-staged mover + deposit kernel lands here; until then the
// tiled family sorts and runs the basic kernels.)
#include "pic_internal.cuh"

namespace pic {

pic_status launch_tiled_step(Ctx *ctx, int s, bool *did_deposit) {
  *did_deposit = false;
  SpeciesStore &sp = ctx->sp[s];
  const int se = ctx->cfg.sort_every;
  if (se > 0 && (ctx->cycle % se == 0 || !sp.sorted)) {
    pic_status st = sort_species(ctx, s);
    if (st != PIC_OK) return st;
  }
  return launch_mover_basic(ctx, s);
}

}  // namespace pic
