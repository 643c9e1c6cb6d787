// TEMPORARY: entry points not implemented yet (replaced as each row lands).
#include "nat_internal.cuh"
#define NOT_YET(name) return nat::fail(NAT_ERR_INVALID_ARG, "%s: not implemented yet", name)
extern "C" {
nat_status nat_mc_sample(const nat_mesh*, const nat_geom*, int64_t, uint64_t, uint64_t, double*, int32_t*, nat_stream_t) { NOT_YET("nat_mc_sample"); }
size_t nat_mc_op_workspace(nat_prec, int64_t, int) { return 0; }
nat_status nat_mc_rhs(nat_prec, int64_t, const double*, int, const double*, const void*, double, double, void*, void*, size_t, nat_stream_t) { NOT_YET("nat_mc_rhs"); }
nat_status nat_mc_apply(nat_prec, int64_t, const double*, int, const double*, const void*, double, void*, void*, size_t, nat_stream_t) { NOT_YET("nat_mc_apply"); }
nat_status nat_mc_check_coincident(int64_t, const double*, int64_t*, void*, size_t, nat_stream_t) { NOT_YET("nat_mc_check_coincident"); }
size_t nat_mc_workspace(nat_prec, int64_t, int, int) { return 0; }
nat_status nat_mc_surface_pressure(const nat_mesh*, const nat_geom*, int, const double*, const void*, const nat_mc_opts*, nat_prec, double, int, double*, int32_t*, void*, void*, size_t, nat_solve_info*, nat_stream_t) { NOT_YET("nat_mc_surface_pressure"); }
}
