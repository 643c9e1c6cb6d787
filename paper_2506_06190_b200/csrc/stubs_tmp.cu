// TEMPORARY: entry points not implemented yet (replaced as each row lands).
#include "nat_internal.cuh"
#define NOT_YET(name) return nat::fail(NAT_ERR_INVALID_ARG, "%s: not implemented yet", name)
extern "C" {
nat_status nat_bem_near_count(const nat_mesh*, const nat_geom*, const nat_quad_opts*, int64_t, int64_t, int64_t*, int64_t*, nat_stream_t) { NOT_YET("nat_bem_near_count"); }
nat_status nat_bem_near_build(const nat_mesh*, const nat_geom*, const nat_quad_opts*, int64_t, int64_t, const int64_t*, int32_t*, uint8_t*, nat_stream_t) { NOT_YET("nat_bem_near_build"); }
size_t nat_bem_assemble_workspace(int64_t, int64_t, int) { return 0; }
nat_status nat_bem_assemble(const nat_mesh*, const nat_geom*, const nat_quad_opts*, const int64_t*, const int32_t*, const uint8_t*, double, nat_prec, int64_t, int64_t, int, const void*, void*, int64_t, void*, void*, size_t, nat_stream_t) { NOT_YET("nat_bem_assemble"); }
nat_status nat_bem_matvec(nat_prec, int64_t, int64_t, const void*, int64_t, const void*, void*, nat_stream_t) { NOT_YET("nat_bem_matvec"); }
nat_status nat_comm_unique_id(uint8_t*) { NOT_YET("nat_comm_unique_id"); }
nat_status nat_comm_create_from_id(nat_comm**, const uint8_t*, int, int) { NOT_YET("nat_comm_create_from_id"); }
nat_status nat_comm_destroy(nat_comm*) { NOT_YET("nat_comm_destroy"); }
size_t nat_bem_solve_workspace(nat_prec, int64_t, int64_t, int) { return 0; }
nat_status nat_bem_solve(nat_comm*, nat_prec, int64_t, int64_t, int64_t, const void*, int64_t, const void*, void*, double, int, void*, size_t, nat_solve_info*, nat_stream_t) { NOT_YET("nat_bem_solve"); }
nat_status nat_mc_sample(const nat_mesh*, const nat_geom*, int64_t, uint64_t, uint64_t, double*, int32_t*, nat_stream_t) { NOT_YET("nat_mc_sample"); }
size_t nat_mc_op_workspace(nat_prec, int64_t, int) { return 0; }
nat_status nat_mc_rhs(nat_prec, int64_t, const double*, int, const double*, const void*, double, double, void*, void*, size_t, nat_stream_t) { NOT_YET("nat_mc_rhs"); }
nat_status nat_mc_apply(nat_prec, int64_t, const double*, int, const double*, const void*, double, void*, void*, size_t, nat_stream_t) { NOT_YET("nat_mc_apply"); }
nat_status nat_mc_check_coincident(int64_t, const double*, int64_t*, void*, size_t, nat_stream_t) { NOT_YET("nat_mc_check_coincident"); }
size_t nat_mc_workspace(nat_prec, int64_t, int, int) { return 0; }
nat_status nat_mc_surface_pressure(const nat_mesh*, const nat_geom*, int, const double*, const void*, const nat_mc_opts*, nat_prec, double, int, double*, int32_t*, void*, void*, size_t, nat_solve_info*, nat_stream_t) { NOT_YET("nat_mc_surface_pressure"); }
}
