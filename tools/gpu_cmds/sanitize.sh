timeout 600 python tools/sanitize_smoke.py
# compute-sanitizer is refused on the graft GPU pool; on other machines:
#   compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck python tools/sanitize_smoke.py
