@foo bar
@data
1,2:3,4
